"""Debug helper: multi-rank (host communicator, one GPU) solves vs the oracle, error per rank
and slice.  python tools/mr_debug.py P name n nt solver"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import tempfile  # noqa: E402

import synth  # noqa: E402
from test_dist_cpu import _spawn  # noqa: E402
from test_gpu_multirank import SOLVERS, _worker  # noqa: E402

if __name__ == "__main__":
    P, name, sv = int(sys.argv[1]), sys.argv[2], sys.argv[5]
    n, nt = (None, None) if sys.argv[3] == "-" else (int(sys.argv[3]), int(sys.argv[4]))
    import oracle as orc

    d = tempfile.mkdtemp()
    _spawn(_worker, P, name, n, nt, (sv,), d)
    cfg = synth.CONFIGS[name] if n is None else synth.CONFIGS[name].scaled(n, nt)
    s = orc.spec(cfg)
    u0 = synth.initial_condition(cfg)
    ref = getattr(orc, ("cplx_" if cfg.is_complex else "") + sv)
    Uo, st, its, _ = ref(s, u0, tol=cfg.tol, maxit=50, **SOLVERS[sv])
    got = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(P)]
    U = np.concatenate([g["U_" + sv] for g in got])
    sc = np.abs(Uo).max()
    print(name, P, sv, "its", [int(g["its_" + sv][0]) for g in got], its)
    for t in range(cfg.nt):
        e = np.abs(U[t] - Uo[t])
        idx = np.unravel_index(np.argmax(e), e.shape)
        print(t, "err/scale %.3e" % (e.max() / sc), "at", idx, "slice max", "%.3e" % np.abs(Uo[t]).max())
