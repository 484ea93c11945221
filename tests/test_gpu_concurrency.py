"""Two plans used at the same time from two host threads, each on its own CUDA stream (the
library's per-device caches -- shared-memory opt-ins, tensor maps, the K1 / line variant
choices -- are process-wide): both solves match the oracle exactly as when run alone."""
from __future__ import annotations

import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

DEV = torch.device("cuda:0")


def relmax(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def test_two_plans_two_streams_two_threads(orc):
    cases = [("c5", 255, 16, "fixed_point"), ("c2", 63, 64, "gmres"), ("c3", 127, 32, "fixed_point"),
             ("c7se", 63, 16, "gmres")]
    cfgs = [synth.CONFIGS[n].scaled(m, nt) for n, m, nt, _ in cases]
    want = []
    for cfg, (_, _, _, sv) in zip(cfgs, cases):
        s = orc.spec(cfg)
        u0 = synth.initial_condition(cfg)
        kw = {"restart": 20} if sv == "gmres" else {}
        ref = getattr(orc, ("cplx_" if cfg.is_complex else "") + sv)
        Uo, st, its, _ = ref(s, u0, tol=cfg.tol, maxit=50, **kw)
        assert st == 0
        want.append((Uo, its))
    out, errs = [None] * len(cases), []

    def run(i):
        try:
            cfg, sv = cfgs[i], cases[i][3]
            stream = torch.cuda.Stream(DEV)
            with torch.cuda.stream(stream):
                plan = Plan(Problem.from_config(cfg), krylov_vectors=21, stream=stream)
                u0 = torch.from_numpy(np.ascontiguousarray(synth.initial_condition(cfg))).to(DEV)
                kw = {"restart": 20} if sv == "gmres" else {}
                for _ in range(3):  # several solves per thread, interleaving with the others
                    U, rep = getattr(plan, sv + "_solve")(u0, tol=cfg.tol, maxit=50, **kw)
                stream.synchronize()
                out[i] = (U.cpu().numpy(), rep["iterations"])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for (U, its), (Uo, its_o), c in zip(out, want, cases):
        assert its == its_o, c
        assert relmax(U, Uo) < 1e-9, c
