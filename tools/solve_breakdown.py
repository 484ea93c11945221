"""Where a small fixed-point solve's time goes: CUDA events around the setup (DST of u0 and
of the initial guess), each sweep + norm read, and the final IDST of U, on the resident
state (the pieces expd_fixed_point_solve runs), for c1 / c2."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


out = {}
for name in sys.argv[1:] or ["c1", "c2"]:
    cfg = synth.CONFIGS[name]
    plan = Plan(Problem.from_config(cfg))
    u0 = torch.from_numpy(synth.initial_condition(cfg)).cuda()
    U = torch.zeros((cfg.nt,) + cfg.shape, dtype=torch.float64, device="cuda")
    rows = []
    for rep in range(6):
        U.zero_()
        e = [ev() for _ in range(6)]
        torch.cuda.synchronize()
        e[0].record()
        plan.load_state(u0, U)
        e[1].record()
        plan.sweep()
        plan.sweep_norm2()
        e[2].record()
        plan.sweep()
        plan.sweep_norm2()
        e[3].record()
        plan.store_state(U)
        e[4].record()
        plan.set_zero_guess(True)  # the solve from U = 0 without transforming the guess
        _, r = plan.fixed_point_solve(u0, U, tol=cfg.tol)
        plan.set_zero_guess(False)
        e[5].record()
        torch.cuda.synchronize()
        rows.append([e[i].elapsed_time(e[i + 1]) for i in range(5)] + [r["sweeps"]])
    best = min(rows, key=lambda x: sum(x[:4]))
    out[name] = {"load_state_ms": best[0], "sweep1_ms": best[1], "sweep2_ms": best[2], "store_state_ms": best[3],
                 "fixed_point_solve_ms": best[4], "sweeps": best[5],
                 "byte_floor_sweep_ms": 16 * cfg.nst / 6557.4e9 * 1e3}
    del plan
print(json.dumps(out))
