"""Fixed-point solve time with the device-side loop (CUDA-graph WHILE node) against the
host-driven loop (EXPD_DEVICE_LOOP=0), device-resident, CUDA events around the C-ABI call
(includes the setup DST of u0 and the final IDST of U, which both loops share)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c1", "c2"]:
    cfg = synth.CONFIGS[name]
    plan = Plan(Problem.from_config(cfg))
    u0 = torch.from_numpy(synth.initial_condition(cfg)).cuda()
    U = torch.zeros((cfg.nt,) + cfg.shape, dtype=torch.float64, device="cuda")
    plan.set_zero_guess(True)  # PAPER.md:895's zero initial guess, no transform of U on entry
    res = {}
    for mode in ("1", "0"):
        os.environ["EXPD_DEVICE_LOOP"] = mode
        for _ in range(3):
            U.zero_()
            plan.fixed_point_solve(u0, U, tol=cfg.tol)
        ts = []
        for _ in range(20):
            U.zero_()  # the zero initial guess
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            _, rep = plan.fixed_point_solve(u0, U, tol=cfg.tol)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        res["device_loop" if mode == "1" else "host_loop"] = {"median_ms": ts[len(ts) // 2], "min_ms": ts[0],
                                                            "sweeps": rep["sweeps"]}
    # the byte floor of the solve's sweeps (16 B/dof each at the measured HBM copy rate) and
    # of its setup DST of u0 + final IDST of U (16 B/dof of one space-time array)
    res["byte_floor_sweeps_ms"] = 16 * cfg.nst / 6557.4e9 * 1e3 * res["device_loop"]["sweeps"]
    res["byte_floor_solve_ms"] = res["byte_floor_sweeps_ms"] + 16 * cfg.nst / 6557.4e9 * 1e3
    out[name] = res
    del plan
print(json.dumps(out))
