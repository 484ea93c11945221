"""Every BASELINE.json config on one GPU through the C-ABI: fixed-point / Picard and (linear)
GMRES solves from U = 0, iteration counts, residual histories, device time and
DOF-iterations/s.  Writes one JSON line per (config, solver)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5", "c3if", "c5if", "c1bdf2", "c2bdf2", "c6se", "c7se", "c7bdf2"]
for name in names:
    cfg = synth.CONFIGS[name]
    u0 = torch.from_numpy(synth.initial_condition(cfg)).cuda()
    for solver in cfg.solvers:
        kv = 0 if solver != "gmres" else (21 if cfg.nst < 2e8 else 4)
        tol = cfg.tol
        plan = Plan(Problem.from_config(cfg), krylov_vectors=kv)
        prob = Problem.from_config(cfg)
        U = torch.zeros((cfg.nt,) + cfg.shape, dtype=prob.dtype, device="cuda")
        run = (lambda: plan.fixed_point_solve(u0, U, tol=tol, maxit=100)) if solver != "gmres" else \
              (lambda: plan.gmres_solve(u0, U, tol=tol, restart=min(20, kv - 1), maxit=100))
        run()  # warm-up (first solve builds the sweep graph)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        U.zero_()
        e0.record()
        _, rep = run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        passes = rep["sweeps"] if solver != "gmres" else rep["iterations"] + 1
        print(json.dumps({"config": name, "solver": solver, "n": cfg.n, "dim": cfg.dim, "nt": cfg.nt,
                          "n_st": cfg.nst, "tol": tol, "iterations": rep["iterations"],
                          "converged": rep["converged"], "hist": [float(f"{h:.3e}") for h in rep["hist"]],
                          "solve_ms": round(ms, 3), "loop_s": rep.get("seconds"),
                          "dof_iter_per_s": cfg.nst * passes / (ms * 1e-3)}), flush=True)
        del plan, U
        torch.cuda.empty_cache()
