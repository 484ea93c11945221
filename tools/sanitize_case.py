"""Small cases for compute-sanitizer (one tool per gpurun call, tools/gpu_sanitize.sh):
every kernel family of the hot path at reduced sizes, through the C-ABI.

  stage 3 TMA line kernels M = 256 and M = 2048 (x-pass, fused y [V, N, V]), K1 k_time_tma in
  its ETD2 / ETD1 / linear / complex forms, the GMRES vector kernels, the reductions."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

which = sys.argv[1:] or ["c5s", "c5big", "c3s", "c1", "c2s", "c7s"]


def T(x):
    return torch.from_numpy(x).cuda()


for name in which:
    if name == "c5s":      # ETD2 Picard, 255^2 x 16: line kernels M = 256, K1 ETD2 form
        cfg = synth.CONFIGS["c5"].scaled(255, 16)
        plan = Plan(Problem.from_config(cfg))
        U, rep = plan.fixed_point_solve(T(synth.initial_condition(cfg)), tol=1e-12, maxit=3)
    elif name == "c5big":  # one ETD2 sweep at n + 1 = 2048 (the bench's line kernels), nt = 4
        cfg = synth.CONFIGS["c5"].scaled(2047, 4)
        plan = Plan(Problem.from_config(cfg))
        U, rep = plan.fixed_point_solve(T(synth.initial_condition(cfg)), tol=1e-12, maxit=1)
    elif name == "c3s":    # ETD1 Picard, 63^2 x 128 (K1 Nt = 128 variant)
        cfg = synth.CONFIGS["c3"].scaled(63, 128)
        plan = Plan(Problem.from_config(cfg))
        U, rep = plan.fixed_point_solve(T(synth.initial_condition(cfg)), tol=1e-12, maxit=5)
    elif name == "c1":     # 1D linear, fixed point + GMRES
        cfg = synth.CONFIGS["c1"]
        plan = Plan(Problem.from_config(cfg), krylov_vectors=4)
        u0 = T(synth.initial_condition(cfg))
        plan.fixed_point_solve(u0, tol=cfg.tol)
        U, rep = plan.gmres_solve(u0, tol=cfg.tol, restart=3)
    elif name == "c2s":    # 2D linear 63^2 x 64, fixed point + GMRES + BiCGStab
        cfg = synth.CONFIGS["c2"].scaled(63, 64)
        plan = Plan(Problem.from_config(cfg), krylov_vectors=6)
        u0 = T(synth.initial_condition(cfg))
        plan.fixed_point_solve(u0, tol=cfg.tol)
        plan.gmres_solve(u0, tol=cfg.tol, restart=3)
        U, rep = plan.bicgstab_solve(u0, tol=cfg.tol)
    elif name == "c7s":    # complex coefficients 2D 63^2 x 16 (K1 complex form, split / merge)
        cfg = synth.CONFIGS["c7se"].scaled(63, 16)
        plan = Plan(Problem.from_config(cfg), krylov_vectors=4)
        U, rep = plan.gmres_solve(T(synth.initial_condition(cfg)), tol=cfg.tol, restart=3)
    torch.cuda.synchronize()
    print(name, rep["iterations"], rep["status"], flush=True)
    del plan
