"""One c4 GMRES solve (3D 255^3 x 64, linear) for profiling the K6/K7 vector kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

cfg = synth.CONFIGS["c4"]
plan = Plan(Problem.from_config(cfg), krylov_vectors=4)
u0 = torch.from_numpy(synth.initial_condition(cfg)).cuda()
for _ in range(2):
    U, rep = plan.gmres_solve(u0, tol=cfg.tol, restart=3, maxit=20)
torch.cuda.synchronize()
print(rep["iterations"], rep["converged"])
