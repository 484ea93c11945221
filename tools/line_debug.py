"""Smallest exercise of the TMA line kernels (tuning / debugging aid): V of random
physical slices at n = 255 (strided-axis line kernel) and V N V of DST coefficients
(x-axis + fused strided line kernels), checked against the CPU oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

dim, n = int(sys.argv[1]), int(sys.argv[2])
which = sys.argv[3] if len(sys.argv) > 3 else "dst"
cfg = synth.Config("t", dim, n, 1.0, 1.0, 1.0, 8, 1e-2, q=(0.0, 0.0, 0.0, -1.0), scheme=1)
plan = Plan(Problem.from_config(cfg))
s = oracle.spec(cfg)
x = np.random.default_rng(1).standard_normal(cfg.shape) / (np.sqrt(cfg.N) if which == "nl" else 1.0)
xt = torch.from_numpy(x).cuda()
if which == "dst":
    got = plan.dst(xt).cpu().numpy()
    want = oracle.dst(s, x)
else:
    got = plan.nonlin_hat(xt).cpu().numpy()
    want = oracle.dst(s, oracle.nonlin(s, oracle.dst(s, x)))
torch.cuda.synchronize()
err = np.abs(got - want).max() / np.abs(want).max()
print(f"{which} dim={dim} n={n}: rel err {err:.3e}", flush=True)
