"""Launch each TMA line-kernel family a few times on c5's spectral state (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
plan = Plan(Problem.from_config(cfg))
plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
for which in (4, 5, 6):
    print(which, plan.debug_kernel_ms(which, 2, 2))
torch.cuda.synchronize()
