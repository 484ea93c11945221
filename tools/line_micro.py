"""TMA line-kernel device times on c5's spectral state (us per slice, 8-slice launches)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
plan = Plan(Problem.from_config(cfg))
plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
out = {}
for which, label in ((4, "rows"), (5, "cols"), (6, "cols_nl")):
    out[label] = round(1e3 * plan.debug_kernel_ms(which, 8, 10) / 8, 2)
print(json.dumps(out))
