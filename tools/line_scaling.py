"""Per-slice device time of the TMA line kernels vs the slices per launch (1 .. 256) on c5's
spectral state: where does the fused strided pass lose when a launch spans many slices?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

cfg = synth.CONFIGS["c5"]
plan = Plan(Problem.from_config(cfg))
plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
out = {}
for which, label in ((4, "rows"), (6, "cols_nl")):
    for ns in (4, 16, 32, 64, 128, 256):
        out[f"{label}_{ns}"] = round(1e3 * plan.debug_kernel_ms(which, ns, 3) / ns, 2)
print(json.dumps(out))
