import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2603_04350_b200 import Plan, Problem
cfg = synth.CONFIGS["c5"]
plan = Plan(Problem.from_config(cfg))
plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
out = {}
for which, label in ((4, "rows"), (6, "cols_nl")):
    for ns in (1, 2, 3):
        out[f"{label}_{ns}"] = round(1e3 * plan.debug_kernel_ms(which, ns, 20) / ns, 2)
print(json.dumps(out))
