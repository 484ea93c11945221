import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2603_04350_b200 import Plan, Problem
cfg = synth.CONFIGS[sys.argv[1]] if len(sys.argv) < 3 else synth.CONFIGS[sys.argv[1]].scaled(int(sys.argv[2]), int(sys.argv[3]))
plan = Plan(Problem.from_config(cfg))
u0 = torch.from_numpy(synth.initial_condition(cfg)).cuda()
plan.load_state(u0, None); torch.cuda.synchronize(); print("load ok", flush=True)
for k in range(3):
    plan.sweep(); torch.cuda.synchronize(); print("sweep", k, plan.sweep_norm2(), flush=True)
