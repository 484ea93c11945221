import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from dataclasses import replace
from paper_2603_04350_b200 import Plan, Problem
cfgs = [synth.CONFIGS[n] for n in ("c4", "c2", "c7se", "c7bdf2", "c5", "c3")]
cfgs.append(replace(synth.CONFIGS["c5"], name="c5lin", q=()))
cfgs.append(replace(synth.CONFIGS["c5"], name="c5bdf2", q=(), scheme=3))
for cfg in cfgs:
    plan = Plan(Problem.from_config(cfg))
    plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
    ms = plan.debug_kernel_ms(3, 1, 10)
    bpd = 32 if cfg.is_complex else (24 if cfg.q else 16)
    print(f"{cfg.name} nt={cfg.nt} K1 {ms:.4f} ms {bpd * cfg.nst / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del plan; torch.cuda.empty_cache()
