"""K1 device time and algorithmic GB/s per config (tuning aid): python tools/k1_cfgs.py c5 c7se ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import Plan, Problem  # noqa: E402

for name in sys.argv[1:] or ["c5"]:
    cfg = synth.CONFIGS[name]
    plan = Plan(Problem.from_config(cfg))
    plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
    ms = plan.debug_kernel_ms(3, 1, 10)
    bpd = 32 if cfg.is_complex else (24 if cfg.q else 16)
    print(f"{os.environ.get('EXPD_K1V', '2562')} {name} nt={cfg.nt} K1 {ms:.4f} ms "
          f"{bpd * cfg.nst / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del plan
    torch.cuda.empty_cache()
