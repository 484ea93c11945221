"""Per-kernel device times on a config's spectral state (tuning aid, not a benchmark)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_04350_b200 import ExpdError, Plan, Problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = synth.CONFIGS[name]
plan = Plan(Problem.from_config(cfg))
u0 = torch.from_numpy(synth.initial_condition(cfg)).cuda()
plan.load_state(u0, None)
res = {"config": name}
for which, label in ((0, "rows"), (1, "cols"), (2, "cols_nl"), (4, "line_rows"), (5, "line_cols"), (6, "line_cols_nl")):
    for ns in (1, 2, 8):
        try:
            res[f"{label}_x{ns}"] = plan.debug_kernel_ms(which, ns, 10) / ns
        except ExpdError as e:
            res[f"{label}_x{ns}"] = str(e)[:60]
res["k1"] = plan.debug_kernel_ms(3, 1, 5)
print(json.dumps(res))
