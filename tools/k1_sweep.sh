#!/bin/bash
# K1 variants (EXPD_K1_PIPE / EXPD_K1V): correctness on small cases + c5 K1 time
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for v in ${K1VS:-"2 0" "3 2561" "3 2562" "3 1281" "3 1282"}; do
  set -- $v
  EXPD_K1_PIPE=$1 EXPD_K1V=$2 timeout 300 python -m pytest tests -q -m gpu -x -k "precond_apply_parity or fixed_point_parity or gmres_parity" 2>&1 | tail -1 | sed "s/^/pipe$1 v$2 /"
  EXPD_K1_PIPE=$1 EXPD_K1V=$2 timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2603_04350_b200 import Plan, Problem
for name in ('c5','c3','c4' if False else 'c2'):
    cfg = synth.CONFIGS[name]
    plan = Plan(Problem.from_config(cfg))
    plan.load_state(torch.from_numpy(synth.initial_condition(cfg)).cuda(), None)
    print('pipe$1 v$2', name, 'K1 ms', round(plan.debug_kernel_ms(3, 1, 5), 4), flush=True)
    del plan
"
done
