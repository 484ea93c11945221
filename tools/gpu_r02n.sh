#!/bin/bash
# r02n: K1 variant A/B on the small linear config c2 (Nt = 64) and on c4
tag=${1:-r02n}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for cfg in c2 c4; do for v in 2562 1282 2561; do
  EXPD_K1V=$v timeout 600 python bench.py --config $cfg --no-cpu --no-e2e --steps 20 > $O/${tag}_${cfg}_$v.json 2>$O/${tag}_${cfg}_$v.err
  python -c "
import json; d=json.loads(open('$O/${tag}_${cfg}_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg $v sweep_ms', round(d['ms_per_step'],4), 'k1', round(k['k1']['launch_ms'],4), round(k['k1']['frac'],3))" || tail -3 $O/${tag}_${cfg}_$v.err
done; done
for v in 2562 1282; do EXPD_K1V=$v timeout 300 python tools/loop_timing.py c2 > $O/${tag}_loop_$v.json 2>&1; echo "$v $(tail -1 $O/${tag}_loop_$v.json)"; done
