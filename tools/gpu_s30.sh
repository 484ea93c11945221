#!/bin/bash
# s30: this session's kernel changes on one box: the library of 355c937 (session start:
# _variants/libexpd_start.so, built from that commit) against the final code, c5 and c3, alternating
tag=${1:-s30}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for cfg in c5 c3; do
for v in start final start final start final; do
  if [ $v = final ]; then E=""; else E="EXPD_LIB=_variants/libexpd_$v.so"; fi
  env $E timeout 600 python bench.py --config $cfg --no-cpu --no-e2e > $O/${tag}_${cfg}_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_${cfg}_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg $v: sweep', round(d['ms_per_step'],4), 'k1', round(k['k1']['launch_ms'],4), 's3', round(k['stage3_ms'],4), 'resid', d.get('residual_norm_last'), d['clocks']['sm_mhz'])"
done
done
