#!/bin/bash
# s21: line kernels at 4 CTAs per SM (one buffer, 128 registers: -DEXPD_LINE_REGS=128, 60-68 B of
# spills) against the defaults (two buffers, 3 CTAs per SM, 168 registers)
tag=${1:-s21}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for v in default r128 default r128; do
  if [ $v = default ]; then E=""; else E="EXPD_LIB=_variants/libexpd_r128.so EXPD_ROWV=1 EXPD_COLV=11"; fi
  env $E timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['launch_ms'],3), 'y', round(k['line_y_nl']['launch_ms'],3), d['clocks']['sm_mhz'])"
done
