#!/bin/bash
# s10: stage-3 chunk size re-measured with the transposed strided store (EXPD_CHUNK_MB)
tag=${1:-s10}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for mb in 512 256 1024 768 384 512; do
  EXPD_CHUNK_MB=$mb timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$mb.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$mb.json').read().strip().splitlines()[-1]); k=d['kernels']
print('chunk $mb MB: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['launch_ms'],3), 'y', round(k['line_y_nl']['launch_ms'],3), d['clocks']['sm_mhz'])"
done
