#!/bin/bash
# r02k: stage-3 chunk size A/B (EXPD_CHUNK_MB) -- DRAM traffic (power) vs launch tails
tag=${1:-r02k}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for mb in 512 1024 2048 4096 9000 1024 2048 9000; do
  EXPD_CHUNK_MB=$mb timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$mb.json 2>$O/${tag}_bench_$mb.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$mb.json').read().strip().splitlines()[-1]); k=d['kernels']
print('chunk $mb MB sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks'])"
done
