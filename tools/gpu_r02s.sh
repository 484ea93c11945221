#!/bin/bash
# r02s: what the write-after-read barriers of the line transform cost (EXPD_EXP_NOWAR drops
# them: the results are wrong, only the timing is meaningful)
tag=${1:-r02s}
O=gpurun_out; mkdir -p $O
L=paper_2603_04350_b200
run() { local lab=$1 lib=$2
  EXPD_LIB=$lib timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_$lab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_$lab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$lab sweep', round(d['ms_per_step'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do run base $L/libexpd.so; run nowar $L/libexpd_nowar.so; done
