#!/bin/bash
# r02t: split arrive / wait write-after-read barriers in the line transform (WarMbar, default)
# vs one __syncthreads each (WarSync, -DEXPD_WAR_MODE=0): parity of the line kernels, then c5 / c3
tag=${1:-r02t}
O=gpurun_out; mkdir -p $O
L=paper_2603_04350_b200
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "dst or nonlin or sweep or fixed_point or c5 or line or max_line" > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/${tag}_pytest.log
run() { local cfg=$1 lab=$2 lib=$3
  EXPD_LIB=$lib timeout 600 python bench.py --config $cfg --no-cpu --no-e2e > $O/${tag}_${cfg}_$lab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_${cfg}_$lab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg $lab sweep', round(d['ms_per_step'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do run c5 mbar $L/libexpd.so; run c5 sync $L/libexpd_warsync.so; done
for i in 1 2; do run c3 mbar $L/libexpd.so; run c3 sync $L/libexpd_warsync.so; done
