#!/bin/bash
# r02u: ping-pong line kernels (two buffers alternating roles, no write-after-read barriers,
# no prefetch): parity with EXPD_COLV=13 EXPD_ROWV=3, then c5 / c3 timing against the defaults
tag=${1:-r02u}
O=gpurun_out; mkdir -p $O
EXPD_COLV=13 EXPD_ROWV=3 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "dst or nonlin or sweep or fixed_point or c5 or line or max_line or c4" > $O/${tag}_pytest.log 2>&1; echo "pytest (pp) exit $?"; tail -2 $O/${tag}_pytest.log
run() { local cfg=$1 lab=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --no-cpu --no-e2e > $O/${tag}_${cfg}_$lab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_${cfg}_$lab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg $lab sweep', round(d['ms_per_step'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do
  run c5 base X=1; run c5 colpp EXPD_COLV=13; run c5 rowpp EXPD_ROWV=3; run c5 bothpp EXPD_COLV=13 EXPD_ROWV=3
done
run c3 base X=1; run c3 bothpp EXPD_COLV=13 EXPD_ROWV=3; run c3 base2 X=1; run c3 bothpp2 EXPD_COLV=13 EXPD_ROWV=3
