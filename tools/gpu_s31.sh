#!/bin/bash
# s31: knobs re-measured on the final code: stage-3 chunk size (EXPD_CHUNK_MB) and the K1 tile
# loads' L2 promotion (EXPD_K1_PROMO), c5
tag=${1:-s31}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for e in "EXPD_CHUNK_MB=512" "EXPD_CHUNK_MB=256" "EXPD_CHUNK_MB=1024" "EXPD_K1_PROMO=2" "EXPD_K1_PROMO=3" "EXPD_CHUNK_MB=512"; do
  env $e timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$e: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'y', round(k['line_y_nl']['launch_ms'],3), d['clocks']['sm_mhz'])"
done
