#!/bin/bash
# r02r: K1 ring twiddle reads through the shared window (LDS) vs the former generic pointer
# (LD.E): c5 (Nt = 256), c3 and c7se (Nt = 128), alternating
tag=${1:-r02r}
O=gpurun_out; mkdir -p $O
L=paper_2603_04350_b200
run() { local cfg=$1 lab=$2 lib=$3
  EXPD_LIB=$lib timeout 600 python bench.py --config $cfg --no-cpu --no-e2e > $O/${tag}_${cfg}_$lab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_${cfg}_$lab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg $lab sweep', round(d['ms_per_step'],4), 'k1', round(k['k1']['launch_ms'],4), 'k1 frac', round(k['k1']['frac'],3), d['clocks']['sm_mhz'])"; }
for i in 1 2; do
  run c5 lds $L/libexpd.so; run c5 generic $L/libexpd_gtw256.so
  run c3 lds $L/libexpd.so; run c3 generic $L/libexpd_gtw128.so
  run c7se lds $L/libexpd.so; run c7se generic $L/libexpd_gtw128.so
done
