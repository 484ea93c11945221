#!/bin/bash
# s33: the warp-per-pair K1's refill point (EXPD_WP_LATE_REFILL 0 / 1 / 2 as variant libraries):
# parity of the Nt = 256 Picard tests on each, then c5 sweeps, alternating
tag=${1:-s33}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for v in late1 late2; do
  EXPD_LIB=_variants/libexpd_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "k1_nt256" -p no:cacheprovider > $O/${tag}_pytest_$v.log 2>&1; echo "pytest $v exit $?"; tail -1 $O/${tag}_pytest_$v.log
done
for v in default late1 late2 default late1 late2; do
  if [ $v = default ]; then E=""; else E="EXPD_LIB=_variants/libexpd_$v.so"; fi
  env $E timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'resid', d.get('residual_norm_last'), d['clocks']['sm_mhz'])"
done
