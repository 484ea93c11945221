#!/bin/bash
# s28: the last prefix's cross-warp barrier deferred to the pre-output barrier (EXPD_LINE_DEFER,
# default 1): parity of the line / stage-3 / Picard tests, A/B against -DEXPD_LINE_DEFER=0
tag=${1:-s28}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -q -m gpu -x -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/${tag}_pytest.log
for v in nodefer default nodefer default; do
  if [ $v = default ]; then E=""; else E="EXPD_LIB=_variants/libexpd_$v.so"; fi
  env $E timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['launch_ms'],3), 'y', round(k['line_y_nl']['launch_ms'],3), 'resid', d.get('residual_norm_last'), d['clocks']['sm_mhz'])"
done
