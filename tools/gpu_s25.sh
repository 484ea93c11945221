#!/bin/bash
# s25: the hybrid buffer schedule of the line kernels (EXPD_LINE_HY=1): parity of the line /
# stage-3 / Picard tests with it forced, then c5 sweeps A/B against the default
tag=${1:-s25}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
EXPD_LINE_HY=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x -k "dst or nonlin or tail or fixed_point_parity or sweep or k1_nt256 or c5" -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest (HY) exit $?"; tail -2 $O/${tag}_pytest.log
for v in 0 1 0 1; do
  EXPD_LINE_HY=$v timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>$O/${tag}_c5_$v.err
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('HY=$v: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['launch_ms'],3), 'y', round(k['line_y_nl']['launch_ms'],3), 'resid', d.get('residual_norm_last'), d['clocks']['sm_mhz'])" || tail -5 $O/${tag}_c5_$v.err
done
