#!/bin/bash
# s12: the strided passes' tail-row parity tests; A/B of the line kernels' sequential twiddle
# powers (-DEXPD_LINE_TWSEQ, _variants/libexpd_twseq.so built by tools/build_variant.sh)
tag=${1:-s12}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tail" -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest tail exit $?"; tail -2 $O/${tag}_pytest.log
for v in default twseq default twseq; do
  if [ $v = default ]; then L=""; else L="EXPD_LIB=_variants/libexpd_$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['launch_ms'],3), 'y', round(k['line_y_nl']['launch_ms'],3), d['clocks']['sm_mhz'])"
done
