#!/bin/bash
# r02f: k_line2 (two threads per radix-16 job) parity + A/B against k_line (EXPD_LINE2=0) and the
# 3-CTA/SM register-light variant
tag=${1:-r02f}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
bash tools/build_variant.sh k_line.cu /tmp/libexpd_l2m3.so -DEXPD_LINE2_MINB=3 -DEXPD_LINE2_TWSEQ -DEXPD_LINE2_LAZY_A > $O/${tag}_variant.log 2>&1 || echo VARIANT FAILED
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "nonlin or dst or sweep or fixed_point or c5_full or max_line or smoke" > $O/${tag}_pytest.log 2>&1; echo "pytest line2 exit $?"; tail -3 $O/${tag}_pytest.log
EXPD_LIB=/tmp/libexpd_l2m3.so timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "nonlin or c5_full or fixed_point_parity" > $O/${tag}_pytest_m3.log 2>&1; echo "pytest m3 exit $?"; tail -2 $O/${tag}_pytest_m3.log
for v in new old m3 new old m3; do
  unset EXPD_LIB; unset EXPD_LINE2
  [ $v = old ] && export EXPD_LINE2=0
  [ $v = m3 ] && export EXPD_LIB=/tmp/libexpd_l2m3.so
  timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$v.json 2>$O/${tag}_bench_$v.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v sweep', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'])" || tail -5 $O/${tag}_bench_$v.err
done
