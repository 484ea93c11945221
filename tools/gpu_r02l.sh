#!/bin/bash
tag=${1:-r02l}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "sweep or fixed_point or c5_full or max_line or c3 or device_loop or fuzz_picard or opt_in" > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/${tag}_pytest.log
for v in 1 0 1 0 1 0; do
  EXPD_S3_FULLX=$v timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$v.json 2>$O/${tag}_bench_$v.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('fullx $v sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'], d['gpu_launches'])" || tail -3 $O/${tag}_bench_$v.err
done
