#!/bin/bash
# K1 ring variant (EXPD_K1V=5123): parity with it forced, bench A/B against the default
tag=${1:-r02c}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
EXPD_K1V=5123 timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "precond or residual or fixed_point or gmres or bicgstab or sweep or device_loop or c5_full or cplx or fuzz" > $O/${tag}_pytest_ring.log 2>&1; echo "pytest ring exit $?"; tail -3 $O/${tag}_pytest_ring.log
for v in 2562 5123; do
EXPD_K1V=$v timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$v.json 2>$O/${tag}_bench_$v.err; echo "bench $v exit $?"
python -c "
import json; d=json.loads(open('$O/${tag}_bench_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v sweep', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'k1', round(k['k1']['launch_ms'],3), round(k['k1']['frac'],3), 's3', round(k['stage3_ms'],3))"
done
for v in 2562 5123; do
EXPD_K1V=$v timeout 600 python bench.py --config c4 --no-cpu --no-e2e --steps 10 > $O/${tag}_bench_c4_$v.json 2>&1; python -c "
import json; d=json.loads(open('$O/${tag}_bench_c4_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('c4 $v sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), round(k['k1']['frac'],3))"
EXPD_K1V=$v timeout 600 python bench.py --config c3 --no-cpu --no-e2e --steps 10 > $O/${tag}_bench_c3_$v.json 2>&1; python -c "
import json; d=json.loads(open('$O/${tag}_bench_c3_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('c3 $v sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), round(k['k1']['frac'],3))"
done
timeout 300 python tools/loop_timing.py c1 c2 > $O/${tag}_loop_timing.json 2>&1; echo "loop timing exit $?"; cat $O/${tag}_loop_timing.json | tail -2
