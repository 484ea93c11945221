#!/bin/bash
# r02h: line kernels with the on-the-fly pre-processing weights: parity + bench
tag=${1:-r02h}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "nonlin or dst or sweep or fixed_point or fullsize or max_line or c3 or smoke or fuzz_picard" > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/${tag}_pytest.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$i.json 2>$O/${tag}_bench_$i.err
python -c "
import json; d=json.loads(open('$O/${tag}_bench_$i.json').read().strip().splitlines()[-1]); k=d['kernels']
fam={n: round(k[n]['ms_per_step'],3) for n in ('line_x','line_y_nl','stage3_persistent') if n in k}
print('sweep', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), fam, d['clocks']['sm_mhz'])"
done
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/${tag}_bench_c3.json 2>&1; EXPD_S3P=1 timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/${tag}_bench_c3_s3p.json 2>&1
for f in c3 c3_s3p; do python -c "
import json; d=json.loads(open('$O/${tag}_bench_$f.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$f sweep', round(d['ms_per_step'],4), 'k1', round(k['k1']['launch_ms'],4), 's3', round(k['stage3_ms'],4))"; done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*2048, .int.0," -s 40 -c 1 -o $O/${tag}_prof_row $CMD > $O/${tag}_ncu_row.log 2>&1; echo "ncu row exit $?"
