#!/bin/bash
# r02d: full GPU suite with the new defaults (ring K1 at Nt = 256, swizzled strided output),
# the strided-output A/B, the device-loop timing, ncu launch list + full captures
tag=${1:-r02d}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }

timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/${tag}_pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -3 $O/${tag}_pytest_gpu.log
for lib in default default; do
  if [ $lib = compact ]; then export EXPD_LIB=/tmp/libexpd_compact.so; else unset EXPD_LIB; fi
  timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$lib.json 2>$O/${tag}_bench_$lib.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$lib.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$lib sweep', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'])"
done
unset EXPD_LIB
timeout 300 python tools/loop_timing.py c1 c2 > $O/${tag}_loop_timing.json 2>&1; echo "loop timing exit $?"; tail -1 $O/${tag}_loop_timing.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${tag}_launches.csv $CMD > $O/${tag}_ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_time_ring" -s 2 -c 1 -o $O/${tag}_prof_k1ring $CMD > $O/${tag}_ncu_k1.log 2>&1; echo "ncu k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*bool.1" -s 20 -c 1 -o $O/${tag}_prof_colnl $CMD > $O/${tag}_ncu_colnl.log 2>&1; echo "ncu colnl exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*2048, .int.0," -s 40 -c 1 -o $O/${tag}_prof_row $CMD > $O/${tag}_ncu_row.log 2>&1; echo "ncu row exit $?"
ls -la $O | grep $tag | head -30
