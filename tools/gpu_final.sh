#!/bin/bash
# End-of-session GPU round: the whole GPU suite, smoke, the default bench line (CPU baseline and
# e2e included), the reference arm, the c3 / c4-GMRES lines, the ncu launch list of the bench
# command and --set full captures of the dominant kernels.  Usage: bash tools/gpu_final.sh <tag>
tag=${1:-final}
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/${tag}_build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > $O/${tag}_pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -16 $O/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${tag}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/${tag}_smoke.log
timeout 900 python bench.py > $O/${tag}_bench.json 2> $O/${tag}_bench.err; echo "bench exit $?"
python -c "
import json; d=json.loads(open('$O/${tag}_bench.json').read().strip().splitlines()[-1]); k=d['kernels']
print('sweep', round(d['ms_per_step'],3), 'value', d['value'], 'frac', round(d['roofline']['frac'],4), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/${tag}_bench_ref.json 2>&1; echo "ref exit $?"; tail -c 300 $O/${tag}_bench_ref.json
timeout 600 python bench.py --config c3 --no-cpu > $O/${tag}_bench_c3.json 2>&1; echo "c3 exit $?"
timeout 900 python bench.py --config c4 --solver gmres --steps 3 --no-cpu > $O/${tag}_bench_c4gmres.json 2>&1; echo "c4 gmres exit $?"
timeout 600 python bench.py --config c7se --no-cpu --steps 10 > $O/${tag}_bench_c7se.json 2>&1; echo "c7se exit $?"
timeout 300 python tools/loop_timing.py c1 c2 > $O/${tag}_loop_timing.json 2>&1
timeout 300 python tools/solve_breakdown.py c1 c2 > $O/${tag}_solve_breakdown.json 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/${tag}_launches.csv $CMD > $O/${tag}_ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_time_(ring|wp)" -s 2 -c 1 -o $O/${tag}_prof_k1 $CMD > $O/${tag}_ncu_k1.log 2>&1; echo "ncu k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*bool.1" -s 20 -c 1 -o $O/${tag}_prof_colnl $CMD > $O/${tag}_ncu_colnl.log 2>&1; echo "ncu colnl exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*2048, .int.0," -s 2 -c 1 -o $O/${tag}_prof_row $CMD > $O/${tag}_ncu_row.log 2>&1; echo "ncu row exit $?"
gzip -f $O/${tag}_prof_*.ncu-rep  # keep the copy-back under the 64 MiB limit (tools/promote_final.sh unpacks)
