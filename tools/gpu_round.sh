#!/bin/bash
# One GPU visit: parity tests, bench, per-kernel micro timings, ncu launch list and a
# full ncu capture of the top kernels.  Usage: bash tools/gpu_round.sh <tag>
tag=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/${tag}_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > $O/${tag}_pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -3 $O/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${tag}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/${tag}_smoke.log
timeout 600 python bench.py > $O/${tag}_bench.json 2> $O/${tag}_bench.err; echo "bench exit $?"; tail -c 3000 $O/${tag}_bench.json
timeout 300 python tools/kernel_micro.py c5 > $O/${tag}_micro.json 2>&1; echo "micro exit $?"; cat $O/${tag}_micro.json | tail -3
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > $O/${tag}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${tag}_launches.csv $CMD > $O/${tag}_ncu_launch.log 2>&1
echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_time' -s 0 -c 1 -o $O/${tag}_prof_k1 $CMD > $O/${tag}_ncu_full_k1.log 2>&1
echo "ncu full k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_rows|k_cols' -s 4 -c 3 -o $O/${tag}_prof_dst $CMD > $O/${tag}_ncu_full_dst.log 2>&1
echo "ncu full dst exit $?"
ls -la $O
