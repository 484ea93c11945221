#!/bin/bash
# s14: ncu of the warp-per-pair K1 (EXPD_K1V=5124) and of the ring, plus the launch list of both
tag=${1:-s14}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
for v in 0 5124; do
EXPD_K1V=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/${tag}_launches_$v.csv $CMD > $O/${tag}_ncu_launch_$v.log 2>&1; echo "ncu launches $v exit $?"
EXPD_K1V=$v timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_time_(ring|wp)" -s 2 -c 1 -o $O/${tag}_prof_k1_$v $CMD > $O/${tag}_ncu_k1_$v.log 2>&1; echo "ncu k1 $v exit $?"
done
