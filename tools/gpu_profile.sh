#!/bin/bash
# One profiling visit: plain bench, ncu launch list of the same command, and full ncu
# captures (one launch each) of K1 and the two stage-3 line-kernel families.
tag=${1:-r01}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > $O/${tag}_plain.json 2> $O/${tag}_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${tag}_launches.csv $CMD > $O/${tag}_ncu_launch.log 2>&1
echo "launch list exit $?"
timeout 300 $CMD > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_time_tma" -s 2 -c 1 -o $O/${tag}_prof_k1 $CMD > $O/${tag}_ncu_k1.log 2>&1
echo "k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*2048, .int.0," -s 40 -c 1 -o $O/${tag}_prof_row $CMD > $O/${tag}_ncu_row.log 2>&1
echo "row exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*bool.1" -s 20 -c 1 -o $O/${tag}_prof_colnl $CMD > $O/${tag}_ncu_colnl.log 2>&1
echo "colnl exit $?"
ls -la $O | grep $tag
