#!/bin/bash
# Copy one GPU round of tools/gpu_final.sh (gpurun_out/<tag>_*) into profiles/r02/*_final* and
# rebuild the summaries (ncu --set full summaries, launch shares, profiles/ncu_traffic.json).
# Usage: bash tools/promote_final.sh <tag>
tag=$1; O=gpurun_out; P=profiles/r02
set -e
for f in $O/${tag}_prof_*.ncu-rep.gz; do [ -e "$f" ] && gunzip -kf "$f"; done
tail -1 $O/${tag}_bench.json > $P/bench_final.json
tail -1 $O/${tag}_bench_ref.json > $P/bench_reference_final.json
tail -1 $O/${tag}_bench_c3.json > $P/bench_final_c3.json
tail -1 $O/${tag}_bench_c4gmres.json > $P/bench_final_c4_gmres.json
tail -1 $O/${tag}_bench_c7se.json > $P/bench_final_c7se.json
cp $O/${tag}_pytest_gpu.log $P/pytest_gpu_final.log
cp $O/${tag}_smoke.log $P/smoke_final.log
tail -1 $O/${tag}_loop_timing.json > $P/loop_timing_final.json
tail -1 $O/${tag}_solve_breakdown.json > $P/solve_breakdown_final.json
python tools/ncu_summary.py $O/${tag}_prof_k1.ncu-rep > $P/ncu_full_final_k1.txt
python tools/ncu_summary.py $O/${tag}_prof_colnl.ncu-rep > $P/ncu_full_final_colnl.txt
python tools/ncu_summary.py $O/${tag}_prof_row.ncu-rep > $P/ncu_full_final_row.txt
cp $O/${tag}_launches.csv $P/ncu_launches_final.csv
python tools/launch_shares.py $O/${tag}_launches.csv > $P/ncu_launch_shares_final.txt
python tools/update_traffic.py $tag
echo promoted $tag
