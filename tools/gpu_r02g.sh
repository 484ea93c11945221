#!/bin/bash
# r02g: the persistent stage 3 (k_stage3p): parity, A/B against the chunked passes (EXPD_S3P=0),
# ring size / role split sweeps, ncu DRAM traffic of the persistent launch; solve breakdown c1/c2
tag=${1:-r02g}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "sweep or fixed_point or c5_full or max_line or c3 or device_loop or smoke or fuzz_picard" > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/${tag}_pytest.log
run() {  # label, env...
  local lab=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$lab.json 2>$O/${tag}_bench_$lab.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$lab.json').read().strip().splitlines()[-1]); k=d['kernels']
fam={n: round(k[n]['ms_per_step'],3) for n in ('line_x','line_y_nl','stage3_persistent') if n in k}
print('$lab sweep', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), fam, d['clocks']['sm_mhz'])" || tail -3 $O/${tag}_bench_$lab.err
}
run chunked EXPD_S3P=0
run s3p EXPD_S3P=1
run s3p_k3 EXPD_S3P_K=3
run s3p_k6 EXPD_S3P_K=6
run s3p_32_84 EXPD_S3P_SPLIT=32,84
run s3p_38_72 EXPD_S3P_SPLIT=38,72
run chunked2 EXPD_S3P=0
run s3p2 EXPD_S3P=1
timeout 300 python tools/solve_breakdown.py c1 c2 > $O/${tag}_solve_breakdown.json 2>&1; echo "breakdown exit $?"; tail -1 $O/${tag}_solve_breakdown.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_stage3p" -s 2 -c 1 -o $O/${tag}_prof_s3p $CMD > $O/${tag}_ncu_s3p.log 2>&1; echo "ncu s3p exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/${tag}_launches.csv $CMD > $O/${tag}_ncu_launch.log 2>&1; echo "ncu launches exit $?"
