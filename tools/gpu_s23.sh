#!/bin/bash
# s23: warp-per-pair K1 with the Û tile kept intact (scratch in the N̂ tile + a pad area, two group
# barriers, u_t re-read): parity, A/B against the ring (EXPD_K1V=5123), ncu
tag=${1:-s23}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -m gpu -x -k "fixed_point_parity or residual_parity or device_loop or k1_nt256 or 256" -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/${tag}_pytest.log
for v in 5123 0 5123 0; do
  EXPD_K1V=$v timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>$O/${tag}_c5_$v.err
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('K1V=$v: sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), 'resid', d.get('residual_norm_last'), d['clocks']['sm_mhz'])" || tail -5 $O/${tag}_c5_$v.err
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_time_wp" -s 2 -c 1 -o $O/${tag}_prof_k1 $CMD > $O/${tag}_ncu_k1.log 2>&1; echo "ncu k1 exit $?"
