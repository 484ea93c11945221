#!/bin/bash
# s9: the transposed strided-axis store (k_line TS, default) -- GPU parity of the line / stage-3 /
# sweep tests, then the c5 / c3 sweeps A/B against the compacted layout (EXPD_COLTS=0)
tag=${1:-s9}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/${tag}_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -q -m gpu -x -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/${tag}_pytest.log
for v in 1 0 1 0; do
  EXPD_COLTS=$v timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c5_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('c5 TS=$v sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), {x: (round(y['launch_ms'],3) if isinstance(y, dict) and 'launch_ms' in y else None) for x, y in k.items()}, d['clocks']['sm_mhz'])"
done
for v in 1 0; do
  EXPD_COLTS=$v timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/${tag}_c3_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c3_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('c3 TS=$v sweep', round(d['ms_per_step'],4), 's3', round(k['stage3_ms'],4))"
done
