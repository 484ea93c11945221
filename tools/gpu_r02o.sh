#!/bin/bash
# r02o: re-tune the line-kernel variants on the current code (EXPD_COLV for the fused strided
# pass, EXPD_ROWV for the x pass)
tag=${1:-r02o}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() { local lab=$1; shift; env "$@" timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_$lab.json 2>$O/${tag}_$lab.err
  python -c "
import json; d=json.loads(open('$O/${tag}_$lab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$lab sweep', round(d['ms_per_step'],3), 's3', round(k['stage3_ms'],3), 'x', round(k['line_x']['ms_per_step'],3), 'y', round(k['line_y_nl']['ms_per_step'],3), d['clocks']['sm_mhz'])" || tail -2 $O/${tag}_$lab.err; }
run base X=1
run colv11 EXPD_COLV=11
run colv21 EXPD_COLV=21
run colv22 EXPD_COLV=22
run rowv1 EXPD_ROWV=1
run base2 X=1
run colv11b EXPD_COLV=11
