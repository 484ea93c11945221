#!/bin/bash
# r02p: physical <-> spectral x pass through re-pitch + TMA row pass: GPU suite, the S-lit
# comparison (precond_apply with physical I/O), small-solve breakdown and e2e, A/B against
# EXPD_PHYS_ROWS=1 (the k_rows path)
tag=${1:-r02p}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/${tag}_pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -3 $O/${tag}_pytest_gpu.log
for v in 0 1; do
  EXPD_PHYS_ROWS=$v timeout 600 python tools/slit_compare.py c3 c5 > $O/${tag}_slit_$v.json 2>/dev/null; echo "slit $v exit $?"
  EXPD_PHYS_ROWS=$v timeout 300 python tools/solve_breakdown.py c1 c2 > $O/${tag}_solve_breakdown_$v.json 2>&1
  EXPD_PHYS_ROWS=$v timeout 900 python bench.py --no-cpu > $O/${tag}_bench_$v.json 2> $O/${tag}_bench_$v.err; echo "bench $v exit $?"
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$v.json').read().strip().splitlines()[-1])
s=json.loads(open('$O/${tag}_slit_$v.json').read())
print('$v sweep', round(d['ms_per_step'],3), 'e2e', d['e2e']['value'], 'spec_apply', {k: round(v['s_spec_precond_apply_ms'],3) for k,v in s.items()}, 'lit', {k: round(v['s_lit_ms']['total'],3) for k,v in s.items()})"
  cat $O/${tag}_solve_breakdown_$v.json
done
