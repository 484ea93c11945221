#!/bin/bash
# r02q: the ring K1 at Nt = 128 (two middle jobs per thread): parity with EXPD_K1V=5123 on the
# whole GPU suite, then c3 / c7se / c5 bench lines A/B against the default (1282 at Nt = 128)
tag=${1:-r02q}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
EXPD_K1V=5123 timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/${tag}_pytest_ring.log 2>&1; echo "pytest (K1V=5123) exit $?"; tail -3 $O/${tag}_pytest_ring.log
for cfg in c3 c7se; do for v in 1282 5123 1282 5123; do
  EXPD_K1V=$v timeout 600 python bench.py --config $cfg --no-cpu --no-e2e > $O/${tag}_${cfg}_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_${cfg}_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$cfg $v sweep', round(d['ms_per_step'],4), 'k1', round(k['k1']['launch_ms'],4), 'k1 frac', round(k['k1']['frac'],3), 'frac', round(d['roofline']['frac'],3))"
done; done
