#!/bin/bash
# r02v: the ring K1 on two-stage plans (Nt = 16 / 32 / 64; EXPD_K1V=5123 forces it): parity of
# the GPU suite with it forced, then c4 GMRES steps and c2 sweeps against the 256-thread TMA kernel
tag=${1:-r02v}
O=gpurun_out; mkdir -p $O
EXPD_K1V=5123 timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/${tag}_pytest_ring.log 2>&1; echo "pytest (K1V=5123) exit $?"; tail -2 $O/${tag}_pytest_ring.log
for v in 2562 5123 2562 5123; do
  EXPD_K1V=$v timeout 900 python bench.py --config c4 --solver gmres --steps 3 --no-cpu > $O/${tag}_c4_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c4_$v.json').read().strip().splitlines()[-1])
print('c4 gmres $v ms/step', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'steps', [round(x,3) for x in d['roofline']['step_ms']])"
  EXPD_K1V=$v timeout 600 python bench.py --config c2 --no-cpu --no-e2e > $O/${tag}_c2_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/${tag}_c2_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('c2 $v sweep', round(d['ms_per_step'],4), 'k1', round(k['k1']['launch_ms'],4), 'k1 frac', round(k['k1']['frac'],3))"
done
