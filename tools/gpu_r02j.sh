#!/bin/bash
tag=${1:-r02j}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/${tag}_pytest.log
timeout 900 python bench.py --no-cpu > $O/${tag}_bench.json 2>$O/${tag}_bench.err; echo "bench exit $?"
python -c "
import json; d=json.loads(open('$O/${tag}_bench.json').read().strip().splitlines()[-1]); k=d['kernels']
print('sweep', round(d['ms_per_step'],3), 'value', d['value'], 'frac', round(d['roofline']['frac'],4), 'e2e', d['e2e'])" || tail -5 $O/${tag}_bench.err
timeout 300 python tools/solve_breakdown.py c1 c2 > $O/${tag}_solve_breakdown.json 2>&1; tail -1 $O/${tag}_solve_breakdown.json
