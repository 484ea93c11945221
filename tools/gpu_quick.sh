#!/bin/bash
# quick GPU visit: build, parity tests (optionally filtered), kernel micro timings, bench
tag=${1:-q}; filt=${2:-}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/${tag}_build.log; exit 1; }
if [ -n "$filt" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$filt" > $O/${tag}_pytest.log 2>&1; else timeout 1200 python -m pytest tests -x -q -m gpu > $O/${tag}_pytest.log 2>&1; fi
echo "pytest exit $?"; tail -15 $O/${tag}_pytest.log
timeout 300 python tools/kernel_micro.py c5 > $O/${tag}_micro.json 2>&1; echo "micro exit $?"; cat $O/${tag}_micro.json | tail -3
timeout 600 python bench.py --no-cpu > $O/${tag}_bench.json 2> $O/${tag}_bench.err; echo "bench exit $?"; cat $O/${tag}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels'], d['roofline']['frac'], d['e2e'])" 2>&1 | tail -3; tail -3 $O/${tag}_bench.err
