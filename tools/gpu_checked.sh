#!/bin/bash
# The GPU suite on the bounds-checked library (-DEXPD_CHECKS: device-side EXPD_CHECK asserts on
# shared-memory positions, TMA item coordinates, K1 store indices, the re-pitch rows; a failed
# check prints and traps), in place of compute-sanitizer, which this pool does not allow.
tag=${1:-checked}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -m paper_2603_04350_b200.build --checked >> $O/${tag}_build.log 2>&1 || { echo CHECKED BUILD FAILED; exit 1; }
EXPD_LIB=$PWD/paper_2603_04350_b200/libexpd_checked.so python -c "
import os
from paper_2603_04350_b200 import expd
expd.load_library()
print('loaded:', [l.split()[-1] for l in open('/proc/self/maps') if 'libexpd' in l][:1])" > $O/${tag}_which_lib.txt 2>&1; cat $O/${tag}_which_lib.txt
EXPD_LIB=$PWD/paper_2603_04350_b200/libexpd_checked.so timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider \
  > $O/${tag}_pytest_checked.log 2>&1; echo "pytest (checked library) exit $?"; tail -3 $O/${tag}_pytest_checked.log
grep -c "expd check failed" $O/${tag}_pytest_checked.log
EXPD_LIB=$PWD/paper_2603_04350_b200/libexpd_checked.so timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/${tag}_bench_checked.json 2>&1; echo "bench (checked) exit $?"
