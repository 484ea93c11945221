#!/bin/bash
# line kernels: correctness at several sizes + c5 micro timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for a in "2 255 nl" "2 511 nl" "2 2047 nl" "3 255 nl" "2 2047 dst" "3 255 dst"; do timeout 120 python tools/line_debug.py $a 2>&1 | tail -1; done
timeout 120 python tools/line_micro.py c5 2>&1 | tail -1
EXPD_COLV=11 timeout 120 python tools/line_micro.py c5 2>&1 | tail -1
