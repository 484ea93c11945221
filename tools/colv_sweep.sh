#!/bin/bash
# correctness + micro timing of the strided-axis line-kernel variants (EXPD_COLV)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for v in ${COLVS:-12 22 11 21 41}; do
  for a in "2 2047 nl" "2 255 nl" "3 255 nl"; do EXPD_COLV=$v timeout 120 python tools/line_debug.py $a 2>&1 | grep -v "^  \|^$" | tail -1 | sed "s/^/v$v /"; done
  EXPD_COLV=$v timeout 200 python tools/kernel_micro.py c5 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v', {k: (round(v*1e3,1) if isinstance(v,float) else v) for k,v in d.items() if 'line' in k})"
done
