#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for v in "EXPD_ROWV=2 EXPD_COLV=11" "EXPD_ROWV=1 EXPD_COLV=12" "EXPD_ROWV=2 EXPD_COLV=21" "EXPD_ROWV=2 EXPD_COLV=22" "EXPD_ROWV=2 EXPD_COLV=41"; do
  echo "$v $(env $v timeout 120 python tools/line_micro.py c5 2>&1 | tail -1)"
done
