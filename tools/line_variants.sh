#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for lib in paper_2603_04350_b200/libexpd.so tools/libexpd_twseq.so; do
  for v in "EXPD_ROWV=2 EXPD_COLV=11" "EXPD_ROWV=1 EXPD_COLV=11" "EXPD_ROWV=1 EXPD_COLV=12"; do
    echo "$lib $v $(env EXPD_LIB=$lib $v timeout 120 python tools/line_micro.py c5 2>&1 | tail -1) $(env EXPD_LIB=$lib $v timeout 120 python tools/line_debug.py 2 2047 nl 2>&1 | tail -1)"
  done
done
