#!/bin/bash
# One compute-sanitizer tool per call (the profiling guide: several tools in one call once left
# the GPU unusable).  Usage: bash tools/gpu_sanitize.sh <memcheck|racecheck|synccheck|initcheck> <tag> [cases]
tool=$1; tag=${2:-r02}; shift 2
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
extra=""
[ "$tool" = "memcheck" ] && extra="--leak-check full"
timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
  python tools/sanitize_case.py "$@" > $O/${tag}_sanitize_${tool}.log 2>&1
echo "sanitize $tool exit $?"; tail -15 $O/${tag}_sanitize_${tool}.log
