#!/bin/bash
# Build an A/B variant of libexpd.so: recompile ONE source with extra flags and relink with the
# default objects.  Usage: bash tools/build_variant.sh <source.cu> <out.so> <nvcc flags...>
# (run after the default build; load it with EXPD_LIB=<out.so>)
src=$1; out=$2; shift 2
B=paper_2603_04350_b200/_build
flags=$(head -1 $B/$(basename $src).o.log | sed 's/ -c .*//' | cut -d' ' -f2-)
mkdir -p /tmp/expd_variant
nvcc $flags "$@" -c paper_2603_04350_b200/csrc/$src -o /tmp/expd_variant/$src.o || exit 1
objs=$(ls $B/*.o | grep -v "/$src.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out $objs /tmp/expd_variant/$src.o -lcudart -ldl && echo "built $out"
