#!/bin/bash
# registers / spills of every kernel in one compiled object's ptxas log
grep -A3 "Compiling entry" paper_2603_04350_b200/_build/$1.o.log | grep -E "registers|spill|Compiling" | paste - - - | sed 's/ptxas info    : //g;s/Compiling entry function .._ZN4expd//;s/EEEv14CUtensorMap_stS1_NS_8LineArgsE. for .sm_100a.//;s/ bytes cumulative stack size//' | cut -c1-180
