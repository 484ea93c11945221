O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_line.*2048, .int.0," -s 2 -c 1 -o $O/r02final3_prof_row $CMD > $O/r02final3_ncu_row.log 2>&1; echo "ncu row exit $?"
