#!/bin/bash
# Round-2 GPU visit: build, the whole GPU suite (no -x: every failure is listed), smoke, the
# default bench line, the c3 Picard line and the c4 GMRES Arnoldi-step line.
tag=${1:-r02a}
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/${tag}_build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > $O/${tag}_pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -25 $O/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${tag}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/${tag}_smoke.log
timeout 900 python bench.py > $O/${tag}_bench.json 2> $O/${tag}_bench.err; echo "bench exit $?"; tail -c 1500 $O/${tag}_bench.json; tail -3 $O/${tag}_bench.err
timeout 600 python bench.py --config c3 --no-cpu > $O/${tag}_bench_c3.json 2> $O/${tag}_bench_c3.err; echo "bench c3 exit $?"; tail -c 600 $O/${tag}_bench_c3.json
timeout 600 python bench.py --config c4 --solver gmres --steps 3 > $O/${tag}_bench_c4gmres.json 2> $O/${tag}_bench_c4gmres.err; echo "bench c4 gmres exit $?"; tail -c 800 $O/${tag}_bench_c4gmres.json; tail -3 $O/${tag}_bench_c4gmres.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/${tag}_bench_ref.json 2>&1; echo "ref exit $?"; tail -c 600 $O/${tag}_bench_ref.json
