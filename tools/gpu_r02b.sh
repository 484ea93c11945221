tag=r02b
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "nonlin or dst or sweep or fixed_point or fullsize or smoke" -p no:cacheprovider > $O/${tag}_pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/${tag}_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench.json 2>$O/${tag}_bench.err; echo "bench exit $?"
python -c "
import json; d=json.loads(open('$O/${tag}_bench.json').read().strip().splitlines()[-1]); k=d['kernels']
print('sweep', d['ms_per_step'], 'frac', d['roofline']['frac'], 'k1', k['k1']['launch_ms'], 's3', k['stage3_ms'], 'x', k['line_x']['ms_per_step'], 'y', k['line_y_nl']['ms_per_step'])"
bash tools/gpu_sanitize.sh racecheck $tag c5s c5big c3s
