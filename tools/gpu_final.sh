#!/bin/bash
# End-of-round GPU visit: full parity suite, smoke, default bench (with e2e and the CPU
# baseline), the reference arm, the complex bench lines and every config's solve report.
tag=${1:-r01f}
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/${tag}_build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > $O/${tag}_pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -3 $O/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${tag}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/${tag}_smoke.log
timeout 900 python bench.py > $O/${tag}_bench.json 2> $O/${tag}_bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${tag}_bench_ref.json 2> $O/${tag}_bench_ref.err; echo "bench ref exit $?"
for c in c7se c7bdf2 c4; do timeout 600 python bench.py --config $c --no-cpu > $O/${tag}_bench_$c.json 2> $O/${tag}_bench_$c.err; echo "bench $c exit $?"; done
timeout 1200 python tools/configs_report.py > $O/${tag}_configs.jsonl 2> $O/${tag}_configs.err; echo "configs exit $?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/*_bench*.json")):
    if "r01f" not in f: continue
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d.get("ms_per_step"), "%.3g" % d["value"], (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("clocks", {}).get("sm_mhz") if isinstance(d.get("clocks"), dict) else None)
    except Exception as e:
        print(f, "ERR", e)
PY
