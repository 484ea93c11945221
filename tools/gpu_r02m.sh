#!/bin/bash
# r02m: K1 ring release by mbarrier (default) vs named barrier (-DEXPD_K1_RELEASE_BAR), promo A/B
tag=${1:-r02m}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
bash tools/build_variant.sh k_time_n256.cu /tmp/libexpd_k1bar.so -DEXPD_K1_RELEASE_BAR > $O/${tag}_variant.log 2>&1 || echo VARIANT FAILED
for v in mbar bar mbar bar; do
  if [ $v = bar ]; then export EXPD_LIB=/tmp/libexpd_k1bar.so; else unset EXPD_LIB; fi
  timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_$v.json 2>$O/${tag}_bench_$v.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_$v.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), d['clocks']['sm_mhz'])" || tail -3 $O/${tag}_bench_$v.err
done
unset EXPD_LIB
for p in 0 3; do EXPD_K1_PROMO=$p timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_p$p.json 2>&1; python -c "
import json; d=json.loads(open('$O/${tag}_bench_p$p.json').read().strip().splitlines()[-1]); k=d['kernels']
print('promo $p sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), d['clocks']['sm_mhz'])"; done
