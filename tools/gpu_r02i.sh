#!/bin/bash
# r02i: K1 L2-promotion A/B (EXPD_K1_PROMO 0 / 2 / 3) with ncu DRAM bytes of the K1 launch
tag=${1:-r02i}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for p in 3 0 2 1 3 0; do
  EXPD_K1_PROMO=$p timeout 600 python bench.py --no-cpu --no-e2e > $O/${tag}_bench_p$p.json 2>$O/${tag}_bench_p$p.err
  python -c "
import json; d=json.loads(open('$O/${tag}_bench_p$p.json').read().strip().splitlines()[-1]); k=d['kernels']
print('promo $p sweep', round(d['ms_per_step'],3), 'k1', round(k['k1']['launch_ms'],3), 's3', round(k['stage3_ms'],3), d['clocks']['sm_mhz'])"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
for p in 3 0; do
EXPD_K1_PROMO=$p timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:k_time_ring --csv --log-file $O/${tag}_k1_p$p.csv $CMD > /dev/null 2>&1; echo "ncu p$p exit $?"
done
