# hist8 tuning: ring group G (2/4/8) and walk window S (6/8/12), C2 + 4096 u8 sweep
for v in "" g2 g8 s6 s12; do
  if [ -n "$v" ]; then export TMB_LIB=paper_2507_19926_b200/libtilemedian_b200_$v.so; else unset TMB_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_c2_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b_c2_$v.json').read().strip().splitlines()[-1]); print('$v C2', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'])"
  timeout 300 python tools/sweep.py --size 4096 --bits 8 --k 15 17 21 25 33 49 75 --kernels histogram --reps 10 2>&1 | python -c "
import sys,json
print('$v', [ (d['k'], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
done
