# round-2 bench lines (every config, fresh process each), reference arm, k sweep (L2 flushed, clocked)
mkdir -p gpurun_out/r2b
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b/bench_c2_k17.json 2> gpurun_out/r2b/bench_c2_k17.err
for cfg in "c1 3" "c3 3" "c3 17" "c3 27" "c3 49" "c3 75" "c4 25" "c4 49" "c4 75" "c5 9" "c5 33"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --k $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b/bench_$1_k$2.json 2> gpurun_out/r2b/bench_$1_k$2.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b/bench_reference_c2.json 2>&1
for f in gpurun_out/r2b/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
c=d.get('config',{}); r=d.get('roofline') or {}
print('$f'.split('/')[-1], c.get('kernel'), round(d['value'],3), 'ms', round(d['ms_per_step'],3), 'e2e', round((d.get('e2e') or {}).get('value',0) or 0,2), r.get('bound'), round(r.get('frac') or 0,3), d.get('clocks',{}).get('sm_mhz'), d.get('parity'))
" 2>&1 | tail -1; done
KS="3 5 7 9 11 13 15 17 19 21 23 25 27 29 31 33 35 37 39 41 43 45 47 49 51 53 55 57 59 61 63 65 67 69 71 73 75"
timeout 1500 python tools/sweep.py --size 4096 --bits 8 16 32 --k $KS --variants auto --reps 10 > gpurun_out/r2b/sweep_4096_auto.jsonl 2> gpurun_out/r2b/sweep.err; wc -l gpurun_out/r2b/sweep_4096_auto.jsonl
