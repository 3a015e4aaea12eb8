# all-kernel fuzz, then ncu + bench lines + patterns for the rank configs (kernel changed)
timeout 400 python tools/fuzz_rank.py --seconds 240 --seed 11 --all-kernels 2>&1 | tail -3
mkdir -p gpurun_out/ncu_r2d gpurun_out/r2e
for cfg in "c3 27 rank 16777216" "c3 49 rank 16777216" "c3 75 rank 16777216" "c4 25 rank 67108864" "c4 49 rank 67108864" "c4 75 rank 67108864"; do
  set -- $cfg
  CMD="ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o gpurun_out/r2d_$1_k$2 python bench.py --config $1 --k $2 --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/ncu_r2d/$1_k$2.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2d_$1_k$2.ncu-rep --samples $4 --config $1 --k $2 --source "$CMD (B200, round 2, final kernels)" --out gpurun_out/ncu_r2d/ncu_$1_k$2.json > /dev/null 2>&1
  python tools/ncu_lines.py gpurun_out/r2d_$1_k$2.ncu-rep --top 40 > gpurun_out/ncu_r2d/lines_$1_k$2.txt 2>&1
  echo "$cfg $(python -c "import json; d=json.load(open('gpurun_out/ncu_r2d/ncu_$1_k$2.json')); print(d['warp_instructions_per_sample'], d['issue_active_pct'], d['duration_ms_under_ncu'])" 2>&1)"
  rm -f gpurun_out/r2d_$1_k$2.ncu-rep
done
cp gpurun_out/ncu_r2d/ncu_*.json profiles/
for cfg in "c3 27" "c3 49" "c3 75" "c4 25" "c4 49" "c4 75"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --k $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e/bench_$1_k$2.json 2> gpurun_out/r2e/bench_$1_k$2.err
done
for f in gpurun_out/r2e/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
c=d.get('config',{}); r=d.get('roofline') or {}
print('$f'.split('/')[-1], c.get('kernel'), round(d['value'],3), 'ms', round(d['ms_per_step'],3), 'e2e', round((d.get('e2e') or {}).get('value',0) or 0,2), r.get('bound'), round(r.get('frac') or 0,3), d.get('clocks',{}).get('sm_mhz'))
" 2>&1 | tail -1; done
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant gentle smooth --reps 3 > gpurun_out/r2e/patterns_c3_u16_4096.jsonl 2>&1
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random gradient impulse constant narrow16 gentle --reps 3 > gpurun_out/r2e/patterns_c4_u32_8192.jsonl 2>&1
KS="23 25 27 29 31 33 35 37 39 41 43 45 47 49 51 53 55 57 59 61 63 65 67 69 71 73 75"
timeout 1200 python tools/sweep.py --size 4096 --bits 16 32 --k $KS --variants auto --reps 10 > gpurun_out/r2e/sweep_4096_rank.jsonl 2> gpurun_out/r2e/sweep.err; wc -l gpurun_out/r2e/sweep_4096_rank.jsonl
