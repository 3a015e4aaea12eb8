# full suite + ncu refresh for the hist8 configs + their bench lines
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread 2>&1 | grep -v "^\.\+$" | tail -3
mkdir -p gpurun_out/ncu_r2c gpurun_out/r2d
for cfg in "c2 17 hist8 90316800" "c5 33 hist8 1073741824"; do
  set -- $cfg
  CMD="ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o gpurun_out/r2c_$1_k$2 python bench.py --config $1 --k $2 --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/ncu_r2c/$1_k$2.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2c_$1_k$2.ncu-rep --samples $4 --config $1 --k $2 --source "$CMD (B200, round 2, final kernels)" --out gpurun_out/ncu_r2c/ncu_$1_k$2.json > /dev/null 2>&1
  python tools/ncu_lines.py gpurun_out/r2c_$1_k$2.ncu-rep --top 40 > gpurun_out/ncu_r2c/lines_$1_k$2.txt 2>&1
  echo "$cfg $(python -c "import json; d=json.load(open('gpurun_out/ncu_r2c/ncu_$1_k$2.json')); print(d['warp_instructions_per_sample'], d['issue_active_pct'], d['dram_read_mb'], d['dram_write_mb'])" 2>&1)"
  rm -f gpurun_out/r2c_$1_k$2.ncu-rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_r2c/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cp gpurun_out/ncu_r2c/ncu_*.json profiles/
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d/bench_c2_k17.json 2> gpurun_out/r2d/bench_c2_k17.err
timeout 600 python bench.py --config c5 --k 33 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d/bench_c5_k33.json 2> gpurun_out/r2d/bench_c5_k33.err
timeout 600 python bench.py --config c5 --k 9 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d/bench_c5_k9.json 2> gpurun_out/r2d/bench_c5_k9.err
for f in gpurun_out/r2d/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
c=d.get('config',{}); r=d.get('roofline') or {}
print('$f'.split('/')[-1], c.get('kernel'), round(d['value'],3), 'ms', round(d['ms_per_step'],3), 'e2e', round((d.get('e2e') or {}).get('value',0) or 0,2), r.get('bound'), round(r.get('frac') or 0,3), r.get('traffic'), d.get('clocks',{}).get('sm_mhz'), d.get('parity'))
" 2>&1 | tail -1; done
