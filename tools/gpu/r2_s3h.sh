# ncu --set full, one launch per config, summarised on the box (reports are ~10 MB each)
mkdir -p gpurun_out/ncu_r2
for cfg in "c2 17 hist8 90316800" "c3 49 rank 16777216" "c3 75 rank 16777216" "c4 25 rank 67108864" "c4 49 rank 67108864" "c4 75 rank 67108864" "c5 9 obl 1073741824" "c5 33 hist8 1073741824" "c1 3 med3 262144" "c3 3 med3 16777216" "c3 17 obl 16777216" "c3 27 rank 16777216"; do
  set -- $cfg
  CMD="ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o gpurun_out/r2_$1_k$2 python bench.py --config $1 --k $2 --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/ncu_r2/$1_k$2.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2_$1_k$2.ncu-rep --samples $4 --config $1 --k $2 --source "$CMD (B200, round 2)" --out gpurun_out/ncu_r2/ncu_$1_k$2.json > /dev/null 2>&1
  ncu -i gpurun_out/r2_$1_k$2.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_r2/src_$1_k$2.csv 2>/dev/null
  gzip -f gpurun_out/ncu_r2/src_$1_k$2.csv
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('gpurun_out/ncu_r2/ncu_$1_k$2.json')); print(d['warp_instructions_per_sample'], d['issue_active_pct'], d['duration_ms_under_ncu'])" 2>&1)"
  case "$1_k$2" in c2_k17|c4_k75) ;; *) rm -f gpurun_out/r2_$1_k$2.ncu-rep ;; esac
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_r2/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/ncu_r2/launches_c2.csv
du -sh gpurun_out
