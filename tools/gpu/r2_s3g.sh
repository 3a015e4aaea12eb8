# ncu --set full, one launch per config (source-level counts), for profiles/ncu_*.json
for cfg in "c2 17 hist8" "c3 49 rank" "c3 75 rank" "c4 25 rank" "c4 49 rank" "c4 75 rank" "c5 9 obl" "c5 33 hist8" "c1 3 med3" "c3 3 med3" "c3 17 obl"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o gpurun_out/r2_$1_k$2 python bench.py --config $1 --k $2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_$1_k$2.log 2>&1
  echo "$cfg rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/r2_launches_c2.csv
