mkdir -p gpurun_out/r2f
for cfg in "c1 3" "c3 3" "c3 17"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --k $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f/bench_$1_k$2.json 2> gpurun_out/r2f/bench_$1_k$2.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f/bench_reference_c2.json 2>&1
tail -c 300 gpurun_out/r2f/bench_c1_k3.json
