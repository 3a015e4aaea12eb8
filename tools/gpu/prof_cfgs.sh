set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__cycles_elapsed.avg,launch__registers_per_thread,launch__grid_size
for cfg in "c3 49 rank" "c3 75 rank" "c4 25 rank" "c4 49 rank" "c4 75 rank" "c1 3 med3" "c3 3 med3"; do
  set -- $cfg
  ncu --metrics $M --clock-control none -k regex:$3 -s 3 -c 1 --csv python bench.py --config $1 --k $2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$1_k$2.csv 2>/dev/null
done
ls -la gpurun_out/ncu_*.csv
