ncu --set full --clock-control none --import-source on -k regex:hist8 -s 4 -c 1 -o gpurun_out/c2_hist python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg --clock-control none -k regex:hist8 -s 4 -c 2 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_metrics.csv 2>/dev/null
tail -3 gpurun_out/prof_c2.log
