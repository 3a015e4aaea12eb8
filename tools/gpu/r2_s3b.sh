# ncu full capture of the current C2 hist8 kernel (source-level counts)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist8 -s 4 -c 1 -o gpurun_out/c2_hist_s3b python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c2_s3b.log 2>&1; tail -2 gpurun_out/prof_c2_s3b.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_s3b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches_c2_s3b.csv
