ncu --set full --clock-control none --import-source on -k regex:rank_kernel -s 1 -c 1 -o gpurun_out/rk16_75b python tools/one.py --bits 16 --k 75 --kernel rank --reps 2 > gpurun_out/prof_rank.log 2>&1
tail -2 gpurun_out/prof_rank.log
