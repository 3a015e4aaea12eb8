ncu --set full --clock-control none --import-source on -k regex:hist8 -s 1 -c 1 -o gpurun_out/h3_17 python tools/one.py --bits 8 --k 17 --kernel histogram --reps 2 > gpurun_out/prof_hist.log 2>&1
tail -2 gpurun_out/prof_hist.log
