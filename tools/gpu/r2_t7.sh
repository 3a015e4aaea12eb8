timeout 600 python -m pytest tests -m gpu -x -q -k "hist or c2 or random_vs_oracle or golden or planes" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c2_r7.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_r7.json')); print(d['value'], d['e2e']['value'], d['clocks'])"
timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 5 9 13 15 17 19 21 23 25 --kernels histogram --reps 10 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist8 -s 4 -c 1 -o gpurun_out/c2_hist_r2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_c2.log 2>&1; tail -2 gpurun_out/prof_c2.log
