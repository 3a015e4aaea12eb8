timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c2_r8.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_r8.json')); print('C2', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
TMB_LIB=paper_2507_19926_b200/libtilemedian_b200_prof.so timeout 600 python tools/rank_prof.py 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rank_kernel -c 1 -o gpurun_out/c3_rank49_r2 python tools/one.py --bits 16 --k 49 --kernel rank --size 4096 --reps 1 > gpurun_out/prof_c3.log 2>&1; tail -1 gpurun_out/prof_c3.log
