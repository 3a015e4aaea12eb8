timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c2_r6.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_r6.json')); print(d['value'], d['e2e']['value'], d['e2e_pinned_cabi']['value'], d['clocks'])"
timeout 600 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient --reps 3 2>&1
timeout 600 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random --reps 3 2>&1
timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 15 17 25 33 49 75 --reps 10 2>&1
