timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant gentle --reps 3 2>&1 | tee gpurun_out/patterns_4096_u16_r4.jsonl
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random gradient impulse constant narrow16 gentle --reps 3 2>&1 | tee gpurun_out/patterns_8192_u32_r4.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c2_r4.json
cat gpurun_out/bench_c2_r4.json
