timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 2>&1 | tail -40
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant smooth gentle --reps 3 2>&1 | tee gpurun_out/patterns_4096_u16_r3.jsonl
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random gradient impulse constant narrow16 gentle --reps 3 2>&1 | tee gpurun_out/patterns_8192_u32_r3.jsonl
