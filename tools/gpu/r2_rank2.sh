timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python tools/patterns.py --size 1024 --bits 16 32 --k 27 49 75 --patterns random gradient impulse constant narrow16 smooth gentle --reps 3 --check 4 2>&1 | tee gpurun_out/patterns_1024_r2.jsonl
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant smooth gentle --reps 3 --check 3 2>&1 | tee gpurun_out/patterns_4096_u16_r2.jsonl
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random gradient impulse constant narrow16 gentle --reps 3 --check 2 2>&1 | tee gpurun_out/patterns_8192_u32_r2.jsonl
