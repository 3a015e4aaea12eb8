set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -2
timeout 600 python tools/patterns.py --size 1024 --bits 16 32 --k 27 49 75 --patterns random gradient impulse constant narrow16 smooth --reps 3 2>&1 | tee gpurun_out/patterns_1024_r0.jsonl
