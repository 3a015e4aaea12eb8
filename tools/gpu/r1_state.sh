set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1s2_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r1s2_bench.json 2> gpurun_out/r1s2_bench.err
timeout 900 python tools/sweep.py --size 4096 --bits 8 16 32 --k 3 5 7 9 11 13 15 17 19 21 23 25 27 29 31 33 41 49 61 75 --variants auto oblivious aware > gpurun_out/r1s2_sweep.jsonl 2> gpurun_out/r1s2_sweep.err
cat gpurun_out/r1s2_pytest.txt gpurun_out/r1s2_bench.json
