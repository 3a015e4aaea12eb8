timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/rank_pytest.txt
cat gpurun_out/rank_pytest.txt
timeout 900 python tools/sweep.py --size 4096 --bits 16 32 --k 9 17 25 29 33 41 49 61 75 --kernels rank > gpurun_out/rank_sweep.jsonl 2> gpurun_out/rank_sweep.err
cut -c1-110 gpurun_out/rank_sweep.jsonl; tail -3 gpurun_out/rank_sweep.err
