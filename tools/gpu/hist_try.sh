set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/hist_pytest.txt
timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 3 5 7 9 11 13 15 17 19 21 25 31 33 41 49 61 75 --kernels histogram oblivious > gpurun_out/hist_sweep.jsonl 2> gpurun_out/hist_sweep.err
cat gpurun_out/hist_pytest.txt gpurun_out/hist_sweep.jsonl
