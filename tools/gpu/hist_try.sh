timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/hist_pytest.txt
timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 3 5 7 9 11 13 15 17 19 21 25 31 33 41 49 61 75 --kernels histogram > gpurun_out/hist_sweep.jsonl 2> gpurun_out/hist_sweep.err
cat gpurun_out/hist_pytest.txt; cut -c1-120 gpurun_out/hist_sweep.jsonl; tail -3 gpurun_out/hist_sweep.err
