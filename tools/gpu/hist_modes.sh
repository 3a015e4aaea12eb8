for m in 0 1 2; do
echo "== mode $m" >> gpurun_out/hm_pytest.txt
TMB_HIST_MODE=$m timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2 >> gpurun_out/hm_pytest.txt
TMB_HIST_MODE=$m timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 3 5 9 13 17 21 25 33 49 75 --kernels histogram > gpurun_out/hm_sweep_$m.jsonl 2>&1
done
cat gpurun_out/hm_pytest.txt; for m in 0 1 2; do echo mode $m; cut -c1-110 gpurun_out/hm_sweep_$m.jsonl; done
