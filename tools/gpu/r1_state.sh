nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/st_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/st_bench.json 2> gpurun_out/st_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/st_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/st_pytest.txt gpurun_out/st_bench.json; tail -3 gpurun_out/st_bench.err
