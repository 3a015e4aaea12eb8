timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/host_probe.py 2>&1 | tail -8
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_c2_r5.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_r5.json')); print(d['value'], d['e2e'], d['e2e_pinned_cabi']['value'], d['clocks'], d.get('parity'))"
