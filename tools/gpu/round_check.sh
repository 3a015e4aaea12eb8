timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; cut -c1-250 gpurun_out/rc_bench.json; python -c "
import json; d=json.load(open('gpurun_out/rc_bench.json')); print('issue', d.get('roofline_issue')); print('traffic', d['roofline']['traffic'], 'cpu', d['cpu_baseline']['value'], 'clocks', d['clocks'])"
