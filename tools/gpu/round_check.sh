timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; python -c "
import json; d=json.load(open('gpurun_out/rc_bench.json')); print('C2', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3), 'issue', round(d['roofline_issue']['frac'],3), 'launches', d['gpu_launches'], 'clk', d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | cut -c1-200
