# final round-2 check: full GPU suite, smoke, default bench, reference arm
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread 2>&1 | grep -v "^\.\+$" | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; python -c "
import json; d=json.load(open('gpurun_out/final_bench.json')); print('C2', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'pageable', round(d['e2e_pageable']['value'],2), 'issue', round(d['roofline']['frac'],3), 'traffic', d['roofline']['traffic'], 'launches', d['gpu_launches'], d['parity'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2>&1; tail -c 400 gpurun_out/final_ref.json
