# round-2 session-3 state check: gpu tests, smoke, C2 bench, rank data sensitivity
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt.txt 2>&1; tail -3 gpurun_out/pt.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -c 600 gpurun_out/b_c2.json
python -c "
import json; d=json.load(open('gpurun_out/b_c2.json')); print('C2', round(d['value'],2), 'e2e', d['e2e']['value'], 'pinned', d['e2e_pinned_cabi']['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks'], d.get('parity'))"
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant gentle smooth --reps 3 2>&1 | tee gpurun_out/patterns_4096_u16.jsonl | cut -c1-200
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random gradient impulse constant narrow16 gentle --reps 3 2>&1 | tee gpurun_out/patterns_8192_u32.jsonl | cut -c1-200
