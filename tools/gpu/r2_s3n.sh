# hist8: select-chain walk packing + incremental ring pointers
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or planes or c2 or c5 or golden or random_vs_oracle or edge or strided or tall or rank" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C2', round(d['value'],2), d['clocks']['sm_mhz'])"
done
timeout 300 python tools/sweep.py --size 4096 --bits 8 --k 15 17 21 25 33 49 75 --kernels histogram --reps 10 2>&1 | python -c "
import sys,json
print([ (d['k'], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
