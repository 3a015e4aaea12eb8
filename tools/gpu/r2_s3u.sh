# rank: one row pointer per fetch + compile-time key modes
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread -k "rank or c3 or c4 or golden or random_vs_oracle or ties or bands or multi or fuzz or rect" 2>&1 | grep -v "^\.\+$" | tail -2
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse gentle --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random impulse gentle --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
timeout 400 python tools/fuzz_rank.py --seconds 120 --seed 3 2>&1 | tail -2
