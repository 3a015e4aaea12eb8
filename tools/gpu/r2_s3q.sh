# rank work-list fix: the former hang, every rect case, full suite (thread timeouts), patterns
timeout 60 python tools/dbg_rect2.py 32,25,127,157,301 2>&1 | tail -1
timeout 300 python tools/dbg_rect.py 2>&1 | grep -c " ok"
timeout 300 python tools/dbg_rect.py 2>&1 | grep -v " ok" | tail -3
timeout 1500 python -m pytest tests -m gpu -q --timeout 120 --timeout-method thread 2>&1 | grep -v "^\.\+$" | tail -8
timeout 900 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant gentle --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
timeout 900 python tools/patterns.py --size 8192 --bits 32 --k 25 49 75 --patterns random impulse narrow16 gentle --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
