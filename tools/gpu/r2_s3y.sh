for v in "" r176 "" r176; do
  if [ -n "$v" ]; then export TMB_LIB=paper_2507_19926_b200/libtilemedian_b200_$v.so; else unset TMB_LIB; fi
  timeout 600 python tools/patterns.py --size 4096 --bits 16 --k 49 75 --patterns random gentle impulse --reps 5 2>&1 | python -c "
import sys,json
print('$v', [(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
  timeout 600 python tools/patterns.py --size 8192 --bits 32 --k 49 75 --patterns random --reps 3 2>&1 | python -c "
import sys,json
print('$v', [(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
done
