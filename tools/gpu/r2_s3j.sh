# rank: interleaved emit + warp-aggregated place (product) vs emit-only (remit) vs round-start (rold)
timeout 900 python -m pytest tests -m gpu -x -q -k "rank or c3 or c4 or golden or random_vs_oracle or ties or bands or multi" 2>&1 | tail -2
for v in "" remit rold; do
  if [ -n "$v" ]; then export TMB_LIB=paper_2507_19926_b200/libtilemedian_b200_$v.so; else unset TMB_LIB; fi
  echo "== $v"
  timeout 600 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse gentle --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
  timeout 600 python tools/patterns.py --size 8192 --bits 32 --k 25 75 --patterns random impulse gentle --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
done
