for v in base H4; do
  cp variants/lib_$v.so paper_2507_19926_b200/libtilemedian_b200.so
  echo "$v: $(timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 15 17 19 21 --kernels histogram --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d:%.1f'%(d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))") C2: $(timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],2))")"
done
