for v in base S; do
  cp variants/lib_$v.so paper_2507_19926_b200/libtilemedian_b200.so
  echo "$v: $(timeout 600 python tools/sweep.py --size 4096 --bits 16 32 --k 15 17 19 21 23 25 27 --kernels oblivious --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d/%d:%.1f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))")"
done
