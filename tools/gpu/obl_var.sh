for v in base P Q; do
  cp variants/lib_$v.so paper_2507_19926_b200/libtilemedian_b200.so
  echo "$v: $(timeout 600 python tools/sweep.py --size 4096 --bits 8 16 32 --k 5 7 9 11 13 --kernels oblivious --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d/%d:%.1f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))")"
done
