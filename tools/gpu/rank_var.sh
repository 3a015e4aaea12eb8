for v in base C3k; do
  cp variants/lib_$v.so paper_2507_19926_b200/libtilemedian_b200.so
  echo "$v: $(timeout 600 python tools/sweep.py --size 4096 --bits 16 32 --k 47 49 55 61 67 75 --kernels rank --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d/%d:%.2f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))")"
done
