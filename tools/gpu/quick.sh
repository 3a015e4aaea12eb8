timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 9 13 15 17 21 25 33 49 75 --kernels histogram --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d/%d:%.1f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))"
timeout 600 python tools/sweep.py --size 4096 --bits 16 32 --k 29 33 49 75 --kernels rank --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d/%d:%.2f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], d['roofline']['frac'], 'e2e', d['e2e']['value'])"
