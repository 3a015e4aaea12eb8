timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -k "rank or multipass" 2>&1 | tail -2
timeout 600 python tools/sweep.py --size 4096 --bits 16 32 --k 27 29 33 41 49 61 75 --kernels rank --reps 10 2>/dev/null | python -c "import json,sys; print(' '.join('%d/%d:%.2f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, sys.stdin)))"
