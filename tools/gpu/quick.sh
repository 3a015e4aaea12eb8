timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "host" 2>&1 | tail -1
for nb in 1 2 4 8 16 32; do TMB_HOST_BANDS=$nb timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bands $nb e2e', round(d['e2e']['value'],2))"; done
