timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "host_entry" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], 'e2e', d['e2e']['value'])"
