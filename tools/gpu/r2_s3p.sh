# rank rect + full suite + smoke + perf check of square rank/hist
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+" | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C2', round(d['value'],2), d['clocks']['sm_mhz'])"
timeout 600 python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random --reps 3 2>&1 | python -c "
import sys,json
print([(d['k'], d['pattern'][:4], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
python - <<'PY'
import torch
from paper_2507_19926_b200 import _lib
lib = _lib.load()
n = 4096
res = []
for bits, tdt in ((16, torch.uint16), (32, torch.uint32)):
    src = torch.randint(0, 1 << min(bits, 31), (n, n), dtype=torch.int64, device="cuda").to(tdt); dst = torch.empty_like(src)
    esz = bits // 8
    for kw, kh in ((9, 41), (41, 9), (25, 75), (75, 25)):
        for kern in ("rank", "select"):
            prev = lib.tm_force_kernel(_lib.KERNEL_CODES[kern])
            s = torch.cuda.current_stream().cuda_stream
            run = lambda: _lib.check(lib.tm_median2d_band(src.data_ptr(), n * esz, n, 0, n, dst.data_ptr(), n * esz, n, 1, bits, kw, kh, 0, s))
            run(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); [run() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
            res.append((bits, kw, kh, kern, round(3 * n * n / e0.elapsed_time(e1) / 1e6, 2)))
            lib.tm_force_kernel(prev)
print("rect 4096^2 Gpx/s", res)
PY
