# rectangular 8-bit kernels on the histogram sweep; square path regression check
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C2', round(d['value'],2), d['clocks']['sm_mhz'])"
done
timeout 300 python tools/sweep.py --size 4096 --bits 8 --k 15 17 21 25 33 49 75 --kernels histogram --reps 10 2>&1 | python -c "
import sys,json
print([ (d['k'], d['gpx_s']) for d in map(json.loads, sys.stdin)])"
python - <<'PY'
import torch, json
from paper_2507_19926_b200 import _lib
lib = _lib.load()
n = 4096
src = torch.randint(0, 256, (n, n), dtype=torch.uint8, device="cuda"); dst = torch.empty_like(src)
res = []
for kw, kh in ((9, 31), (31, 9), (17, 33), (33, 17), (5, 75), (75, 5)):
    for kern in ("histogram", "select"):
        prev = lib.tm_force_kernel(_lib.KERNEL_CODES[kern])
        s = torch.cuda.current_stream().cuda_stream
        run = lambda: _lib.check(lib.tm_median2d_band(src.data_ptr(), n, n, 0, n, dst.data_ptr(), n, n, 1, 8, kw, kh, 0, s))
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); [run() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
        res.append((kw, kh, kern, round(5 * n * n / e0.elapsed_time(e1) / 1e6, 2)))
        lib.tm_force_kernel(prev)
print("rect 4096^2 u8 Gpx/s", res)
PY
