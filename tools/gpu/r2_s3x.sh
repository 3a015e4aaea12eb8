# square windows 77..127 on the data-aware sweeps
timeout 900 python -m pytest tests -m gpu -q -k "above_75 or hist or rank or golden" --timeout 300 --timeout-method thread 2>&1 | grep -v "^\.\+$" | tail -2
timeout 400 python tools/fuzz_rank.py --seconds 150 --seed 31 2>&1 | tail -1
python - <<'PY'
import torch
from paper_2507_19926_b200 import _lib
lib = _lib.load()
n = 4096
res = []
for bits, tdt in ((8, torch.uint8), (16, torch.uint16), (32, torch.uint32)):
    src = torch.randint(0, 1 << min(bits, 31), (n, n), dtype=torch.int64, device="cuda").to(tdt); dst = torch.empty_like(src)
    esz = bits // 8
    for k in (77, 101, 127):
        for kern in ("auto", "multipass"):
            prev = lib.tm_force_kernel(0 if kern == "auto" else _lib.KERNEL_CODES[kern])
            name = lib.tm_kernel_name(lib.tm_dispatch_query(bits, k, k, 0)).decode()
            s = torch.cuda.current_stream().cuda_stream
            run = lambda: _lib.check(lib.tm_median2d(src.data_ptr(), n * esz, dst.data_ptr(), n * esz, n, n, bits, k, 0, s))
            run(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); [run() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
            res.append((bits, k, name, round(3 * n * n / e0.elapsed_time(e1) / 1e6, 2)))
            lib.tm_force_kernel(prev)
print("k>75 4096^2 Gpx/s", res)
PY
