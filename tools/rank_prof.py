"""Per-phase cycle split of the rank kernel (library built with -DTMB_RANK_PROFILE)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19926_b200 import _lib
lib = _lib.load()
lib.tm_force_kernel(5)
TDT = {16: torch.uint16, 32: torch.uint32}
arr = (ctypes.c_ulonglong * 8)()
for bits in (16, 32):
    for k in (25, 49, 75):
        n = 4096
        src = torch.randint(0, 1 << min(bits, 31), (n, n), device="cuda", dtype=torch.int64).to(TDT[bits])
        dst = torch.empty_like(src)
        s = torch.cuda.current_stream().cuda_stream
        _lib.check(lib.tm_median2d(src.data_ptr(), n * bits // 8, dst.data_ptr(), n * bits // 8, n, n, bits, k, 0, s))
        torch.cuda.synchronize()
        lib.tm_rank_profile(arr)
        _lib.check(lib.tm_median2d(src.data_ptr(), n * bits // 8, dst.data_ptr(), n * bits // 8, n, n, bits, k, 0, s))
        torch.cuda.synchronize()
        lib.tm_rank_profile(arr)
        tot = sum(arr[:5])
        names = ["range(coarse)", "count-scan", "place-scan", "bucket-sort", "fine"]
        print(bits, k, " ".join(f"{nm}={arr[i]/tot*100:.1f}%" for i, nm in enumerate(names)))
