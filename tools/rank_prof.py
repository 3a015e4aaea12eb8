"""Per-phase cycle split of the rank kernel.

    TMB_LIB=paper_2507_19926_b200/libtilemedian_b200_prof.so python tools/rank_prof.py

Needs the library built with -DTMB_RANK_PROFILE (TMB_NVCC_EXTRA, into its own
TMB_BUILD_DIR / TMB_LIB_OUT).  Phases (RANK_T marks in tm_rank.cuh): guess scan
+ range sweep, count scan, candidate placement, bucket sort, fine sweep (with
the per-pixel candidate selection; slices and interval sweeps land there too).
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19926_b200 import _lib  # noqa: E402
from paper_2507_19926_b200.synth import render  # noqa: E402

lib = _lib.load()
lib.tm_force_kernel(5)
arr = (ctypes.c_ulonglong * 8)()
names = ["range", "count", "place", "sort", "fine"]
for bits, n in ((16, 4096), (32, 8192)):
    for pat in ("random", "gentle"):
        src = render(pat, (n, n), bits)
        dst = torch.empty_like(src)
        for k in (27, 49, 75):
            s = torch.cuda.current_stream().cuda_stream
            esz = bits // 8
            _lib.check(lib.tm_median2d(src.data_ptr(), n * esz, dst.data_ptr(), n * esz, n, n, bits, k, 0, s))
            torch.cuda.synchronize()
            lib.tm_rank_profile(arr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.tm_median2d(src.data_ptr(), n * esz, dst.data_ptr(), n * esz, n, n, bits, k, 0, s))
            e1.record()
            torch.cuda.synchronize()
            lib.tm_rank_profile(arr)
            tot = sum(arr[:5]) or 1
            print(bits, pat, k, f"{n * n / e0.elapsed_time(e1) / 1e6:.2f} Gpx/s (profiled build)",
                  " ".join(f"{nm}={arr[i] / tot * 100:.1f}%" for i, nm in enumerate(names)), flush=True)
