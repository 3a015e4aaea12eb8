"""Host path: pinned vs pageable, per-call times, in one process (TMB_HOST_TRACE=1 for phases)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19926_b200 import _lib, filter_planes  # noqa: E402

H, W, C = 4480, 6720, 3
lib = _lib.load()
img = np.random.default_rng(0).integers(0, 256, (H, W, C), dtype=np.uint8)
hin = torch.from_numpy(img).pin_memory()
hout = torch.empty(img.shape, dtype=torch.uint8).pin_memory()


def cabi(a, b):
    _lib.check(lib.tm_median2d_host(a, W * C, b, W * C, W, H, C, 8, 17, 17, 0, 0))


def timed(name, fn, n=5):
    fn()
    out = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        out.append(round(1e3 * (time.perf_counter() - t0), 2))
    print(name, out, flush=True)


timed("pinned->pinned", lambda: cabi(hin.data_ptr(), hout.data_ptr()))
timed("dropin pageable", lambda: filter_planes(img, 17))
timed("pinned->pinned again", lambda: cabi(hin.data_ptr(), hout.data_ptr()))
res = None
def loop():
    global res
    res = filter_planes(img, 17)
timed("dropin pageable (kept)", loop)
timed("pinned->pinned third", lambda: cabi(hin.data_ptr(), hout.data_ptr()))
