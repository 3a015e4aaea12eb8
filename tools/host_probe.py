"""Host-path timing probe: where does a drop-in numpy call spend its time?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19926_b200 import _lib, filter_planes  # noqa: E402
from paper_2507_19926_b200.engine import pinned_empty  # noqa: E402


def t(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


H, W, C = 4480, 6720, 3
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
img = np.random.default_rng(0).integers(0, 256, (H, W, C), dtype=np.uint8)
print("pinned_empty ms", t(lambda: pinned_empty(img.shape, img.dtype)))
dst = np.empty_like(img)
print("np.copyto 90MB ms", t(lambda: np.copyto(dst, img)))
print("filter_planes pageable ms", t(lambda: filter_planes(img, 17)))
pin = torch.from_numpy(img).pin_memory().numpy()
print("filter_planes pinned-in ms", t(lambda: filter_planes(pin, 17)))
lib = _lib.load()
out_pg = np.empty_like(img)
out_pin = torch.empty(img.shape, dtype=torch.uint8).pin_memory().numpy()
for name, a, b in (("pageable->pageable", img, out_pg), ("pageable->pinned", img, out_pin),
                   ("pinned->pinned", pin, out_pin), ("pinned->pageable", pin, out_pg)):
    def run():
        _lib.check(lib.tm_median2d_host(a.ctypes.data, W * C, b.ctypes.data, W * C, W, H, C, 8,
                                        17, 17, 0, 0))
    print("tm_median2d_host", name, "ms", t(run))
for th in ("1", "4", "8"):
    pass
x = torch.from_numpy(img).cuda()
torch.cuda.synchronize()
print("torch pageable H2D ms", t(lambda: (torch.from_numpy(img).cuda(), torch.cuda.synchronize())))
print("torch pinned H2D ms", t(lambda: (torch.from_numpy(pin).cuda(non_blocking=True), torch.cuda.synchronize())))
cudart = torch.cuda.cudart()
buf = np.random.default_rng(1).integers(0, 256, (H, W, C), dtype=np.uint8)
def reg():
    rc = cudart.cudaHostRegister(buf.ctypes.data, buf.nbytes, 0)
    rc2 = cudart.cudaHostUnregister(buf.ctypes.data)
print("cudaHostRegister+Unregister 90MB ms", t(reg))
import threading
def mt_copy(nt):
    src = img.reshape(-1); d = dst.reshape(-1); n = src.size
    def part(i):
        a, b = n * i // nt, n * (i + 1) // nt
        np.copyto(d[a:b], src[a:b])
    th = [threading.Thread(target=part, args=(i,)) for i in range(nt)]
    [x.start() for x in th]; [x.join() for x in th]
for nt in (2, 4, 8, 16):
    print("np copy threads", nt, "ms", t(lambda: mt_copy(nt)))
