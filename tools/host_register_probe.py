"""Cost of pinning a pageable numpy image in place (cudaHostRegister) versus
staging it through pinned memory: the two ways the drop-in can feed the DMA
engines from a user's pageable array.

    python tools/host_register_probe.py
"""
import ctypes
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
try:
    cudart = ctypes.CDLL("libcudart.so")
except OSError:
    import glob
    import os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = ctypes.CDLL(cands[0])

torch.cuda.init()
for mb in (8, 90, 360):
    a = np.random.default_rng(0).integers(0, 256, mb << 20, dtype=np.uint8)
    for it in range(3):
        t0 = time.perf_counter()
        rc = cudart.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 0)
        t1 = time.perf_counter()
        rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
        t2 = time.perf_counter()
        pin = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True).numpy()
        t3 = time.perf_counter()
        np.copyto(pin, a)
        t4 = time.perf_counter()
        print(f"{mb} MB: register {1e3 * (t1 - t0):.2f} ms (rc {rc}), unregister {1e3 * (t2 - t1):.2f} ms, "
              f"1-thread copy to pinned {1e3 * (t4 - t3):.2f} ms", flush=True)
