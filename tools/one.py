"""Run one (bits, k, kernel) configuration a few times (for ncu captures).

    python tools/one.py --bits 8 --k 17 --kernel histogram --size 4096 --reps 3
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19926_b200 import _lib  # noqa: E402

TDT = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=8)
    ap.add_argument("--k", type=int, default=17)
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--size", type=int, nargs="+", default=[4096])
    ap.add_argument("--channels", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    h, w = (a.size[0], a.size[-1])
    lib = _lib.load()
    if a.kernel:
        lib.tm_force_kernel(_lib.KERNEL_CODES[a.kernel])
    g = torch.Generator(device="cuda").manual_seed(42)
    src = torch.randint(0, 1 << min(a.bits, 31), (h, w * a.channels), generator=g, device="cuda",
                        dtype=torch.int64).to(TDT[a.bits])
    dst = torch.empty_like(src)
    esz = a.bits // 8
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(a.reps):
        _lib.check(lib.tm_median2d_band(src.data_ptr(), w * a.channels * esz, h, 0, h, dst.data_ptr(),
                                        w * a.channels * esz, w, a.channels, a.bits, a.k, a.k, 0, s))
    torch.cuda.synchronize()
    print("kernel", lib.tm_kernel_name(lib.tm_dispatch_query(a.bits, a.k, a.k, 0)).decode())


if __name__ == "__main__":
    main()
