"""Data-sensitivity timing: Gpx/s per (bits, k, pattern) on device-resident images.

    python tools/patterns.py --size 4096 --bits 16 --k 27 49 75 --patterns random gradient impulse constant

Patterns: paper_2507_19926_b200.synth (the reference generator's patterns plus
narrow16 / gentle / smooth), rendered on the device with a seeded generator.  Timing: CUDA events on the launching stream, L2 flushed
(256 MiB write) before every rep, median of --reps; SM clocks sampled via NVML.
Optional --check compares a few random rows against the C oracle (banded).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_19926_b200 import _lib  # noqa: E402
from paper_2507_19926_b200.synth import render  # noqa: E402

TDT = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}


def make(pattern: str, h: int, w: int, bits: int, seed: int = 42) -> torch.Tensor:
    return render(pattern, (h, w), bits, seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, nargs="+", default=[4096])
    ap.add_argument("--bits", type=int, nargs="+", default=[16])
    ap.add_argument("--k", type=int, nargs="+", default=[27, 49, 75])
    ap.add_argument("--patterns", nargs="+", default=["random", "gradient", "impulse", "constant"])
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", type=int, default=0, help="rows to verify against the C oracle")
    a = ap.parse_args()
    h, w = a.size[0], a.size[-1]
    lib = _lib.load()
    lib.tm_force_kernel(_lib.KERNEL_CODES[a.kernel] if a.kernel else 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    try:
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:
        hnd = None
    for bits in a.bits:
        esz = bits // 8
        for pat in a.patterns:
            if pat == "narrow16" and bits < 32:
                continue
            src = make(pat, h, w, bits)
            dst = torch.empty_like(src)
            s = torch.cuda.current_stream().cuda_stream
            for k in a.k:
                kern = lib.tm_kernel_name(lib.tm_dispatch_query(bits, k, k, 0)).decode()

                def run():
                    _lib.check(lib.tm_median2d(src.data_ptr(), w * esz, dst.data_ptr(), w * esz,
                                               w, h, bits, k, 0, s))
                run()
                torch.cuda.synchronize()
                times, clk = [], []
                for _ in range(a.reps):
                    flush.fill_(1)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run()
                    e1.record()
                    if hnd is not None:
                        clk.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
                    e1.synchronize()
                    times.append(e0.elapsed_time(e1))
                ms = float(np.median(times))
                rec = {"bits": bits, "k": k, "pattern": pat, "kernel": kern, "size": [h, w],
                       "ms": round(ms, 4), "gpx_s": round(h * w / ms / 1e6, 3),
                       "sm_mhz": int(np.median(clk)) if clk else None}
                if a.check:
                    from oracle import oracle_median_filter_c
                    img = src.cpu().numpy()
                    out = dst.cpu().numpy()
                    rng = np.random.default_rng(k)
                    rows = sorted(set([0, h - 1] + list(rng.integers(0, h, a.check))))
                    bad = 0
                    for y in rows:
                        y0, y1 = max(0, y - k // 2), min(h, y + k // 2 + 1)
                        ref = oracle_median_filter_c(np.ascontiguousarray(img[y0:y1]), k)[y - y0]
                        # the crop replicates rows at y0 / y1 - 1, which are true edges only there;
                        # rows with a full window are unaffected
                        bad += int((ref != out[y]).sum())
                    rec["check_rows"] = len(rows)
                    rec["mismatches"] = bad
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
