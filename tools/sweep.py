"""Kernel sweep: Gpx/s per (dtype, k, variant) on device-resident images.

    python tools/sweep.py --size 4096 --bits 8 16 32 --k 3 5 7 9 11 --variants auto

Times the C ABI on torch CUDA buffers with CUDA events (warm-up, then the
median of --reps launches, L2 flushed with a 256 MiB write before each timed
launch), samples SM clocks and throttle reasons during every point (bench.py's
ClockSampler), and prints one JSON object per point including the ALU-roofline
fraction against W(k) (the reference op model) and the measured min/max issue
peak (profiles/r01_minmax_microbench.txt), and the HBM roofline against
MEASURED_PEAKS.json.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19926_b200 import _lib  # noqa: E402
from paper_2507_19926_b200.program import op_model  # noqa: E402
from bench import ClockSampler, _peaks  # noqa: E402

MINMAX_PEAK = 18.6e12  # thread-level VIMNMX/s, measured (148 SM x 64/clk x 1.965 GHz)
TDT = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--bits", type=int, nargs="+", default=[8, 16, 32])
    ap.add_argument("--k", type=int, nargs="+", default=[3, 5, 7, 9, 11])
    ap.add_argument("--variants", nargs="+", default=["auto"])
    ap.add_argument("--kernels", nargs="+", default=None,
                    help="force kernels by name (oblivious, aware, select, histogram, ...) "
                         "instead of iterating variants")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lib = _lib.load()
    n = a.size
    g = torch.Generator(device="cuda").manual_seed(42)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    hbm_gbs = float(_peaks().get("hbm_gbs", 6650.0))
    for bits in a.bits:
        src = torch.randint(0, 1 << min(bits, 31), (n, n), generator=g, device="cuda",
                            dtype=torch.int64).to(TDT[bits])
        dst = torch.empty_like(src)
        esz = bits // 8
        for k in a.k:
            W = op_model(k)["minmax_per_pixel"]
            runs = ([("forced:" + kn, kn) for kn in a.kernels] if a.kernels
                    else [(v, None) for v in a.variants])
            for v, forced in runs:
                code = _lib.VARIANT_CODES["auto" if forced else v]
                lib.tm_force_kernel(_lib.KERNEL_CODES[forced] if forced else 0)
                kern = lib.tm_kernel_name(lib.tm_dispatch_query(bits, k, k, code)).decode()
                if forced and kern != forced:
                    continue
                s = torch.cuda.current_stream().cuda_stream
                def run():
                    _lib.check(lib.tm_median2d(src.data_ptr(), n * esz, dst.data_ptr(), n * esz,
                                               n, n, bits, k, code, s))
                for _ in range(3):
                    run()
                torch.cuda.synchronize()
                times = []
                with ClockSampler(torch.cuda.current_device()) as clk:
                    for _ in range(a.reps):
                        flush.fill_(1)  # evict the image from L2 (untimed)
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        run()
                        e1.record()
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1))
                ms = float(np.median(times))
                gpx = n * n / ms / 1e6
                lanes = 2 if bits < 32 else 1
                roof_alu = MINMAX_PEAK * lanes / W / 1e9
                roof_hbm = hbm_gbs / (2 * esz)
                cs = clk.summary()
                print(json.dumps({"bits": bits, "k": k, "variant": v, "kernel": kern,
                                  "ms": round(ms, 4), "gpx_s": round(gpx, 2),
                                  "roof_gpx": round(min(roof_alu, roof_hbm), 1),
                                  "frac": round(gpx / min(roof_alu, roof_hbm), 3),
                                  "hbm_frac": round(gpx / roof_hbm, 3),
                                  "sm_mhz": cs.get("sm_mhz"), "clk_reasons": cs.get("reasons"),
                                  "l2": "flushed"}), flush=True)


if __name__ == "__main__":
    main()
