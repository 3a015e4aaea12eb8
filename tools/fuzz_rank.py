"""Randomised parity fuzzing of the data-aware kernels (rank for 16/32-bit,
histogram for 8-bit) against the C oracle, with a hang watchdog.

    python tools/fuzz_rank.py --seconds 240 [--seed 1]

Each case draws a dtype, a square or rectangular window, an image shape and a
value distribution (uniform, narrow bands, a few distinct values, impulse noise
of random density over gradients or smooth fields, step edges, clipped noise,
mixtures), runs the kernel the dispatcher picks for "auto" (forcing the
data-aware kernel), and compares with oracle/median_oracle.c.  Prints one line
per failure and a summary; exits 3 on a hang (watchdog), 1 on a mismatch.
"""
import argparse
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle_median_filter_c  # noqa: E402
from paper_2507_19926_b200 import KernelSpec, _lib  # noqa: E402

TDT = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}
state = {"t": time.time(), "case": None}


def watchdog(limit):
    while True:
        time.sleep(1)
        if time.time() - state["t"] > limit:
            print("HANG", state["case"], flush=True)
            os._exit(3)


def draw_image(rng, bits, h, w):
    mx = (1 << bits) - 1
    kind = rng.choice(["uniform", "narrow", "few", "impulse", "steps", "smooth", "mix", "clip"])
    ys, xs = np.mgrid[0:h, 0:w].astype(np.float64)
    if kind == "uniform":
        img = rng.integers(0, mx, (h, w), endpoint=True, dtype=np.uint64)
    elif kind == "narrow":
        base = int(rng.integers(0, mx))
        span = int(rng.choice([1, 3, 50, 126, 127, 300, 5000, 1 << 20]))
        img = np.clip(base + rng.integers(0, span + 1, (h, w)), 0, mx).astype(np.uint64)
    elif kind == "few":
        vals = rng.integers(0, mx, int(rng.integers(1, 6)), endpoint=True)
        img = rng.choice(vals, (h, w)).astype(np.uint64)
    elif kind == "impulse":
        slope = float(rng.choice([0.0, 1.0, 9.0, 200.0]))
        base = (xs + ys) * slope + rng.integers(0, max(1, mx // 2))
        img = np.clip(base, 0, mx).astype(np.uint64)
        d = float(rng.uniform(0.05, 0.6))
        hit = rng.random((h, w)) < d
        salt = rng.random((h, w)) < 0.5
        img[hit & salt] = mx
        img[hit & ~salt] = 0
    elif kind == "steps":
        levels = rng.integers(0, mx, 4, endpoint=True)
        img = levels[((xs // rng.integers(3, 40)) + (ys // rng.integers(3, 40))).astype(np.int64) % 4]
        img = img.astype(np.uint64)
    elif kind == "smooth":
        f = float(rng.uniform(20, 600))
        base = (np.sin(xs / f) * np.cos(ys / (f * 0.7)) + 1) * 0.45 * mx
        noise = rng.normal(0, float(rng.choice([0, 3, 200])) * mx / 65535, (h, w))
        img = np.clip(base + noise, 0, mx).astype(np.uint64)
    elif kind == "clip":
        img = np.clip(rng.normal(mx / 2, mx / 4, (h, w)), 0, mx).astype(np.uint64)
        img[rng.random((h, w)) < 0.4] = rng.choice([0, mx])
    else:  # mix: left half uniform, right half narrow
        img = rng.integers(0, mx, (h, w), endpoint=True, dtype=np.uint64)
        img[:, w // 2:] = (mx // 3) + rng.integers(0, 40, (h, w - w // 2))
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    return kind, img.astype(dt)


def run(img, bits, kw, kh, kernel):
    lib = _lib.load()
    dev = torch.from_numpy(img.astype(np.int64)).to(TDT[bits]).cuda()
    out = torch.empty_like(dev)
    h, w = img.shape
    pitch = w * img.itemsize
    prev = lib.tm_force_kernel(_lib.KERNEL_CODES[kernel] if kernel else 0)
    try:
        got = lib.tm_kernel_name(lib.tm_dispatch_query(bits, kw, kh, 0)).decode()
        assert kernel is None or got == kernel, (got, kernel)
        _lib.check(lib.tm_median2d_band(dev.data_ptr(), pitch, h, 0, h, out.data_ptr(), pitch, w, 1,
                                        bits, kw, kh, 0, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
    finally:
        lib.tm_force_kernel(prev)
    return out.cpu().numpy().astype(img.dtype)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--hang", type=float, default=20)
    ap.add_argument("--all-kernels", action="store_true",
                    help="also draw k <= 27 windows for the oblivious / med3 kernels and "
                         "small windows for select (auto routing, not forced)")
    a = ap.parse_args()
    threading.Thread(target=watchdog, args=(a.hang,), daemon=True).start()
    rng = np.random.default_rng(a.seed)
    t_end = time.time() + a.seconds
    n = bad = 0
    while time.time() < t_end:
        bits = int(rng.choice([8, 16, 16, 32, 32]))
        kw = int(rng.integers(1, 38)) * 2 + 1
        kh = kw if rng.random() < 0.6 else int(rng.integers(1, 64)) * 2 + 1
        if rng.random() < 0.1:  # square windows beyond 75 (up to the ABI's 127)
            kw = kh = int(rng.integers(38, 64)) * 2 + 1
        kernel = "histogram" if bits == 8 else "rank"
        if a.all_kernels and rng.random() < 0.5:
            # whatever "auto" picks (med3 / oblivious / select / data-aware)
            kw = int(rng.integers(1, 14)) * 2 + 1
            kh = kw if rng.random() < 0.7 else int(rng.integers(1, 14)) * 2 + 1
            kernel = None
        elif kw * kh < 81:
            continue
        h = int(rng.integers(1, 400))
        w = int(rng.integers(1, 400))
        kind, img = draw_image(rng, bits, h, w)
        state["case"] = (bits, kw, kh, h, w, kind, n)
        state["t"] = time.time()
        out = run(img, bits, kw, kh, kernel)
        ref = oracle_median_filter_c(img, KernelSpec(kw, kh))
        n += 1
        if not np.array_equal(out, ref):
            bad += 1
            print("MISMATCH", state["case"], int((out != ref).sum()), flush=True)
    print(f"fuzz: {n} cases, {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
