"""Debug helper: one forced kernel vs the C oracle on small images, mismatch stats."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import TestImageSpec, generate, oracle_median_filter_c  # noqa: E402
from test_kernels_gpu import run_forced  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="histogram")
    ap.add_argument("--bits", type=int, default=8)
    ap.add_argument("--k", type=int, nargs="+", default=[3, 9, 13, 17, 33])
    ap.add_argument("--shape", type=int, nargs=2, default=[157, 301])
    a = ap.parse_args()
    for k in a.k:
        img = generate(TestImageSpec("random", a.shape[1], a.shape[0], a.bits, seed=k))
        got = run_forced(a.kernel, img, k)
        ref = oracle_median_filter_c(img, k)
        bad = np.argwhere(got != ref)
        print(f"k={k} mismatches={len(bad)}", flush=True)
        if len(bad):
            ys, xs = bad[:, 0], bad[:, 1]
            print("  rows", np.unique(ys)[:20], "cols", np.unique(xs)[:20])
            y, x = bad[0]
            print("  first", (y, x), "got", got[y, x], "ref", ref[y, x])


if __name__ == "__main__":
    main()


def characterise(kernel="histogram", bits=8, k=9, shape=(157, 301), seg=32, strip=128):
    """Map of mismatches per (row segment, column strip) and rank error of the first ones."""
    img = generate(TestImageSpec("random", shape[1], shape[0], bits, seed=k))
    got = run_forced(kernel, img, k)
    ref = oracle_median_filter_c(img, k)
    bad = got != ref
    H, W = shape
    grid = np.zeros(((H + seg - 1) // seg, (W + strip - 1) // strip), int)
    for y, x in np.argwhere(bad):
        grid[y // seg, x // strip] += 1
    print("mismatch map (rows=segments, cols=strips):\n", grid)
    h = k // 2
    pad = np.pad(img, h, mode="edge")
    r = (k * k + 1) // 2
    for y, x in np.argwhere(bad)[:6]:
        win = pad[y:y + k, x:x + k].ravel()
        lt = int((win < got[y, x]).sum())
        le = int((win <= got[y, x]).sum())
        print(f"  ({y},{x}) got {got[y, x]} ref {ref[y, x]}: got covers ranks ({lt}, {le}], want {r}")
