"""Restatement of the reference's brute-force median filter and test images.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* ``oracle_median_filter_np``: numpy restatement of
  ``/root/reference/pkg/src/tilemedian/reference.py:26-43``: replicate-pad
  (``np.pad(mode="edge")``, :37-38), all k_h x k_w windows (:39-40) and a
  partition at rank (k_w*k_h+1)/2 - 1 (:41-43).  Processed in row bands so
  the H*W*k^2 window copy stays bounded; the bands
  are exact because each band re-reads +-k_h/2 halo rows of the original
  image and replication only ever happens at the true image edges.
* ``oracle_median_filter_c``: the same selection in C
  (``oracle/median_oracle.c``), multi-threaded, used for large parity checks
  and as the CPU baseline (``kind: "port"``).
* ``generate`` / ``TestImageSpec`` / ``compare_images``: restatement of the
  reference's deterministic test-image generator (``reference.py:46-126``,
  Philox keyed by the seed, :74-75) so the GPU box -- which has no
  /root/reference -- produces the very same synthetic inputs.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

_HERE = os.path.dirname(os.path.abspath(__file__))


def _kernel_sides(k) -> tuple[int, int]:
    """(k_w, k_h) for an int or any object with k_w/k_h (KernelSpec)."""
    if hasattr(k, "k_w"):
        kw, kh = int(k.k_w), int(k.k_h)
    else:
        kw = kh = int(k)
    for side in (kw, kh):
        if side < 3 or side % 2 == 0:
            raise ValueError(f"kernel sides must be odd and >= 3, got {kw}x{kh}")
    return kw, kh


def oracle_median_filter_np(image, k, band_rows: int | None = None) -> np.ndarray:
    """Exact median filter, edge-replicated borders (reference.py:26-43)."""
    img = np.asarray(image)
    if img.ndim != 2:
        raise ValueError("expected a 2-D image")
    kw, kh = _kernel_sides(k)
    hw, hh = kw // 2, kh // 2
    n = kw * kh
    rank = (n + 1) // 2 - 1
    H, W = img.shape
    if band_rows is None:
        # keep the window copy around 64 MiB
        band_rows = max(1, (64 << 20) // max(1, W * n * img.itemsize))
    padded_x = np.pad(img, ((0, 0), (hw, hw)), mode="edge")
    out = np.empty_like(img)
    for y0 in range(0, H, band_rows):
        y1 = min(H, y0 + band_rows)
        rows = np.clip(np.arange(y0 - hh, y1 + hh), 0, H - 1)
        block = padded_x[rows]
        win = sliding_window_view(block, (kh, kw)).reshape(y1 - y0, W, n)
        out[y0:y1] = np.partition(win, rank, axis=2)[:, :, rank]
    return out


_C_LIB = None


def load_c_oracle():
    """Load (building if needed) ``oracle/liboracle.so``."""
    global _C_LIB
    if _C_LIB is not None:
        return _C_LIB
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "median_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        import subprocess
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    lib = ctypes.CDLL(path)
    lib.oracle_median2d.restype = ctypes.c_int
    lib.oracle_median2d.argtypes = [
        ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
        ctypes.c_int, ctypes.c_int, ctypes.c_int]
    _C_LIB = lib
    return lib


def oracle_median_filter_c(image, k, rows=None, threads: int | None = None) -> np.ndarray:
    """C oracle.  ``rows=(y0, y1)`` filters just that band (output has y1-y0 rows)."""
    img = np.asarray(image)
    if img.ndim != 2:
        raise ValueError("expected a 2-D image")
    if img.dtype not in (np.uint8, np.uint16, np.uint32):
        raise TypeError(f"oracle supports uint8/16/32, got {img.dtype}")
    img = np.ascontiguousarray(img)
    kw, kh = _kernel_sides(k)
    H, W = img.shape
    y0, y1 = (0, H) if rows is None else (int(rows[0]), int(rows[1]))
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    full = np.empty((H, W), dtype=img.dtype) if (y0, y1) == (0, H) else None
    if full is None:
        band = np.empty((y1 - y0, W), dtype=img.dtype)
        # dst pointer offset so that row y lands at band[y - y0]
        base = band.ctypes.data - y0 * W * img.itemsize
        dst = ctypes.c_void_p(base)
    else:
        band = full
        dst = ctypes.c_void_p(band.ctypes.data)
    rc = load_c_oracle().oracle_median2d(
        ctypes.c_void_p(img.ctypes.data), W, dst, W, W, H, img.itemsize * 8,
        kw, kh, y0, y1, int(threads))
    if rc != 0:
        raise ValueError("oracle_median2d rejected its arguments")
    return band


def oracle_median_filter(image, k) -> np.ndarray:
    """Default oracle: C for supported dtypes, numpy otherwise."""
    img = np.asarray(image)
    if img.ndim == 2 and img.dtype in (np.uint8, np.uint16, np.uint32):
        return oracle_median_filter_c(img, k)
    return oracle_median_filter_np(img, k)


def banded_oracle(image, k, y0: int, y1: int, threads: int | None = None) -> np.ndarray:
    """Rows [y0, y1) of the exact filter of ``image`` (halo re-read, exact)."""
    return oracle_median_filter_c(image, k, rows=(y0, y1), threads=threads)


# ---------------------------------------------------------------------------
# deterministic test images (reference.py:46-99)

_DTYPES = {8: np.uint8, 16: np.uint16, 32: np.uint32}
PATTERNS = ("constant", "gradient", "random", "impulse")


@dataclass(frozen=True)
class TestImageSpec:
    """Recipe for a reproducible test image (reference.py:50-71)."""

    __test__ = False

    pattern: str
    width: int
    height: int
    depth: int = 8
    seed: int = 0
    density: float = 0.3

    def __post_init__(self):
        if self.pattern not in PATTERNS:
            raise ValueError(f"unknown pattern {self.pattern!r} (expected one of {PATTERNS})")
        if self.depth not in _DTYPES:
            raise ValueError(f"unsupported depth {self.depth} (expected 8, 16, or 32)")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be positive")
        if not 0.0 <= self.density <= 1.0:
            raise ValueError("density must be within [0, 1]")


def generate(spec: TestImageSpec) -> np.ndarray:
    """Render ``spec`` exactly like reference.py:78-99 (Philox keyed by seed)."""
    dtype = _DTYPES[spec.depth]
    top = np.iinfo(dtype).max
    h, w = spec.height, spec.width
    if spec.pattern == "constant":
        return np.full((h, w), 1 << (spec.depth - 1), dtype=dtype)
    diag = (np.arange(h)[:, None] + np.arange(w)[None, :]) & top
    if spec.pattern == "gradient":
        return diag.astype(dtype)
    gen = np.random.Generator(np.random.Philox(key=spec.seed))
    if spec.pattern == "random":
        return gen.integers(0, top, size=(h, w), endpoint=True, dtype=dtype)
    img = diag.astype(dtype)
    hit = gen.random(size=img.shape) < spec.density
    salt = gen.random(size=img.shape) < 0.5
    img[hit & salt] = top
    img[hit & ~salt] = 0
    return img


@dataclass(frozen=True)
class ImageComparison:
    equal: bool
    mismatches: int
    max_abs_diff: int
    first_diff: tuple[int, int] | None

    def __bool__(self) -> bool:
        return self.equal


def compare_images(a, b) -> ImageComparison:
    """Pixel-exact comparison (reference.py:113-126)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    d = a.astype(np.int64) - b.astype(np.int64)
    bad = np.argwhere(d != 0)
    if len(bad) == 0:
        return ImageComparison(True, 0, 0, None)
    return ImageComparison(False, int(len(bad)), int(np.abs(d).max()),
                           (int(bad[0][0]), int(bad[0][1])))
