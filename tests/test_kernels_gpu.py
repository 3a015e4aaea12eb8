"""Every exact kernel, forced through the C ABI, against the CPU oracle (GPU).

The dispatch table picks one kernel per (dtype, k); this file pins each
kernel on its own (``tm_force_kernel``) so a kernel that auto does not pick
today is still bit-exact when a later table change routes to it.  Patterns
follow the reference's test images (reference.py:78-99): random, constant,
impulse (salt and pepper on a gradient) and low-entropy ties.
"""
import numpy as np
import pytest
import torch

from oracle import TestImageSpec, generate, oracle_median_filter_c

pytestmark = pytest.mark.gpu

from paper_2507_19926_b200 import KernelSpec, _lib  # noqa: E402

TDT = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}


def run_forced(kernel: str, img: np.ndarray, k: int) -> np.ndarray:
    lib = _lib.load()
    bits = img.dtype.itemsize * 8
    dev = torch.from_numpy(img.astype(np.int64)).to(TDT[bits]).cuda()
    if img.ndim == 2:
        h, w = img.shape
        ch = 1
    else:
        h, w, ch = img.shape
    out = torch.empty_like(dev)
    prev = lib.tm_force_kernel(_lib.KERNEL_CODES[kernel])
    try:
        assert lib.tm_kernel_name(lib.tm_dispatch_query(bits, k, k, 0)).decode() == kernel
        stream = torch.cuda.current_stream().cuda_stream
        rc = lib.tm_median2d_band(dev.data_ptr(), w * ch * img.itemsize, h, 0, h, out.data_ptr(),
                                  w * ch * img.itemsize, w, ch, bits, k, k, 0, stream)
        _lib.check(rc)
    finally:
        lib.tm_force_kernel(prev)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(img.dtype)


def images(bits, h, w, seed):
    yield "random", generate(TestImageSpec("random", w, h, bits, seed=seed))
    yield "impulse", generate(TestImageSpec("impulse", w, h, bits, seed=seed, density=0.3))
    yield "gradient", generate(TestImageSpec("gradient", w, h, bits, seed=seed))
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    yield "constant", np.full((h, w), np.iinfo(dt).max // 3, dtype=dt)
    ties = np.random.default_rng(seed).integers(0, 3, size=(h, w)).astype(dt)
    yield "ties", (ties * (np.iinfo(dt).max // 2)).astype(dt)
    yield "extremes", np.random.default_rng(seed).choice(
        np.array([0, np.iinfo(dt).max], dtype=dt), size=(h, w))


HIST_KS = [3, 5, 9, 15, 17, 21, 31, 33, 47, 75]


@pytest.mark.parametrize("k", HIST_KS)
def test_histogram_u8_patterns(k):
    for name, img in images(8, 157, 301, seed=k):
        assert np.array_equal(run_forced("histogram", img, k), oracle_median_filter_c(img, k)), (name, k)


@pytest.mark.parametrize("shape", [(1, 1), (1, 200), (200, 1), (3, 5), (130, 129), (257, 700)])
def test_histogram_u8_shapes(shape):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    img = rng.integers(0, 256, size=shape, dtype=np.uint8)
    for k in (3, 17, 41):
        assert np.array_equal(run_forced("histogram", img, k), oracle_median_filter_c(img, k)), (shape, k)


def test_histogram_u8_interleaved_planes():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (150, 333, 3), dtype=np.uint8)
    for k in (5, 17, 27):
        out = run_forced("histogram", img, k)
        for c in range(3):
            ref = oracle_median_filter_c(np.ascontiguousarray(img[..., c]), k)
            assert np.array_equal(out[..., c], ref), (k, c)


def test_histogram_u8_tall_image_many_segments():
    """Tall enough that the launcher splits columns into several row segments."""
    img = generate(TestImageSpec("random", 140, 3000, 8, seed=9))
    for k in (7, 25):
        assert np.array_equal(run_forced("histogram", img, k), oracle_median_filter_c(img, k)), k


def test_histogram_u8_wide_short_image_pieces_span_strips():
    """Wide and short: the launcher's equal pieces per warp are shorter than a
    strip's rows or span several strips (sub-items with their own builds)."""
    img = np.random.default_rng(21).integers(0, 256, (100, 60000), dtype=np.uint8)
    for k in (9, 17):
        assert np.array_equal(run_forced("histogram", img, k), oracle_median_filter_c(img, k)), k


@pytest.mark.parametrize("ch", [2, 4, 5])
def test_histogram_u8_continuous_pieces_channels(ch):
    """Large interleaved images take the equal-piece split with groups of
    (adjacent strips x channels) warps; 2, 4 and 5 channels give different
    group shapes (5: one strip per group) and partial last strip blocks."""
    from oracle import banded_oracle
    rng = np.random.default_rng(ch)
    img = rng.integers(0, 256, (4480, 6720, ch), dtype=np.uint8)  # the C2 frame size
    out = run_forced("histogram", img, 17)
    for c in range(ch):
        plane = np.ascontiguousarray(img[..., c])
        for y0 in (0, 1100, 2239, 4480 - 48):  # edges and piece / strip boundaries
            ref = banded_oracle(plane, 17, y0, y0 + 48)
            assert np.array_equal(out[y0:y0 + 48, :, c], ref), (ch, c, y0)


RANK_KS = [3, 9, 17, 29, 33, 47, 75]


@pytest.mark.parametrize("bits", [16, 32])
@pytest.mark.parametrize("k", RANK_KS)
def test_rank_patterns(bits, k):
    for name, img in images(bits, 157, 301, seed=k):
        assert np.array_equal(run_forced("rank", img, k), oracle_median_filter_c(img, k)), (bits, name, k)


@pytest.mark.parametrize("bits", [16, 32])
@pytest.mark.parametrize("shape", [(1, 1), (1, 200), (200, 1), (3, 5), (130, 129), (257, 300)])
def test_rank_shapes(bits, shape):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1] + bits)
    dt = {16: np.uint16, 32: np.uint32}[bits]
    img = rng.integers(0, np.iinfo(dt).max, size=shape, dtype=dt, endpoint=True)
    for k in (3, 17, 41):
        assert np.array_equal(run_forced("rank", img, k), oracle_median_filter_c(img, k)), (shape, k)


@pytest.mark.parametrize("bits", [16, 32])
def test_rank_high_entropy_narrow_band(bits):
    """Many distinct candidates in a narrow value band: rank bins + fine scan,
    and the candidate-overflow split (smooth ramp + small noise)."""
    rng = np.random.default_rng(bits)
    dt = {16: np.uint16, 32: np.uint32}[bits]
    h, w = 150, 260
    ramp = np.linspace(1000, 1200 if bits == 16 else 5000, w)[None, :] + np.zeros((h, 1))
    scale = 1 if bits == 16 else 1 << 12
    img = ((ramp + rng.integers(0, 300, size=(h, w))) * scale).astype(dt)
    for k in (29, 51):
        assert np.array_equal(run_forced("rank", img, k), oracle_median_filter_c(img, k)), k


def test_rank_interleaved_planes_u16():
    rng = np.random.default_rng(6)
    img = rng.integers(0, 65536, (90, 170, 3), dtype=np.uint16)
    for k in (9, 31):
        out = run_forced("rank", img, k)
        for c in range(3):
            ref = oracle_median_filter_c(np.ascontiguousarray(img[..., c]), k)
            assert np.array_equal(out[..., c], ref), (k, c)


@pytest.mark.parametrize("bits", [8, 16, 32])
def test_multipass_kernel(bits):
    """The GPU restatement of the reference's multi-pass aware engine (kept as
    a forced-only kernel) stays exact."""
    for name, img in images(bits, 97, 131, seed=bits):
        for k in (9, 25):
            assert np.array_equal(run_forced("multipass", img, k), oracle_median_filter_c(img, k)), (name, k)


@pytest.mark.parametrize("bits", [8, 16, 32])
def test_med3_patterns_and_shapes(bits):
    for name, img in images(bits, 157, 301, seed=3):
        assert np.array_equal(run_forced("med3", img, 3), oracle_median_filter_c(img, 3)), name
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    rng = np.random.default_rng(bits)
    for shape in [(1, 1), (1, 9), (9, 1), (2, 2), (3, 17), (70, 1031), (513, 64), (5, 8)]:
        img = rng.integers(0, np.iinfo(dt).max, size=shape, dtype=dt, endpoint=True)
        assert np.array_equal(run_forced("med3", img, 3), oracle_median_filter_c(img, 3)), shape


def test_med3_interleaved_and_band():
    rng = np.random.default_rng(33)
    img = rng.integers(0, 256, (90, 77, 3), dtype=np.uint8)
    out = run_forced("med3", img, 3)
    for c in range(3):
        assert np.array_equal(out[..., c], oracle_median_filter_c(np.ascontiguousarray(img[..., c]), 3))
    # band entry point: output rows of a source with halo rows
    lib = _lib.load()
    full = rng.integers(0, 65536, (200, 256), dtype=np.uint16)
    ref = oracle_median_filter_c(full, 3)
    dev = torch.from_numpy(full.astype(np.int32)).to(torch.uint16).cuda()
    prev = lib.tm_force_kernel(_lib.KERNEL_CODES["med3"])
    try:
        for y0, y1 in ((0, 37), (37, 38), (38, 150), (150, 200)):
            s0, s1 = max(0, y0 - 1), min(200, y1 + 1)
            src = dev[s0:s1].contiguous()
            dst = torch.empty((y1 - y0, 256), dtype=torch.uint16, device="cuda")
            _lib.check(lib.tm_median2d_band(src.data_ptr(), 512, s1 - s0, y0 - s0, y1 - y0,
                                            dst.data_ptr(), 512, 256, 1, 16, 3, 3, 0, None))
            torch.cuda.synchronize()
            assert np.array_equal(dst.cpu().numpy().astype(np.uint16), ref[y0:y1]), (y0, y1)
    finally:
        lib.tm_force_kernel(prev)


# rectangular k_w x k_h windows on the 8-bit histogram sweep: both CPL
# layouts (k_w x k_h < 512 with k_w <= 21 -> 3 columns per lane), tall and
# wide windows, heights beyond 75, a window taller than the image
RECT_KS = [(3, 27), (27, 3), (5, 17), (17, 5), (21, 23), (21, 25), (15, 31), (31, 15),
           (75, 3), (3, 75), (25, 121), (75, 127), (9, 127)]


def run_rect(img: np.ndarray, kw: int, kh: int) -> np.ndarray:
    """auto variant through the C ABI (the reference's Python front end only
    accepts rectangular kernels whose sides cover its root tile)."""
    lib = _lib.load()
    assert lib.tm_kernel_name(lib.tm_dispatch_query(8, kw, kh, 0)).decode() == "histogram"
    dev = torch.from_numpy(img).cuda()
    out = torch.empty_like(dev)
    h, w = img.shape
    _lib.check(lib.tm_median2d_band(dev.data_ptr(), w, h, 0, h, out.data_ptr(), w, w, 1, 8, kw, kh, 0,
                                    torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("kw,kh", RECT_KS)
def test_histogram_u8_rect(kw, kh):
    for name, img in images(8, 157, 301, seed=kw * 1000 + kh):
        ref = oracle_median_filter_c(img, KernelSpec(kw, kh))
        assert np.array_equal(run_rect(img, kw, kh), ref), (name, kw, kh)


def test_histogram_u8_rect_window_taller_than_image():
    img = np.random.default_rng(4).integers(0, 256, (60, 230), dtype=np.uint8)
    for kw, kh in ((9, 127), (41, 101)):
        assert np.array_equal(run_rect(img, kw, kh), oracle_median_filter_c(img, KernelSpec(kw, kh)))


def test_histogram_u8_rect_drop_in():
    """filter_image / filter_planes with a KernelSpec (torch and numpy inputs)."""
    from paper_2507_19926_b200 import dispatch_query, filter_image, filter_planes
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, (230, 410, 3), dtype=np.uint8)
    for kw, kh in ((9, 31), (21, 23), (31, 15)):
        assert dispatch_query(np.uint8, KernelSpec(kw, kh), "auto") == "histogram"
        out = filter_planes(img, KernelSpec(kw, kh))  # numpy drop-in (host path)
        for c in range(3):
            plane = np.ascontiguousarray(img[..., c])
            ref = oracle_median_filter_c(plane, KernelSpec(kw, kh))
            assert np.array_equal(out[..., c], ref), (kw, kh, c)
            got = filter_image(torch.from_numpy(plane).cuda(), KernelSpec(kw, kh)).cpu().numpy()
            assert np.array_equal(got, ref), (kw, kh, c)


RANK_RECT_KS = [(5, 17), (17, 5), (9, 33), (33, 9), (27, 49), (49, 27), (75, 3), (3, 75), (25, 127)]


def run_rect_any(img: np.ndarray, kw: int, kh: int, expect: str) -> np.ndarray:
    lib = _lib.load()
    bits = img.dtype.itemsize * 8
    assert lib.tm_kernel_name(lib.tm_dispatch_query(bits, kw, kh, 0)).decode() == expect
    dev = torch.from_numpy(img.astype(np.int64)).to(TDT[bits]).cuda()
    out = torch.empty_like(dev)
    h, w = img.shape
    pitch = w * img.itemsize
    _lib.check(lib.tm_median2d_band(dev.data_ptr(), pitch, h, 0, h, out.data_ptr(), pitch, w, 1, bits,
                                    kw, kh, 0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(img.dtype)


@pytest.mark.parametrize("bits", [16, 32])
@pytest.mark.parametrize("kw,kh", RANK_RECT_KS)
def test_rank_rect(bits, kw, kh):
    """16/32-bit rectangular windows on the rank sweeps (run-time height)."""
    for name, img in images(bits, 157, 301, seed=kw * 1000 + kh):
        ref = oracle_median_filter_c(img, KernelSpec(kw, kh))
        assert np.array_equal(run_rect_any(img, kw, kh, "rank"), ref), (bits, name, kw, kh)


def test_rect_small_windows_use_select():
    img = np.random.default_rng(2).integers(0, 1 << 16, (90, 130), dtype=np.uint16)
    for kw, kh in ((3, 5), (5, 9), (3, 25)):
        ref = oracle_median_filter_c(img, KernelSpec(kw, kh))
        assert np.array_equal(run_rect_any(img, kw, kh, "select"), ref), (kw, kh)


def test_data_aware_fuzz_short():
    """A short randomised run of tools/fuzz_rank.py (value distributions that
    stress the rank work-list: narrow bands, few values, impulse densities,
    steps, smooth fields, mixtures; square and rectangular windows)."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_rank.py"), "--seconds", "20",
                        "--seed", "7"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "0 mismatches" in p.stdout
