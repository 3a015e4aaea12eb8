"""Bit-exact parity of the CUDA path against the reference (GPU required).

Every test here calls the product through its public boundary -- the Python
drop-in ``filter_image`` / ``filter_planes`` or the C ABI directly -- and
compares with (a) golden digests produced by the reference itself
(tests/golden/make_golden.py) and (b) the CPU oracle restatement (oracle/),
which tests/test_oracle_golden.py pins to those same goldens.
"""
import ctypes

import numpy as np
import pytest

from golden_util import GOLDEN, digest, load, spec_of
from oracle import TestImageSpec, banded_oracle, generate, oracle_median_filter_c

pytestmark = pytest.mark.gpu

import paper_2507_19926_b200 as tmb  # noqa: E402
from paper_2507_19926_b200 import KernelSpec, filter_image, filter_planes  # noqa: E402


def test_golden_matrix_all_variants():
    """Reference's 264-cell matrix, each cell through its own variant."""
    images = {}
    for cell in load("matrix.json"):
        key = (cell["pattern"], cell["width"], cell["height"], cell["depth"])
        if key not in images:
            images[key] = generate(spec_of(cell))
        out = filter_image(images[key], cell["k"], cell["variant"])
        assert digest(out) == cell["output"], cell


@pytest.mark.parametrize("variant", ["auto", "oblivious", "aware", "oracle"])
def test_golden_sweep_k3_to_k75(variant):
    for cell in load("sweep.json")["square"]:
        k = cell["k"]
        if variant == "aware" and k < 9:
            continue
        out = filter_image(generate(spec_of(cell)), k, variant)
        assert digest(out) == cell["output"], (variant, cell["depth"], cell["pattern"], k)


def test_golden_rect_kernels():
    for cell in load("sweep.json")["rect"]:
        img = generate(spec_of(cell))
        kern = KernelSpec(cell["k_w"], cell["k_h"])
        if cell["output"].startswith("ValueError"):
            with pytest.raises(ValueError, match=cell["output"][len("ValueError: "):]):
                filter_image(img, kern, "oblivious")
        else:
            assert digest(filter_image(img, kern, "oblivious")) == cell["output"], cell
            assert digest(filter_image(img, kern, "oracle")) == cell["output"], cell


def test_config1_full_golden():
    z = np.load(f"{GOLDEN}/c1_u8_512_k3.npz")
    assert np.array_equal(filter_image(z["input"], 3), z["output"])


@pytest.mark.parametrize("bits", [8, 16, 32])
@pytest.mark.parametrize("k", [3, 5, 7, 9, 11, 13, 15, 17, 21, 25, 33])
def test_random_vs_oracle(bits, k):
    img = generate(TestImageSpec("random", 301, 157, bits, seed=1000 + k))
    ref = oracle_median_filter_c(img, k)
    for variant in ("auto", "oblivious", "oracle") + (("aware",) if k >= 9 else ()):
        assert np.array_equal(filter_image(img, k, variant), ref), (bits, k, variant)


@pytest.mark.parametrize("bits", [8, 16, 32])
def test_ties_low_entropy(bits):
    rng = np.random.default_rng(bits)
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    for k in (3, 5, 9, 11, 19, 27):
        img = rng.integers(0, 3, size=(83, 129), dtype=dt)
        if bits > 8:
            img = (img * np.iinfo(dt).max // 2).astype(dt)  # extremes + middle
        ref = oracle_median_filter_c(img, k)
        assert np.array_equal(filter_image(img, k), ref), (bits, k)


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (2, 3), (5, 300), (300, 5), (97, 61)])
def test_edge_shapes(shape):
    rng = np.random.default_rng(sum(shape))
    for dt in (np.uint8, np.uint16, np.uint32):
        img = rng.integers(0, np.iinfo(dt).max, size=shape, dtype=dt, endpoint=True)
        for k in (3, 9, 25):
            assert np.array_equal(filter_image(img, k), oracle_median_filter_c(img, k)), (dt, k)


def test_strided_views():
    img = generate(TestImageSpec("random", 200, 150, 16, seed=3))
    view = img[::2, 1::3]
    assert np.array_equal(filter_image(view, 5), oracle_median_filter_c(np.ascontiguousarray(view), 5))
    flipped = img[::-1]
    assert np.array_equal(filter_image(flipped, 3), oracle_median_filter_c(np.ascontiguousarray(flipped), 3))


def test_filter_planes_interleaved():
    rng = np.random.default_rng(10)
    img = rng.integers(0, 256, (67, 45, 3), dtype=np.uint8)
    for k in (3, 9, 17):
        out = filter_planes(img, k)
        assert out.shape == img.shape and out.dtype == img.dtype
        for c in range(3):
            assert np.array_equal(out[..., c], oracle_median_filter_c(np.ascontiguousarray(img[..., c]), k))


def test_monotone_invariance():
    """test_acceptance.py:146-160: filtering commutes with increasing relabelling."""
    rng = np.random.default_rng(0)
    lut = np.cumsum(rng.integers(1, 200, size=256)).astype(np.uint16)
    for _ in range(4):
        img = rng.integers(0, 256, size=(48, 48), dtype=np.uint8)
        for k in (3, 9, 25):
            assert np.array_equal(filter_image(lut[img], k), lut[filter_image(img, k)])


def test_torch_cuda_tensors_zero_copy():
    import torch
    img = generate(TestImageSpec("random", 256, 130, 8, seed=11))
    t = torch.from_numpy(img).cuda()
    out = filter_image(t, 9)
    assert out.is_cuda and out.dtype == torch.uint8 and out.shape == t.shape
    assert np.array_equal(out.cpu().numpy(), oracle_median_filter_c(img, 9))
    for bits, tdt in ((16, torch.uint16), (32, torch.uint32)):
        im = generate(TestImageSpec("random", 77, 66, bits, seed=12))
        tt = torch.from_numpy(im.astype(np.int64)).to(tdt).cuda() if bits == 32 else \
            torch.from_numpy(im.astype(np.int32)).to(tdt).cuda()
        got = filter_image(tt, 5)
        assert np.array_equal(got.cpu().numpy().astype(np.int64),
                              oracle_median_filter_c(im, 5).astype(np.int64))


def test_band_api_is_exact():
    """tm_median2d_band over bands with +-k/2 halos equals the whole image."""
    import torch
    from paper_2507_19926_b200 import _lib
    lib = _lib.load()
    img = generate(TestImageSpec("random", 190, 203, 16, seed=21))
    k, h = 11, 5
    full = oracle_median_filter_c(img, k)
    dev = torch.from_numpy(img.astype(np.int32)).to(torch.uint16).cuda()
    H, W = img.shape
    got = np.empty_like(img)
    for y0, y1 in ((0, 50), (50, 51), (51, 140), (140, 203)):
        s0, s1 = max(0, y0 - h), min(H, y1 + h)
        src = dev[s0:s1].contiguous()
        dst = torch.empty((y1 - y0, W), dtype=torch.uint16, device="cuda")
        rc = lib.tm_median2d_band(src.data_ptr(), W * 2, s1 - s0, y0 - s0, y1 - y0,
                                  dst.data_ptr(), W * 2, W, 1, 16, k, k, 0, None)
        _lib.check(rc)
        torch.cuda.synchronize()
        got[y0:y1] = dst.cpu().numpy().astype(np.uint16)
    assert np.array_equal(got, full)


def test_host_entry_point_pitches():
    from paper_2507_19926_b200 import _lib
    lib = _lib.load()
    img = generate(TestImageSpec("random", 100, 40, 8, seed=2))
    big = np.zeros((40, 128), np.uint8)
    big[:, :100] = img
    out = np.zeros((40, 160), np.uint8)
    rc = lib.tm_median2d_host(big.ctypes.data, 128, out.ctypes.data, 160, 100, 40, 1, 8, 7, 7, 0, 0)
    _lib.check(rc)
    assert np.array_equal(out[:, :100], oracle_median_filter_c(img, 7))
    assert not out[:, 100:].any()


def test_counter_and_checksums_aware():
    img = np.zeros((48, 48), dtype=np.uint8)
    c = tmb.ComparisonCounter()
    filter_image(img, 23, "auto", counter=c)
    assert c.total > 0
    lines = []
    out = filter_image(generate(TestImageSpec("random", 40, 40, 8, seed=1)), 9, "aware",
                       checksums=lines)
    assert lines and all(l.startswith("pass=finalize") for l in lines)


@pytest.mark.parametrize("bits,k", [(16, 3), (16, 17), (16, 41), (32, 25), (8, 9), (8, 33)])
def test_full_size_bands_vs_oracle(bits, k):
    """Config-scale images: border and random interior bands vs the banded oracle."""
    n = {8: 2048, 16: 2048, 32: 1536}[bits]
    img = generate(TestImageSpec("random", n, n, bits, seed=42))
    out = filter_image(img, k)
    rng = np.random.default_rng(k)
    bands = [(0, 8), (n - 8, n)] + [(y, y + 4) for y in rng.integers(8, n - 12, size=3)]
    for y0, y1 in bands:
        ref = banded_oracle(img, k, int(y0), int(y1))
        assert np.array_equal(out[y0:y1], ref), (y0, y1)
    # columns at the left/right border are inside every band checked above


@pytest.mark.parametrize("bits,k,shape", [(8, 17, (1100, 257, 3)), (16, 41, (900, 190)),
                                          (32, 75, (530, 97)), (8, 3, (2049, 64))])
def test_host_entry_point_pipelined_bands(bits, k, shape):
    """tm_median2d_host splits tall images into row bands pipelined over three
    streams; halos cross band boundaries (k/2 > band height for k = 75)."""
    from paper_2507_19926_b200 import _lib
    lib = _lib.load()
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    rng = np.random.default_rng(k)
    img = rng.integers(0, np.iinfo(dt).max, size=shape, dtype=dt, endpoint=True)
    h, w = shape[:2]
    ch = shape[2] if len(shape) == 3 else 1
    out = np.zeros_like(img)
    rc = lib.tm_median2d_host(img.ctypes.data, img.strides[0], out.ctypes.data, out.strides[0],
                              w, h, ch, bits, k, k, 0, 0)
    _lib.check(rc)
    for c in range(ch):
        plane = img[..., c] if ch > 1 else img
        got = out[..., c] if ch > 1 else out
        assert np.array_equal(got, oracle_median_filter_c(np.ascontiguousarray(plane), k)), c


@pytest.mark.parametrize("bits", [8, 16, 32])
def test_kernels_above_75(bits):
    """k = 77..127: auto / aware run the data-aware sweeps (histogram for
    8-bit, rank for 16/32-bit), oblivious / oracle the per-pixel selection
    kernel -- all exact."""
    img = generate(TestImageSpec("random", 90, 70, bits, seed=77))
    for k in (77, 101, 127):
        ref = oracle_median_filter_c(img, k)
        for variant in ("auto", "aware", "oblivious", "oracle"):
            assert np.array_equal(filter_image(img, k, variant), ref), (k, variant)
