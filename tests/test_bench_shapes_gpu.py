"""Parity at the exact benchmarked shapes, on every reference test pattern (GPU).

BASELINE.json's configs C2-C5 at their full sizes, through the public
drop-in (``filter_planes`` / ``filter_image`` on numpy, host path with its
band pipeline; the torch path for the 1 GiB C5 image), with the launch
geometry the bench uses.  A full-size oracle is infeasible (SURVEY.md
section 8c: up to 1.4 TB of windows), so every run is checked on the 2 border
row bands plus 8 random interior bands against the banded C oracle -- exact
because replicate padding then applies only at the true image edges
(oracle.banded_oracle).  Patterns: the reference generator's random,
gradient, impulse (density 0.3) and constant (reference.py:78-99).
"""
import numpy as np
import pytest

from oracle import TestImageSpec, banded_oracle, generate

pytestmark = pytest.mark.gpu

from paper_2507_19926_b200 import filter_image, filter_planes  # noqa: E402

PATTERNS = ("random", "gradient", "impulse", "constant")


def _bands(h: int, k: int, seed: int, n_interior: int = 8, rows: int = 2):
    rng = np.random.default_rng(seed)
    edge = min(h, max(4, k // 2 + 2))
    out = [(0, edge), (h - edge, h)]
    for y in rng.integers(edge, max(edge + 1, h - edge - rows), size=n_interior):
        out.append((int(y), int(y) + rows))
    return out


def _check_bands(img, out, k, seed):
    for y0, y1 in _bands(img.shape[0], k, seed):
        ref = banded_oracle(img, k, y0, y1)
        assert np.array_equal(out[y0:y1], ref), (k, y0, y1, int((out[y0:y1] != ref).sum()))


@pytest.mark.parametrize("pattern", PATTERNS)
def test_c2_rgb_30mp_k17(pattern):
    """C2: 4480 x 6720 x 3 uint8 interleaved, k = 17, through filter_planes."""
    h, w = 4480, 6720
    img = np.stack([generate(TestImageSpec(pattern, w, h, 8, seed=42 + c)) for c in range(3)], -1)
    out = filter_planes(img, 17)
    assert out.shape == img.shape and out.dtype == img.dtype
    for c in range(3):
        _check_bands(np.ascontiguousarray(img[..., c]), np.ascontiguousarray(out[..., c]), 17, c)


@pytest.mark.parametrize("pattern", PATTERNS)
def test_c3_u16_4096(pattern):
    """C3: 4096^2 uint16 over the k sweep's corners and the dispatch crossovers."""
    img = generate(TestImageSpec(pattern, 4096, 4096, 16, seed=42))
    for k in (3, 17, 27, 49, 75):
        _check_bands(img, filter_image(img, k), k, k)


@pytest.mark.parametrize("pattern", PATTERNS + ("narrow16",))
def test_c4_u32_8192(pattern):
    """C4: 8192^2 uint32, the data-aware regime k = 25..75.  ``narrow16``:
    uniform values below 2^16 stored as uint32 (depth / 16-bit data in a wide
    container -- every sample shares the top bits)."""
    if pattern == "narrow16":
        rng = np.random.default_rng(5)
        img = rng.integers(0, 1 << 16, size=(8192, 8192), dtype=np.uint32)
    else:
        img = generate(TestImageSpec(pattern, 8192, 8192, 32, seed=42))
    for k in (25, 49, 75):
        _check_bands(img, filter_image(img, k), k, k)


@pytest.mark.parametrize("pattern", PATTERNS)
def test_c5_u8_32768(pattern):
    """C5: 32768^2 uint8 (1 GiB) at k = 9 and 33 through the torch path (the
    image is generated on the device; the banded oracle reads row bands)."""
    import torch
    h = w = 32768
    dev = "cuda"
    ys = torch.arange(h, device=dev, dtype=torch.int32)[:, None]
    xs = torch.arange(w, device=dev, dtype=torch.int32)[None, :]
    g = torch.Generator(device=dev).manual_seed(42)
    if pattern == "constant":
        t = torch.full((h, w), 128, device=dev, dtype=torch.uint8)
    elif pattern == "random":
        t = torch.randint(0, 256, (h, w), generator=g, device=dev, dtype=torch.uint8)
    else:
        t = ((xs + ys) & 255).to(torch.uint8)
        if pattern == "impulse":
            u = torch.randint(0, 20, (h, w), generator=g, device=dev, dtype=torch.uint8)
            t[u < 3] = 255  # 15 % salt
            t[(u >= 3) & (u < 6)] = 0  # 15 % pepper
    del xs, ys
    for k in (9, 33):
        out = filter_image(t, k)
        torch.cuda.synchronize()
        hh = k // 2
        for y0, y1 in _bands(h, k, k, n_interior=8, rows=2):
            s0, s1 = max(0, y0 - hh), min(h, y1 + hh)
            img = t[s0:s1].cpu().numpy()
            ref = banded_oracle(img, k, y0 - s0, y1 - s0)
            # the crop's own edges replicate only where they are the image's
            got = out[y0:y1].cpu().numpy()
            assert np.array_equal(got, ref), (pattern, k, y0, y1)
        del out
    del t
    torch.cuda.empty_cache()
