"""Synthetic images rendered on the device (bench inputs, data-sensitivity runs).

The patterns are the reference generator's (reference.py:78-99): ``constant``
(1 << (bits - 1)), ``gradient`` ((x + y) & max), ``random`` (uniform over the
dtype) and ``impulse`` (the gradient with 30 % salt and pepper), drawn with a
seeded torch generator instead of Philox (the bench needs the shapes and
value statistics, not the reference's exact bits; parity tests use the
reference's own generator, oracle.generate).  Extra patterns for the
data-aware kernels: ``narrow16`` (uniform below 2^16 in a wider dtype),
``gentle`` / ``smooth`` (a smooth field with a maximum slope of ~9 / ~95
values per pixel at 16 bits plus Gaussian noise of sigma 200, both scaled with
the dtype range).
"""
from __future__ import annotations

PATTERNS = ("random", "gradient", "impulse", "constant", "narrow16", "gentle", "smooth")


def render(pattern: str, shape, bits: int, seed: int = 42, device="cuda"):
    """A (H, W) or (H, W, C) tensor of uint{bits} on ``device``; channel c of
    a multi-channel image is drawn with seed + c."""
    import torch
    if len(shape) == 3:
        return torch.stack([render(pattern, shape[:2], bits, seed + c, device)
                            for c in range(shape[2])], dim=-1)
    h, w = (int(s) for s in shape)
    tdt = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}[bits]
    mx = (1 << bits) - 1
    g = torch.Generator(device=device).manual_seed(seed)
    if pattern == "constant":
        return torch.full((h, w), 1 << (bits - 1), device=device, dtype=torch.int64).to(tdt)
    if pattern == "random":
        return torch.randint(0, mx + 1, (h, w), generator=g, device=device,
                             dtype=torch.int64).to(tdt)
    if pattern == "narrow16":
        return torch.randint(0, 1 << 16, (h, w), generator=g, device=device,
                             dtype=torch.int64).to(tdt)
    ys = torch.arange(h, device=device, dtype=torch.int64)[:, None]
    xs = torch.arange(w, device=device, dtype=torch.int64)[None, :]
    if pattern in ("gradient", "impulse"):
        t = (xs + ys) & mx
        if pattern == "impulse":
            hit = torch.rand((h, w), generator=g, device=device) < 0.3
            salt = torch.rand((h, w), generator=g, device=device) < 0.5
            t = torch.where(hit & salt, torch.full_like(t, mx), t)
            t = torch.where(hit & ~salt, torch.zeros_like(t), t)
        return t.to(tdt)
    if pattern in ("gentle", "smooth"):
        fx, fy, amp = (1500.0, 1100.0, 0.2) if pattern == "gentle" else (517.0, 311.0, 0.45)
        base = (torch.sin(xs / fx) * torch.cos(ys / fy) + 1.0) * amp * mx
        noise = torch.randn((h, w), generator=g, device=device) * 200.0 * mx / 65535
        return (base + noise + 0.05 * mx).clamp(0, mx).to(torch.int64).to(tdt)
    raise ValueError(f"unknown pattern {pattern!r} (expected one of {PATTERNS})")


def generate_host(pattern: str, width: int, height: int, depth: int = 8, seed: int = 0,
                  density: float = 0.3):
    """The reference's test image, bit for bit (reference.py:78-99): numpy,
    Philox keyed by ``seed`` -- the command line's ``synth:`` inputs."""
    import numpy as np
    if pattern not in ("constant", "gradient", "random", "impulse"):
        raise ValueError(f"unknown pattern {pattern!r} "
                         "(expected one of ('constant', 'gradient', 'random', 'impulse'))")
    if depth not in (8, 16, 32):
        raise ValueError(f"unsupported depth {depth} (expected 8, 16, or 32)")
    if width < 1 or height < 1:
        raise ValueError("image dimensions must be positive")
    if not 0.0 <= density <= 1.0:
        raise ValueError("density must be within [0, 1]")
    dtype = {8: np.uint8, 16: np.uint16, 32: np.uint32}[depth]
    top = np.iinfo(dtype).max
    if pattern == "constant":
        return np.full((height, width), 1 << (depth - 1), dtype=dtype)
    ramp = ((np.arange(height)[:, None] + np.arange(width)[None, :]) & top).astype(dtype)
    if pattern == "gradient":
        return ramp
    rng = np.random.Generator(np.random.Philox(key=seed))
    if pattern == "random":
        return rng.integers(0, top, size=(height, width), endpoint=True, dtype=dtype)
    hit = rng.random(size=ramp.shape) < density
    salt = rng.random(size=ramp.shape) < 0.5
    ramp[hit & salt] = top
    ramp[hit & ~salt] = 0
    return ramp
