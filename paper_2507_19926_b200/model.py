"""Shape-only work models of the reference engines (host side, no pixels).

The reference instruments its engines with data-independent comparison
counts; they are part of its public API (``ComparisonCounter``,
``comparison_count``; aware.py:31-45, 135-160, 495-506) and of the
roofline definition (W(k), oblivious.py:303-326 -- see ``program.op_model``).
The B200 kernels do different (and fewer) operations, so these numbers are
*models*: they are computed here in closed form from the image shape, the
kernel size and the band plan, exactly as the reference's aware engine would
accumulate them (aware.py:239-413, band plan aware.py:437-463), so that
``filter_image(..., "aware", counter=c)`` ticks like the reference
(test_engine.py:28-32).
"""
from __future__ import annotations

from .geometry import retention_window, root_tile_size
from .networks import make_sorter

AWARE_MIN_KERNEL = 9  # reference aware.py:28


class ComparisonCounter:
    """Accumulates model comparison counts grouped by label (aware.py:31-45)."""

    def __init__(self):
        self.total = 0
        self.by_label: dict[str, int] = {}

    def add(self, label: str, n) -> None:
        n = int(n)
        self.total += n
        self.by_label[label] = self.by_label.get(label, 0) + n

    def absorb(self, other: "ComparisonCounter") -> None:
        for label, n in other.by_label.items():
            self.add(label, n)


def _kway_cost(sizes) -> int:
    """Binary-reduction merge: p + q - 1 per pairwise merge of non-empty runs."""
    sizes = list(sizes)
    cost = 0
    while len(sizes) > 1:
        nxt = []
        for a, b in zip(sizes[0::2], sizes[1::2]):
            if a and b:
                cost += a + b - 1
            nxt.append(a + b)
        if len(sizes) % 2:
            nxt.append(sizes[-1])
        sizes = nxt
    return cost


def _trimmed_merge_cost(p: int, q: int, out: int) -> int:
    return min(p + q - 1, out + (min(p, q) + 1).bit_length())


def _sorter_cost(n: int) -> int:
    return len(make_sorter(n)) if n > 1 else 0


def validate_aware_root(k: int, root) -> int:
    """Root tile side of the aware engine (aware.py:228-236)."""
    if k % 2 == 0 or k < AWARE_MIN_KERNEL:
        raise ValueError(
            f"data-aware engine handles odd k >= {AWARE_MIN_KERNEL}; "
            f"got {k} (small kernels belong to the oblivious engine)")
    t = max(root_tile_size(k), 2) if root is None else int(root)
    if t < 2 or t & (t - 1) or t > k:
        raise ValueError(f"root tile side must be a power of two in [2, {k}], got {t}")
    return t


def peak_bytes(k: int, t: int, W: int, band_rows: int, itemsize: int) -> int:
    """The reference's buffer bound for a band of root-tile rows (aware.py:416-434)."""
    H_band = band_rows * t
    n_cx, n_cy = -(-W // t), band_rows
    n_y = H_band + k
    peak, s = 0, t
    while s >= 2:
        c = k - s + 1
        win = retention_window(k * k, c * c)
        level = n_cx * n_y * c + n_cy * W * c + n_cy * n_cx * win.count
        if s == 2:
            level += H_band * W * (win.count + 2 * k - 1)
        peak = max(peak, level)
        n_cx, n_cy, s = 2 * n_cx, 2 * n_cy, s // 2
    return peak * itemsize


def aware_bands(H: int, W: int, k: int, t: int, itemsize: int, workers: int = 1,
                slice_budget=None) -> list[tuple[int, int]]:
    """Band plan in root-tile rows (aware.py:455-463)."""
    n_ty = -(-H // t)
    band_rows = n_ty
    if slice_budget is not None:
        band_rows = 1
        while band_rows < n_ty and peak_bytes(k, t, W, band_rows + 1, itemsize) <= slice_budget:
            band_rows += 1
    if workers > 1:
        band_rows = min(band_rows, max(1, -(-n_ty // workers)))
    return [(a, min(a + band_rows, n_ty)) for a in range(0, n_ty, band_rows)]


def aware_band_counts(H: int, W: int, k: int, t: int, ty0: int, ty1: int,
                      counter: ComparisonCounter) -> None:
    """Model counts of one band (pass_init / pass_extend_level / pass_finalize)."""
    half = k // 2
    c = k - t + 1
    n_tx = -(-W // t)
    n_cy = ty1 - ty0
    py0 = ty0 * t
    n_y = min(H - 1, ty1 * t - 1 + half) - max(0, py0 - half) + 1
    n_total = k * k
    if c > 1:
        counter.add("rowsort", _sorter_cost(c) * n_tx * n_y)
        counter.add("colsort", _sorter_cost(c) * n_cy * W)
    counter.add("core", _kway_cost((c,) * c) * n_cy * n_tx)
    win = retention_window(n_total, c * c)
    n_cand = win.count
    s, n_cx = t, n_tx
    while s > 2:
        g = s // 2
        c = k - s + 1
        c2 = c + g
        counter.add("pack", _kway_cost((c,) * g) * n_cy * 2 * n_cx)
        w = retention_window(n_total, c2 * c)
        counter.add("cand", _trimmed_merge_cost(n_cand, g * c, w.count) * n_cy * 2 * n_cx)
        n_cand = w.count
        if g > 1:
            counter.add("cornerpack", _sorter_cost(g) * 2 * n_cx * n_y)
        counter.add("extend", (c + g - 1) * 2 * n_cx * n_y)
        counter.add("pack", _kway_cost((c2,) * g) * 2 * n_cy * 2 * n_cx)
        w2 = retention_window(n_total, c2 * c2)
        counter.add("cand", _trimmed_merge_cost(n_cand, g * c2, w2.count) * 2 * n_cy * 2 * n_cx)
        n_cand = w2.count
        if g > 1:
            counter.add("cornerpack", _sorter_cost(g) * 2 * n_cy * W)
        counter.add("extend", (c + g - 1) * 2 * n_cy * W)
        n_cy, n_cx, s = 2 * n_cy, 2 * n_cx, g
    c = k - 1
    out_h = min(n_cy * 2, H - py0)
    counter.add("finalize", (n_cand + c - 1 + c + n_cand + 2 * c) * out_h * W)


def aware_counts(H: int, W: int, k: int, root=None, itemsize: int = 1, workers: int = 1,
                 slice_budget=None, counter: ComparisonCounter | None = None) -> ComparisonCounter:
    counter = ComparisonCounter() if counter is None else counter
    t = validate_aware_root(k, root)
    for ty0, ty1 in aware_bands(H, W, k, t, itemsize, workers, slice_budget):
        sub = ComparisonCounter()
        aware_band_counts(H, W, k, t, ty0, ty1, sub)
        counter.absorb(sub)
    return counter


def comparison_count(k, shape=(128, 128), root=None) -> dict:
    """Model comparisons per pixel (aware.py:495-506)."""
    c = aware_counts(shape[0], shape[1], int(k), root)
    return {"k": int(k), "comparisons_per_pixel": c.total / (shape[0] * shape[1]),
            "by_label": dict(c.by_label), "total": c.total}
