"""Tile geometry of hierarchical tiling (build-time and host-side only).

This is the index arithmetic the CUDA kernels embody; the code generator
(``codegen.py``) and the host dispatcher use it, nothing here runs per pixel.
Semantics follow the reference's ``geometry.py`` (cited per function) so that
generated programs walk exactly the reference's split schedule:

* pixel (x, y), x to the right, y down; a tile anchored at (x0, y0) of
  t_w x t_h owns [x0, x0+t_w) x [y0, y0+t_h);
* a tile splits its width when t_w >= t_h, else its height
  (geometry.py:84-86, section 3.1);
* footprint = union of the tile's windows, core = their intersection, with
  t-1 extra columns/rows per side and (t-1)^2 corner cells per quadrant
  (geometry.py:114-228, Fig. 4).
"""
from __future__ import annotations

from dataclasses import dataclass


def _pow2(v: int) -> bool:
    return v > 0 and not (v & (v - 1))


@dataclass(frozen=True)
class KernelSpec:
    """Odd k_w x k_h window (reference geometry.py:25-58)."""

    k_w: int
    k_h: int

    def __post_init__(self) -> None:
        if any(s < 3 or s % 2 == 0 for s in (self.k_w, self.k_h)):
            raise ValueError(
                f"kernel sides must be odd and >= 3, got {self.k_w}x{self.k_h}")

    @classmethod
    def square(cls, k: int) -> "KernelSpec":
        return cls(k, k)

    @property
    def half_w(self) -> int:
        return self.k_w // 2

    @property
    def half_h(self) -> int:
        return self.k_h // 2

    @property
    def count(self) -> int:
        return self.k_w * self.k_h

    @property
    def median_rank(self) -> int:
        """1-based rank of the median."""
        return (self.count + 1) // 2


def as_kernel(k) -> KernelSpec:
    """int or KernelSpec-like (anything with k_w/k_h) -> KernelSpec."""
    if isinstance(k, KernelSpec):
        return k
    if hasattr(k, "k_w") and hasattr(k, "k_h"):
        return KernelSpec(int(k.k_w), int(k.k_h))
    return KernelSpec.square(int(k))


@dataclass(frozen=True)
class TileDims:
    """Power-of-two tile sides plus depth in the split tree (geometry.py:61-81)."""

    t_w: int
    t_h: int
    depth: int = 0

    def __post_init__(self) -> None:
        if not (_pow2(self.t_w) and _pow2(self.t_h)):
            raise ValueError(f"tile sides must be powers of two, got {self.t_w}x{self.t_h}")
        if self.depth < 0:
            raise ValueError("depth must be non-negative")

    @property
    def area(self) -> int:
        return self.t_w * self.t_h

    @property
    def is_leaf(self) -> bool:
        return self.t_w == 1 and self.t_h == 1

    def split(self) -> "TileDims":
        """Child dims: halve the width when t_w >= t_h, else the height."""
        if self.t_w >= self.t_h:
            return TileDims(self.t_w // 2, self.t_h, self.depth + 1)
        return TileDims(self.t_w, self.t_h // 2, self.depth + 1)

    @property
    def axis(self) -> str:
        """'h' when the next split halves the width (geometry.py:84-86)."""
        return "h" if self.t_w >= self.t_h else "v"


def root_tile_size(k: int) -> int:
    """t(k) = 2**(floor(log2 k) - 1) (geometry.py:89-97, section 4.2)."""
    if k < 3 or k % 2 == 0:
        raise ValueError(f"kernel side must be odd and >= 3, got {k}")
    return 1 << (int(k).bit_length() - 2)


@dataclass(frozen=True)
class Window:
    """Ranks (1-based, among the seen values) that can still hold the median.

    After ``n_seen`` of ``n_total`` values with m unseen, the median is among
    seen ranks [max(1, r-m), min(n_seen, r)] (geometry.py:231-269,
    PAPER.md Fig. 3 "forgetfulness").
    """

    n_total: int
    n_seen: int
    lo: int
    hi: int

    @property
    def count(self) -> int:
        return self.hi - self.lo + 1

    @property
    def d_lo(self) -> int:
        return self.lo - 1


def retention_window(n_total: int, n_seen: int) -> Window:
    if n_total < 1 or n_total % 2 == 0:
        raise ValueError(f"n_total must be odd and positive, got {n_total}")
    if not 1 <= n_seen <= n_total:
        raise ValueError(f"n_seen must be in [1, {n_total}], got {n_seen}")
    r = (n_total + 1) // 2
    unseen = n_total - n_seen
    return Window(n_total, n_seen, max(1, r - unseen), min(n_seen, r))


@dataclass(frozen=True)
class Region:
    """Footprint partition of one tile (geometry.py:203-228).

    Coordinates are relative to the tile anchor.  ``core`` is
    (x0, y0, w, h); extra columns sit left/right of the core at core height,
    extra rows above/below at core width.
    """

    anchor: tuple[int, int]
    dims: TileDims
    kernel: KernelSpec

    @property
    def fp_x0(self) -> int:
        return self.anchor[0] - self.kernel.half_w

    @property
    def fp_y0(self) -> int:
        return self.anchor[1] - self.kernel.half_h

    @property
    def fp_w(self) -> int:
        return self.kernel.k_w + self.dims.t_w - 1

    @property
    def fp_h(self) -> int:
        return self.kernel.k_h + self.dims.t_h - 1

    @property
    def core_x0(self) -> int:
        return self.anchor[0] + self.dims.t_w - 1 - self.kernel.half_w

    @property
    def core_y0(self) -> int:
        return self.anchor[1] + self.dims.t_h - 1 - self.kernel.half_h

    @property
    def core_w(self) -> int:
        return self.kernel.k_w - self.dims.t_w + 1

    @property
    def core_h(self) -> int:
        return self.kernel.k_h - self.dims.t_h + 1

    def core_xs(self) -> range:
        return range(self.core_x0, self.core_x0 + self.core_w)

    def core_ys(self) -> range:
        return range(self.core_y0, self.core_y0 + self.core_h)

    def extra_xs(self) -> list[int]:
        return (list(range(self.fp_x0, self.core_x0))
                + list(range(self.core_x0 + self.core_w, self.fp_x0 + self.fp_w)))

    def extra_ys(self) -> list[int]:
        return (list(range(self.fp_y0, self.core_y0))
                + list(range(self.core_y0 + self.core_h, self.fp_y0 + self.fp_h)))

    def corners(self) -> list[tuple[int, int]]:
        return [(x, y) for y in self.extra_ys() for x in self.extra_xs()]


def region(anchor, dims: TileDims, kernel: KernelSpec) -> Region:
    if dims.t_w > kernel.k_w or dims.t_h > kernel.k_h:
        raise ValueError(
            f"tile {dims.t_w}x{dims.t_h} larger than kernel {kernel.k_w}x{kernel.k_h}")
    return Region(tuple(anchor), dims, kernel)


@dataclass(frozen=True)
class Child:
    """One child of a split (geometry.py:272-338).

    ``gained``: the parent extra columns (h split) or rows (v split) that join
    the child core; ``grown``: per surviving run of the other orientation, the
    parent corner cells it absorbs; ``corners``: corner cells kept as corners.
    """

    region: Region
    gained: tuple[int, ...]
    grown: tuple[tuple[int, tuple[tuple[int, int], ...]], ...]
    corners: tuple[tuple[int, int], ...]


def split(parent: Region) -> tuple[str, tuple[Child, Child]]:
    dims = parent.dims
    if dims.is_leaf:
        raise ValueError("cannot split a 1x1 tile")
    axis = dims.axis
    cd = dims.split()
    ax, ay = parent.anchor
    if axis == "h":
        anchors = ((ax, ay), (ax + cd.t_w, ay))
    else:
        anchors = ((ax, ay), (ax, ay + cd.t_h))
    kids = []
    for a in anchors:
        ch = region(a, cd, parent.kernel)
        if axis == "h":
            old = set(parent.core_xs())
            gained = tuple(x for x in ch.core_xs() if x not in old)
            grown = tuple((y, tuple((x, y) for x in gained)) for y in ch.extra_ys())
        else:
            old = set(parent.core_ys())
            gained = tuple(y for y in ch.core_ys() if y not in old)
            grown = tuple((x, tuple((x, y) for y in gained)) for x in ch.extra_xs())
        kids.append(Child(ch, gained, grown, tuple(ch.corners())))
    return axis, (kids[0], kids[1])


def tile_grid(width: int, height: int, dims: TileDims) -> tuple[int, int]:
    """Number of root tiles (cols, rows) covering an image (geometry.py:341-361)."""
    if width < 1 or height < 1:
        raise ValueError(f"image dims must be positive, got {width}x{height}")
    return -(-width // dims.t_w), -(-height // dims.t_h)
