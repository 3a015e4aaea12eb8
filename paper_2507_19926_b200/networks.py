"""Comparator networks for the generated selection programs (build time only).

A network is a tuple of (i, j) compare-exchange pairs over ``n`` wires: after
the pair, wire i holds min and wire j holds max (ties never move a value,
reference networks.py:79-81).  Pruning to single-sided MIN/MAX ops is not done
here: the program builder (``program.py``) works in SSA form, where global
dead-code elimination performs exactly the reference's backward pruning
(networks.py:297-328, oblivious.py:240-255).

Constructions are the standard published ones, realised with the same
pad-and-drop rule as the reference (networks.py:129-162) so comparator
counts agree with the reference's op model:

* ``oddeven_sort``   -- Batcher's odd-even merge sort (networks.py:164-170);
* ``oddeven_merge``  -- Batcher's odd-even merge of two sorted runs of any
  sizes: first run padded in front with -inf, second behind with +inf, to a
  common power of two (networks.py:173-191);
* ``multiway_merge`` -- balanced binary reduction of two-way merges
  (networks.py:199-231);
* ``pairwise_sort``  -- Parberry's pairwise sorting network
  (networks.py:234-262), used above 64 wires (``make_sorter``, :265-279).
"""
from __future__ import annotations

from functools import lru_cache

Net = tuple[tuple[int, int], ...]


def _pow2_at_least(n: int) -> int:
    p = 1
    while p < n:
        p <<= 1
    return p


def _merge_positions(n: int) -> list[tuple[int, int]]:
    """Odd-even merge of the two sorted halves of n = 2^m positions.

    Iterative form: distance d runs n/2, n/4, ..., 1.  At d = n/2 every i is
    compared with i + d; below that, positions i and i + d are compared when
    i sits in an odd slot of its 2d-block pattern (Knuth 5.3.4 exercise 11).
    """
    out: list[tuple[int, int]] = []
    half = n // 2
    d = half
    while d >= 1:
        if d == half:
            out.extend((i, i + d) for i in range(half))
        else:
            # compare positions a, a+d where a = d + 2d*m + r, r < d
            for base in range(d, n - d, 2 * d):
                for r in range(d):
                    a = base + r
                    if a + d < n:
                        out.append((a, a + d))
        d //= 2
    return out


def _sort_positions(n: int) -> list[tuple[int, int]]:
    """Odd-even merge sort of n = 2^m positions: sort halves, then merge."""
    out: list[tuple[int, int]] = []
    size = 2
    while size <= n:
        for start in range(0, n, size):
            out.extend((start + a, start + b) for a, b in _merge_positions(size))
        size *= 2
    return out


@lru_cache(maxsize=None)
def oddeven_sort(n: int) -> Net:
    if n < 0:
        raise ValueError("n must be non-negative")
    if n <= 1:
        return ()
    m = _pow2_at_least(n)
    # +inf pads sit at positions >= n: comparators touching them never move
    return tuple((a, b) for a, b in _sort_positions(m) if b < n)


@lru_cache(maxsize=None)
def oddeven_merge(p: int, q: int) -> Net:
    """Merge a sorted p-run on wires [0, p) with a sorted q-run on [p, p+q)."""
    if p < 0 or q < 0:
        raise ValueError("run lengths must be non-negative")
    if p == 0 or q == 0:
        return ()
    half = _pow2_at_least(max(p, q))
    lead = half - p  # -inf pads in front of run A

    def wire(pos: int):
        if pos < lead:
            return None
        if pos < half:
            return pos - lead
        if pos < half + q:
            return p + pos - half
        return None

    out = []
    for a, b in _merge_positions(2 * half):
        wa, wb = wire(a), wire(b)
        if wa is not None and wb is not None:
            out.append((wa, wb))
    return tuple(out)


@lru_cache(maxsize=None)
def multiway_merge(sizes: tuple[int, ...]) -> Net:
    """Merge back-to-back sorted runs by pairwise reduction, rounds of pairs."""
    runs = []
    off = 0
    for s in sizes:
        if s < 0:
            raise ValueError("run sizes must be non-negative")
        if s:
            runs.append((off, s))
        off += s
    ops: list[tuple[int, int]] = []
    while len(runs) > 1:
        nxt = []
        for a in range(0, len(runs) - 1, 2):
            (o1, l1), (o2, l2) = runs[a], runs[a + 1]
            ops.extend((o1 + i, o1 + j) for i, j in oddeven_merge(l1, l2))
            nxt.append((o1, l1 + l2))
        if len(runs) % 2:
            nxt.append(runs[-1])
        runs = nxt
    return tuple(ops)


def _pairwise_positions(pos: list[int]) -> list[tuple[int, int]]:
    n = len(pos)
    if n <= 1:
        return []
    out = [(pos[i], pos[i + 1]) for i in range(0, n, 2)]
    out += _pairwise_positions(pos[0::2])
    out += _pairwise_positions(pos[1::2])
    s = n // 4
    while s >= 1:
        out += [(pos[2 * j + 1], pos[2 * (j + s)]) for j in range(n // 2 - s)]
        s //= 2
    return out


@lru_cache(maxsize=None)
def pairwise_sort(n: int) -> Net:
    if n < 0:
        raise ValueError("n must be non-negative")
    if n <= 1:
        return ()
    m = _pow2_at_least(n)
    return tuple((a, b) for a, b in _pairwise_positions(list(range(m))) if a < n and b < n)


def make_sorter(n: int) -> Net:
    """Full sorter policy: Batcher up to 64 wires, pairwise above."""
    return oddeven_sort(n) if n <= 64 else pairwise_sort(n)


def apply_network(net: Net, values: list) -> list:
    """Scalar evaluation (tests / verification)."""
    v = list(values)
    for i, j in net:
        if v[j] < v[i]:
            v[i], v[j] = v[j], v[i]
    return v


def to_text(net: Net, n: int) -> str:
    """Reference network-file text (networks.py:603-641): WIRES / CE lines."""
    return "\n".join([f"WIRES {n}"] + [f"CE {i} {j}" for i, j in net]) + "\n"
