"""Build-time generator and work models pinned against the reference's numbers."""
import json
import random

import pytest

from golden_util import load
from paper_2507_19926_b200 import networks as nets
from paper_2507_19926_b200.geometry import (KernelSpec, TileDims, region, retention_window,
                                            root_tile_size, split)
from paper_2507_19926_b200.model import comparison_count
from paper_2507_19926_b200.program import build_program, op_model

MODEL = load("model.json")


def test_network_sizes_match_reference():
    for key, size in MODEL["nets"].items():
        if key.startswith("batcher"):
            got = len(nets.oddeven_sort(int(key[7:])))
        elif key.startswith("pairwise"):
            got = len(nets.pairwise_sort(int(key[8:])))
        elif key.startswith("merge"):
            p, q = map(int, key[5:].split(","))
            got = len(nets.oddeven_merge(p, q))
        else:
            got = len(nets.multiway_merge(tuple(map(int, key[5:].split(",")))))
        assert got == size, key


def test_networks_sort_and_merge():
    rnd = random.Random(0)
    for n in range(1, 80):
        net = nets.make_sorter(n)
        for _ in range(10):
            x = [rnd.randrange(6) for _ in range(n)]
            assert nets.apply_network(net, x) == sorted(x)
    for p in range(0, 13):
        for q in range(0, 13):
            for _ in range(5):
                a = sorted(rnd.randrange(5) for _ in range(p))
                b = sorted(rnd.randrange(5) for _ in range(q))
                assert nets.apply_network(nets.oddeven_merge(p, q), a + b) == sorted(a + b)


def test_zero_one_exhaustive_small():
    # zero-one principle: a network sorts all inputs iff it sorts all 0/1 inputs
    for n in range(2, 13):
        net = nets.make_sorter(n)
        for m in range(1 << n):
            x = [(m >> i) & 1 for i in range(n)]
            assert nets.apply_network(net, x) == sorted(x)


@pytest.mark.parametrize("k", list(range(3, 77, 2)))
def test_op_model_matches_reference(k):
    """W(k): the reference's min/max per pixel (oblivious.py:303-326)."""
    om = op_model(k)
    assert om["minmax_per_pixel"] == pytest.approx(MODEL["W"][str(k)], abs=1e-9)


def test_op_model_other_roots():
    for key, ref in MODEL["ops"].items():
        if "@" not in key:
            continue
        k, t = key.split("@")
        tw, th = map(int, t.split("x"))
        assert op_model(int(k), TileDims(tw, th))["minmax_per_pixel"] == pytest.approx(
            ref["minmax_per_pixel"], abs=1e-9), key


def test_program_is_exact_on_random_footprints():
    """run the SSA program on random footprints vs brute force (test_oblivious.py:142-151)."""
    rnd = random.Random(1)
    for k, (tw, th) in ((3, (2, 2)), (5, (4, 2)), (7, (4, 2)), (9, (4, 4)), (9, (4, 2))):
        prog = build_program(k, TileDims(tw, th))
        reg = region((0, 0), prog.tile, prog.kernel)
        for trial in range(40):
            hi = 8 if trial % 2 else 1000  # low entropy exercises ties
            fp = {(x, y): rnd.randrange(hi) for x in range(reg.fp_x0, reg.fp_x0 + reg.fp_w)
                  for y in range(reg.fp_y0, reg.fp_y0 + reg.fp_h)}
            val = {}
            for v, node in enumerate(prog.values):
                if node[0] == "pix":
                    val[v] = fp[(node[1], node[2])]
                elif node[0] == "col":
                    col = sorted(fp[(node[1], y)] for y in reg.core_ys())
                    val[v] = col[node[2]]
                else:
                    a, b = val.get(node[1]), val.get(node[2])
                    if a is not None and b is not None:
                        val[v] = min(a, b) if node[0] == "min" else max(a, b)
            for y in range(th):
                for x in range(tw):
                    win = sorted(fp[(x + dx, y + dy)] for dx in range(-(k // 2), k // 2 + 1)
                                 for dy in range(-(k // 2), k // 2 + 1))
                    assert val[prog.outputs[y][x]] == win[len(win) // 2], (k, x, y)


def test_retention_schedule_golden_k9():
    """test_acceptance.py:78-99: the compiled program walks the frozen schedule."""
    frozen = {36: (1, 36), 48: (8, 41), 64: (24, 41), 72: (32, 41), 81: (41, 41)}
    for n, (lo, hi) in frozen.items():
        w = retention_window(81, n)
        assert (w.lo, w.hi) == (lo, hi)
    prog = build_program(9)
    walked = sorted({(seen, (lo, hi)) for _, seen, lo, hi in prog.trace})
    assert walked == sorted(frozen.items())


def test_retention_windows_golden():
    for n_total, table in MODEL["windows"].items():
        for n, (lo, hi) in table.items():
            w = retention_window(int(n_total), int(n))
            assert (w.lo, w.hi) == (lo, hi)


def test_root_sizes_golden():
    for k, t in MODEL["root"].items():
        assert root_tile_size(int(k)) == t
    assert [root_tile_size(k) for k in (3, 9, 15, 31)] == [1, 4, 4, 8]


def test_split_geometry_k9():
    """test_acceptance.py:78-84: 4x4 -> 2x4 -> 2x2 and the cores they expose."""
    reg = region((0, 0), TileDims(4, 4), KernelSpec.square(9))
    assert (reg.core_w, reg.core_h) == (6, 6)
    axis, kids = split(reg)
    assert axis == "h" and (kids[0].region.core_w, kids[0].region.core_h) == (8, 6)
    axis2, grand = split(kids[0].region)
    assert axis2 == "v" and (grand[0].region.core_w, grand[0].region.core_h) == (8, 8)
    assert len(kids[0].gained) == 2 and len(grand[0].gained) == 2


def test_comparison_counts_frozen():
    """Frozen aware totals (test_aware.py:262-275)."""
    assert comparison_count(9, (64, 64))["total"] == 419072 == MODEL["aware"]["9"]
    assert comparison_count(19, (64, 64))["total"] == 1025984 == MODEL["aware"]["19"]


def test_kernel_spec_validation():
    with pytest.raises(ValueError, match="odd"):
        KernelSpec(4, 3)
    with pytest.raises(ValueError, match="powers of two"):
        TileDims(3, 4)
    with pytest.raises(ValueError, match="larger than kernel"):
        region((0, 0), TileDims(4, 4), KernelSpec(3, 9))
