"""Data-oblivious selection programs in SSA form (build time only).

``build_program(k, tile)`` produces the straight-line min/max program one CUDA
thread runs for one root tile of the oblivious kernel.  It follows the
hierarchical-tiling recursion of the reference (oblivious.py:124-237,
PAPER.md sections 3.3-3.4):

1. inputs are the tile footprint's raw pixels and the footprint columns
   sorted at core height -- the column sorts are done cooperatively by the
   whole CTA and shared between horizontally adjacent tiles, so they are
   program *inputs* (oblivious.py:133-144, 368-376);
2. extra rows are sorted per tile (oblivious.py:146-151);
3. the core columns are merged (multiway merge) and immediately trimmed to
   the retention window (oblivious.py:155-163, geometry.py:259-269);
4. every split merges the gained runs into a pack, merges the pack with the
   candidate window (trimmed again), and grows the surviving runs of the other
   orientation by their sorted corner cells (oblivious.py:167-227);
5. at each 1x1 leaf the window is a single value -- the median.

Every comparator becomes a ``min`` and a ``max`` SSA value; global dead-code
elimination from the leaf medians is the reference's backward pruning
(oblivious.py:240-255): a compare-exchange with one dead side becomes a single
min or max, one with both sides dead disappears.

``op_model(k)`` reproduces the reference's op model W(k)
(oblivious.py:303-326): min/max instructions per pixel with column sorts
amortised over t_w; the test-suite pins it against the reference's numbers.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import networks as nets
from .geometry import (KernelSpec, Region, TileDims, as_kernel, region,
                       retention_window, root_tile_size, split)

MAX_TILE_AREA = 256       # reference oblivious.py:49
RECORD = None             # netexport: list collecting every network application
DRIVER_ROOT_CAP = 16      # reference oblivious.py:50


@dataclass
class Program:
    kernel: KernelSpec
    tile: TileDims
    # value table: index -> tuple; ('pix', x, y) | ('col', x, i) | ('min'|'max', a, b)
    values: list = field(default_factory=list)
    outputs: list = field(default_factory=list)  # [t_h][t_w] value ids
    _memo: dict = field(default_factory=dict)
    trace: list = field(default_factory=list)    # (label, seen, lo, hi) per candidate merge
    leaf_order: list = field(default_factory=list)  # (x, y) of leaves in split-tree DFS order
    labels: dict = field(default_factory=dict)      # value id -> (stage kind, node depth)
    stage_of: dict = field(default_factory=dict)    # value id -> network application index
    n_stages: int = 0
    companions: dict = field(default_factory=dict)  # stage -> sibling stages to emit with it
    root_cand: list = field(default_factory=list)   # value ids of the root candidate window
    root_rows: dict = field(default_factory=dict)   # y -> value ids of the root's sorted extra rows
    _label: tuple = ("input", -1)

    cse: bool = True

    def _mk(self, node: tuple) -> int:
        if not self.cse and node[0] in ("min", "max"):
            self.values.append(node)
            return len(self.values) - 1
        got = self._memo.get(node)
        if got is None:
            got = len(self.values)
            self.values.append(node)
            self._memo[node] = got
        return got

    def pix(self, x: int, y: int) -> int:
        return self._mk(("pix", x, y))

    def col(self, x: int, i: int) -> int:
        return self._mk(("col", x, i))

    def run(self, net, wires: list[int], label=None, runs=None) -> list[int]:
        """Apply network ``net`` to ``wires``; ``runs`` = the sorted input runs
        of a merge (None for a sort) -- what the stage claims, for netexport."""
        w = list(wires)
        lab = label or self._label
        st = self.n_stages
        self.n_stages += 1
        if RECORD is not None:
            RECORD.append((self, lab, tuple(net), None if runs is None else tuple(runs),
                           tuple(wires)))
        for i, j in net:
            a, b = w[i], w[j]
            w[i] = self._mk(("min", a, b))
            w[j] = self._mk(("max", a, b))
            for v in (w[i], w[j]):
                self.labels.setdefault(v, lab)
                self.stage_of.setdefault(v, st)
        return w

    # ---- analysis -----------------------------------------------------
    def live(self) -> list[bool]:
        alive = [False] * len(self.values)
        stack = [v for row in self.outputs for v in row]
        while stack:
            v = stack.pop()
            if alive[v]:
                continue
            alive[v] = True
            node = self.values[v]
            if node[0] in ("min", "max"):
                stack.append(node[1])
                stack.append(node[2])
        return alive

    def minmax_count(self) -> int:
        alive = self.live()
        return sum(1 for v, node in enumerate(self.values)
                   if alive[v] and node[0] in ("min", "max"))

    def input_counts(self) -> dict:
        alive = self.live()
        out = {"pix": 0, "col": 0}
        for v, node in enumerate(self.values):
            if alive[v] and node[0] in out:
                out[node[0]] += 1
        return out

    def colsort_minmax(self) -> int:
        """Min/max per full column sort at core height (all CEs kept)."""
        return 2 * len(nets.make_sorter(self.kernel.k_h - self.tile.t_h + 1))

    def order(self) -> list[int]:
        """Demand-driven emission order: post-order DFS from the leaf medians.

        Each live min/max is emitted right before its first consumer needs
        it, leaf by leaf, which keeps live ranges short (the DAG is tree-like:
        siblings share their ancestors' candidate windows and runs).  Inputs
        are not listed; the code generator loads them at first use.
        """
        done = [False] * len(self.values)
        out: list[int] = []
        leaves = self.leaf_order or [(x, y) for y in range(self.tile.t_h)
                                     for x in range(self.tile.t_w)]
        for (lx, ly) in leaves:
            root = self.outputs[ly][lx]
            if True:
                stack = [(root, False)]
                while stack:
                    v, expanded = stack.pop()
                    if done[v]:
                        continue
                    node = self.values[v]
                    if node[0] not in ("min", "max"):
                        done[v] = True
                        continue
                    if expanded:
                        done[v] = True
                        out.append(v)
                    else:
                        stack.append((v, True))
                        stack.append((node[2], False))
                        stack.append((node[1], False))
        return out

    def stage_order(self, eager: bool = True) -> list[int]:
        """Demand-driven over network applications, creation order inside each.

        Post-order DFS over the stage DAG from the leaf medians (split-tree
        order): a stage (one sorting/merging network) is emitted right before
        the first stage that needs it, and its comparators in network order,
        which keeps a merge's live set at its wire count instead of the
        ~2x that per-output demand order costs.
        """
        alive = self.live()
        ops_of: dict[int, list[int]] = {}
        preds: dict[int, set] = {}
        for v, node in enumerate(self.values):
            if not alive[v] or node[0] not in ("min", "max"):
                continue
            st = self.stage_of[v]
            ops_of.setdefault(st, []).append(v)
            for a in (node[1], node[2]):
                sa = self.stage_of.get(a)
                if sa is not None and sa != st:
                    preds.setdefault(st, set()).add(sa)
        done = set()
        out: list[int] = []
        leaves = self.leaf_order or [(x, y) for y in range(self.tile.t_h)
                                     for x in range(self.tile.t_w)]
        for (lx, ly) in leaves:
            root = self.stage_of.get(self.outputs[ly][lx])
            if root is None:
                continue
            stack = [(root, False)]
            while stack:
                st, expanded = stack.pop()
                if st in done:
                    continue
                if expanded:
                    done.add(st)
                    out.extend(ops_of.get(st, ()))
                    # eager siblings: a split's second candidate merge runs right
                    # after the first, so the parent window dies before descending
                    for comp in self.companions.get(st, ()) if eager else ():
                        if comp not in done:
                            stack.append((comp, False))
                else:
                    stack.append((st, True))
                    for p in sorted(preds.get(st, ()), reverse=True):
                        if p not in done:
                            stack.append((p, False))
        return out

    def peak_live(self, order=None) -> int:
        """Peak simultaneously-live values (inputs count from first use)."""
        order = self.order() if order is None else order
        pos = {v: i for i, v in enumerate(order)}
        first, last = {}, {}
        for i, v in enumerate(order):
            node = self.values[v]
            for a in (node[1], node[2]):
                first.setdefault(a, i)
                last[a] = i
        end = len(order)
        for row in self.outputs:
            for v in row:
                last[v] = end
        events = []
        for v in set(first) | set(pos):
            start = pos.get(v, first.get(v))
            events.append((start, 1))
            events.append((last.get(v, start) + 0.5, -1))
        events.sort()
        cur = peak = 0
        for _, d in events:
            cur += d
            peak = max(peak, cur)
        return peak


def build_program(k, tile=None, cse: bool = True, remat: bool = False,
                  trim: bool = False) -> Program:
    """Selection program for kernel ``k`` and root tile ``tile`` (TileDims or side).

    ``remat``: the second child of every split sorts its grown runs straight
    from the raw pixels (shared-memory inputs) instead of merging its
    parent's computed runs with the absorbed corners, so no computed run of
    the parent stays live across the first child's subtree.  Costs a little
    more min/max (sort(n) instead of merge(n - g, g)), cuts the DFS live
    state -- the quantity that decides whether a tile fits in 255 registers.
    """
    kern = as_kernel(k)
    if tile is None:
        tile = min(root_tile_size(max(kern.k_w, kern.k_h)), DRIVER_ROOT_CAP)
    dims = tile if isinstance(tile, TileDims) else TileDims(int(tile), int(tile))
    if dims.area > MAX_TILE_AREA:
        raise ValueError(f"tile {dims.t_w}x{dims.t_h} exceeds {MAX_TILE_AREA} outputs")
    root = region((0, 0), dims, kern)
    prog = Program(kern, dims, cse=cse)
    n_total = kern.count

    # a run = (sorted SSA values, raw cells it covers, computed?)
    col_runs = {x: ([prog.col(x, i) for i in range(root.core_h)],
                    [(x, y) for y in root.core_ys()], False)
                for x in range(root.fp_x0, root.fp_x0 + root.fp_w)}
    row_sorter = nets.make_sorter(root.core_w)
    row_runs = {}
    for y in root.extra_ys():
        cells = [(x, y) for x in root.core_xs()]
        row_runs[y] = (prog.run(row_sorter, [prog.pix(*c) for c in cells], ("rowsort", 0)),
                       cells, True)
    corners = {c: prog.pix(*c) for c in root.corners()}

    seen = root.core_w * root.core_h
    win = retention_window(n_total, seen)
    flat = [v for x in root.core_xs() for v in col_runs[x][0]]
    merged = prog.run(nets.multiway_merge((root.core_h,) * root.core_w), flat, ("core", 0),
                      runs=(root.core_h,) * root.core_w)
    cand = merged[win.lo - 1: win.hi]
    prog.root_cand = list(cand)
    prog.root_rows = {y: list(r[0]) for y, r in row_runs.items()}
    prog.trace.append(("core", seen, win.lo, win.hi))
    leaves: dict = {}

    def descend(reg: Region, cols, rows, corn, cand, d_lo, seen):
        if reg.dims.is_leaf:
            assert seen == n_total and len(cand) == 1
            leaves[reg.anchor] = cand[0]
            return
        axis, kids = split(reg)
        cand_stages = []
        for ki, kid in enumerate(kids):
            dep = kid.region.dims.depth
            src = cols if axis == "h" else rows
            runs = [src[key][0] for key in kid.gained]
            if len(runs) == 1:
                pack = runs[0]
            else:
                sizes = tuple(len(r) for r in runs)
                pack = prog.run(nets.multiway_merge(sizes), [v for r in runs for v in r],
                                ("pack", dep), runs=sizes)
            seen2 = seen + len(pack)
            w = retention_window(n_total, seen2)
            lo, hi = w.lo - 1 - d_lo, w.hi - 1 - d_lo
            assert 0 <= lo <= hi < len(cand) + len(pack)
            ca, pa = list(cand), list(pack)
            if trim:
                # drop inputs that provably sit above / below the kept window:
                # x[i] lands at merged position i .. i + len(other)
                lo_a = max(0, lo - len(pa))          # cand[i], i < lo_a: always below
                lo_b = max(0, lo - len(ca))
                ca = ca[lo_a: hi + 1]
                pa = pa[lo_b: hi + 1]
                lo, hi = lo - lo_a - lo_b, hi - lo_a - lo_b
            both = prog.run(nets.oddeven_merge(len(ca), len(pa)), ca + pa, ("cand", dep),
                            runs=(len(ca), len(pa)))
            cand_stages.append(prog.n_stages - 1)
            if len(cand_stages) == 2:
                prog.companions[cand_stages[0]] = [cand_stages[1]]
            kid_cand = both[lo: hi + 1]
            prog.trace.append((f"cand {kid.region.dims.t_w}x{kid.region.dims.t_h}",
                               seen2, w.lo, w.hi))
            other = rows if axis == "h" else cols
            grown = {}
            for key, cells in kid.grown:
                base, bcells, computed = other[key]
                allcells = list(bcells) + list(cells)
                if remat and ki == 1 and computed:
                    vals = prog.run(nets.make_sorter(len(allcells)),
                                    [prog.pix(*c) for c in allcells], ("rowsort", dep))
                else:
                    add = [corn[c] for c in cells]
                    if len(add) > 1:
                        add = prog.run(nets.make_sorter(len(add)), add, ("cornersort", dep))
                    vals = prog.run(nets.oddeven_merge(len(base), len(add)), base + add,
                                    ("extend", dep), runs=(len(base), len(add)))
                grown[key] = (vals, allcells, True)
            if axis == "h":
                kcols = {x: cols[x] for x in kid.region.extra_xs()}
                krows = grown
            else:
                kcols = grown
                krows = {y: rows[y] for y in kid.region.extra_ys()}
            descend(kid.region, kcols, krows, {c: corn[c] for c in kid.corners},
                    kid_cand, w.lo - 1, seen2)

    descend(root, {x: col_runs[x] for x in root.extra_xs()}, row_runs, corners,
            cand, win.lo - 1, seen)
    prog.outputs = [[leaves[(x, y)] for x in range(dims.t_w)] for y in range(dims.t_h)]
    prog.leaf_order = list(leaves)
    return prog


def op_model(k, tile=None) -> dict:
    """Reference op model: min/max per pixel, column sorts amortised over t_w."""
    prog = build_program(k, tile, cse=False)
    t_w, t_h = prog.tile.t_w, prog.tile.t_h
    per_tile = prog.minmax_count() + t_w * prog.colsort_minmax()
    return {"k": prog.kernel.k_w, "tile": (t_w, t_h),
            "minmax_per_tile_shared": per_tile,
            "minmax_per_pixel": per_tile / (t_w * t_h),
            "program_minmax": prog.minmax_count()}
