"""Thread-pair selection programs: one root tile per PAIR of threads.

For kernels whose per-tile live state does not fit in 255 registers (k >= 15
on 4x4 root tiles, SURVEY.md section 7 "hard part 1"), a root tile is split
between the two threads of a lane pair (lane ^ 1), following the first split
of the tile recursion (section 3.4):

1. root phase, work split in two structurally identical halves:
   * each thread merges HALF of the core columns (multiway merge, full);
   * the halves are exchanged with ``__shfl_xor_sync(.., 1)`` and both threads
     run the same pruned two-way merge of (own, other) down to the core's
     retention window -- merge(A, B) and merge(B, A) give the same values, so
     the instruction stream is identical on both threads;
   * each thread sorts half of the extra rows (top rows / bottom rows, a
     translation in y), rows are exchanged and put back in geometric order
     with one SEL per value;
2. child phase: thread r runs child r's subtree of the first (horizontal)
   split.  The right child is the mirror image of the left child (x -> t_w-1-x),
   and every comparator acts on value multisets, so both threads execute the
   left child's program; the right thread reads its inputs and writes its
   outputs through mirrored addresses.

Per thread that is ~1/2 of the root work (+ the final core merge run twice)
plus one child subtree, with a live state of ~210 values at k = 17 instead of
~320 for the whole tile, so the tile runs without spills.
"""
from __future__ import annotations

from . import networks as nets
from .geometry import TileDims, region, retention_window
from .program import Program, build_program


def _emit_network_block(prog: Program, names: dict, body: list, load_fn) -> None:
    """Emit the live min/max ops of ``prog`` in creation (network) order."""
    alive = prog.live()
    for v, node in enumerate(prog.values):
        if not alive[v] or node[0] not in ("min", "max"):
            continue
        ops = []
        for a in (node[1], node[2]):
            if a not in names:
                names[a] = load_fn(a)
            ops.append(names[a])
        fn = "mn" if node[0] == "min" else "mx"
        names[v] = f"p{v}_{len(body)}"
        body.append(f"    const uint32_t {names[v]} = IO::{fn}({ops[0]}, {ops[1]});")


def emit_pair_program(k: int, tw: int, th: int, name: str) -> tuple[str, dict]:
    dims = TileDims(tw, th)
    if dims.axis != "h" or tw < 2:
        raise ValueError("pair programs split the root tile horizontally")
    full = build_program(k, dims)
    kern = full.kernel
    root = region((0, 0), dims, kern)
    if root.core_w % 2:
        raise ValueError("core width must be even")
    hw = root.core_w // 2
    body: list[str] = []
    stats = {"minmax": 0, "xchg": 0, "sel": 0}

    # ---- 1a. half core merge (thread r: core columns [r*hw, r*hw + hw)) -------
    half = Program(kern, dims)
    xs = list(root.core_xs())[:hw]
    flat = [half.col(x, i) for x in xs for i in range(root.core_h)]
    hvals = half.run(nets.multiway_merge((root.core_h,) * hw), flat, ("core-half", 0),
                     runs=(root.core_h,) * hw)
    half.outputs = [hvals]
    names: dict = {}

    def load_core(v):
        _, x, i = half.values[v]
        nm = f"c{x + 64}_{i}"
        body.append(f"    const uint32_t {nm} = io.col_t({x}, {i});")
        return nm

    _emit_network_block(half, names, body, load_core)
    own = [names[v] for v in hvals]
    stats["minmax"] += half.minmax_count()
    # ---- 1b. exchange halves, merge (own, other) to the core window -----------
    other = []
    for i, nm in enumerate(own):
        body.append(f"    const uint32_t o{i} = io.xchg({nm});")
        other.append(f"o{i}")
    stats["xchg"] += len(own)
    n = len(own)
    fin = Program(kern, dims)
    a_ids = [fin.pix(0, i) for i in range(n)]      # placeholders: own half
    b_ids = [fin.pix(1, i) for i in range(n)]      # placeholders: other half
    merged = fin.run(nets.oddeven_merge(n, n), a_ids + b_ids, ("core-pair", 0), runs=(n, n))
    win = retention_window(kern.count, root.core_w * root.core_h)
    cand_ids = merged[win.lo - 1: win.hi]
    fin.outputs = [cand_ids]
    fnames: dict = {}
    for i in range(n):
        fnames[a_ids[i]] = own[i]
        fnames[b_ids[i]] = other[i]
    _emit_network_block(fin, fnames, body, lambda v: (_ for _ in ()).throw(KeyError(v)))
    stats["minmax"] += fin.minmax_count()
    cand_names = [fnames[v] for v in cand_ids]
    assert len(cand_names) == len(full.root_cand)

    # ---- 1c. extra rows: thread r sorts the top (r=0) / bottom (r=1) rows ------
    ys = root.extra_ys()
    top = ys[: th - 1]
    bottom = ys[th - 1:]
    shift = bottom[0] - top[0]
    assert [y + shift for y in top] == bottom
    rows_prog = Program(kern, dims)
    row_ids = {}
    for y in top:
        row_ids[y] = rows_prog.run(nets.make_sorter(root.core_w),
                                   [rows_prog.pix(x, y) for x in root.core_xs()], ("rowsort", 0))
    rows_prog.outputs = [[v for y in top for v in row_ids[y]]]
    rnames: dict = {}

    def load_row(v):
        _, x, y = rows_prog.values[v]
        nm = f"w{x + 64}_{y + 64}"
        body.append(f"    const uint32_t {nm} = io.pix_t({x}, {y});")
        return nm

    _emit_network_block(rows_prog, rnames, body, load_row)
    stats["minmax"] += rows_prog.minmax_count()
    row_names = {}
    for j, y in enumerate(top):
        yb = y + shift
        tops, bots = [], []
        for i, v in enumerate(row_ids[y]):
            mine = rnames[v]
            oth = f"x{j}_{i}"
            body.append(f"    const uint32_t {oth} = io.xchg({mine});")
            # r = 0 owns the top row, r = 1 the bottom row
            body.append(f"    const uint32_t t{j}_{i} = io.sel({mine}, {oth});")
            body.append(f"    const uint32_t b{j}_{i} = io.sel({oth}, {mine});")
            tops.append(f"t{j}_{i}")
            bots.append(f"b{j}_{i}")
        row_names[y] = tops
        row_names[yb] = bots
        stats["xchg"] += len(tops)
        stats["sel"] += 2 * len(tops)

    # ---- 2. child phase: left child's subtree, mirrored for thread 1 -----------
    leaves = [(x, y) for (x, y) in full.leaf_order if x < tw // 2]
    outs = full.outputs
    full.outputs = [[outs[y][x] for x in range(tw // 2)] for y in range(th)]
    full.leaf_order = leaves
    root_vals = {v for v, lab in full.labels.items() if lab[1] == 0}
    order = [v for v in full.stage_order(eager=True) if v not in root_vals]
    cnames: dict = {}
    for i, v in enumerate(full.root_cand):
        cnames[v] = cand_names[i]
    for y, ids in full.root_rows.items():
        for i, v in enumerate(ids):
            cnames[v] = row_names[y][i]

    def ref(v):
        if v in cnames:
            return cnames[v]
        node = full.values[v]
        if node[0] == "pix":
            nm = f"m{node[1] + 64}_{node[2] + 64}"
            body.append(f"    const uint32_t {nm} = io.pix_m({node[1]}, {node[2]});")
        elif node[0] == "col":
            nm = f"n{node[1] + 64}_{node[2]}"
            body.append(f"    const uint32_t {nm} = io.col_m({node[1]}, {node[2]});")
        else:
            raise KeyError(v)
        cnames[v] = nm
        return nm

    where = {}
    for y, row in enumerate(full.outputs):
        for x, v in enumerate(row):
            where.setdefault(v, []).append((x, y))
    for v in order:
        kind, a, b = full.values[v]
        ra, rb = ref(a), ref(b)
        fn = "mn" if kind == "min" else "mx"
        cnames[v] = f"q{v}"
        body.append(f"    const uint32_t q{v} = IO::{fn}({ra}, {rb});")
        stats["minmax"] += 1
        for (x, y) in where.get(v, ()):
            body.append(f"    io.out_m({x}, {y}, q{v});")
    full.outputs = outs
    head = [f"// generated by paper_2507_19926_b200/pairgen.py -- do not edit",
            f"// kernel {k}x{k}, root tile {tw}x{th} split over a thread pair: "
            f"{stats['minmax']} min/max per thread, {stats['xchg']} shuffles, {stats['sel']} selects",
            f"struct {name} {{",
            "  static constexpr int kSpillSlots = 0;",
            "  static constexpr int kPair = 1;",
            f"  static constexpr int kCoreHalf = {hw};",
            f"  static constexpr int kRowShift = {shift};",
            "  template <class IO>",
            "  __device__ __forceinline__ static void run(IO& io) {"]
    return "\n".join(head + body + ["  }", "};", ""]), stats
