"""CUDA code generator for the oblivious selection programs (build time).

Emits, under ``csrc/gen/``:

* ``colsort.cuh``       -- ``ColSortN`` structs: full sorting networks for the
  cooperative column sorts (network policy of ``networks.make_sorter``);
* ``obl_<cfg>.cuh``     -- one ``Prog_*`` struct per (kernel, root tile): the
  pruned straight-line min/max program of ``program.build_program`` in
  demand-driven order, loading each input from shared memory at first use;
* ``obl_inst_<bits>.cu`` -- kernel instantiations + launchers per dtype;
* ``dispatch.inc``      -- the (bits, k) -> launcher table used by the C ABI.

The per-k configuration (root tile per thread, CTA shape) lives in
``OBLIVIOUS_CONFIGS``; ``tools/`` scripts and the bench can override it.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

from . import networks as nets
from .geometry import TileDims
from .program import build_program

HERE = os.path.dirname(os.path.abspath(__file__))
GEN_DIR = os.path.join(HERE, "csrc", "gen")


@dataclass(frozen=True)
class OblConfig:
    k: int
    tw: int
    th: int
    bx: int  # tiles per CTA row (per lane)
    by: int  # tile rows per CTA (per lane); == tw for conflict-free loads
    regs: int = 0  # register budget for program values; 0 = no explicit spilling
    pair: bool = False  # split each root tile over a thread pair (pairgen.py)

    @property
    def name(self) -> str:
        return f"k{self.k}_t{self.tw}x{self.th}" + ("p" if self.pair else "")

    @property
    def threads(self) -> int:
        return self.bx * self.by


# Square kernels served by the register-resident oblivious kernel.
OBLIVIOUS_CONFIGS = {
    3: OblConfig(3, 2, 2, 64, 2),
    5: OblConfig(5, 4, 4, 32, 4),  # 4x4: +5 % over 4x2 (round-1 config search)
    7: OblConfig(7, 4, 4, 32, 4),  # 4x4: +2 %
    9: OblConfig(9, 4, 2, 32, 4),
    11: OblConfig(11, 4, 4, 64, 4),  # 4x4: +7 %, 64-wide CTA +7 %; k = 9 stays 4x2 (4x4: -11 %)
    13: OblConfig(13, 4, 4, 64, 4),  # 64-wide CTA: +9 %
    15: OblConfig(15, 4, 4, 32, 4, pair=True),  # pair: +32 % over one thread per tile
    # k >= 15: a 4x4 root tile's live state exceeds the register file of one
    # thread -- split each tile over a thread pair (pairgen.py)
    17: OblConfig(17, 4, 4, 32, 4, pair=True),
    19: OblConfig(19, 4, 4, 32, 4, pair=True),
    21: OblConfig(21, 4, 4, 32, 4, pair=True),
    23: OblConfig(23, 4, 4, 32, 4, pair=True),
    25: OblConfig(25, 4, 4, 32, 4, pair=True),
    27: OblConfig(27, 4, 4, 32, 4, pair=True),
}

DTYPES = {8: "uint8_t", 16: "uint16_t", 32: "uint32_t"}


def configs_from_env():
    """TMB_OBL_CONFIGS="17:4x4:32x4,15:4x4:32x4" overrides the table (experiments)."""
    spec = os.environ.get("TMB_OBL_CONFIGS")
    if not spec:
        return dict(OBLIVIOUS_CONFIGS)
    out = {}
    for item in spec.split(","):
        parts = item.split(":")
        k, t, b = parts[:3]
        regs = int(parts[3]) if len(parts) > 3 and parts[3] != "p" else 0
        pair = "p" in parts[3:]
        tw, th = map(int, t.split("x"))
        bx, by = map(int, b.split("x"))
        out[int(k)] = OblConfig(int(k), tw, th, bx, by, regs, pair)
    return out


def dtypes_from_env():
    spec = os.environ.get("TMB_DTYPES")
    if not spec:
        return dict(DTYPES)
    return {int(b): DTYPES[int(b)] for b in spec.split(",")}


def emit_colsort(n: int) -> str:
    lines = [f"struct ColSort{n} {{",
             "  template <class L>",
             f"  __device__ __forceinline__ static void run(uint32_t (&v)[{n}]) {{"]
    for i, j in nets.make_sorter(n):
        lines.append(f"    {{ const uint32_t a = v[{i}], b = v[{j}]; "
                     f"v[{i}] = L::mn(a, b); v[{j}] = L::mx(a, b); }}")
    lines += ["  }", "};", ""]
    return "\n".join(lines)


def allocate(prog, order, budget: int):
    """Linear-scan placement of SSA values with an explicit shared-memory spill.

    Walks the emission order keeping at most ``budget`` values in registers.
    When full it evicts the value whose next use is furthest away (Belady):
    program inputs (raw pixels, sorted columns) are simply dropped and
    re-read from their home in shared memory; computed values are stored once
    into a per-thread spill slot (slot-major, thread-fastest layout: conflict
    free) and reloaded before their next use.  Returns an event list for the
    emitter and the number of spill slots.  ``budget <= 0`` disables it.
    """
    INF = float("inf")
    uses: dict[int, list[int]] = {}
    pos_of = {}
    for i, v in enumerate(order):
        pos_of[v] = i
        _, a, b = prog.values[v]
        uses.setdefault(a, []).append(i)
        uses.setdefault(b, []).append(i)
    outputs = {v for row in prog.outputs for v in row}
    ptr = {v: 0 for v in uses}

    def next_use(v, i):
        lst = uses.get(v, ())
        k = ptr.get(v, 0)
        while k < len(lst) and lst[k] < i:
            k += 1
        ptr[v] = k
        return lst[k] if k < len(lst) else INF

    regs: set[int] = set()
    slot_of: dict[int, int] = {}
    free_slots: list[int] = []
    n_slots = 0
    events = []

    def is_input(v):
        return prog.values[v][0] in ("pix", "col")

    def evict(i, keep):
        nonlocal n_slots
        best, best_d = None, -1
        for r in regs:
            if r in keep:
                continue
            d = next_use(r, i)
            # dropping an input is cheaper than spilling: prefer it on ties
            key = (d, 1 if is_input(r) else 0)
            if best is None or key > best_d:
                best, best_d = r, key
        regs.discard(best)
        if not is_input(best) and best not in slot_of and best_d[0] != INF:
            if free_slots:
                sl = free_slots.pop()
            else:
                sl = n_slots
                n_slots += 1
            slot_of[best] = sl
            events.append(("spill", best, sl))

    def ensure(v, i, keep):
        if v in regs:
            return
        if budget > 0:
            while len(regs) >= budget:
                evict(i, keep)
        if is_input(v):
            events.append(("load", v))
        else:
            events.append(("reload", v, slot_of[v]))
        regs.add(v)

    for i, v in enumerate(order):
        _, a, b = prog.values[v]
        ensure(a, i, {a, b})
        ensure(b, i, {a, b})
        if budget > 0:
            while len(regs) >= budget:
                evict(i, {a, b})
        events.append(("op", v))
        regs.add(v)
        for x in (a, b):
            if next_use(x, i + 1) == INF:
                regs.discard(x)
                if x in slot_of:
                    free_slots.append(slot_of.pop(x))
        if v in outputs:
            events.append(("out", v))
            if next_use(v, i + 1) == INF:
                regs.discard(v)
    return events, n_slots


def emit_program(cfg: OblConfig) -> tuple[str, dict]:
    prog = build_program(cfg.k, TileDims(cfg.tw, cfg.th))
    order = prog.stage_order(eager=True)
    name = f"Prog_{cfg.name}"
    events, n_slots = allocate(prog, order, cfg.regs)
    where = {}
    for y, row in enumerate(prog.outputs):
        for x, v in enumerate(row):
            where[v] = (x, y)
    cur: dict[int, str] = {}
    body = []
    counter = [0]
    stats = {"minmax": 0, "loads": 0, "spills": 0, "reloads": 0}

    def fresh(v):
        counter[0] += 1
        nm = f"r{counter[0]}"
        cur[v] = nm
        return nm

    for ev in events:
        kind = ev[0]
        if kind == "load":
            v = ev[1]
            node = prog.values[v]
            fn = "pix" if node[0] == "pix" else "col"
            body.append(f"    const uint32_t {fresh(v)} = io.{fn}({node[1]}, {node[2]});")
            stats["loads"] += 1
        elif kind == "reload":
            v, sl = ev[1], ev[2]
            body.append(f"    const uint32_t {fresh(v)} = io.reload({sl});")
            stats["reloads"] += 1
        elif kind == "spill":
            v, sl = ev[1], ev[2]
            body.append(f"    io.spill({sl}, {cur[v]});")
            stats["spills"] += 1
        elif kind == "op":
            v = ev[1]
            op, a, b = prog.values[v]
            fn = "mn" if op == "min" else "mx"
            ra, rb = cur[a], cur[b]
            body.append(f"    const uint32_t {fresh(v)} = IO::{fn}({ra}, {rb});")
            stats["minmax"] += 1
        else:  # out
            v = ev[1]
            x, y = where[v]
            body.append(f"    io.out({x}, {y}, {cur[v]});")
    head = [f"// generated by paper_2507_19926_b200/codegen.py -- do not edit",
            f"// kernel {cfg.k}x{cfg.k}, root tile {cfg.tw}x{cfg.th}: {stats['minmax']} min/max per"
            f" tile, {stats['loads']} input loads, {stats['spills']} spills / {stats['reloads']}"
            f" reloads over {n_slots} slots (register budget {cfg.regs})",
            f"struct {name} {{",
            f"  static constexpr int kSpillSlots = {n_slots};",
            "  static constexpr int kPair = 0;",
            "  static constexpr int kCoreHalf = 0;",
            "  static constexpr int kRowShift = 0;",
            "  template <class IO>",
            "  __device__ __forceinline__ static void run(IO& io) {"]
    stats.update({"peak_live": prog.peak_live(order), "colsort_minmax": prog.colsort_minmax(),
                  "slots": n_slots})
    return "\n".join(head + body + ["  }", "};", ""]), stats


def _write(path: str, text: str) -> None:
    old = None
    if os.path.exists(path):
        with open(path) as f:
            old = f.read()
    if old != text:
        with open(path, "w") as f:
            f.write(text)


def generate(configs=None) -> dict:
    """Write all generated sources; returns per-config stats."""
    configs = configs_from_env() if configs is None else dict(configs)
    dtypes = dtypes_from_env()
    os.makedirs(GEN_DIR, exist_ok=True)
    stats = {}
    col_lens = sorted({c.k - c.th + 1 for c in configs.values()})
    _write(os.path.join(GEN_DIR, "colsort.cuh"),
           "// generated -- column sorting networks\n#pragma once\n#include <cstdint>\n"
           "namespace tmb {\n" + "".join(emit_colsort(n) for n in col_lens) + "}  // namespace tmb\n")
    for cfg in configs.values():
        if cfg.pair:
            from .pairgen import emit_pair_program
            text, st = emit_pair_program(cfg.k, cfg.tw, cfg.th, f"Prog_{cfg.name}")
        else:
            text, st = emit_program(cfg)
        stats[cfg.k] = st
        _write(os.path.join(GEN_DIR, f"obl_{cfg.name}.cuh"),
               "#pragma once\n#include <cstdint>\nnamespace tmb {\n" + text + "}  // namespace tmb\n")
    import glob as _glob
    wanted = set()
    for bits, ctype in DTYPES.items():
        if bits not in dtypes:
            continue
        for cfg in configs.values():
            ch = cfg.k - cfg.th + 1
            fname = f"obl_inst_u{bits}_{cfg.name}.cu"
            wanted.add(fname)
            _write(os.path.join(GEN_DIR, fname), "\n".join([
                "// generated -- oblivious kernel instantiation",
                '#include "../tm_oblivious.cuh"', '#include "../tm_launch.cuh"',
                '#include "colsort.cuh"', f'#include "obl_{cfg.name}.cuh"', "namespace tmb {",
                f"int launch_obl_u{bits}_k{cfg.k}(const Job& job, cudaStream_t s) {{",
                f"  return launch_oblivious<{ctype}, {cfg.k}, {cfg.k}, {cfg.tw}, {cfg.th}, "
                f"{cfg.bx}, {cfg.by}, Prog_{cfg.name}, ColSort{ch}>(job, s);", "}",
                "}  // namespace tmb", ""]))
    for stale in _glob.glob(os.path.join(GEN_DIR, "obl_inst_*.cu")):
        if os.path.basename(stale) not in wanted:
            os.remove(stale)
    decl = ["// generated -- oblivious launch table (included inside namespace tmb)"]
    for bits in dtypes:
        for cfg in configs.values():
            decl.append(f"int launch_obl_u{bits}_k{cfg.k}(const Job&, cudaStream_t);")
    decl.append("static const OblEntry kOblTable[] = {")
    for bits in dtypes:
        for cfg in configs.values():
            decl.append(f"  {{{bits}, {cfg.k}, {cfg.tw}, {cfg.th}, &launch_obl_u{bits}_k{cfg.k}}},")
    decl.append("};")
    _write(os.path.join(GEN_DIR, "dispatch.inc"), "\n".join(decl) + "\n")
    return stats


if __name__ == "__main__":
    for k, st in generate().items():
        print(k, st)
