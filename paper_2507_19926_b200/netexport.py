"""Export the comparator networks the oblivious CUDA kernels run (build-time tooling).

Every network application of every generated selection program (the
``Prog_*`` structs of ``codegen.py`` / ``pairgen.py``: row / corner sorts,
core and pack multiway merges, trimmed candidate merges, run extensions) and
every cooperative column sort (``ColSort*``) is written in the reference's
network-description format (``WIRES n`` / ``CE i j`` / ``MIN i j`` /
``MAX i j``, reference networks.py:603-641) *as the kernel executes it*:
after the program's global dead-code elimination, so a compare-exchange with
one dead side appears as MIN or MAX and fully dead ones are gone (the
reference's backward pruning, networks.py:297-328).  Each file carries its
claim in the reference's vocabulary (networks.py:347-376): the live output
wires must hold those ranks of the inputs -- over every 0/1 input for sorts,
over sorted-run inputs for merges.

``tools/verify_networks.py`` proves the claims with the reference's own
``verify_zero_one`` (networks.py:488-567) and records the results with each
network's SHA-256 in ``tests/golden/networks.json``; ``tests/test_networks_golden.py``
regenerates the networks and pins them to those verified digests.
"""
from __future__ import annotations

import hashlib

from . import networks as nets

CE, MIN, MAX = "CE", "MIN", "MAX"


def _stage_text(prog, label, net, runs, wires, alive) -> tuple[str, dict] | None:
    w = list(wires)
    ops = []
    for i, j in net:
        a, b = w[i], w[j]
        mn = prog._memo.get(("min", a, b))
        mx = prog._memo.get(("max", a, b))
        la = mn is not None and alive[mn]
        lb = mx is not None and alive[mx]
        if la and lb:
            ops.append((CE, i, j))
        elif la:
            ops.append((MIN, i, j))
        elif lb:
            ops.append((MAX, i, j))
        w[i], w[j] = mn, mx
    ranks = [p for p in range(len(w)) if w[p] is not None and alive[w[p]]]
    if not ranks:
        return None
    claim = {"kind": "ranks", "ranks": ranks, "runs": list(runs) if runs else None}
    lines = [f"# {label[0]} stage: live wires carry these ranks of the inputs"
             + (f" (inputs: sorted runs {list(runs)})" if runs else " (any inputs)"),
             f"# ranks {' '.join(map(str, ranks))}",
             f"WIRES {len(w)}"]
    lines += [f"{k} {i} {j}" for k, i, j in ops]
    return "\n".join(lines) + "\n", claim


def _colsort_text(n: int) -> tuple[str, dict]:
    lines = [f"# ColSort{n}: full sort of a column (cooperative column sort)",
             f"WIRES {n}"]
    lines += [f"CE {i} {j}" for i, j in nets.make_sorter(n)]
    return "\n".join(lines) + "\n", {"kind": "sorted", "ranks": None, "runs": None}


def export(configs=None) -> dict:
    """{name: {"text", "claim", "sha256", "wires", "ops", "used_by"}} for every
    distinct network the generated kernels execute."""
    from . import codegen, pairgen, program
    configs = codegen.OBLIVIOUS_CONFIGS if configs is None else configs
    out: dict = {}

    def add(text, claim, user):
        sha = hashlib.sha256(text.encode()).hexdigest()
        for name, e in out.items():
            if e["sha256"] == sha:
                if user not in e["used_by"]:
                    e["used_by"].append(user)
                return
        first = text.splitlines()[0]
        kind = first.split()[1].rstrip(":")
        wires = int([ln for ln in text.splitlines() if ln.startswith("WIRES")][0].split()[1])
        name = f"{kind}_{wires}w_{sha[:10]}"
        out[name] = {"text": text, "claim": claim, "sha256": sha, "wires": wires,
                     "ops": sum(1 for ln in text.splitlines() if ln[:2] in ("CE", "MI", "MA")),
                     "used_by": [user]}

    for cfg in sorted(configs.values(), key=lambda c: c.k):
        rec: list = []
        program.RECORD = rec
        try:
            if cfg.pair:
                pairgen.emit_pair_program(cfg.k, cfg.tw, cfg.th, f"Prog_{cfg.name}")
            else:
                codegen.emit_program(cfg)
        finally:
            program.RECORD = None
        alive_of: dict = {}
        for prog, label, net, runs, wires in rec:
            if id(prog) not in alive_of:
                alive_of[id(prog)] = prog.live()
            got = _stage_text(prog, label, net, runs, wires, alive_of[id(prog)])
            if got is not None:
                add(got[0], got[1], f"Prog_{cfg.name}")
        text, claim = _colsort_text(cfg.k - cfg.th + 1)
        add(text, claim, f"ColSort{cfg.k - cfg.th + 1}")
    return out
