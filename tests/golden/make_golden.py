"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``tilemedian`` (read-only, never copied) and
records what its own public API returns, so the parity tests can pin both the
CPU oracle restatement (oracle/) and the CUDA path without /root/reference:

* ``matrix.json``   -- the reference's 264-cell oracle-equivalence matrix
  (report.py:104-153, test_acceptance.py:33-46): for every cell the blake2b
  digest of the input image and of ``filter_image(img, k, variant)``.
* ``sweep.json``    -- digests of ``filter_image`` for every odd k in 3..75 on
  small odd-shaped images of each depth (oracle/oblivious/aware as the
  reference routes them), plus rectangular KernelSpec cases (oblivious).
* ``c1_u8_512_k3.npz`` -- config 1 in full: input and output arrays.
* ``model.json``    -- the reference's op model W(k) (oblivious.py:303-326),
  root sizes (geometry.py:89-97), retention windows (geometry.py:259-269),
  network sizes (networks.py:164-262) and frozen aware comparison totals
  (aware.py:495-506).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import tilemedian as tm
from tilemedian.geometry import TileDims
from tilemedian.report import matrix_cells

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.blake2b(digest_size=16)
    h.update(str(a.dtype).encode())
    h.update(repr(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def main() -> None:
    cells = []
    images = {}
    for spec, k, variant in matrix_cells("full"):
        if spec not in images:
            images[spec] = tm.generate(spec)
        img = images[spec]
        out = tm.filter_image(img, k, variant)
        assert np.array_equal(out, tm.oracle_median_filter(img, k))
        cells.append({"pattern": spec.pattern, "width": spec.width, "height": spec.height,
                      "depth": spec.depth, "seed": spec.seed, "density": spec.density,
                      "k": k, "variant": variant,
                      "input": digest(img), "output": digest(out)})
    with open(os.path.join(OUT, "matrix.json"), "w") as f:
        json.dump(cells, f, indent=0)
    print("matrix cells", len(cells), file=sys.stderr)

    sweep = []
    for depth, (w, h) in ((8, (45, 38)), (16, (41, 29)), (32, (23, 31))):
        for pattern in ("random", "impulse"):
            spec = tm.TestImageSpec(pattern, w, h, depth, seed=7)
            img = tm.generate(spec)
            for k in range(3, 77, 2):
                out = tm.filter_image(img, k, "oracle" if k > 31 else "auto")
                sweep.append({"pattern": pattern, "width": w, "height": h, "depth": depth,
                              "seed": 7, "density": 0.3, "k": k,
                              "input": digest(img), "output": digest(out)})
    rect = []
    for (kw, kh) in ((3, 5), (5, 3), (9, 11), (7, 3), (3, 9)):
        spec = tm.TestImageSpec("random", 37, 26, 8, seed=3)
        img = tm.generate(spec)
        try:
            out = tm.filter_image(img, tm.KernelSpec(kw, kh), "oblivious")
            res = digest(out)
        except ValueError as exc:  # e.g. default root 4x4 is wider than a 3-wide kernel
            res = "ValueError: " + str(exc)
        rect.append({"k_w": kw, "k_h": kh, "pattern": "random", "width": 37, "height": 26,
                     "depth": 8, "seed": 3, "density": 0.3,
                     "input": digest(img), "output": res})
    with open(os.path.join(OUT, "sweep.json"), "w") as f:
        json.dump({"square": sweep, "rect": rect}, f, indent=0)
    print("sweep cells", len(sweep), len(rect), file=sys.stderr)

    img = tm.generate(tm.TestImageSpec("random", 512, 512, 8, seed=42))
    out = tm.filter_image(img, 3)
    np.savez_compressed(os.path.join(OUT, "c1_u8_512_k3.npz"), input=img, output=out)

    model = {"W": {}, "root": {}, "ops": {}, "windows": {}, "nets": {}, "aware": {}}
    for k in range(3, 77, 2):
        t = min(tm.root_tile_size(k), 16)
        oc = tm.op_count(tm.compile_plan(k, t))
        model["W"][k] = oc["minmax_per_pixel"]
        model["root"][k] = tm.root_tile_size(k)
        model["ops"][k] = {"tile": list(oc["tile"]), "ops_per_tile": oc["ops_per_tile"],
                           "ops_per_tile_shared": oc["ops_per_tile_shared"],
                           "breakdown": {g: list(v) for g, v in oc["breakdown"].items()}}
    for k in (3, 5, 9, 17, 25):
        for (tw, th) in ((1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (8, 8)):
            if tw > k or th > k:
                continue
            oc = tm.op_count(tm.compile_plan(k, TileDims(tw, th)))
            model["ops"][f"{k}@{tw}x{th}"] = {"ops_per_tile": oc["ops_per_tile"],
                                             "minmax_per_pixel": oc["minmax_per_pixel"]}
    for n_total in (9, 25, 81, 289, 5625):
        model["windows"][n_total] = {
            n: [tm.retention_window(n_total, n).lo, tm.retention_window(n_total, n).hi]
            for n in range(1, n_total + 1, max(1, n_total // 97))}
    for n in range(0, 70):
        model["nets"][f"batcher{n}"] = tm.batcher_sort(n).size()
        model["nets"][f"pairwise{n}"] = tm.pairwise_sort(n).size()
    for p in range(0, 20):
        for q in range(0, 20):
            model["nets"][f"merge{p},{q}"] = tm.oddeven_merge(p, q).size()
    for sizes in ((4, 4, 4), (6, 6, 6, 6, 6, 6), (3, 5, 7), (10,) * 10):
        model["nets"]["multi" + ",".join(map(str, sizes))] = tm.multiway_merge(sizes).size()
    for k in (9, 19):
        model["aware"][k] = tm.comparison_count(k, (64, 64))["total"]
    with open(os.path.join(OUT, "model.json"), "w") as f:
        json.dump(model, f, indent=0)
    print("model done", file=sys.stderr)


if __name__ == "__main__":
    main()
