"""Command line: ``python -m paper_2507_19926_b200.cli filter ...`` (reference cli.py:33-56).

``filter`` reads a P5 / P6 / MF32 file (or renders ``synth:PATTERN:WxH:DEPTH``
with the reference's generator), runs the drop-in ``filter_planes`` on the GPU
and writes the result in the matching container -- the reference's
``tilemedian filter`` with the same options, usage errors (exit status 2) and
output line.  ``networks`` writes every comparator network the oblivious
kernels execute in the reference's network-file format (for its
``tilemedian verify --network-file``).
"""
from __future__ import annotations

import argparse
import os
import sys

from . import pnm
from .engine import VARIANTS, filter_planes
from .model import AWARE_MIN_KERNEL
from .synth import generate_host

PATTERNS = ("constant", "gradient", "random", "impulse")


def _synth(token: str, seed: int, density: float):
    parts = token.split(":")
    if len(parts) != 4:
        raise ValueError("expected synth:PATTERN:WxH:DEPTH")
    _, pattern, size, depth = parts
    w, _, h = size.partition("x")
    return generate_host(pattern, int(w), int(h), int(depth), seed=seed, density=density)


def cmd_filter(args, parser) -> int:
    if args.k < 3 or args.k % 2 == 0:
        parser.error(f"--k must be an odd diameter >= 3, got {args.k}")
    if args.variant == "aware" and args.k < AWARE_MIN_KERNEL:
        parser.error(f"the aware engine needs k >= {AWARE_MIN_KERNEL}; "
                     f"use --variant oblivious for k={args.k}")
    try:
        image = (_synth(args.infile, args.seed, args.density) if args.infile.startswith("synth:")
                 else pnm.read_image(args.infile))
    except (OSError, ValueError) as exc:
        parser.error(f"cannot read {args.infile}: {exc}")
    checksums = [] if args.dump_checksums else None
    kw = {"device": args.device}
    if args.devices:
        kw["devices"] = [int(d) for d in args.devices.split(",")]
    out = filter_planes(image, args.k, args.variant, root=args.root, workers=args.workers,
                        slice_budget=args.slice_budget, checksums=checksums, **kw)
    if checksums:
        print("\n".join(checksums))
    pnm.write_image(args.out, out)
    print(f"wrote {args.out}: {out.shape[1]}x{out.shape[0]} "
          f"{out.dtype.name} k={args.k} variant={args.variant}")
    return 0


def cmd_networks(args, parser) -> int:
    from .netexport import export
    os.makedirs(args.dir, exist_ok=True)
    nets = export()
    for name, e in nets.items():
        with open(os.path.join(args.dir, name + ".net"), "w") as f:
            f.write(e["text"])
    print(f"wrote {len(nets)} networks to {args.dir}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="tilemedian-b200",
        description="Exact median filtering on B200 (hierarchical tiling, arXiv 2507.19926).")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("filter", help="median-filter an image file")
    p.add_argument("--in", dest="infile", required=True,
                   help="input image (P5/P6/MF32), or synth:PATTERN:WxH:DEPTH "
                        f"with PATTERN one of {'/'.join(PATTERNS)}")
    p.add_argument("--out", required=True, help="output image path")
    p.add_argument("--k", type=int, required=True, help="odd kernel diameter")
    p.add_argument("--variant", choices=VARIANTS, default="auto")
    p.add_argument("--root", type=int, default=None, help="override the root tile edge length")
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--slice-budget", type=int, default=None, metavar="BYTES",
                   help="device bytes per band of the host path")
    p.add_argument("--seed", type=int, default=0, help="seed for synth: inputs")
    p.add_argument("--density", type=float, default=0.3,
                   help="impulse fraction for synth:impulse inputs")
    p.add_argument("--dump-checksums", action="store_true",
                   help="print the finalize-pass checksums (aware engine)")
    p.add_argument("--device", type=int, default=0, help="GPU ordinal")
    p.add_argument("--devices", default=None, help="comma-separated GPUs: one row band each")
    p.set_defaults(func=cmd_filter)
    p = sub.add_parser("networks", help="write the kernels' comparator networks (.net files)")
    p.add_argument("--dir", required=True)
    p.set_defaults(func=cmd_networks)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    return args.func(args, parser)


if __name__ == "__main__":
    sys.exit(main())
