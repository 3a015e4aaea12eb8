"""Build the CUDA extension in-tree: codegen + nvcc (sm_100a) -> libtilemedian_b200.so.

    python -m paper_2507_19926_b200.build [-j N] [--force]

Object files go to ``paper_2507_19926_b200/_build/``; the shared library to
``paper_2507_19926_b200/libtilemedian_b200.so`` (git-ignored, shipped to the GPU
box by gpurun).  ``-Xptxas -v`` output (registers, spills, shared memory) is
kept in ``_build/ptxas.log``.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

from . import codegen

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
# experiment builds (e.g. TMB_NVCC_EXTRA=-DTMB_RANK_PROFILE) go elsewhere with
# TMB_BUILD_DIR / TMB_LIB_OUT; the product library is libtilemedian_b200.so
BUILD = os.environ.get("TMB_BUILD_DIR", os.path.join(PKG, "_build"))
LIB = os.environ.get("TMB_LIB_OUT", os.path.join(PKG, "libtilemedian_b200.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-diag-suppress", "177",
         *os.environ.get("TMB_NVCC_EXTRA", "").split()]


def _sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "gen", "*.cu")))


def _headers() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(CSRC, "gen", "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "gen", "*.inc"))
                  + glob.glob(os.path.join(PKG, "..", "include", "*.h")))


def _obj(src: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel[:-3] + ".o")


def _compile(src: str) -> tuple[str, str]:
    obj = _obj(src)
    cmd = [NVCC, *ARCH, *FLAGS, "-MD", "-MF", obj[:-2] + ".d", "-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr[-6000:]}")
    return src, p.stderr


def _deps(obj: str) -> list[str] | None:
    """Headers `obj` was compiled against (nvcc -MD), None when unknown."""
    try:
        text = open(obj[:-2] + ".d").read()
    except OSError:
        return None
    text = text.replace("\\\n", " ")
    _, _, rest = text.partition(":")
    return [d for d in rest.split() if d]


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> str:
    codegen.generate()
    os.makedirs(BUILD, exist_ok=True)
    # a change of compiler flags (e.g. TMB_NVCC_EXTRA) rebuilds everything
    stamp = os.path.join(BUILD, "flags.txt")
    flags = " ".join([NVCC, *ARCH, *FLAGS])
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
        with open(stamp, "w") as f:
            f.write(flags)
    newest_hdr = max((os.path.getmtime(h) for h in _headers()), default=0)
    todo = []
    for src in _sources():
        obj = _obj(src)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < os.path.getmtime(src):
            todo.append(src)
            continue
        deps = _deps(obj)
        t_obj = os.path.getmtime(obj)
        if deps is None:
            stale = t_obj < newest_hdr
        else:
            stale = any(not os.path.exists(d) or os.path.getmtime(d) > t_obj for d in deps)
        if stale:
            todo.append(src)
    # the template-heavy data-aware kernels compile longest: start them first so
    # the many small generated files fill the other cores meanwhile
    heavy = ("tm_rank", "tm_hist", "tm_aware", "tm_select")
    todo.sort(key=lambda src: 0 if os.path.basename(src).startswith(heavy) else 1)
    logs = {}
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(jobs) as pool:
            for src, log in pool.map(_compile, todo):
                logs[src] = log
                if verbose:
                    print(f"compiled {os.path.relpath(src, PKG)}", file=sys.stderr)
        with open(os.path.join(BUILD, "ptxas.log"), "a") as f:
            for src, log in logs.items():
                f.write(f"==== {src}\n{log}\n")
    objs = [_obj(s) for s in _sources()]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr[-4000:]}")
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(a.j, a.force, verbose=True))


if __name__ == "__main__":
    main()
