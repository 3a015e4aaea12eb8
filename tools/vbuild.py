"""Experiment builds: recompile a few sources with extra nvcc flags into a
variant library, reusing the product build's objects for everything else.

    python tools/vbuild.py NAME "-DTMB_HIST_WPC=1" csrc/tm_hist.cu [...]

-> paper_2507_19926_b200/libtilemedian_b200_NAME.so (load it with
TMB_LIB=<path>; tools/sweep.py and bench.py go through _lib.load()).
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_19926_b200 import build as B  # noqa: E402


def main():
    name, extra, srcs = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
    B.build()  # the product objects are current
    vdir = os.path.join(B.PKG, "_build_v", name)
    os.makedirs(vdir, exist_ok=True)
    objs = []
    targets = {os.path.abspath(os.path.join(B.PKG, s)) for s in srcs}
    jobs = []
    for src in B._sources():
        obj = B._obj(src)
        if os.path.abspath(src) in targets:
            vobj = os.path.join(vdir, os.path.basename(obj))
            jobs.append([B.NVCC, *B.ARCH, *B.FLAGS, *extra, "-c", src, "-o", vobj])
            objs.append(vobj)
        else:
            objs.append(obj)
    with cf.ThreadPoolExecutor(max(1, len(jobs))) as pool:  # one nvcc per source
        for p in pool.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs):
            if p.returncode:
                raise SystemExit(p.stderr[-4000:])
            with open(os.path.join(vdir, "ptxas.log"), "a") as f:
                f.write(p.stderr)
    lib = os.path.join(B.PKG, f"libtilemedian_b200_{name}.so")
    p = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"],
                       capture_output=True, text=True)
    if p.returncode:
        raise SystemExit(p.stderr[-4000:])
    print(lib)


if __name__ == "__main__":
    main()
