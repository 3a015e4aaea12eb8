"""Executed warp instructions and stall samples per CUDA source line from an
ncu report (``--print-source cuda,sass`` source page): where a kernel's
instructions go, by line of tm_*.cu(h).

    python tools/ncu_lines.py gpurun_out/r2_c4_k75.ncu-rep [--top 40]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True, check=True).stdout
    inst = collections.Counter()
    stall = collections.Counter()
    text = {}
    path = None
    hdr = None
    cur = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            path = row[1].split("/")[-1]
            continue
        if row[0] in ("Function Name",):
            continue
        if row[0] == "Line No":
            hdr = row
            ie = hdr.index("Instructions Executed")
            se = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None:
            continue
        if row[0]:  # a source line row
            cur = (path, int(row[0]))
            text[cur] = row[1].strip()[:80]
        if len(row) > ie and row[2]:
            try:
                inst[cur] += float(row[ie] or 0)
                stall[cur] += float(row[se] or 0)
            except ValueError:
                pass
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"total warp instructions {ti:.0f}")
    for key, n in inst.most_common(a.top):
        print(f"{100 * n / ti:5.1f}% inst {100 * stall[key] / ts:5.1f}% stall  {key[0]}:{key[1]}  {text.get(key, '')}")


if __name__ == "__main__":
    main()
