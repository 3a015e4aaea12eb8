"""Summarise one kernel launch of an ncu report into profiles/ncu_<config>_k<k>.json.

    python tools/ncu_summary.py gpurun_out/c2_hist.ncu-rep --samples 90316800 \
        --config c2 --k 17 --source "ncu --set full ... (command)" [--out profiles/ncu_c2_k17.json]

Reads ``ncu -i <rep> --page raw --csv`` (works without a GPU) and keeps the
numbers the bench and DESIGN.md quote: duration, DRAM bytes, warp
instructions (per sample), IPC, issue-slot and warp occupancy, shared-memory
pipe use, registers, grid, and the top stall reasons per issued instruction.
"""
import argparse
import csv
import io
import json
import subprocess


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units, data = rows[0], rows[1], rows[2:]
    return header, units, data


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--samples", type=int, required=True, help="output samples per launch")
    ap.add_argument("--config", required=True)
    ap.add_argument("--k", type=int, required=True)
    ap.add_argument("--source", default="")
    ap.add_argument("--launch", type=int, default=0, help="row of the report (launch index)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    header, units, data = raw_rows(a.rep)
    row = data[a.launch]
    m = {h: row[i] for i, h in enumerate(header)}
    u = {h: units[i] for i, h in enumerate(header)}

    def g(name, scale=1.0):
        v = num(m.get(name))
        return None if v is None else v * scale

    def bytes_of(name):
        v = num(m.get(name))
        if v is None:
            return None
        unit = u.get(name, "byte").lower()
        mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "b": 1, "kb": 1e3,
                "mb": 1e6, "gb": 1e9}.get(unit, 1)
        return v * mult

    def ms_of(name):
        v = num(m.get(name))
        if v is None:
            return None
        unit = u.get(name, "nsecond").lower()
        return v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                    "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1e-6)

    rd, wr = bytes_of("dram__bytes_read.sum"), bytes_of("dram__bytes_write.sum")
    inst = g("smsp__inst_executed.sum")
    stalls = {}
    for h in header:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            v = num(m[h])
            if v:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
    top = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    res = {
        "source": a.source,
        "kernel": m.get("Kernel Name", m.get("Function Name", "")),
        "config": a.config, "k": a.k,
        "dram_bytes_per_launch": None if rd is None or wr is None else int(rd + wr),
        "dram_read_mb": None if rd is None else round(rd / 1e6, 2),
        "dram_write_mb": None if wr is None else round(wr / 1e6, 2),
        "duration_ms_under_ncu": ms_of("gpu__time_duration.sum"),
        "sm_cycles_elapsed": g("sm__cycles_elapsed.avg"),
        "warp_instructions": inst,
        "warp_instructions_per_sample": None if inst is None else round(inst / a.samples, 3),
        "ipc_per_sm": g("sm__inst_executed.avg.per_cycle_active"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "shared_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "shared_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "registers_per_thread": g("launch__registers_per_thread"),
        "grid_size": g("launch__grid_size"),
        "block_size": g("launch__block_size"),
        "occupancy_limit_shared_mem": g("launch__occupancy_limit_shared_mem"),
        "stall_per_issue_top": top,
        "samples_per_launch": a.samples,
        "note": a.note,
    }
    text = json.dumps(res, indent=2)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
