"""Benchmark of the hot path: exact median filtering on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--k K]
                    [--mode frames|bands] [--impl ours|reference]

Default workload (N=1): BASELINE.json configs[1], the paper's teaser -- a
30-MP RGB photo (4480 x 6720 x 3, uint8, interleaved HWC), every channel
filtered separately with a 17 x 17 median (``filter_planes``).  Synthetic
uniform-random pixels (no datasets offline).  A step is one filter of one
image.  Metric: Gpixel/s counting every channel sample (90.3 M per image),
whole job over all ranks.

Timing: W untimed warm-up steps, then K timed steps; before each timed step
a 512 MiB buffer is written to flush the 126 MB L2 (the input, 90 MB, would
otherwise stay L2-resident), and each step is bracketed by CUDA events on the
launching stream; the timed region is bracketed by a barrier and
torch.cuda.synchronize(); the reported time is the max over ranks.

Multi-GPU (torchrun, NCCL): --mode frames (default) gives every rank its own
frame (batch of frames split across GPUs, no communication, weak scaling);
--mode bands splits ONE image into row bands and exchanges the k/2-row halo
with the neighbours over NCCL before filtering (strong scaling).

Extra keys: roofline (the dominant kernel: the issue roofline from the
config's ncu capture, HBM at k = 3), roofline_model
(W(k) op model), roofline_hbm, e2e (the Python drop-in filter_planes on a
numpy input in pinned host memory, copies included), e2e_pageable (the same
on pageable memory), e2e_pinned_cabi (the raw C ABI), cpu_baseline (the C
oracle port on the host cores, bounded sample, doubling as the parity
self-check), gpu_launches, clocks (NVML sampled during the timed region).

--impl reference times the reference algorithm's CPU implementation (the
oracle port, oracle/median_oracle.c, all host threads) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (height, width, channels, bits, default k, label)
    "c1": (512, 512, 1, 8, 3, "uint8 512x512 grayscale"),
    "c2": (4480, 6720, 3, 8, 17, "uint8 30-MP RGB photo (4480x6720x3 HWC), channels filtered separately"),
    "c3": (4096, 4096, 1, 16, 25, "uint16 4096x4096"),
    "c4": (8192, 8192, 1, 32, 25, "uint32 8192x8192"),
    "c5": (32768, 32768, 1, 8, 9, "uint8 32768x32768 row-band sharded"),
}
METRIC = "Gpixel/s (channel samples) median filter"
MINMAX_PEAK_TPS = 18.6e12   # thread-level VIMNMX per s: profiles/r01_minmax_microbench.txt


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    NVML (pynvml) every 2 ms when available -- the timed region of the default
    run is tens of milliseconds -- else nvidia-smi every 100 ms.
    """

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set of active reasons)
        self._stop = threading.Event()
        self._t = None
        self.source = "nvidia-smi"

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(mx), {n for n, b in bits.items() if r & b}))
            self._stop.wait(0.002)

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) >= 6 and f[0].replace(".", "").isdigit():
                    self.samples.append((float(f[0]), float(f[1]),
                                         {self.NAMES[i] for i in range(4)
                                          if f[i + 2].lower().startswith("active")}))
            except Exception:
                return
            self._stop.wait(0.1)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.source = "nvml"
            try:
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # the first sample lands before the timed region starts (NVML init
        # takes longer than a short timed region)
        t0 = time.time()
        while not self.samples and self._t.is_alive() and time.time() - t0 < 5.0:
            time.sleep(0.001)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted(set().union(*(s[2] for s in self.samples)))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.samples),
                "source": self.source}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def cpu_baseline(cfg, k, seconds=10.0, threads=None, src=None, ours=None):
    """The C oracle port (the reference algorithm, reference.py:26-43) on a
    crop of the workload sized for ~`seconds` of host work, all host threads.

    With ``src`` / ``ours`` (the bench's device input and GPU output) the crop
    is cut from the real input -- rows around the image middle, columns from
    the left edge -- and the oracle's result is compared with the GPU output
    on the same pixels: the bench's parity self-check.
    """
    from oracle import load_c_oracle  # test infrastructure: reported baseline / checker only
    import ctypes
    H, W, C, bits, _, _ = cfg
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    threads = threads or len(os.sched_getaffinity(0))
    lib = load_c_oracle()
    rng = np.random.default_rng(1)
    h = k // 2
    width = min(W, 2048)
    cw = min(W, width + h)          # crop columns (left edge = the image edge)
    valid_w = W if cw == W else cw - h
    check = {"pixels": 0, "mismatches": 0}

    def crop(rows):
        y0 = max(0, H // 2 - rows // 2)
        s0, s1 = max(0, y0 - h), min(H, y0 + rows + h)
        if src is None:
            img = rng.integers(0, np.iinfo(dt).max, size=(s1 - s0, cw, C), dtype=dt, endpoint=True)
        else:
            t = src[s0:s1, :cw]
            img = t.cpu().numpy().astype(dt).reshape(s1 - s0, cw, C)
        return y0, s0, img

    def run(rows, verify=False):
        y0, s0, img = crop(rows)
        planes = [np.ascontiguousarray(img[..., c]) for c in range(C)]
        outs = [np.empty((rows, cw), dtype=dt) for _ in range(C)]
        t0 = time.perf_counter()
        for c in range(C):
            base = outs[c].ctypes.data - (y0 - s0) * cw * planes[c].itemsize
            rc = lib.oracle_median2d(ctypes.c_void_p(planes[c].ctypes.data), cw,
                                     ctypes.c_void_p(base), cw, cw, planes[c].shape[0],
                                     bits, k, k, y0 - s0, y0 - s0 + rows, threads)
            assert rc == 0
        dt_s = time.perf_counter() - t0
        if verify and ours is not None:
            got = ours[y0:y0 + rows, :valid_w].cpu().numpy().astype(dt).reshape(rows, valid_w, C)
            for c in range(C):
                check["pixels"] += rows * valid_w
                check["mismatches"] += int((got[..., c] != outs[c][:, :valid_w]).sum())
        return dt_s

    rows = 8
    dt_s = run(rows)
    while dt_s < 0.25 and rows < H:
        rows = min(H, rows * 4)
        dt_s = run(rows)
    rows = max(1, min(H, int(rows * min(seconds, 2.0) / max(dt_s, 1e-6))))
    # repeat the crop until `seconds` of work; report the median repetition
    reps, total = [], 0.0
    while total < seconds or len(reps) < 3:
        t = run(rows, verify=not reps)
        reps.append(t)
        total += t
    dt_s = statistics.median(reps)
    samples = rows * cw * C
    res = {"value": samples / dt_s / 1e9, "unit": "Gpixel/s", "cores": threads, "kind": "port",
           "cpu_model": cpu_model(),
           "sample": f"{rows}x{cw}x{C} crop of the same workload (rows around the middle, "
                     f"columns from the left edge; uint{bits}, k={k}), median of {len(reps)} "
                     f"repetitions ({total:.1f} s total), oracle/median_oracle.c with {threads} threads",
           "seconds": round(total, 2)}
    if ours is not None:
        res["parity_check"] = dict(check, rows=rows, columns=valid_w, channels=C)
    return res


def reference_python(cfg, k, budget_s=30.0, threads=None):
    """The UNMODIFIED reference package (baseline/_ref/tilemedian, installed by
    pip from /root/reference) on a crop of the workload, on this host's cores:
    its shipped path ``filter_planes(img, k, "auto", workers=n)`` and its
    fastest engine for this k ("aware" for k >= 9, the brute-force oracle below).
    None when baseline/_ref is absent.  Reported beside the C port."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "tilemedian")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import tilemedian  # the reference itself
    H, W, C, bits, _, _ = cfg
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    threads = threads or len(os.sched_getaffinity(0))
    rng = np.random.default_rng(3)
    out = {"cores": threads, "cpu_model": cpu_model(), "unit": "Gpixel/s",
           "source": "baseline/_ref/tilemedian (pip install of /root/reference, unmodified)"}
    best = "aware" if k >= 9 else "oracle"
    t_end = time.perf_counter() + budget_s
    for name, variant in (("shipped_auto", "auto"), ("best_engine", best)):
        side, rec = 32, None
        while time.perf_counter() < t_end:
            h, w = min(H, side), min(W, side)
            img = rng.integers(0, np.iinfo(dt).max, size=(h, w, C) if C > 1 else (h, w),
                               dtype=dt, endpoint=True)
            kw = {"workers": threads} if variant != "oracle" else {}
            t0 = time.perf_counter()
            tilemedian.filter_planes(img, k, variant, **kw)
            dt_s = time.perf_counter() - t0
            rec = {"value": h * w * C / dt_s / 1e9, "variant": variant,
                   "sample": f"{h}x{w}x{C} random crop, one call, {dt_s:.2f} s"}
            if dt_s > budget_s / 8 or (h == H and w == W):
                break
            side *= 2
        out[name] = rec
    return out


def run_reference(args, cfg, k, rank, world):
    """--impl reference: the reference algorithm's CPU path (oracle port), rank 0 only."""
    if rank != 0:
        return
    H, W, C, bits, _, label = cfg
    threads = len(os.sched_getaffinity(0))
    per_step = max(1.0, min(5.0, 120.0 / max(1, args.steps + args.warmup)))
    cal = cpu_baseline(cfg, k, seconds=per_step, threads=threads)
    times = []
    total = args.warmup + args.steps
    for i in range(total):
        r = cpu_baseline(cfg, k, seconds=per_step, threads=threads) if i else cal
        if i >= args.warmup:
            times.append(r)
    v = statistics.median(t["value"] for t in times)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "Gpixel/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * H * W * C / (v * 1e9),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": f"u{bits}", "data": "synthetic (uniform random)",
        "config": {"workload": label, "k": k, "height": H, "width": W, "channels": C,
                   "sample": times[-1]["sample"],
                   "timing": "per step: the crop's median repetition, scaled to the full image "
                             "(ms_per_step); per-pixel cost is size-independent"},
        "cpu_baseline": {"value": v, "unit": "Gpixel/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": times[-1]["sample"]},
        "e2e": {"value": v, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:  # the reference package itself, when baseline/_ref travelled with the repo
        rp = reference_python(cfg, k, threads=threads)
    except Exception as exc:  # reported, never fatal for the arm
        rp = {"error": f"{type(exc).__name__}: {exc}"}
    if rp is not None:
        line["reference_python"] = rp
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--mode", default=None, choices=("frames", "bands"))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--pattern", default="random",
                    help="synthetic input pattern (paper_2507_19926_b200.synth.PATTERNS)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    H, W, C, bits, k_default, label = cfg
    k = args.k or k_default
    mode = args.mode or ("bands" if args.config == "c5" else "frames")

    if args.impl == "reference":
        run_reference(args, cfg, k, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2507_19926_b200 import _lib, bands, filter_planes
    from paper_2507_19926_b200.program import op_model
    from paper_2507_19926_b200.synth import render
    lib = _lib.load()
    tdt = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}[bits]
    esz = bits // 8

    # ---- inputs resident in HBM ------------------------------------------
    if mode == "bands":
        y0, y1 = bands.band_rows(H, world, rank)
        rows = y1 - y0
        band = render(args.pattern, (rows, W, C) if C > 1 else (rows, W), bits, 42 + rank, dev)
        halo = k // 2
        buf, r0 = bands.halo_buffer(band, halo, rank > 0, rank < world - 1)
        del band
        samples_rank = rows * W * C
    else:
        img = render(args.pattern, (H, W, C) if C > 1 else (H, W), bits, 42 + rank, dev)
        out = torch.empty_like(img)
        samples_rank = H * W * C
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    variant = args.variant  # "auto": the C ABI's measured per-(dtype, k) table
    vcode = _lib.VARIANT_CODES[variant]
    kernel = lib.tm_kernel_name(lib.tm_dispatch_query(bits, k, k, vcode)).decode()
    stream = torch.cuda.current_stream(dev)

    def step():
        if mode == "bands":
            bands.exchange_halo(buf, r0, rows, k // 2)
            return bands.filter_band(buf, r0, rows, k, variant)
        rc = lib.tm_median2d_planes(img.data_ptr(), W * C * esz, out.data_ptr(), W * C * esz,
                                    W, H, C, bits, k, vcode, stream.cuda_stream)
        _lib.check(rc)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = lib.tm_launch_count()
    times = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            flush.fill_(1)  # evict the input from L2 (untimed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            times.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = lib.tm_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in times]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    if mode == "bands":
        samples_job = H * W * C
    else:
        samples_job = samples_rank * world
    value = samples_job * args.steps / (total_ms * 1e-3) / 1e9

    # ---- end to end ------------------------------------------------------
    # through the drop-in a user calls, filter_planes(numpy) -> numpy, with the
    # H2D copy of the input, the filter and the D2H copy of the result inside
    # the call (wall clock, max over ranks):
    # (1) e2e: the input in pinned host memory (the package's pinned_empty,
    #     the contract's "inputs from pinned host memory");
    # (2) e2e_pageable: the input in ordinary pageable numpy memory (the copy
    #     threads stage it into pinned buffers -- host-memory bound);
    # (3) e2e_pinned_cabi: the raw C ABI on pinned buffers.
    e2e = None
    e2e_pageable = None
    e2e_pinned = None
    if mode == "frames":
        from paper_2507_19926_b200 import pinned_empty
        nbytes = H * W * C * esz
        n_e2e = max(3, args.steps // 2)

        def time_dropin(host_in):
            res = None
            for _ in range(3):  # the same allocation pattern as the timed loop
                res = filter_planes(host_in, k, variant, device=local)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                res = filter_planes(host_in, k, variant, device=local)
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            del res
            if world > 1:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            return samples_rank * world * n_e2e / float(dt.item()) / 1e9

        host_np = img.cpu().numpy()  # pageable numpy, as a user's image usually is
        host_pin = pinned_empty(host_np.shape, host_np.dtype)
        host_pin[...] = host_np
        e2e = {"value": time_dropin(host_pin), "unit": "Gpixel/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes,
               "path": "filter_planes(numpy) drop-in, input in pinned host memory "
                       "(paper_2507_19926_b200.pinned_empty), output numpy; H2D + filter + "
                       "D2H inside the call, wall clock"}
        e2e_pageable = {"value": time_dropin(host_np), "unit": "Gpixel/s",
                        "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                        "path": "filter_planes(numpy) drop-in, input in pageable memory "
                                "(staged by the copy threads), wall clock"}
        del host_pin
        hin = torch.empty(img.shape, dtype=tdt, pin_memory=True)
        hin.copy_(img)
        hout = torch.empty_like(hin).pin_memory()

        def host_step():
            rc = lib.tm_median2d_host(hin.data_ptr(), W * C * esz, hout.data_ptr(), W * C * esz,
                                      W, H, C, bits, k, k, vcode, local)
            _lib.check(rc)
        for _ in range(2):
            host_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            host_step()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e_pinned = {"value": samples_rank * world * n_e2e / float(e2e_s.item()) / 1e9,
                      "unit": "Gpixel/s", "h2d_bytes_per_step": nbytes,
                      "d2h_bytes_per_step": nbytes,
                      "path": "tm_median2d_host (C ABI) on pinned host buffers"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel -------------------------------------
    peaks = _peaks()
    kern_ms = statistics.median(step_ms)
    lanes = 2 if bits < 32 else 1
    w_k = op_model(k)["minmax_per_pixel"]
    per_launch = samples_rank
    alu_achieved = w_k * per_launch / (kern_ms * 1e-3) / 1e12
    alu_peak = MINMAX_PEAK_TPS * lanes / 1e12
    hbm_achieved = 2 * esz * per_launch / (kern_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}_k{k}.json")  # ncu --set full summary
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline_model = {"bound": "alu", "achieved": alu_achieved, "peak": alu_peak,
                      "unit": "T minmax/s", "frac": alu_achieved / alu_peak, "traffic": traffic,
                      "kernel": kernel,
                      "per_launch": f"W(k)={w_k:.1f} reference min/max per sample x "
                                    f"{per_launch} samples (the reference's op model; the "
                                    "data-aware kernels execute fewer operations)",
                      "peak_source": "measured (profiles/r01_minmax_microbench.txt)"}
    # hardware: instruction issue of the dominant kernel -- ncu-measured warp
    # instructions per sample (committed capture of this config and kernel) x
    # the live sample rate, against 4 warp-instructions/clk/SM x 148 SMs x the
    # sampled SM clock
    roofline_issue = None
    ncu_prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}_k{k}.json")
    if os.path.exists(ncu_prof) and args.pattern == "random":
        with open(ncu_prof) as f:
            npf = json.load(f)
        ips = npf.get("warp_instructions_per_sample")
        ncu_name = {"oblivious": "obl_kernel", "histogram": "hist8_kernel", "rank": "rank_kernel",
                    "med3": "med3_kernel", "multipass": "aware", "select": "select"}.get(kernel, kernel)
        if ips and ncu_name in npf.get("kernel", ""):
            clk_mhz = (clk.summary().get("sm_mhz") or 1965.0)
            achieved_wi = ips * per_launch / (kern_ms * 1e-3) / 1e12
            peak_wi = 4 * 148 * clk_mhz * 1e6 / 1e12
            roofline_issue = {"bound": "issue", "achieved": achieved_wi, "peak": peak_wi,
                              "unit": "T warp-instr/s", "frac": achieved_wi / peak_wi,
                              "traffic": traffic, "kernel": kernel,
                              "per_launch": f"{ips} warp instructions per sample (ncu, "
                                            f"{ncu_prof[len(ROOT) + 1:]}) x {per_launch} samples",
                              "peak_source": "4 warp-instr/clk/SM x 148 SMs x sampled SM clock"}
    roofline_hbm = {"bound": "hbm", "achieved": hbm_achieved, "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s", "frac": hbm_achieved / peaks.get("hbm_gbs", 6650.0),
                    "traffic": traffic, "kernel": kernel,
                    "per_launch": f"2 x {esz} B x {per_launch} samples",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    # primary: HBM for k = 3 (copy-bound), else the hardware issue roofline
    # when a config-matched ncu capture exists, else the op model
    if k < 5:
        roofline = roofline_hbm
    elif roofline_issue is not None:
        roofline = roofline_issue
    else:
        roofline = roofline_model
    line = {
        "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if mode == "bands" else "weak",
        "vs_baseline": None, "dtype": f"u{bits}",
        "data": f"synthetic ({args.pattern}, seeded; paper_2507_19926_b200.synth)",
        "config": {"workload": label, "k": k, "height": H, "width": W, "channels": C,
                   "variant": variant, "kernel": kernel, "mode": mode, "pattern": args.pattern,
                   "l2": "flushed (512 MiB write) before every timed step",
                   "parallelism": f"{mode} x{world}"},
        "roofline": roofline, "roofline_model": roofline_model, "roofline_hbm": roofline_hbm,
        "roofline_issue": roofline_issue,
        "e2e": e2e, "e2e_pageable": e2e_pageable, "e2e_pinned_cabi": e2e_pinned,
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        # the reported CPU baseline, cut from this run's input; its result
        # doubles as the parity self-check of this run's GPU output
        line["cpu_baseline"] = cpu_baseline(cfg, k, src=img if mode == "frames" else None,
                                            ours=out if mode == "frames" else None)
        pc = line["cpu_baseline"].get("parity_check")
        if pc is not None:
            line["parity"] = "ok" if pc["mismatches"] == 0 else f"MISMATCH ({pc['mismatches']} px)"
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
