"""bench.py — throughput of the constant-time bilateral filter on B200.

Workload (BASELINE.json metric "bilateral Mpixel/s and Gpixel·term/s per B200 vs
FP32/SFU roofline; 1/2/4/8 GPUs" — the 1/2/4/8-GPU config is configs[4]):
cfg5, 8192x8192 uint8, box spatial radius 16, sigma_r = 15, N = 118, seeded
synthetic image (synth/).  One step = one whole filter of the image (all
N+1 terms, every pixel).  At N GPUs the image is split into N row bands with
r-row input halos (strong scaling); inputs are placed on each
GPU before timing; there is no collective inside the timed region.

Timing: W untimed warm-up steps; then K timed steps, each preceded by an
untimed L2 flush (256 MiB write); CUDA events on the launching stream around
each step; barrier + cuda synchronize on both sides; max over ranks.

Also measured in the same run: e2e (host buffers through the C-ABI host entry
point, H2D + D2H inside the timed region), the radius sweep r in {4,16,64}
(constant time in r), the roofline fraction of the fused kernel, nvidia-smi
clocks during the timed region, and (rank 0, N=1) the fp64 oracle on a
bounded row band on the host cores (cpu_baseline).

`--impl reference`: the reference arm is the fp64 oracle (oracle/), timed on
host cores on a bounded row band of the same workload per step; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "bilateral Mpixel/s and Gpixel·term/s per B200 vs FP32/SFU roofline; 1/2/4/8 GPUs"
UNIT = "Mpixel/s"
CFG = synth.CONFIGS["cfg5"]
RADIUS = 16
SWEEP = (4, 16, 64)


def algo_instr_per_pixel(N: int, kind: int) -> int:
    """Algorithmic FP32 lane-instructions per output pixel (SURVEY.md §8(d),
    DESIGN.md §6): box: 28 per conjugate pair with omega != 0, 6 for the even-N
    middle term, 3 for the final ratio; q_2: 100 per pair."""
    pairs_nz = (N + 1) // 2
    mid = 1 if N % 2 == 0 else 0
    per = 28 if kind == 0 else 100
    return per * pairs_nz + (6 if kind == 0 else 22) * mid + 3


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML every 10 ms in a thread (nvidia-smi's own loop as the
    fallback)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []          # (sm_mhz, max_mhz, reasons bitmask) from NVML
        self.stop = threading.Event()
        self.t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        g = str(self.gpu)
        if g.startswith("GPU-") or g.startswith("MIG-"):
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(g)
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(int(g))

    def _poll_nvml(self, nv, h):
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, int(get_reasons(h))))
            except Exception:
                pass
            self.stop.wait(0.01)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.t is not None:
            self.t.join(timeout=1)

    def summary(self):
        sm, mx, reasons = [], [], set()
        if self.samples:
            for c, m, bits in self.samples:
                sm.append(float(c))
                mx.append(float(m))
                reasons.update(nm for nm, bit in self.REASONS.items() if bits & bit)
            src = "nvml"
        else:
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            src = "nvidia-smi"
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": src}


def oracle_band_rate(rows: int, radius: int, nthreads: int = 0):
    """fp64 oracle (Algorithm 2) on output rows [0, rows) of the workload image."""
    import oracle
    img = _image()
    t0 = time.perf_counter()
    oracle.bilateral_shiftable(img, radius, CFG.kind, CFG.sigma_r, CFG.N, row_begin=0, row_end=rows,
                               nthreads=nthreads)
    dt = time.perf_counter() - t0
    return rows * CFG.W / dt / 1e6, dt


_IMG = None


def _image():
    global _IMG
    if _IMG is None:
        _IMG = CFG.image()
    return _IMG


def size_oracle_rows(radius: int, target_s: float) -> int:
    rate, _ = oracle_band_rate(128, radius)                   # Mpixel/s probe (~1 s)
    rows = int(target_s * rate * 1e6 / CFG.W)
    return max(8, min(CFG.H, rows))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cores = oracle.max_threads()
    rows = size_oracle_rows(RADIUS, 4.0)
    for _ in range(args.warmup):
        oracle_band_rate(rows, RADIUS)
    times = []
    for _ in range(args.steps):
        _, dt = oracle_band_rate(rows, RADIUS)
        times.append(dt)
    total = sum(times)
    value = args.steps * rows * CFG.W / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"cfg5 8192x8192 box r={RADIUS} sigma_r=15 N=118 (rows 0..{rows} per step)",
                   "H": CFG.H, "W": CFG.W, "radius": RADIUS, "sigma_r": CFG.sigma_r, "N": CFG.N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"output rows [0,{rows}) x {CFG.W} cols of the cfg5 image per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1107_4617_b200 as sf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    sf.load()
    stream = torch.cuda.current_stream()

    H, W, N, s, kind = CFG.H, CFG.W, CFG.N, CFG.sigma_r, CFG.kind
    img_np = _image()
    # row band of this rank (+ input halo), placed before timing
    b0, b1 = rank * H // world, (rank + 1) * H // world

    def band_input(r):
        i0, i1 = max(0, b0 - r), min(H, b1 + r)
        return torch.from_numpy(np.ascontiguousarray(img_np[i0:i1])).to(dev)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = torch.empty((b1 - b0, W), dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def time_steps(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        ms = 0.0
        for _ in range(steps):
            flush.fill_(1.0)                      # untimed L2 flush
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ms += e0.elapsed_time(e1)
        barrier()
        return max_over_ranks(ms)

    # ---- main timed region: r = 16, device-resident input
    timg = band_input(RADIUS)
    launches = []

    def step():
        sf.sf_filter_rows(timg, H, W, b0, b1, RADIUS, kind, s, N, out_band=out, stream=stream)
        launches.append(sf.sf_last_launch_count())

    def _visible_index(i):
        # nvidia-smi -i accepts an index or a UUID; CUDA_VISIBLE_DEVICES may hold either,
        # and the process's device i is the i-th entry of it
        vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
        return vis[i] if i < len(vis) else str(i)
    gpu_index = _visible_index(local if world > 1 else 0)
    with ClockSampler(gpu_index) as clk:
        total_ms = time_steps(step, args.steps, args.warmup)
    clocks = clk.summary()
    launches_timed = sum(launches[args.warmup:])
    ms_per_step = total_ms / args.steps
    value = H * W / (ms_per_step * 1e-3) / 1e6                   # whole-job Mpixel/s
    terms = N + 1
    gpt = value * 1e6 * terms / 1e9                               # Gpixel·term/s

    # ---- roofline of the fused kernel (alu-bound): algorithmic FP32 lane-instr/s
    peaks = load_peaks()
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tis = sm_count * 128 * fmax * 1e6 / 1e12                 # T lane-instr/s at max clock
    ipp = algo_instr_per_pixel(N, kind)
    rows_rank = b1 - b0
    kernel_ms_rank = ms_per_step                                   # one launch per step (max over ranks)
    achieved = ipp * rows_rank * W / (kernel_ms_rank * 1e-3) / 1e12       # per GPU (slowest rank)
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(f"cfg5_r{RADIUS}_n{world}")
    except Exception:
        pass
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_tis,
                "unit": "T FP32 lane-instr/s", "frac": achieved / peak_tis,
                "traffic": traffic,
                "peak_source": f"derived: {sm_count} SMs x 128 FP32 lanes x {fmax:.0f} MHz (sm_max_mhz, "
                               "MEASURED_PEAKS.json) per GPU; B200_PROFILING.md unit counts",
                "algorithmic_instr_per_pixel": ipp,
                "frac_at_observed_clock": (achieved / (sm_count * 128 * clocks["sm_mhz"] * 1e6 / 1e12)
                                           if clocks.get("sm_mhz") else None)}

    # ---- radius sweep (constant time in r), same band split
    sweep = {}
    if not args.no_sweep:
        for r in SWEEP:
            t_r = band_input(r)

            def step_r(t_r=t_r, r=r):
                sf.sf_filter_rows(t_r, H, W, b0, b1, r, kind, s, N, out_band=out, stream=stream)
            sweep[str(r)] = time_steps(step_r, max(2, min(args.steps, 5)), 1) / max(2, min(args.steps, 5))
        vals = list(sweep.values())
        sweep["max_over_min"] = max(vals) / min(vals)

    # ---- e2e through the C-ABI host entry point (pinned host buffers)
    i0, i1 = max(0, b0 - RADIUS), min(H, b1 + RADIUS)
    h_in = torch.from_numpy(np.ascontiguousarray(img_np[i0:i1])).pin_memory()
    h_out = torch.empty((b1 - b0, W), dtype=torch.float32).pin_memory()
    h_in_np, h_out_np = h_in.numpy(), h_out.numpy()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(1):
        sf.sf_filter_rows_host(h_in_np, H, W, b0, b1, RADIUS, kind, s, N, out_band=h_out_np, stream=stream)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sf.sf_filter_rows_host(h_in_np, H, W, b0, b1, RADIUS, kind, s, N, out_band=h_out_np, stream=stream)
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0) / e2e_steps
    e2e = {"value": H * W / e2e_s / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": int(sum_over_ranks(dist, world, dev, (i1 - i0) * W)),
           "d2h_bytes_per_step": int(H * W * 4),
           "how": "sf_filter_rows_host (C-ABI) per rank: pinned host band -> device -> kernel -> host, "
                  "wall clock around the calls, max over ranks"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"cfg5 8192x8192 uint8, box r={RADIUS}, sigma_r=15, N=118, "
                                   f"row bands x{world}",
                       "H": H, "W": W, "radius": RADIUS, "sigma_r": s, "N": N, "terms": terms,
                       "parallelism": f"rowband{world}",
                       "l2": "flushed (256 MiB write) before every timed step"},
            "gpixel_terms_per_s": gpt,
            "radius_sweep_ms": sweep,
            "roofline": roofline,
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches_timed,
        }
        if world == 1 and not args.no_cpu:
            import oracle
            rows = size_oracle_rows(RADIUS, 20.0)
            rate, dt = oracle_band_rate(rows, RADIUS)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": oracle.max_threads(),
                                    "kind": "oracle",
                                    "sample": f"output rows [0,{rows}) x {W} cols of the cfg5 r={RADIUS} "
                                              f"image ({dt:.1f} s, fp64 Algorithm 2, OpenMP)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def sum_over_ranks(dist, world, dev, x):
    if world == 1:
        return x
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return t.item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
