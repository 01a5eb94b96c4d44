"""bench.py — throughput of the constant-time bilateral filter on B200.

Workload (BASELINE.json metric "bilateral Mpixel/s and Gpixel·term/s per B200 vs
FP32/SFU roofline; 1/2/4/8 GPUs" — the 1/2/4/8-GPU config is configs[4]):
cfg5, 8192x8192 uint8, box spatial radius 16, sigma_r = 15, N = 118, seeded
synthetic image (synth/).  One step = one whole filter of the image (all
N+1 terms, every pixel).  At N GPUs the image is split into N row bands with
r-row input halos (strong scaling); inputs are placed on each
GPU before timing; there is no collective inside the timed region.
`--workload cfg4` times config 4 instead (4096^2, r = 16, sigma_r = 10,
N = 264) as the north star's term split: rank i accumulates the partial
(P', Q) of its share of the 133 conjugate pairs (sf_accumulate), one NCCL
reduce sums them on rank 0, which runs sf_finalize — all inside the timed
region.

Launch: `python bench.py --gpus N` with no torchrun environment re-executes
itself under torch.distributed.run (N ranks, 127.0.0.1); under the driver's
torchrun the world size must equal --gpus.  NCCL communicator set-up is
logged (NCCL_DEBUG=INFO, subsystem INIT, to stderr).

Timing: W untimed warm-up steps; then K timed steps, each preceded by an
untimed L2 flush (256 MiB write); CUDA events on the launching stream around
each step; barrier + cuda synchronize on both sides; max over ranks.

Also measured in the same run: e2e (host buffers through the C-ABI host entry
point, H2D + D2H inside the timed region), the radius sweep r in {4,16,64}
(constant time in r), the roofline fraction of the fused kernel (FP32 and
SFU), every other BASELINE config on one GPU (`configs`), nvidia-smi clocks
during the timed region, and (rank 0, N=1) the fp64 oracle on a bounded row
band on the host cores (cpu_baseline).

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


def oracle_band_rate(rows: int, radius: int, nthreads: int = 0, cfg=None):
    """fp64 oracle (Algorithm 2) on output rows [0, rows) of the workload image."""
    import oracle
    cfg = cfg or CFG
    img = _image(cfg)
    t0 = time.perf_counter()
    oracle.bilateral_shiftable(img, radius, cfg.kind, cfg.sigma_r, cfg.N, row_begin=0, row_end=rows,
                               nthreads=nthreads)
    dt = time.perf_counter() - t0
    return rows * cfg.W / dt / 1e6, dt


_IMGS = {}


def _image(cfg=None):
    cfg = cfg or CFG
    if cfg.name not in _IMGS:
        _IMGS[cfg.name] = cfg.image()
    return _IMGS[cfg.name]


def size_oracle_rows(radius: int, target_s: float, cfg=None) -> int:
    """Rows of a bounded oracle sample of about target_s seconds; at least
    32 rows per host core, so the oracle's 32-row bands occupy every core."""
    import oracle
    cfg = cfg or CFG
    rate, _ = oracle_band_rate(128, radius, cfg=cfg)          # Mpixel/s probe (~1 s)
    rows = int(target_s * rate * 1e6 / cfg.W)
    rows = max(rows, 32 * oracle.max_threads())
    return max(8, min(cfg.H, rows))


def workload_cfg(args):
    return synth.CONFIGS[args.workload]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cfg = workload_cfg(args)
    radius = RADIUS if args.workload == "cfg5" else cfg.radius
    cores = oracle.max_threads()
    rows = size_oracle_rows(radius, float(os.environ.get("SF_BENCH_ORACLE_S", "4.0")), cfg)
    for _ in range(args.warmup):
        oracle_band_rate(rows, radius, cfg=cfg)
    times = []
    for _ in range(args.steps):
        _, dt = oracle_band_rate(rows, radius, cfg=cfg)
        times.append(dt)
    total = sum(times)
    value = args.steps * rows * cfg.W / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name} {cfg.H}x{cfg.W} box r={radius} sigma_r={cfg.sigma_r:g} N={cfg.N} "
                               f"(rows 0..{rows} per step)",
                   "H": cfg.H, "W": cfg.W, "radius": radius, "sigma_r": cfg.sigma_r, "N": cfg.N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"output rows [0,{rows}) x {cfg.W} cols of the {cfg.name} image per step "
                                   f"(>= 32 rows per core)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def kernel_stats():
    """Per-launch constants of the default cfg5 kernel from its ncu capture
    (profiles/kernel_stats.json, written by tools/ncu_summary.py --json): DRAM
    bytes and MUFU (XU-pipe) lane-ops per launch.  The bench cannot run ncu
    itself, so these are quoted with the capture they come from."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "kernel_stats.json")))
    except Exception:
        return {}


def bind_host_to_gpu(gpu):
    """Restrict this process to the CPUs NVML reports as local to GPU `gpu`
    (an index or UUID as in CUDA_VISIBLE_DEVICES), before any pinned host
    buffer is allocated, so that the e2e leg's pinned buffers (first touch)
    sit on the GPU's NUMA node.  Returns the number of CPUs bound, or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        g = str(gpu)
        h = (pynvml.nvmlDeviceGetHandleByUUID(g) if g.startswith(("GPU-", "MIG-"))
             else pynvml.nvmlDeviceGetHandleByIndex(int(g)))
        ncpu = os.cpu_count() or 64
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        cpus &= set(os.sched_getaffinity(0))
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return len(cpus)
    except Exception:
        return None


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1107_4617_b200 as sf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: world size {world} != --gpus {args.gpus}", file=sys.stderr)
        return 2
    vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    li = local if world > 1 else 0
    all_cpus = set(os.sched_getaffinity(0))
    host_cpus = bind_host_to_gpu(vis[li] if li < len(vis) else li)
    # SF_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0 over gloo, to
    # exercise the N > 1 code path on a one-GPU box; its timings are not a
    # scaling measurement and its line says so ("diagnostic")
    shared = world > 1 and os.environ.get("SF_BENCH_SHARED_GPU") == "1"
    if shared:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    elif world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 and not shared else 0)
    torch.cuda.set_device(dev)
    sf.load()
    stream = torch.cuda.current_stream()

    cfg = workload_cfg(args)
    radius = RADIUS if args.workload == "cfg5" else cfg.radius
    H, W, N, s, kind = cfg.H, cfg.W, cfg.N, cfg.sigma_r, cfg.kind
    img_np = _image(cfg)
    term_split = args.workload == "cfg4"
    # row band of this rank (+ input halo), placed before timing
    b0, b1 = (0, H) if term_split else (rank * H // world, (rank + 1) * H // world)

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

    # ---- main timed region, device-resident input
    timg = band_input(radius)
    launches = []
    if term_split:
        K = sf.sf_pair_count(N)
        p0, p1 = rank * K // world, (rank + 1) * K // world
        part = torch.empty((2, H, W), dtype=torch.float32, device=dev)      # (num, den) of this rank

        def step():
            sf.sf_accumulate(timg, radius, kind, s, N, p0, p1, num=part[0], den=part[1], stream=stream)
            n = sf.sf_last_launch_count()
            if world > 1 and shared:                                     # gloo: all_reduce of CUDA tensors
                dist.all_reduce(part, op=dist.ReduceOp.SUM)
            elif world > 1:
                dist.reduce(part, dst=0, op=dist.ReduceOp.SUM)             # NCCL, on the current stream
            if rank == 0:
                sf.sf_finalize(part[0], part[1], timg, out=out, stream=stream)
                n += sf.sf_last_launch_count()
            launches.append(n)
    else:
        def step():
            sf.sf_filter_rows(timg, H, W, b0, b1, radius, kind, s, N, out_band=out, stream=stream)
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
    # per GPU: the slowest rank's step covers its band (row split) or all pixels
    # with its share of the pairs (term split, where the reduce is in the step too)
    work_px = (b1 - b0) * W if not term_split else H * W * (p1 - p0) / max(1, K)
    achieved = ipp * work_px / (ms_per_step * 1e-3) / 1e12
    ks = kernel_stats().get(f"{cfg.name}_r{radius}", {}) if world == 1 else {}
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_tis,
                "unit": "T FP32 lane-instr/s", "frac": achieved / peak_tis,
                "traffic": ks.get("dram_bytes_per_launch"),
                "traffic_source": ks.get("source"),
                "peak_source": f"derived: {sm_count} SMs x 128 FP32 lanes x {fmax:.0f} MHz (sm_max_mhz, "
                               "MEASURED_PEAKS.json) per GPU; B200_PROFILING.md unit counts",
                "algorithmic_instr_per_pixel": ipp,
                "frac_at_observed_clock": (achieved / (sm_count * 128 * clocks["sm_mhz"] * 1e6 / 1e12)
                                           if clocks.get("sm_mhz") else None)}
    if ks.get("mufu_lane_ops_per_launch"):
        sfu_peak = sm_count * 16 * fmax * 1e6 / 1e12                # T MUFU lane-ops/s
        sfu_ach = ks["mufu_lane_ops_per_launch"] / (ms_per_step * 1e-3) / 1e12
        roofline["sfu"] = {"achieved": sfu_ach, "peak": sfu_peak, "unit": "T MUFU lane-ops/s",
                           "frac": sfu_ach / sfu_peak,
                           "mufu_per_pixel_pair": ks.get("mufu_per_pixel_pair"),
                           "peak_source": f"{sm_count} SMs x 16 MUFU lanes x {fmax:.0f} MHz "
                                          "(profiles/r01_ubench_b200.txt)"}

    # ---- radius sweep (constant time in r), same band split
    sweep = {}
    if not args.no_sweep and not term_split:
        for r in SWEEP:
            t_r = band_input(r)

            def step_r(t_r=t_r, r=r):
                sf.sf_filter_rows(t_r, H, W, b0, b1, r, kind, s, N, out_band=out, stream=stream)
            sweep[str(r)] = time_steps(step_r, max(2, min(args.steps, 5)), 1) / max(2, min(args.steps, 5))
        vals = list(sweep.values())
        sweep["max_over_min"] = max(vals) / min(vals)

    # ---- e2e through the C-ABI host entry point (pinned host buffers): each
    # step copies its input band in and its output band out; successive steps
    # pipeline (sf_filter_rows_host_async: copies on the copy engines overlap
    # the neighbouring steps' kernels)
    e2e = None
    if not term_split:
        i0, i1 = max(0, b0 - radius), min(H, b1 + radius)
        h_in = torch.from_numpy(np.ascontiguousarray(img_np[i0:i1])).pin_memory()
        h_outs = [torch.empty((b1 - b0, W), dtype=torch.float32).pin_memory() for _ in range(2)]
        h_in_np = h_in.numpy()
        e2e_steps = max(20, args.steps)      # steady state: the first input and last output copy amortise
        sf.sf_filter_rows_host_async(h_in_np, H, W, b0, b1, radius, kind, s, N, h_outs[0].numpy(), stream=stream)
        sf.sf_host_sync()
        barrier()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            sf.sf_filter_rows_host_async(h_in_np, H, W, b0, b1, radius, kind, s, N, h_outs[k % 2].numpy(),
                                         stream=stream)
        sf.sf_host_sync()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        barrier()
        e2e_s = max_over_ranks(e2e_s)
        e2e = {"value": H * W / e2e_s / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(dist, world, dev, (i1 - i0) * W)),
               "d2h_bytes_per_step": int(H * W * 4),
               "steps": e2e_steps,
               "how": "sf_filter_rows_host_async (C-ABI) per rank, back-to-back steps: pinned host band -> "
                      "device -> kernel -> pinned host, copies on the copy engines overlapping the "
                      "neighbouring steps' kernels; wall clock around all steps + sf_host_sync, max over ranks", "host_cpus_bound": host_cpus}

    if term_split:
        # e2e of the term split: each step copies the pinned host image in,
        # accumulates this rank's pairs, reduces, finalizes and copies the
        # result out on rank 0 (synchronous per step)
        h_img = torch.from_numpy(np.ascontiguousarray(img_np)).pin_memory()
        h_out = torch.empty((H, W), dtype=torch.float32).pin_memory()
        e2e_steps = max(3, args.steps)

        def e2e_step():
            timg.copy_(h_img, non_blocking=True)
            step()
            if rank == 0:
                h_out.copy_(out, non_blocking=True)
        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        barrier()
        e2e_s = max_over_ranks(e2e_s)
        e2e = {"value": H * W / e2e_s / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(H * W * world), "d2h_bytes_per_step": int(H * W * 4),
               "steps": e2e_steps,
               "how": "per step: pinned host image -> device (every rank), sf_accumulate + NCCL reduce + "
                      "sf_finalize, result -> pinned host (rank 0); wall clock, max over ranks"}

    # ---- every other BASELINE config on one GPU (rank 0, N = 1)
    configs = {}
    if world == 1 and not args.no_configs:
        configs = time_configs(sf, torch, dev, stream, flush, peak_tis)

    if rank == 0:
        parallelism = f"termsplit{world}" if term_split else f"rowband{world}"
        desc = (f"{cfg.name} {H}x{W} uint8, box r={radius}, sigma_r={s:g}, N={N}, "
                + (f"term split x{world} (sf_accumulate + NCCL reduce + sf_finalize)" if term_split
                   else f"row bands x{world}"))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "H": H, "W": W, "radius": radius, "sigma_r": s, "N": N, "terms": terms,
                       "parallelism": parallelism,
                       "l2": "flushed (256 MiB write) before every timed step"},
            "gpixel_terms_per_s": gpt,
            "radius_sweep_ms": sweep,
            "roofline": roofline,
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches_timed,
        }
        if configs:
            line["configs"] = configs
        if shared:
            line["diagnostic"] = f"{world} ranks shared cuda:0 over gloo (SF_BENCH_SHARED_GPU): code-path check, not a scaling number"
        if world == 1 and not args.no_cpu:
            os.sched_setaffinity(0, all_cpus)      # the CPU baseline uses every host core
            import oracle
            rows = size_oracle_rows(radius, 20.0, cfg)
            rate, dt = oracle_band_rate(rows, radius, cfg=cfg)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": oracle.max_threads(),
                                    "kind": "oracle",
                                    "sample": f"output rows [0,{rows}) x {W} cols of the {cfg.name} r={radius} "
                                              f"image ({dt:.1f} s, fp64 Algorithm 2, OpenMP)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def time_configs(sf, torch, dev, stream, flush, peak_tis):
    """cfg1..cfg4 on their default kernels, one GPU, device-resident input,
    L2 flushed before each timed launch, median of 5 (CUDA events); cfg4 also
    as the term split's accumulate + finalize."""
    res = {}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return sorted(ts)[reps // 2]

    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        c = synth.CONFIGS[name]
        img = torch.from_numpy(_image(c)).to(dev)
        o = torch.empty((c.H, c.W), dtype=torch.float32, device=dev)
        ms = timed(lambda: sf.sf_filter(img, c.radius, c.kind, c.sigma_r, c.N, out=o, stream=stream))
        ipp = algo_instr_per_pixel(c.N, c.kind)
        mpx = c.H * c.W / (ms * 1e-3) / 1e6
        res[name] = {"H": c.H, "W": c.W, "radius": c.radius, "spatial": "box" if c.kind == 0 else "q2",
                     "sigma_r": c.sigma_r, "N": c.N, "ms": ms, "Mpixel_s": mpx,
                     "Gpixel_term_s": mpx * 1e6 * (c.N + 1) / 1e9,
                     "fp32_frac": ipp * c.H * c.W / (ms * 1e-3) / 1e12 / peak_tis}
        if name == "cfg4":
            K = sf.sf_pair_count(c.N)
            num = torch.empty_like(o)
            den = torch.empty_like(o)

            def split():
                sf.sf_accumulate(img, c.radius, c.kind, c.sigma_r, c.N, 0, K, num=num, den=den, stream=stream)
                sf.sf_finalize(num, den, img, out=o, stream=stream)
            ms2 = timed(split)
            res["cfg4_term_split_1gpu"] = {"ms": ms2, "Mpixel_s": c.H * c.W / (ms2 * 1e-3) / 1e6,
                                           "how": "sf_accumulate (all pairs) + sf_finalize"}
    return res


def sum_over_ranks(dist, world, dev, x):
    if world == 1:
        return x
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return t.item()


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this script as N ranks under
    torch.distributed.run on 127.0.0.1 (one process per GPU)."""
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg5", "cfg4"],
                    help="cfg5: row bands (default, the metric's 1/2/4/8-GPU config); cfg4: term split + NCCL reduce")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    # NCCL communicator set-up is logged (nranks per communicator), on stderr
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
