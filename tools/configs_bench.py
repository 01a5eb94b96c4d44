"""Time every BASELINE.json config (synth.CONFIGS) through the C-ABI on one
GPU: device-resident input, CUDA events, median of 5 after warm-up, L2 flushed
between launches.  cfg4 is also timed as the term split on one GPU
(sf_accumulate over all pairs + sf_finalize).  One JSON line per case with
Mpixel/s, Gpixel.term/s and the fraction of the FP32 roofline (algorithmic
lane-instr per pixel as bench.py)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench
import paper_1107_4617_b200 as sf
import synth

peak = torch.cuda.get_device_properties(0).multi_processor_count * 128 * 1965e6
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for name, c in synth.CONFIGS.items():
    img = torch.from_numpy(c.image()).cuda()
    out = torch.empty((c.H, c.W), dtype=torch.float32, device="cuda")
    cases = [("filter", lambda: sf.sf_filter(img, c.radius, c.kind, c.sigma_r, c.N, out=out), c.N + 1)]
    if name == "cfg4":
        num = torch.empty_like(out)
        den = torch.empty_like(out)
        K = sf.sf_pair_count(c.N)

        def termsplit():
            sf.sf_accumulate(img, c.radius, c.kind, c.sigma_r, c.N, 0, K, num=num, den=den)
            sf.sf_finalize(num, den, img, out=out)
        cases.append(("accumulate+finalize", termsplit, c.N + 1))

        def fused():                                  # the fused term split's per-rank path
            num.zero_()
            den.zero_()
            sf.sf_accumulate_add(img, c.radius, c.kind, c.sigma_r, c.N, 0, K, num, den)
            sf.sf_finalize(num, den, img, out=out)
        cases.append(("zero+accumulate_add+finalize", fused, c.N + 1))
    if name in ("cfg4", "cfg5"):
        for eps in (1e-6, 1e-4):
            kept = c.N + 1 - 2 * sf.sf_truncation_n0(c.N, eps)
            cases.append((f"truncated eps={eps:g}",
                          lambda eps=eps: sf.sf_filter_truncated(img, c.radius, c.kind, c.sigma_r, c.N, eps, out=out),
                          kept))
    for how, fn, terms in cases:
        ms = timed(fn)
        px = c.H * c.W
        # algorithmic work of the terms actually evaluated (terms - 1 = N' of
        # an order-N' expansion with the same pair structure)
        ipp = bench.algo_instr_per_pixel(terms - 1, c.kind)
        print(json.dumps({"config": name, "how": how, "H": c.H, "W": c.W, "r": c.radius, "kind": c.kind,
                          "N": c.N, "terms": terms, "ms": round(ms, 4), "mpix_s": round(px / ms / 1e3, 1),
                          "gpix_term_s": round(px * terms / ms / 1e6, 1),
                          "frac": round(ipp * px / (ms * 1e-3) / peak, 4)}), flush=True)
