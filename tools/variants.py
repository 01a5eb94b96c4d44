"""A/B timing of the kernel variants (SF_VARIANT=v1|v3|v4) on the
cfg5 workload (8192x8192, sigma_r=15, N=118) at several radii.  One JSON line
per (variant, radius): CUDA-event time per filter, Mpixel/s, and the fraction
of the FP32 roofline (algorithmic 1661 lane-instr/pixel, bench.py).
usage: SF_VARIANT=v4 python tools/variants.py [H W] [r ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_1107_4617_b200 as sf
import synth

args = [int(a) for a in sys.argv[1:]]
H, W = (args[0], args[1]) if len(args) >= 2 else (8192, 8192)
radii = args[2:] or [4, 16, 64]
s, N = 15.0, 118
img = torch.from_numpy(synth.gen_image(H, W, 5, 10.0)).cuda()
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
peak = torch.cuda.get_device_properties(0).multi_processor_count * 128 * 1965e6
for r in radii:
    sf.sf_filter(img, r, 0, s, N, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sf.sf_filter(img, r, 0, s, N, out=out)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"variant": os.environ.get("SF_VARIANT", "default"), "H": H, "W": W, "r": r,
                      "ms": round(ms, 3), "mpix_s": round(H * W / ms / 1e3, 1),
                      "frac": round(1661 * H * W / (ms * 1e-3) / peak, 4),
                      "checksum": float(out.double().mean())}), flush=True)
