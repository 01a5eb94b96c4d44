"""Event-timing floor probe: what a tiny launch costs between two CUDA events
after the bench's 256 MiB L2 flush, with and without the launch pre-queued
behind a GPU-side delay (torch.cuda._sleep), for an empty fill_ and for cfg1."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1107_4617_b200 as sf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
small = torch.empty(16, dtype=torch.float32, device=dev)
c = synth.CONFIGS["cfg1"]


def timed(fn, mode, reps=21):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if mode in ("flush", "flush+sleep"):
            flush.fill_(1.0)
        if mode in ("sleep", "flush+sleep"):
            torch.cuda._sleep(200000)          # ~100 us of GPU spin: the launch below is queued before e0 runs
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return {"median_us": ts[reps // 2], "min_us": ts[0]}


out = {}
from bench import _image  # noqa: E402
img = torch.from_numpy(_image(c)).to(dev)
o = torch.empty((c.H, c.W), dtype=torch.float32, device=dev)
for mode in ("none", "flush", "sleep", "flush+sleep"):
    out[mode] = {"fill16": timed(lambda: small.fill_(0.0), mode),
                 "cfg1": timed(lambda: sf.sf_filter(img, c.radius, c.kind, c.sigma_r, c.N, out=o, stream=stream), mode)}
print(json.dumps(out, indent=1))
