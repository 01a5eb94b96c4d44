"""CUDA-event time (median of 5, L2 flushed) of sf_filter on a named config.
usage: python tools/time_cfg.py cfg5 16 [cfg4 16 ...]   (env SF_VARIANT etc. apply)"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import synth

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
a = sys.argv[1:]
for name, r in zip(a[::2], a[1::2]):
    r = int(r)
    c = synth.CONFIGS[name]
    img = torch.from_numpy(c.image()).cuda()
    out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
    fn = lambda: sf.sf_filter(img, r, c.kind, c.sigma_r, c.N, out=out)
    fn(); torch.cuda.synchronize()
    ts, td = [], []
    for _ in range(5):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        # device time alone: the host's call overhead hidden behind a spin kernel
        flush.fill_(1.0)
        torch.cuda._sleep(400000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        td.append(e0.elapsed_time(e1))
    print(json.dumps({"cfg": name, "r": r, "env": {k: v for k, v in os.environ.items() if k.startswith("SF_")},
                      "ms": round(sorted(ts)[2], 4), "device_ms": round(sorted(td)[2], 4)}), flush=True)
