"""CUDA-event time (median of 7, L2 flushed, host call hidden behind a spin
kernel) of sf_filter on small synthetic images — the crossover between the
small-image kernel (box_small.cuh) and the band sweep (v7).
usage: SF_VARIANT=vs|v7m python tools/small_sweep.py H W r sigma_r N [H W r sigma_r N ...]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import synth

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
a = sys.argv[1:]
for i in range(0, len(a), 5):
    H, W, r, s, N = int(a[i]), int(a[i + 1]), int(a[i + 2]), float(a[i + 3]), int(a[i + 4])
    img = torch.from_numpy(synth.gen_image(H, W, 1, 10.0)).cuda()
    out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
    fn = lambda: sf.sf_filter(img, r, 0, s, N, out=out)
    fn(); torch.cuda.synchronize()
    ts, td = [], []
    for _ in range(7):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        flush.fill_(1.0)
        torch.cuda._sleep(400000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        td.append(e0.elapsed_time(e1))
    print(json.dumps({"H": H, "W": W, "r": r, "N": N, "variant": os.environ.get("SF_VARIANT", "default"),
                      "ms": round(sorted(ts)[3], 4), "device_ms": round(sorted(td)[3], 4)}), flush=True)
