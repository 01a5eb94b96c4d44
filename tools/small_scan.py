"""Device time (spin-kernel hidden host overhead, L2 flushed, median of 7) of
sf_filter on small images against N, H, W: separates the fixed cost of a
launch from the per-pair cost.  usage: python tools/small_scan.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import synth

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def dev_ms(fn, reps=7):
    fn(); torch.cuda.synchronize()
    td = []
    for _ in range(reps):
        flush.fill_(1.0)
        torch.cuda._sleep(400000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        td.append(e0.elapsed_time(e1))
    return sorted(td)[reps // 2]


cases = [(256, 256, 5, N) for N in (2, 4, 8, 16, 30, 60, 118)] + \
        [(H, 256, 5, 30) for H in (16, 32, 64, 128, 512)] + [(256, W, 5, 30) for W in (64, 128, 512, 1024)]
for H, W, r, N in cases:
    img = torch.from_numpy(synth.gen_image(H, W, 1, 10.0)).cuda()
    out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
    s = 170.0 / N ** 0.5
    ms = dev_ms(lambda: sf.sf_filter(img, r, 0, s, N, out=out))
    print(json.dumps({"H": H, "W": W, "r": r, "N": N, "pairs": sf.sf_pair_count(N),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("SF_")}, "device_us": round(ms * 1e3, 1)}), flush=True)
# an empty-ish reference: a torch kernel launch after the spin
x = torch.empty(16, device="cuda")
print(json.dumps({"torch_fill_16_us": round(dev_ms(lambda: x.fill_(1.0)) * 1e3, 1)}))
