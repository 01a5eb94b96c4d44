"""Device time of the cfg2 parameters (r = 8, sigma_r = 20, N = 66) against
the image height (W = 1920): the slope is the steady-state cost, the
intercept the fixed and segment-start costs.  usage: python tools/cfg2_scan.py"""
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


r, s, N = int(os.environ.get("R", 8)), float(os.environ.get("S", 20.0)), int(os.environ.get("NN", 66))
for H in (272, 544, 1080, 2160, 4320, 8640):
    img = torch.from_numpy(synth.gen_image(H, 1920, 1, 10.0)).cuda()
    out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
    ms = dev_ms(lambda: sf.sf_filter(img, r, 0, s, N, out=out))
    print(json.dumps({"H": H, "W": 1920, "r": r, "N": N, "device_us": round(ms * 1e3, 1),
                      "ns_per_px_pair": round(ms * 1e6 / (H * 1920 * sf.sf_pair_count(N)) * 1e3, 3)}), flush=True)
