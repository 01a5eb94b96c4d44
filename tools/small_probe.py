"""Where the small-image time goes: CUDA-event times (median of 9) of a tiny
torch op and of sf_filter at several N, with and without the L2 flush."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import synth

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
img = torch.from_numpy(synth.gen_image(256, 256, 1, 10.0)).cuda()
out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
small = torch.empty(16, device="cuda")


def t(fn, fl):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(9):
        if fl:
            flush.fill_(1.0)
        torch.cuda._sleep(200000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(sorted(ts)[4] * 1000, 2)


for fl in (True, False):
    print(json.dumps({"flush": fl, "what": "small.fill_", "us": t(lambda: small.fill_(1.0), fl)}))
    for (s, N) in ((300.0, 2), (30.0, 30), (15.0, 118)):
        print(json.dumps({"flush": fl, "what": f"sf_filter r=5 N={N} {os.environ.get('SF_VARIANT', 'default')}",
                          "us": t(lambda: sf.sf_filter(img, 5, 0, s, N, out=out), fl)}))
