import os, sys, json
sys.path.insert(0, '.')
import torch, paper_1107_4617_b200 as sf, synth
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
img = torch.from_numpy(synth.gen_image(256, 256, 1, 10.0)).cuda()
out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
for N in (2, 30):
    s = 170.0 / N ** 0.5
    fn = lambda: sf.sf_filter(img, 5, 0, s, N, out=out)
    fn(); torch.cuda.synchronize()
    for fl in (True, False):
        td = []
        for _ in range(9):
            if fl: flush.fill_(1.0)
            torch.cuda._sleep(400000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            td.append(e0.elapsed_time(e1))
        print(json.dumps({"N": N, "flush": fl, "us": round(sorted(td)[4] * 1e3, 1)}))
    # back to back 50 launches, no flush
    torch.cuda._sleep(4000000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): fn()
    e1.record(); e1.synchronize()
    print(json.dumps({"N": N, "b2b_us": round(e0.elapsed_time(e1) / 50 * 1e3, 1)}))
