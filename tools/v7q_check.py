"""v7q bring-up: parity of the separable q_M band sweep (M = 1..4) against the
fp64 oracle on small images, the sigma_s-fitted variant, and timings of
config 3 (q_2) and a q_4 filter of the same size.  usage: python tools/v7q_check.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1107_4617_b200 as sf
import oracle
import synth

worst = 0.0
H, W, N, s = 150, 530, 30, 30.0
img = synth.gen_image(H, W, 77, 10.0)
t = torch.from_numpy(img).cuda()
for M in (1, 2, 3, 4):
    for r in (1, 2, 5, 10, 16, 24):
        kind = sf.SF_SPATIAL_QM(M)
        out = sf.sf_filter(t, r, kind, s, N).cpu().numpy().astype(np.float64)
        ref = oracle.bilateral_shiftable(img, r, kind, s, N)
        e = np.abs(out - ref)
        worst = max(worst, float(e.max()))
        print(json.dumps({"M": M, "r": r, "max": float(e.max()), "mean": float(e.mean())}), flush=True)
for M, ss in ((2, 3.0), (4, 5.0)):
    r = 10
    try:
        out = sf.sf_filter_spatial_sigma(t, r, ss, M, s, N).cpu().numpy().astype(np.float64)
        ref = oracle.bilateral_shiftable(img, r, sf.SF_SPATIAL_QM(M), s, N, beta=oracle.spatial_beta(ss, M))
        e = np.abs(out - ref)
        worst = max(worst, float(e.max()))
        print(json.dumps({"sigma_s": ss, "M": M, "r": r, "max": float(e.max()), "mean": float(e.mean())}), flush=True)
    except Exception as ex:  # report, keep going
        print(json.dumps({"sigma_s": ss, "M": M, "error": str(ex)}), flush=True)
print(json.dumps({"worst": worst}), flush=True)

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
c = synth.CONFIGS["cfg3"]
img3 = torch.from_numpy(c.image()).cuda()
o3 = torch.empty(img3.shape, dtype=torch.float32, device="cuda")
for M in (2, 1, 3, 4):
    kind = c.kind if M == 2 else sf.SF_SPATIAL_QM(M)
    fn = lambda: sf.sf_filter(img3, c.radius, kind, c.sigma_r, c.N, out=o3)
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.fill_(1.0)
        torch.cuda._sleep(400000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"cfg3_size": True, "M": M, "env": {k: v for k, v in os.environ.items() if k.startswith("SF_")},
                      "ms": round(sorted(ts)[2], 4)}), flush=True)
