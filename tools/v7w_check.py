"""Parity of the wide large-radius kernel (SF_VARIANT=v7w) against the fp64
oracle: every radius 25..64 on a 150 x 530 image, plus a speck image
(reading R16's hard case) at r = 32 and 64."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import oracle, synth

H, W, N, s = 150, 530, 30, 30.0
img = synth.gen_image(H, W, 77, 10.0)
t = torch.from_numpy(img).cuda()
worst = 0.0
for r in range(25, 65):
    out = sf.sf_filter(t, r, 0, s, N).cpu().numpy().astype(np.float64)
    e = np.abs(out - oracle.bilateral_shiftable(img, r, 0, s, N))
    worst = max(worst, float(e.max()))
    if e.max() > 0.05 or e.mean() > 0.005:
        print("FAIL r", r, float(e.max()), float(e.mean()), flush=True)
print("radii 25..64 worst max-abs", worst, flush=True)
rng = np.random.default_rng(5)
sp = np.full((600, 700), 255, np.uint8)
sp.flat[rng.choice(sp.size, sp.size // 200, replace=False)] = 0
ts = torch.from_numpy(sp).cuda()
for r in (32, 64):
    out = sf.sf_filter(ts, r, 0, 15.0, 118).cpu().numpy().astype(np.float64)
    e = np.abs(out - oracle.bilateral_shiftable(sp, r, 0, 15.0, 118))
    print("speck r", r, "max", float(e.max()), "mean", float(e.mean()), flush=True)
