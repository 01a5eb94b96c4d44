"""Quick v5c check: small image, r = 33, 48, 64 against the oracle, then one cfg5 r = 64 timing."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1107_4617_b200 as sf
import oracle, synth
img = synth.gen_image(150, 530, 77, 10.0)
t = torch.from_numpy(img).cuda()
for r in (33, 48, 64):
    out = sf.sf_filter(t, r, 0, 30.0, 30).cpu().numpy()
    ref = oracle.bilateral_shiftable(img, r, 0, 30.0, 30)
    e = np.abs(out - ref)
    print("r", r, "max", e.max(), "mean", e.mean(), flush=True)
