"""Where do the sampled full-size parity errors sit (row/col, rows mod 16)?"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1107_4617_b200 as m
import synth, oracle
name, r = sys.argv[1], int(sys.argv[2])
c = synth.CONFIGS[name]
img = c.image()
H, W = img.shape
timg = torch.from_numpy(img).cuda()
out = m.sf_filter(timg, r, c.kind, c.sigma_r, c.N).cpu().numpy()
_, den = m.sf_accumulate(timg, r, c.kind, c.sigma_r, c.N, 0, m.sf_pair_count(c.N))
d = den.flatten()
low = torch.topk(d, 2000, largest=False).indices.cpu().numpy()
rnd = np.random.default_rng(1234).choice(H * W, 6000, replace=False)
idx = np.unique(np.concatenate([low, rnd])).astype(np.int64)
ref = oracle.bilateral_direct(img, r, c.kind, c.sigma_r, c.N, idx=idx)
err = np.abs(out.ravel()[idx] - ref)
print("max", err.max(), "mean", err.mean())
o = np.argsort(-err)[:15]
dd = d.cpu().numpy()
for i in o:
    y, x = divmod(int(idx[i]), W)
    print(f"y={y} x={x} y%16={y%16} err={err[i]:.4f} got={out.ravel()[idx[i]]:.3f} ref={ref[i]:.3f} den={dd[idx[i]]:.3f} f={img[y,x]}")
