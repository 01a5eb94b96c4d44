"""Running-sum drift stress (reading R15): uniform-noise images
(every pixel an outlier, denominators near 1) at the drift-capped segment
lengths, sampled parity at the smallest denominators against the oracle."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1107_4617_b200 as sf
import oracle

CASES = [("noise", 4096, 2048, 16, 15.0, 118), ("noise", 4096, 1024, 16, 10.0, 264),
         ("stars", 8192, 1024, 16, 15.0, 118), ("stars", 8192, 1024, 4, 15.0, 118),
         ("stars", 4096, 1024, 16, 10.0, 264), ("stars", 8192, 1024, 64, 15.0, 118),
         ("holes", 8192, 1024, 16, 15.0, 118), ("stars", 4096, 1024, 12, 25.0, 43)]
for (kind_img, H, W, r, s, N) in CASES:
    rng = np.random.default_rng(7)
    if kind_img == "noise":
        img = rng.integers(0, 256, (H, W), dtype=np.uint8)
    else:   # flat 0 (or 255) background with 0.5 % isolated 255 (0) specks: denominators ~1 at the specks
        img = np.full((H, W), 0 if kind_img == "stars" else 255, dtype=np.uint8)
        m = rng.random((H, W)) < 0.005
        img[m] = 255 if kind_img == "stars" else 0
    t = torch.from_numpy(img).cuda()
    out = sf.sf_filter(t, r, 0, s, N).cpu().numpy().ravel()
    _, den = sf.sf_accumulate(t, r, 0, s, N, 0, sf.sf_pair_count(N))
    low = torch.topk(den.flatten(), 1500, largest=False).indices.cpu().numpy()
    rnd = rng.choice(H * W, 1500, replace=False)
    idx = np.unique(np.concatenate([low, rnd])).astype(np.int64)
    ref = oracle.bilateral_direct(img, r, 0, s, N, idx=idx)
    err = np.abs(out[idx] - ref)
    print(json.dumps({"image": kind_img, "H": H, "W": W, "r": r, "sigma_r": s, "N": N, "max_abs": float(err.max()),
                      "mean_abs": float(err.mean()), "min_den": float(den.min())}), flush=True)
