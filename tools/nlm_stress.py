"""NLM precision on speck images (flat background, 0.5 % isolated specks):
sampled parity at the smallest-weight pixels is not available for NLM, so the
whole image is compared with the oracle (small images)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1107_4617_b200 as sf
import oracle

for kind_img, p, r, h, rho, n in [("stars", 1, 5, 60.0, 1.0, 15), ("stars", 2, 5, 60.0, 1.0, 15), ("holes", 2, 8, 80.0, 0.7, 9),
                                  ("stars", 3, 3, 150.0, 0.8, 7)]:
    rng = np.random.default_rng(3)
    img = np.full((160, 300), 0 if kind_img == "stars" else 255, dtype=np.uint8)
    img[rng.random(img.shape) < 0.005] = 255 if kind_img == "stars" else 0
    got = sf.sf_nlm(torch.from_numpy(img).cuda(), r, p, h, rho, n).cpu().numpy().astype(np.float64)
    ref = oracle.nlm_shiftable(img, r, p, h, rho, n)
    err = np.abs(got - ref)
    print(json.dumps({"image": kind_img, "p": p, "r": r, "max_abs": float(err.max()), "mean_abs": float(err.mean())}), flush=True)
