"""One NLM call (after warm-up) for ncu captures: python tools/profile_nlm.py H W r p h rho n"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_1107_4617_b200 as sf
import synth

H, W, r, p = (int(a) for a in sys.argv[1:5])
h, rho, n = float(sys.argv[5]), float(sys.argv[6]), int(sys.argv[7])
img = torch.from_numpy(synth.gen_image(H, W, 5, 10.0)).cuda()
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
for _ in range(2):
    sf.sf_nlm(img, r, p, h, rho, n, out=out)
torch.cuda.synchronize()
print("ok", float(out.mean()))
