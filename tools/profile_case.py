"""Run one filter call (after warm-up) for ncu captures.
usage: python tools/profile_case.py H W radius kind sigma_r N [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_1107_4617_b200 as sf
import synth

H, W, r, kind = (int(a) for a in sys.argv[1:5])
s, N = float(sys.argv[5]), int(sys.argv[6])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
img = torch.from_numpy(synth.gen_image(H, W, 5, 10.0)).cuda()
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
for _ in range(reps):
    sf.sf_filter(img, r, kind, s, N, out=out)
torch.cuda.synchronize()
print("ok", float(out.mean()))
