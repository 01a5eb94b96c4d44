"""One small filter call for the hang/parity matrix (tools/gpu_diag.sh):
prints max-abs vs the fp64 oracle.  usage: python tools/hangcheck.py H W r N sigma_r"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_1107_4617_b200 as sf
import synth

H, W, r, N = (int(a) for a in sys.argv[1:5])
s = float(sys.argv[5])
img = synth.gen_image(H, W, 7, 10.0)
out = sf.sf_filter(torch.from_numpy(img).cuda(), r, 0, s, N)
torch.cuda.synchronize()
ref = oracle.bilateral_shiftable(img, r, 0, s, N)
print(os.environ.get("SF_VARIANT"), H, W, r, N, "max_abs", float(np.abs(out.cpu().numpy() - ref).max()))
