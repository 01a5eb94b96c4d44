"""One sf_filter call on a named config (after a warm-up call) for ncu captures.
usage: python tools/prof_cfg.py cfg3 [radius] [M]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import synth

c = synth.CONFIGS[sys.argv[1]]
r = int(sys.argv[2]) if len(sys.argv) > 2 else c.radius
kind = sf.SF_SPATIAL_QM(int(sys.argv[3])) if len(sys.argv) > 3 else c.kind
img = torch.from_numpy(c.image()).cuda()
out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
for _ in range(2):
    sf.sf_filter(img, r, kind, c.sigma_r, c.N, out=out)
torch.cuda.synchronize()
