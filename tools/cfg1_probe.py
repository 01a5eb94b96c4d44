"""A handful of sf_filter calls on cfg1-sized images for an ncu launch list
(kernel durations without the event floor).  usage: python tools/cfg1_probe.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1107_4617_b200 as sf
import synth

img = torch.from_numpy(synth.gen_image(256, 256, 1, 10.0)).cuda()
out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
for N in (2, 30, 118):
    s = 170.0 / N ** 0.5
    for _ in range(3):
        sf.sf_filter(img, 5, 0, s, N, out=out)
torch.cuda.synchronize()
