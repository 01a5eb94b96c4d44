"""Timings of the §8(f) extensions on one GPU (CUDA events, median of 5, L2
flushed) on a 2048 x 2048 synthetic image: Algorithm 1 spatial filters (box,
q_2, q_4), the q_M bilateral (M = 1..4 on the v7q band sweep, 6 on the tile
kernel), the sigma_s-fitted spatial kernel, term truncation (f1) against the
full expansion, the polynomial range kernel (f3, fp64) and the shiftable NLM
with p = 1, 2, 3 (f4).  One JSON line per case: ms, Mpixel/s, terms
evaluated per pixel, Gpixel.term/s."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_1107_4617_b200 as sf
import synth

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


H = W = 2048
img = torch.from_numpy(synth.gen_image(H, W, 3, 10.0)).cuda()
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
N0P = sf.sf_nmin_poly(40.0)
cases = [
    ("spatial box r=10 (Alg. 1)", lambda: sf.sf_spatial_filter(img, 10, 0, out=out), 1),
    ("spatial q_2 r=10 (Alg. 1)", lambda: sf.sf_spatial_filter(img, 10, 1, out=out), 1),
    ("spatial q_4 r=10 (Alg. 1)", lambda: sf.sf_spatial_filter(img, 10, sf.SF_SPATIAL_QM(4), out=out), 1),
    ("bilateral q_1 r=10 s=40 N=17", lambda: sf.sf_filter(img, 10, sf.SF_SPATIAL_QM(1), 40.0, 17, out=out), 18),
    ("bilateral q_2 r=10 s=40 N=17 (cfg3)", lambda: sf.sf_filter(img, 10, 1, 40.0, 17, out=out), 18),
    ("bilateral q_3 r=10 s=40 N=17", lambda: sf.sf_filter(img, 10, sf.SF_SPATIAL_QM(3), 40.0, 17, out=out), 18),
    ("bilateral q_4 r=10 s=40 N=17", lambda: sf.sf_filter(img, 10, sf.SF_SPATIAL_QM(4), 40.0, 17, out=out), 18),
    ("bilateral q_6 r=10 s=40 N=17 (tile kernel)", lambda: sf.sf_filter(img, 10, sf.SF_SPATIAL_QM(6), 40.0, 17, out=out), 18),
    ("bilateral sigma_s=5 M=4 r=10 s=40 N=17", lambda: sf.sf_filter_spatial_sigma(img, 10, 5.0, 4, 40.0, 17, out=out), 18),
    ("bilateral box r=16 s=10 N=264", lambda: sf.sf_filter(img, 16, 0, 10.0, 264, out=out), 265),
    ("truncated box r=16 s=10 N=264 eps=1e-6", lambda: sf.sf_filter_truncated(img, 16, 0, 10.0, 264, 1e-6, out=out),
     265 - 2 * sf.sf_truncation_n0(264, 1e-6)),
    (f"poly p_N box r=8 s=40 N={N0P} (fp64)", lambda: sf.sf_filter_poly(img, 8, 40.0, N0P, out=out), 2 * N0P + 2),
    ("nlm p=1 r=5 h=60 n=15", lambda: sf.sf_nlm(img, 5, 1, 60.0, 1.0, 15, out=out), 16),
    ("nlm p=2 r=5 h=60 n=15", lambda: sf.sf_nlm(img, 5, 2, 60.0, 1.0, 15, out=out), 256),
    ("nlm p=3 r=5 h=150 n=7", lambda: sf.sf_nlm(img, 5, 3, 150.0, 0.8, 7, out=out), 512),
]
for name, fn, terms in cases:
    ms = timed(fn)
    print(json.dumps({"case": name, "H": H, "W": W, "ms": round(ms, 4), "mpix_s": round(H * W / ms / 1e3, 1),
                      "terms": terms, "gpix_term_s": round(H * W * terms / ms / 1e6, 1),
                      "launches": sf.sf_last_launch_count()}), flush=True)
