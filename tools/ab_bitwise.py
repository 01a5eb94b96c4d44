"""Bitwise comparison of sf_filter between the in-tree library and an A/B
build (SF_LIB_OVERRIDE in a child process): a change of synchronisation only
must leave every output bit unchanged.
usage: python tools/ab_bitwise.py tools/_ab/libsf_X.so [H W r sigma_r N ...]"""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1107_4617_b200 as sf, synth
a = sys.argv[3:]
outs = []
for i in range(0, len(a), 5):
    H, W, r, s, N = int(a[i]), int(a[i+1]), int(a[i+2]), float(a[i+3]), int(a[i+4])
    img = torch.from_numpy(synth.gen_image(H, W, 3, 10.0)).cuda()
    outs.append(sf.sf_filter(img, r, 0, s, N).cpu().numpy().ravel())
np.save(sys.argv[2], np.concatenate(outs))
"""
lib = sys.argv[1]
cases = sys.argv[2:] or ["2048", "2048", "16", "15", "118", "1080", "1920", "8", "20", "66", "777", "1333", "24", "10", "264",
                         "4096", "4096", "4", "15", "118"]
res = []
for env_lib in (None, lib):
    env = dict(os.environ)
    env.pop("SF_LIB_OVERRIDE", None)
    if env_lib:
        env["SF_LIB_OVERRIDE"] = env_lib
    dst = f"/tmp/ab_bitwise_{len(res)}.npy"
    subprocess.run([sys.executable, "-c", CHILD, ROOT, dst] + cases, env=env, check=True, timeout=600)
    res.append(np.load(dst))
same = np.array_equal(res[0].view(np.uint32), res[1].view(np.uint32))
print({"lib": lib, "bitwise_equal": bool(same), "max_abs_diff": float(np.max(np.abs(res[0] - res[1])))})
