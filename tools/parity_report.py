"""Full-size element-wise parity report: GPU (C-ABI) vs fp64 oracle (Algorithm 2)
for every BASELINE config (cfg5 at r = 4, 16, 64).  Prints one JSON line per case."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_1107_4617_b200 as sf
import synth


def main():
    cases = [(n, c.radius) for n, c in synth.CONFIGS.items() if n != "cfg5"] + [("cfg5", r) for r in (4, 16, 64)]
    only = sys.argv[1:]
    for name, r in cases:
        if only and name not in only:
            continue
        c = synth.CONFIGS[name]
        img = c.image()
        t0 = time.perf_counter()
        ref, num, den = oracle.bilateral_shiftable(img, r, c.kind, c.sigma_r, c.N, return_parts=True)
        t_or = time.perf_counter() - t0
        out = sf.sf_filter(torch.from_numpy(img).cuda(), r, c.kind, c.sigma_r, c.N)
        torch.cuda.synchronize()
        err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
        i = int(np.argmax(err))
        print(json.dumps({"case": f"{name} r={r}", "max_abs": float(err.max()), "mean_abs": float(err.mean()),
                          "p99_99": float(np.quantile(err, 0.9999)), "worst_pixel": i,
                          "den_at_worst": float(den.flat[i]), "min_den": float(den.min()),
                          "oracle_s": round(t_or, 1), "oracle_threads": oracle.max_threads()}), flush=True)


if __name__ == "__main__":
    main()
