"""f3 precision table: the GPU's fp64 Chebyshev-basis Algorithm 2
(sf_filter_poly) and the oracle's fp64 monomial-basis Algorithm 2 against the
brute-force Eq.(3) with phi_p, per order N = N0(sigma_r); one JSON line each.
usage: python tools/poly_errors.py > profiles/r02_poly_errors.jsonl"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1107_4617_b200 as sf
import oracle, synth

img = synth.gen_image(256, 256, 1, 10.0)
t = torch.from_numpy(img).cuda()
for sigma in (60.0, 40.0, 30.0, 20.0, 15.0, 10.0):
    N = sf.sf_nmin_poly(sigma)
    r = 5
    ref = oracle.bilateral_direct(img, r, 0, sigma, N, range_kind=3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = sf.sf_filter_poly(t, r, sigma, N)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0)
    got = got.cpu().numpy().astype(np.float64)
    mono = oracle.bilateral_poly_shiftable(img, r, sigma, N) if N <= 160 else None
    line = {"sigma_r": sigma, "N": N, "terms": 2 * N + 1, "image": "cfg1-like 256x256 seed 1", "r": r,
            "gpu_chebyshev_fp64_max_abs": float(np.abs(got - ref).max()),
            "gpu_chebyshev_fp64_mean_abs": float(np.abs(got - ref).mean()),
            "oracle_monomial_fp64_max_abs": float(np.abs(mono - ref).max()) if mono is not None else None,
            "gpu_ms_incl_table": round(ms, 3)}
    print(json.dumps(line), flush=True)
