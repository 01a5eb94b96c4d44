"""GPU parity of every kernel variant (SF_VARIANT = v1 | v4 | v5 | v5m | v7 | v7m,
DESIGN.md §5) against the fp64 oracle, each in its own process (the variant
is read once per process).  The default dispatch is covered by
test_gpu_parity.py; this file keeps the non-default variants honest, with a
timeout so that a deadlocked kernel fails instead of hanging the suite."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1107_4617_b200 as sf, synth
H, W, r, N, s, seed, kind = (int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]),
                             float(sys.argv[6]), int(sys.argv[7]), int(sys.argv[9]))
img = synth.gen_image(H, W, seed, 10.0)
out = sf.sf_filter(torch.from_numpy(img).cuda(), r, kind, s, N)
torch.cuda.synchronize()
np.save(sys.argv[8], out.cpu().numpy())
"""


CASES = [(v, r, 0) for v in ["v1", "v4", "v5", "v5m", "v7", "v7m", "vs"] for r in [4, 5, 8, 10, 16]] + \
        [(v, r, 1) for v in ["v1", "default"] for r in [4, 5, 8, 10, 16]]   # q_2: tile kernel / band sweep


@pytest.mark.parametrize("variant,r,kind", CASES)
def test_variant_parity(variant, r, kind, tmp_path):
    H, W, N, s, seed = 203, 517, 66, 20.0, 300 + r
    dst = str(tmp_path / "out.npy")
    env = dict(os.environ)
    env.pop("SF_VARIANT", None)
    if variant != "default":
        env["SF_VARIANT"] = variant
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(H), str(W), str(r), str(N), str(s), str(seed), dst,
                    str(kind)], env=env, check=True, timeout=120)
    got = np.load(dst).astype(np.float64)
    ref = oracle.bilateral_shiftable(synth.gen_image(H, W, seed, 10.0), r, kind, s, N)
    err = np.abs(got - ref)
    assert err.max() <= 0.05 and err.mean() <= 0.005, (variant, r, kind, err.max(), err.mean())


CHILD_RADII = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1107_4617_b200 as sf, synth
H, W, N, s, seed = 150, 530, 30, 30.0, 77
img = torch.from_numpy(synth.gen_image(H, W, seed, 10.0)).cuda()
outs = [sf.sf_filter(img, r, 0, s, N).cpu().numpy() for r in range(1, 65)]
np.save(sys.argv[2], np.stack(outs))
"""


@pytest.mark.parametrize("variant", ["default", "v5", "v5m", "v7", "v7m", "v7w"])
def test_every_radius_1_to_64(variant, tmp_path):
    """The band-sweep kernels are instantiated for every radius: v5 for
    1..64 (v5_dispatch.h), v7 for 1..24 (v7_dispatch.h; larger radii fall
    back to v5), each with the outgoing rows by rotation (v5 / v7, R <= 32)
    and by MUFU (v5m / v7m); each one against the oracle on a 150 x 530
    image (2-4 column strips with a ragged last one, 10 row batches)."""
    dst = str(tmp_path / "radii.npy")
    env = dict(os.environ)
    env.pop("SF_VARIANT", None)
    if variant != "default":
        env["SF_VARIANT"] = variant
    subprocess.run([sys.executable, "-c", CHILD_RADII, ROOT, dst], env=env, check=True, timeout=300)
    got = np.load(dst).astype(np.float64)
    img = synth.gen_image(150, 530, 77, 10.0)
    for r in range(1, 65):
        ref = oracle.bilateral_shiftable(img, r, 0, 30.0, 30)
        err = np.abs(got[r - 1] - ref)
        assert err.max() <= 0.05 and err.mean() <= 0.005, (variant, r, err.max(), err.mean())


CHILD_NLM = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1107_4617_b200 as sf, synth
img = torch.from_numpy(synth.gen_image(150, 300, 91, 10.0)).cuda()
outs = [sf.sf_nlm(img, r, p, 90.0, 0.8, 9).cpu().numpy() for p in (1, 2, 3) for r in (3, 5)]
np.save(sys.argv[2], np.stack(outs))
"""


@pytest.mark.parametrize("variant", ["default", "v1"])
def test_nlm_band_sweep_and_tile(variant, tmp_path):
    """sf_nlm on both of its kernels — the band sweep (default) and the tile
    kernel (SF_VARIANT=v1) — against the oracle, p = 1..3."""
    dst = str(tmp_path / "nlm.npy")
    env = dict(os.environ)
    env.pop("SF_VARIANT", None)
    if variant != "default":
        env["SF_VARIANT"] = variant
    subprocess.run([sys.executable, "-c", CHILD_NLM, ROOT, dst], env=env, check=True, timeout=300)
    got = np.load(dst).astype(np.float64)
    img = synth.gen_image(150, 300, 91, 10.0)
    i = 0
    for p in (1, 2, 3):
        for r in (3, 5):
            ref = oracle.nlm_shiftable(img, r, p, 90.0, 0.8, 9)
            err = np.abs(got[i] - ref)
            assert err.max() <= 0.05 and err.mean() <= 0.005, (variant, p, r, err.max(), err.mean())
            i += 1


PS_CASES = [(256, 256, 5, 30, 30.0), (40, 700, 8, 66, 20.0), (130, 200, 16, 264, 10.0), (17, 1000, 13, 118, 15.0)]


@pytest.mark.parametrize("ps", [1, 2, 3, 4])
@pytest.mark.parametrize("H,W,r,N,s", PS_CASES)
def test_pair_split(ps, H, W, r, N, s, tmp_path):
    """The v7 pair split (ps CTAs of a cluster per unit, each over a pair
    subrange, DSMEM reduction of (Q, P')): forced by SF_V7_PS = ps, uneven
    subranges included (16 / 3, 133 / 4 pairs)."""
    seed = 40 + r
    dst = str(tmp_path / "out.npy")
    env = dict(os.environ)
    env["SF_VARIANT"] = "v7m"          # (the default dispatch sends the small cases to box_small)
    env["SF_V7_PS"] = str(ps)
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(H), str(W), str(r), str(N), str(s), str(seed), dst, "0"],
                   env=env, check=True, timeout=120)
    got = np.load(dst).astype(np.float64)
    ref = oracle.bilateral_shiftable(synth.gen_image(H, W, seed, 10.0), r, 0, s, N)
    err = np.abs(got - ref)
    assert err.max() <= 0.05 and err.mean() <= 0.005, (ps, H, W, r, err.max(), err.mean())
