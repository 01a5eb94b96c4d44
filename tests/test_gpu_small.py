"""GPU parity of the small-image kernel (box_small.cuh, "vs": tile x pair
groups, rotation across pairs) against the fp64 oracle.

The kernel is the default for box radii 1..8 on images of at most one wave
of its 16 x 32 tiles (config 1); SF_VARIANT=vs forces it on larger images so
that its tile seams, ragged tiles and every radius are checked.  Each case
runs in its own process (the variant is read once per process)."""
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
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1107_4617_b200 as sf, synth
H, W, N, s, seed, noise = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5]), int(sys.argv[6]), float(sys.argv[7])
radii = [int(x) for x in sys.argv[9].split(",")]
img = torch.from_numpy(synth.gen_image(H, W, seed, noise)).cuda()
outs = []
for r in radii:
    outs.append(sf.sf_filter(img, r, 0, s, N).cpu().numpy())
    # the term split's partials over two pair ranges, summed, then finalized
    K = sf.sf_pair_count(N)
    n1, d1 = sf.sf_accumulate(img, r, 0, s, N, 0, K // 3)
    n2, d2 = sf.sf_accumulate(img, r, 0, s, N, K // 3, K)
    outs.append(sf.sf_finalize(n1 + n2, d1 + d2, img).cpu().numpy())
    # a row band [H/3, 2H/3) from its input rows plus r halo rows
    b0, b1 = H // 3, max(H // 3 + 1, 2 * H // 3)
    i0, i1 = max(0, b0 - r), min(H, b1 + r)
    band = sf.sf_filter_rows(img[i0:i1].contiguous(), H, W, b0, b1, r, 0, s, N).cpu().numpy()
    full = np.full((H, W), np.nan, dtype=np.float32)
    full[b0:b1] = band
    outs.append(full)
np.save(sys.argv[8], np.stack(outs))
"""


def _run(tmp_path, H, W, N, s, seed, radii, variant="vs", noise=10.0):
    dst = str(tmp_path / "out.npy")
    env = dict(os.environ)
    env.pop("SF_VARIANT", None)
    if variant:
        env["SF_VARIANT"] = variant
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(H), str(W), str(N), str(s), str(seed), str(noise), dst,
                    ",".join(map(str, radii))], env=env, check=True, timeout=180)
    return np.load(dst).astype(np.float64)


def _check(got, img, radii, s, N):
    for i, r in enumerate(radii):
        ref = oracle.bilateral_shiftable(img, r, 0, s, N)
        for j, what in enumerate(("filter", "accumulate+finalize", "row band")):
            g = got[3 * i + j]
            m = np.isfinite(g)
            err = np.abs(g[m] - ref[m])
            assert m.any() and err.max() <= 0.05 and err.mean() <= 0.005, (r, what, err.max(), err.mean())


@pytest.mark.parametrize("H,W,N,s", [(203, 517, 30, 30.0), (61, 95, 67, 20.0), (130, 200, 264, 10.0)])
def test_small_kernel_every_radius(H, W, N, s, tmp_path):
    """radii 1..8 on ragged shapes (partial tiles in both directions), even and
    odd N, N = 264 (133 pairs, uneven pair groups); filter, term split, row band."""
    radii = list(range(1, 9))
    seed = 500 + H
    got = _run(tmp_path, H, W, N, s, seed, radii)
    _check(got, synth.gen_image(H, W, seed, 10.0), radii, s, N)


def test_small_kernel_tiny_images(tmp_path):
    """images smaller than one tile, r = min(H, W) - 1 (the largest the
    reflect-101 boundary allows), fewer pairs than pair groups (N = 2: 2 pairs)."""
    for (H, W, r, N, s) in [(9, 9, 8, 30, 30.0), (3, 40, 2, 30, 30.0), (20, 5, 4, 2, 300.0), (1 + 16, 33, 8, 4, 200.0)]:
        seed = 7 + H + W
        got = _run(tmp_path, H, W, N, s, seed, [r])
        _check(got, synth.gen_image(H, W, seed, 10.0), [r], s, N)


def test_small_default_dispatch_cfg1_specks(tmp_path):
    """the default dispatch on a config-1-sized speck image (flat 255, 0.5 %
    zero specks: reading R16's hard case) stays within the bar."""
    H = W = 256
    rng = np.random.default_rng(11)
    img = np.full((H, W), 255, np.uint8)
    img.flat[rng.choice(H * W, H * W // 200, replace=False)] = 0
    dst = str(tmp_path / "speck.npy")
    np.save(str(tmp_path / "img.npy"), img)
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1107_4617_b200 as sf
img = torch.from_numpy(np.load(sys.argv[2])).cuda()
np.save(sys.argv[3], np.stack([sf.sf_filter(img, r, 0, 30.0, 30).cpu().numpy() for r in (1, 5, 8)]))
"""
    env = dict(os.environ)
    env.pop("SF_VARIANT", None)
    subprocess.run([sys.executable, "-c", code, ROOT, str(tmp_path / "img.npy"), dst], env=env, check=True,
                   timeout=120)
    got = np.load(dst).astype(np.float64)
    for i, r in enumerate((1, 5, 8)):
        err = np.abs(got[i] - oracle.bilateral_shiftable(img, r, 0, 30.0, 30))
        assert err.max() <= 0.05 and err.mean() <= 0.005, (r, err.max(), err.mean())
