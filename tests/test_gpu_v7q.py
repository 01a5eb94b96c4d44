"""GPU parity of the v7q band sweep (box_v7q.cuh): Algorithm 2
with the separable spatial kernel w1(u) = cos(beta u)^M, M = 1..4 (the q_M
family; config 3 is M = 2), r = 1..24, against the fp64
oracle element by element at BASELINE.json's bar (max-abs 0.05, mean-abs
0.005).  Covers every frequency count F = ceil(M/2), the odd-M kernels without
a zero frequency, window spans of one to several lane segments (Q = 0..5),
ragged strips, the sigma_s-fitted beta (Eq. (7)) and the
term-split partials."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
MAX_ABS, MEAN_ABS = 0.05, 0.005


def sf():
    import paper_1107_4617_b200 as m
    return m


def check(got, ref, what):
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(np.isfinite(got)), what
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (what, err.max(), err.mean())


@pytest.mark.parametrize("M", [1, 2, 3, 4])
@pytest.mark.parametrize("r", [1, 2, 5, 7, 10, 13, 16, 21, 24])
def test_qm_band_sweep(M, r):
    H, W, N, s = 150, 530, 30, 30.0
    img = synth.gen_image(H, W, 100 + r, 10.0)
    kind = sf().SF_SPATIAL_QM(M)
    got = sf().sf_filter(torch.from_numpy(img).cuda(), r, kind, s, N).cpu().numpy()
    check(got, oracle.bilateral_shiftable(img, r, kind, s, N), (M, r))


@pytest.mark.parametrize("H,W", [(40, 1000), (333, 517), (17, 64)])
def test_q2_shapes(H, W):
    """config 3's kernel (q_2, r = 10, sigma_r = 40, N = 17) on ragged shapes."""
    img = synth.gen_image(H, W, 7, 10.0)
    got = sf().sf_filter(torch.from_numpy(img).cuda(), 10, 1, 40.0, 17).cpu().numpy()
    check(got, oracle.bilateral_shiftable(img, 10, 1, 40.0, 17), (H, W))


@pytest.mark.parametrize("M,sigma_s", [(2, 8.0), (4, 5.0), (3, 6.0)])
def test_sigma_s_fitted(M, sigma_s):
    H, W, r, N, s = 120, 400, 10, 30, 30.0
    img = synth.gen_image(H, W, 3, 10.0)
    got = sf().sf_filter_spatial_sigma(torch.from_numpy(img).cuda(), r, sigma_s, M, s, N).cpu().numpy()
    ref = oracle.bilateral_shiftable(img, r, sf().SF_SPATIAL_QM(M), s, N, beta=oracle.spatial_beta(sigma_s, M))
    check(got, ref, (M, sigma_s))


def test_q2_term_split():
    """num/den partials (centred at SF_CENTER) over two pair ranges + finalize."""
    m = sf()
    H, W, r, N, s = 200, 480, 10, 66, 20.0
    img = synth.gen_image(H, W, 9, 10.0)
    t = torch.from_numpy(img).cuda()
    K = m.sf_pair_count(N)
    n1, d1 = m.sf_accumulate(t, r, 1, s, N, 0, K // 3)
    n2, d2 = m.sf_accumulate(t, r, 1, s, N, K // 3, K)
    got = m.sf_finalize(n1 + n2, d1 + d2, t).cpu().numpy()
    check(got, oracle.bilateral_shiftable(img, r, 1, s, N), "term split")


def test_q2_speck_image():
    """reading R16's hard case on the q_2 kernel: flat 255 with 0.5 % zero specks."""
    rng = np.random.default_rng(5)
    img = np.full((512, 640), 255, dtype=np.uint8)
    img[rng.random(img.shape) < 0.005] = 0
    got = sf().sf_filter(torch.from_numpy(img).cuda(), 10, 1, 15.0, 118).cpu().numpy()
    check(got, oracle.bilateral_shiftable(img, 10, 1, 15.0, 118), "specks")
