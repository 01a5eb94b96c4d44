"""GPU parity of f3, the polynomial range kernel (sf_filter_poly, fp64
Chebyshev-basis Algorithm 2): against the brute-force oracle (Eq.(3) with
phi_p, O1) element by element, at the validity threshold N0 of sigma_r in
{40, 30, 20, 15} (N = 21, 37, 82, 145) — including the orders where the
paper's monomial basis is useless in fp64 (tests/test_oracle_pins.py) — and
on a speck image."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 0.05, 0.005


@pytest.mark.parametrize("sigma_r", [40.0, 30.0, 20.0, 15.0])
@pytest.mark.parametrize("r", [3, 8, 16, 24])
def test_poly_vs_bruteforce(sigma_r, r):
    import paper_1107_4617_b200 as sf
    N = sf.sf_nmin_poly(sigma_r)
    assert N == oracle.nmin_poly(sigma_r)
    img = synth.gen_image(131, 197, 60 + r, 10.0)       # several tiles, ragged edges
    got = sf.sf_filter_poly(torch.from_numpy(img).cuda(), r, sigma_r, N).cpu().numpy().astype(np.float64)
    ref = oracle.bilateral_direct(img, r, 0, sigma_r, N, range_kind=3)
    err = np.abs(got - ref)
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (sigma_r, r, err.max(), err.mean())


def test_poly_speck_image_and_errors():
    import paper_1107_4617_b200 as sf
    rng = np.random.default_rng(3)
    img = np.full((96, 128), 255, np.uint8)
    img[rng.random(img.shape) < 0.01] = 0
    got = sf.sf_filter_poly(torch.from_numpy(img).cuda(), 8, 30.0, 37).cpu().numpy().astype(np.float64)
    ref = oracle.bilateral_direct(img, 8, 0, 30.0, 37, range_kind=3)
    assert np.abs(got - ref).max() <= MAX_ABS
    t = torch.zeros((8, 8), dtype=torch.uint8, device="cuda")
    with pytest.raises(sf.SFError):                     # N below the validity threshold
        sf.sf_filter_poly(t, 2, 30.0, 36)
    with pytest.raises(sf.SFError):                     # radius beyond SF_MAX_POLY_RADIUS
        sf.sf_filter_poly(torch.zeros((80, 80), dtype=torch.uint8, device="cuda"), 33, 30.0, 37)
