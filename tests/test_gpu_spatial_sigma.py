"""GPU parity of f2's Gaussian-fitted separable spatial kernel
(sf_filter_spatial_sigma / sf_spatial_filter_sigma: w1(u) =
cos(u/(sigma_s sqrt M))^M, Eq.(7) with T = pi sigma_s/2) against the fp64
oracle (Algorithm 2 with the same spatial expansion), element by element."""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("r,sigma_s,M", [(5, 2.0, 3), (10, 3.0, 5), (10, 6.0, 2), (16, 4.0, 8), (24, 8.0, 6)])
def test_bilateral_spatial_sigma(r, sigma_s, M):
    import paper_1107_4617_b200 as sf
    assert M >= sf.sf_spatial_mmin(r, sigma_s) == oracle.spatial_mmin(r, sigma_s)
    img = synth.gen_image(150, 211, 80 + r, 10.0)
    got = sf.sf_filter_spatial_sigma(torch.from_numpy(img).cuda(), r, sigma_s, M, 30.0, 30).cpu().numpy()
    ref = oracle.bilateral_shiftable(img, r, 100 + M, 30.0, 30, beta=oracle.spatial_beta(sigma_s, M))
    err = np.abs(got.astype(np.float64) - ref)
    assert err.max() <= 0.05 and err.mean() <= 0.005, (r, sigma_s, M, err.max(), err.mean())


def test_algorithm1_spatial_sigma_and_errors():
    import paper_1107_4617_b200 as sf
    img = synth.gen_image(120, 130, 9, 10.0)
    r, ss, M = 8, 3.0, 4
    got = sf.sf_spatial_filter_sigma(torch.from_numpy(img).cuda(), r, ss, M).cpu().numpy()
    ref = oracle.bilateral_shiftable(img, r, 100 + M, 30.0, 0, beta=oracle.spatial_beta(ss, M))
    assert np.abs(got - ref).max() <= 0.05
    t = torch.from_numpy(img).cuda()
    with pytest.raises(sf.SFError):          # M below the validity order
        sf.sf_filter_spatial_sigma(t, 16, 2.0, 2, 30.0, 30)
    with pytest.raises(sf.SFError):          # M beyond the walker's 8
        sf.sf_filter_spatial_sigma(t, 4, 2.0, 9, 30.0, 30)
