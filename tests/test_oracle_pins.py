"""Pins of the fp64 oracle against the paper and mathematics (not against itself).

Each test names the passage (PAPER.md line, section/equation/algorithm) or the
mathematical fact it checks.  A plausible mistake in the oracle — a dropped
term, a wrong sign of omega_n, a wrong coefficient, a wrong boundary, a
transposed operand, weighting by f(x) instead of f(x-y), the wrong sigma
scaling — fails at least one of these.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view
from scipy import ndimage

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ORDERS = [1, 2, 3, 17, 30, 66, 118, 264]


# ---------------------------------------------------------------- Eq.(1) ----

@pytest.mark.parametrize("N", ORDERS)
def test_coefficients_are_exact_binomials(N):
    """c_n = C(N,n)/2^N (binomial expansion of ((e^{jx}+e^{-jx})/2)^N), exact
    rational arithmetic; sum c_n = 1 (phi(0) = 1, PAPER.md:202 q_N(0)=1)."""
    om, c = oracle.expansion(N, 20.0)
    for n in range(N + 1):
        exact = float(Fraction(math.comb(N, n), 2 ** N))
        assert c[n] == pytest.approx(exact, rel=1e-15, abs=0.0)
    assert math.fsum(c) == pytest.approx(1.0, abs=1e-15)
    gamma = 1.0 / (20.0 * math.sqrt(N))
    # omega_n = (2n - N) gamma: antisymmetric, step 2 gamma
    assert np.allclose(om, (2 * np.arange(N + 1) - N) * gamma, rtol=0, atol=1e-15)
    assert np.allclose(om + om[::-1], 0.0, atol=1e-15)


@pytest.mark.parametrize("N,sigma", [(1, 300.0), (2, 200.0), (17, 40.0), (30, 30.0),
                                     (66, 20.0), (118, 15.0), (264, 10.0)])
def test_shiftability_identity(N, sigma):
    """Eq.(1): phi(t - tau) = sum_n d_n(tau) phi_n(t) with
    d_n(tau) = c_n e^{-j omega_n tau}, phi_n(t) = e^{j omega_n t}, at 1000 random
    (t, tau) in [-255, 255]^2; |err| <= 1e-12 * sum|d_n|."""
    rng = np.random.default_rng(N)
    t = rng.uniform(-255, 255, 1000)
    tau = rng.uniform(-255, 255, 1000)
    om, c = oracle.expansion(N, sigma)
    lhs = np.array([oracle.range_kernel(a - b, sigma, N) for a, b in zip(t, tau)])
    d = c[None, :] * np.exp(-1j * om[None, :] * tau[:, None])
    rhs = (d * np.exp(1j * om[None, :] * t[:, None])).sum(axis=1)
    assert np.max(np.abs(rhs.imag)) < 1e-12
    assert np.max(np.abs(lhs - rhs.real)) < 1e-12 * 1.0   # sum |d_n| = sum c_n = 1


def test_cosine_shift_identity_N1():
    """PAPER.md:36 (Sec. 1): cos(x - tau) = cos(tau)cos(x) + sin(tau)sin(x).
    With N = 1 the expansion has omega = -/+gamma, c = 1/2 and its conjugate pair
    must reduce to exactly that identity."""
    sigma = 50.0
    om, c = oracle.expansion(1, sigma)
    gamma = 1.0 / sigma
    assert om[0] == pytest.approx(-gamma) and om[1] == pytest.approx(gamma)
    assert c[0] == 0.5 and c[1] == 0.5
    rng = np.random.default_rng(0)
    for x, tau in rng.uniform(-255, 255, (200, 2)):
        pair = sum(c[n] * np.exp(-1j * om[n] * tau) * np.exp(1j * om[n] * x) for n in range(2))
        X, TAU = gamma * x, gamma * tau
        assert pair.real == pytest.approx(math.cos(TAU) * math.cos(X) + math.sin(TAU) * math.sin(X),
                                          abs=1e-15)
        assert oracle.range_kernel(x - tau, sigma, 1) == pytest.approx(math.cos(X - TAU), abs=1e-13)


# ----------------------------------------------------- N0 rule (Sec. 3.1) ----

def test_nmin_golden():
    """N0 = ceil((2T/(pi sigma))^2): SPEC.md:95 example and the five config
    orders of BASELINE.json (tests/golden/nmin.json, each case cited)."""
    cases = json.load(open(os.path.join(GOLDEN, "nmin.json")))["cases"]
    for case in cases:
        assert oracle.nmin(case["sigma_r"]) == case["N0"], case["source"]
    for cfg in synth.CONFIGS.values():
        assert oracle.nmin(cfg.sigma_r) == cfg.N


@pytest.mark.parametrize("sigma", [10.0, 15.0, 20.0, 30.0, 40.0])
def test_kernel_valid_at_nmin(sigma):
    """at N >= N0 the kernel is symmetric,
    non-negative and unimodal on [-T, T]; below N0 the cosine argument leaves
    [-pi/2, pi/2] and unimodality (or non-negativity) fails."""
    N = oracle.nmin(sigma)
    t = np.arange(0, 256)
    v = np.array([oracle.range_kernel(x, sigma, N) for x in t])
    vm = np.array([oracle.range_kernel(-x, sigma, N) for x in t])
    assert np.array_equal(v, vm)
    assert np.all(v >= 0.0) and np.all(np.diff(v) <= 0.0) and v[0] == 1.0
    if N > 1:
        w = np.array([oracle.range_kernel(x, sigma, N - 1) for x in t])
        # odd N-1: negative lobe (may underflow to -0.0); even N-1: a second rise
        assert np.any(np.signbit(w[1:])) or np.any(np.diff(w) > 0.0)


def test_gaussian_limit_rate():
    """Eq.(6): q_N(t/sqrt N) -> Gaussian as N -> infinity.  In
    the sigma_r scaling (reading R1) log cos u = -u^2/2 - u^4/12 - ... gives
    sup_t |phi_N(t) - e^{-t^2/2 sigma^2}| = (4/3) e^{-2} / N + O(1/N^2) = 0.18045/N.
    A wrong gamma (e.g. pi/2T or 1/sigma) breaks both the limit and the rate."""
    sigma = 30.0
    t = np.linspace(-255, 255, 5101)
    closed = 4.0 / 3.0 * math.exp(-2.0)
    prev = None
    for N in [30, 120, 480, 1920]:
        err = max(abs(oracle.range_kernel(x, sigma, N) - oracle.gaussian_kernel(x, sigma)) for x in t)
        assert N * err == pytest.approx(closed, rel=0.03 if N >= 120 else 0.06)
        if prev is not None:
            assert err < prev
        prev = err
    assert oracle.gaussian_kernel(30.0, 30.0) == pytest.approx(math.exp(-0.5), rel=1e-15)


def test_spatial_q2_is_paper_qN():
    """Reading R5: the config-3 spatial weight (1 + cos(pi u/(r+1)))/2 is the
    paper's q_N(u) = cos(pi u / 2T)^N with N = 2, T = r + 1."""
    for r in [1, 4, 10, 16]:
        for u in range(-r, r + 1):
            assert oracle.spatial_weight(u, r, 1) == pytest.approx(
                math.cos(math.pi * u / (2 * (r + 1))) ** 2, abs=1e-15)
            assert oracle.spatial_weight(u, r, 0) == 1.0
        assert oracle.spatial_weight(r + 1, r, 1) == 0.0


# ------------------------------------------------- moving sums ----

def _box_sum_numpy(F, r):
    P = np.pad(F, r, mode="reflect")          # numpy 'reflect' == reflect-101 (R3)
    return sliding_window_view(P, (2 * r + 1, 2 * r + 1)).sum(axis=(2, 3))


@pytest.mark.parametrize("shape,r", [((17, 23), 1), ((31, 16), 5), ((64, 64), 7), ((9, 40), 8),
                                     ((5, 5), 4), ((1, 7), 0)])
def test_moving_sum_exact_on_integers(shape, r):
    """Sum(F,x,T) by recursion equals the library window sum
    exactly on integer images (all partial sums exact in fp64)."""
    rng = np.random.default_rng(r)
    F = rng.integers(-1000, 1000, shape).astype(np.float64)
    assert np.array_equal(oracle.moving_sum(F, r), _box_sum_numpy(F, r))


def test_moving_sum_ones_reflect101():
    """With reflect-101 every window has (2r+1)^2 samples: Sum(1) = (2r+1)^2
    everywhere (the clipped 9/6/4 of SPEC.md:196 is ZeroOutside, not used)."""
    for r in [1, 2, 3]:
        out = oracle.moving_sum(np.ones((7, 9)), r)
        assert np.all(out == (2 * r + 1) ** 2)


# ------------------------------------------------ Eq.(3) and Algorithm 2 ----

SMALL_CASES = [
    # (H, W, r, kind, sigma_r, N, seed)
    (48, 40, 5, 0, 30.0, 30, 1),
    (33, 47, 8, 0, 20.0, 66, 2),
    (40, 40, 10, 1, 40.0, 17, 3),
    (36, 29, 3, 0, 10.0, 264, 4),
    (30, 52, 4, 0, 15.0, 118, 5),
    (25, 25, 24, 0, 30.0, 31, 6),      # r = min(H, W) - 1 (largest allowed radius)
    (21, 34, 6, 1, 20.0, 67, 7),       # q_2 spatial, odd N
    (16, 16, 0, 0, 30.0, 30, 8),       # r = 0: output = input
]


@pytest.mark.parametrize("case", SMALL_CASES)
def test_algorithm2_equals_eq3_bruteforce(case):
    """The reduction of Eq.(3) to moving sums (Alg. 2
    PAPER.md:146-156) is an identity, so Alg. 2 (O2) must equal the literal
    double loop (O1) to fp64 rounding (<= 1e-9 grey levels)."""
    H, W, r, kind, s, N, seed = case
    img = synth.gen_image(H, W, seed, 20.0)
    o1 = oracle.bilateral_direct(img, r, kind, s, N)
    o2, num, den = oracle.bilateral_shiftable(img, r, kind, s, N, return_parts=True)
    assert np.max(np.abs(o1 - o2)) < 1e-9
    if r == 0:
        assert np.array_equal(o1, img.astype(np.float64))
    # denominator >= w(0) phi(0) = 1 when N >= N0 (R3 + R2): no guard needed
    assert np.min(den) >= 1.0 - 1e-9


def test_partial_terms_and_rows_add_up():
    """Alg. 2 step 3 is a sum over (m, n): partial sums over disjoint term
    ranges and row bands must add up to the whole (the term-split and
    row-band decompositions of the multi-GPU path)."""
    img = synth.gen_image(40, 36, 11, 10.0)
    r, kind, s, N = 4, 0, 15.0, 118
    _, num, den = oracle.bilateral_shiftable(img, r, kind, s, N, return_parts=True)
    cut = [0, 20, 59, 90, N + 1]
    pn = sum(oracle.bilateral_shiftable(img, r, kind, s, N, a, b, return_parts=True)[1]
             for a, b in zip(cut[:-1], cut[1:]))
    pd = sum(oracle.bilateral_shiftable(img, r, kind, s, N, a, b, return_parts=True)[2]
             for a, b in zip(cut[:-1], cut[1:]))
    assert np.allclose(pn, num, atol=1e-7, rtol=0) and np.allclose(pd, den, atol=1e-9, rtol=0)
    band = oracle.bilateral_shiftable(img, r, kind, s, N, row_begin=13, row_end=29)
    full = oracle.bilateral_shiftable(img, r, kind, s, N)
    assert np.max(np.abs(band - full[13:29])) < 1e-12


def test_two_level_image_closed_form():
    """Eq.(3) on an image with only two grey levels a, b has the closed form
    (n_a phi(a-f) a + n_b phi(b-f) b) / (n_a phi(a-f) + n_b phi(b-f)) with
    window counts n_a, n_b from a library window sum.  Catches weighting by
    f(x) instead of f(x-y), a wrong window size or a wrong boundary."""
    rng = np.random.default_rng(3)
    a, b = 90, 130
    mask = rng.random((30, 34)) < 0.3
    img = np.where(mask, b, a).astype(np.uint8)
    r, s, N = 3, 30.0, 30
    nb = _box_sum_numpy(mask.astype(np.float64), r)
    na = (2 * r + 1) ** 2 - nb
    gamma = 1.0 / (s * math.sqrt(N))
    f = img.astype(np.float64)
    pa, pb = np.cos(gamma * (a - f)) ** N, np.cos(gamma * (b - f)) ** N
    expect = (na * pa * a + nb * pb * b) / (na * pa + nb * pb)
    for out in (oracle.bilateral_direct(img, r, 0, s, N), oracle.bilateral_shiftable(img, r, 0, s, N)):
        assert np.max(np.abs(out - expect)) < 1e-9


def test_constant_image_unchanged():
    """Eq.(3) normalisation: a constant image is a fixed point."""
    for v in [0, 77, 255]:
        img = np.full((20, 26), v, np.uint8)
        for kind in (0, 1):
            assert np.max(np.abs(oracle.bilateral_shiftable(img, 5, kind, 30.0, 30) - v)) < 1e-10
            assert np.max(np.abs(oracle.bilateral_direct(img, 5, kind, 30.0, 30) - v)) < 1e-12


def test_step_edge_preserved():
    """Edge preservation of the bilateral filter: across a 0|255
    step phi(255) = cos(255/(sigma sqrt N))^N ~ 1e-52..0 at N0, so each side
    keeps its value."""
    img = np.zeros((32, 32), np.uint8)
    img[:, 16:] = 255
    for s, N in [(30.0, 30), (10.0, 264), (15.0, 118)]:
        out = oracle.bilateral_shiftable(img, 5, 0, s, N)
        assert np.max(np.abs(out - img)) < 1e-9


def test_wide_range_kernel_reduces_to_spatial_filter():
    """sigma_r -> infinity with N = N0 = 1: phi -> 1, so Eq.(3) reduces to the
    spatial filter Eq.(2): the box mean, or the q_2-weighted
    mean (library correlate with mode='mirror' == reflect-101)."""
    img = synth.gen_image(40, 44, 9, 10.0)
    f = img.astype(np.float64)
    r = 6
    box = _box_sum_numpy(f, r) / (2 * r + 1) ** 2
    w1 = np.array([oracle.spatial_weight(u, r, 1) for u in range(-r, r + 1)])
    w = np.outer(w1, w1)
    q2 = ndimage.correlate(f, w, mode="mirror") / w.sum()
    for fn in (oracle.bilateral_direct, oracle.bilateral_shiftable):
        assert np.max(np.abs(fn(img, r, 0, 1e9, 1) - box)) < 1e-9
        assert np.max(np.abs(fn(img, r, 1, 1e9, 1) - q2)) < 1e-9


def test_symmetries():
    """Symmetric kernels + flip-symmetric reflect-101: transposes and flips
    commute with the filter; f -> 255 - f maps to 255 - f~; f -> f + c maps to
    f~ + c (phi depends on differences only)."""
    img = synth.gen_image(36, 36, 12, 10.0)
    small = (img.astype(np.int32) * 200 // 255).astype(np.uint8)
    for kind in (0, 1):
        args = (5, kind, 30.0, 30)
        o = oracle.bilateral_shiftable(img, *args)
        assert np.max(np.abs(oracle.bilateral_shiftable(np.ascontiguousarray(img.T), *args) - o.T)) < 1e-9
        assert np.max(np.abs(oracle.bilateral_shiftable(np.ascontiguousarray(img[::-1]), *args) - o[::-1])) < 1e-9
        assert np.max(np.abs(oracle.bilateral_shiftable(np.ascontiguousarray(img[:, ::-1]), *args) - o[:, ::-1])) < 1e-9
        assert np.max(np.abs(oracle.bilateral_shiftable(255 - img, *args) - (255 - o))) < 1e-9
        os_ = oracle.bilateral_shiftable(small, *args)
        assert np.max(np.abs(oracle.bilateral_shiftable(small + 55, *args) - (os_ + 55))) < 1e-9


def test_convexity():
    """With N >= N0 all weights are >= 0, so f~(x) lies within the window's
    [min f, max f]."""
    img = synth.gen_image(40, 40, 13, 20.0)
    r = 4
    out = oracle.bilateral_shiftable(img, r, 0, 10.0, 264)
    P = np.pad(img, r, mode="reflect")
    win = sliding_window_view(P, (2 * r + 1, 2 * r + 1))
    assert np.all(out >= win.min(axis=(2, 3)) - 1e-9)
    assert np.all(out <= win.max(axis=(2, 3)) + 1e-9)


def test_convergence_to_gaussian_bilateral():
    """Eq.(6) at filter level: the raised-cosine bilateral
    filter converges to the Gaussian-range bilateral filter as N grows, with
    error ~ 1/N (N * max|diff| roughly constant)."""
    img = synth.gen_image(24, 24, 1, 10.0)
    r, s = 3, 30.0
    g = oracle.bilateral_direct(img, r, 0, s, 0, range_kind=1)
    errs = []
    for N in [30, 60, 120, 240, 480]:
        errs.append(np.max(np.abs(oracle.bilateral_direct(img, r, 0, s, N) - g)))
    assert all(b < a for a, b in zip(errs, errs[1:]))
    scaled = [N * e for N, e in zip([30, 60, 120, 240, 480], errs)]
    assert max(scaled) / min(scaled) < 1.15


# ---------------------------------------- f1: term truncation

@pytest.mark.parametrize("N,eps", [(30, 1e-3), (118, 1e-6), (264, 1e-6), (264, 1e-8), (17, 0.0)])
def test_truncation_n0_threshold(N, eps):
    """n0 is the first index whose exact binomial weight reaches eps * max c_n
    (exact rational arithmetic), so terms n0..N-n0 are exactly the kept set."""
    n0 = oracle.truncation_n0(N, eps)
    cmax = Fraction(math.comb(N, N // 2), 2 ** N)
    kept = [n for n in range(N + 1) if Fraction(math.comb(N, n), 2 ** N) >= Fraction(eps) * cmax]
    assert kept == list(range(n0, N - n0 + 1))


@pytest.mark.parametrize("N,sigma,eps", [(30, 30.0, 1e-3), (264, 10.0, 1e-6), (118, 15.0, 1e-4)])
def test_truncated_kernel_error_bound(N, sigma, eps):
    """Dropping terms of Eq.(1) changes the kernel by at most the dropped
    weight (triangle inequality, |e^{j w t}| = 1): |phi_eps - phi| <= sum of
    dropped c_n; with nothing dropped phi_eps = phi (to rounding)."""
    n0 = oracle.truncation_n0(N, eps)
    dropped = 2 * sum(float(Fraction(math.comb(N, n), 2 ** N)) for n in range(n0))
    for t in np.linspace(-255, 255, 203):
        full = oracle.range_kernel(t, sigma, N)
        assert abs(oracle.range_kernel_truncated(t, sigma, N, n0) - full) <= dropped + 1e-13
        assert oracle.range_kernel_truncated(t, sigma, N, 0) == pytest.approx(full, abs=1e-13)


@pytest.mark.parametrize("H,W,r,kind,sigma,N,eps", [(29, 37, 4, 0, 10.0, 264, 1e-6),
                                                    (24, 31, 3, 1, 30.0, 30, 1e-2),
                                                    (21, 26, 5, 0, 15.0, 118, 1e-4)])
def test_truncated_algorithm2_equals_bruteforce(H, W, r, kind, sigma, N, eps):
    """Algorithm 2 over the kept terms n0..N-n0 (the term range of O2) equals
    Eq.(3) brute force with the truncated kernel written out as a cosine sum:
    the reduction is exact for any coefficient set."""
    img = synth.gen_image(H, W, 77 + r, 20.0)
    n0 = oracle.truncation_n0(N, eps)
    o2 = oracle.bilateral_shiftable(img, r, kind, sigma, N, n_begin=n0, n_end=N - n0 + 1)
    o1 = oracle.bilateral_direct(img, r, kind, sigma, N, range_kind=2, n0=n0)
    assert np.max(np.abs(o2 - o1)) <= 1e-9


def test_truncated_output_bound():
    """A-posteriori bound per pixel: with delta = dropped weight and
    S = sum_y w(y) = (2r+1)^2 (box), |dP'| <= 255 delta S (P' centred at
    f(x)) and |dQ| <= delta S, so |f~_eps - f~| <= (255 + |f~ - f(x)|) delta S
    / (Q - delta S) wherever Q > delta S."""
    H, W, r, sigma, N, eps = 40, 44, 4, 10.0, 264, 1e-5
    img = synth.gen_image(H, W, 5, 20.0)
    n0 = oracle.truncation_n0(N, eps)
    delta = 2 * sum(float(Fraction(math.comb(N, n), 2 ** N)) for n in range(n0))
    full, _, den = oracle.bilateral_shiftable(img, r, 0, sigma, N, return_parts=True)
    trunc = oracle.bilateral_shiftable(img, r, 0, sigma, N, n_begin=n0, n_end=N - n0 + 1)
    S = (2 * r + 1) ** 2
    ok = den > 2 * delta * S
    bound = (255.0 + np.abs(full - img)) * delta * S / (den - delta * S)
    assert ok.mean() > 0.99
    assert np.all(np.abs(trunc - full)[ok] <= bound[ok] + 1e-9)


# ------------------------- f2: general separable spatial kernels q_M, Algorithm 1

QM = [101, 103, 104, 106, 108]


def test_qM_spatial_weights():
    """q_M(u) = cos(pi u / (2T))^M with T = r+1: q_M(0) = 1,
    positive on the window, products of shiftable kernels add orders
    (q_a q_b = q_{a+b}), and q_2 equals the (1+cos)/2 form
    of config 3 (cos^2(x/2) = (1 + cos x)/2)."""
    for r in (1, 5, 10, 16):
        for u in range(-r, r + 1):
            for a in range(1, 5):
                for b in range(1, 5):
                    qa = oracle.spatial_weight(u, r, 100 + a)
                    qb = oracle.spatial_weight(u, r, 100 + b)
                    assert qa * qb == pytest.approx(oracle.spatial_weight(u, r, 100 + a + b), rel=1e-12)
            assert oracle.spatial_weight(u, r, 102) == pytest.approx(oracle.spatial_weight(u, r, 1), rel=1e-12)
            assert oracle.spatial_weight(u, r, 107) > 0
        assert oracle.spatial_weight(0, r, 105) == 1.0
        assert oracle.spatial_weight(r + 1, r, 103) == 0.0


@pytest.mark.parametrize("kind", [0, 1] + QM)
def test_algorithm1_is_normalised_correlation(kind):
    """Algorithm 1 = the bilateral machinery with an
    order-0 (constant) range kernel: the normalised correlation of f with the
    separable kernel, checked against scipy.ndimage.correlate (mode 'mirror'
    = reflect-101)."""
    H, W, r = 37, 45, 6
    img = synth.gen_image(H, W, 31 + kind, 10.0)
    w1 = np.array([oracle.spatial_weight(u, r, kind) for u in range(-r, r + 1)])
    k2 = np.outer(w1, w1)
    ref = ndimage.correlate(img.astype(np.float64), k2 / k2.sum(), mode="mirror")
    got = oracle.bilateral_shiftable(img, r, kind, 30.0, 0)
    assert np.max(np.abs(got - ref)) <= 1e-9


@pytest.mark.parametrize("kind", QM)
def test_qM_algorithm2_equals_bruteforce(kind):
    """Algorithm 2 with (M+1)^2 spatial terms equals Eq.(3) brute force with the
    q_M spatial weight (the shiftable reduction is exact)."""
    img = synth.gen_image(23, 29, kind, 10.0)
    o2 = oracle.bilateral_shiftable(img, 4, kind, 30.0, 30)
    o1 = oracle.bilateral_direct(img, 4, kind, 30.0, 30)
    assert np.max(np.abs(o2 - o1)) <= 1e-9


# --------------------------------------------- f4: shiftable NLM, tiny patch

@pytest.mark.parametrize("p,rho,h,n", [(1, 1.0, 60.0, 15), (2, 1.0, 60.0, 15), (3, 0.8, 150.0, 7),
                                       (2, 0.0, 60.0, 15)])
def test_nlm_shiftable_equals_bruteforce(p, rho, h, n):
    """The paper's moving-sum algorithm over all (n+1)^p multi-indices
     equals Eq.(approx_multivariate) evaluated literally."""
    img = synth.gen_image(19, 22, 40 + p, 10.0)
    o2 = oracle.nlm_shiftable(img, 3, p, h, rho, n)
    o1 = oracle.nlm_direct(img, 3, p, h, rho, n)
    assert np.max(np.abs(o2 - o1)) <= 1e-9


def test_nlm_p1_is_bilateral_and_rho0_drops_neighbours():
    """p = 1 (patch = the pixel) is the bilateral filter with the raised-cosine
    range kernel of sigma_r = h / sqrt 2 (gamma_1 = 1/(sigma_r sqrt n)); with
    rho = 0 the patch weight g vanishes off the centre, so p = 2, 3 reduce to p = 1."""
    img = synth.gen_image(24, 27, 9, 10.0)
    a = oracle.nlm_direct(img, 4, 1, 60.0, 1.0, 15)
    b = oracle.bilateral_direct(img, 4, 0, 60.0 / math.sqrt(2.0), 15)
    assert np.max(np.abs(a - b)) <= 1e-10
    for p in (2, 3):
        c = oracle.nlm_direct(img, 4, p, 60.0, 0.0, 15)
        assert np.max(np.abs(c - a)) <= 1e-10


def test_nlm_constant_image_and_convergence_to_gaussian_nlm():
    """A constant image is unchanged; as n grows the shiftable kernel tends to
    the Gaussian patch weight exp(-h^-2 sum_k g(u_k) t_k^2) (Eq.(6) per factor,
    PAPER.md:244-247), and the filter to Gaussian NLM at rate ~1/n."""
    assert np.max(np.abs(oracle.nlm_direct(np.full((12, 13), 77, np.uint8), 3, 2, 60.0, 1.0, 15) - 77)) < 1e-10
    img = synth.gen_image(16, 18, 12, 10.0)
    H, W, r, h, rho = 16, 18, 3, 60.0, 1.0
    g = [1.0, math.exp(-1 / (2 * rho * rho))]
    pad = np.pad(img.astype(np.float64), r + 1, mode="reflect")
    ref = np.empty((H, W))
    for y in range(H):
        for x in range(W):
            cy, cx = y + r + 1, x + r + 1
            num = den = 0.0
            for dy in range(-r, r + 1):
                for dx in range(-r, r + 1):
                    zy, zx = cy - dy, cx - dx
                    d = g[0] * (pad[cy, cx] - pad[zy, zx]) ** 2 + g[1] * (pad[cy, cx + 1] - pad[zy, zx + 1]) ** 2
                    wgt = math.exp(-d / h ** 2)
                    num += wgt * pad[zy, zx]
                    den += wgt
            ref[y, x] = num / den
    errs = [np.max(np.abs(oracle.nlm_direct(img, r, 2, h, rho, n) - ref)) for n in (15, 60, 240)]
    assert errs[0] > errs[1] > errs[2]
    assert 2.5 < errs[0] / errs[1] < 6.0 and 2.5 < errs[1] / errs[2] < 6.0


@pytest.mark.parametrize("rho", [0.8, 1.5])
def test_nlm_p3_converges_to_gaussian_nlm_with_offset_u3(rho):
    """p = 3 with rho > 0 (reading R14: u_1 = (0,0), u_2 = (0,1), u_3 = (1,0),
    i.e. the pixel, its right neighbour and the pixel BELOW it; g(u) =
    exp(-|u|^2/(2 rho^2))): the shiftable NLM of Eq.(approx_multivariate)
     tends at rate ~1/n to Gaussian NLM with the weight
    exp(-h^-2 sum_k g(u_k) t_k^2) written out here independently of the
    oracle (which shares nlm_offsets / nlm_gamma between its O1 and O2, so O2 =
    O1 cannot catch an error there).  A wrong u_3 (e.g. (-1,0) or (0,-1)) or a
    wrong g(u_3) moves the oracle off this reference by O(1) grey levels and
    breaks the 1/n convergence."""
    img = synth.gen_image(17, 19, 23, 10.0)
    H, W, r, h = 17, 19, 3, 150.0
    g = [1.0, math.exp(-1 / (2 * rho * rho)), math.exp(-1 / (2 * rho * rho))]
    offs = [(0, 0), (0, 1), (1, 0)]                     # (dy, dx) of u_1, u_2, u_3
    pad = np.pad(img.astype(np.float64), r + 1, mode="reflect")   # numpy reflect = reflect-101
    ref = np.empty((H, W))
    for y in range(H):
        for x in range(W):
            cy, cx = y + r + 1, x + r + 1
            num = den = 0.0
            for dy in range(-r, r + 1):
                for dx in range(-r, r + 1):
                    zy, zx = cy - dy, cx - dx
                    d = sum(gk * (pad[cy + oy, cx + ox] - pad[zy + oy, zx + ox]) ** 2
                            for gk, (oy, ox) in zip(g, offs))
                    wgt = math.exp(-d / h ** 2)
                    num += wgt * pad[zy, zx]
                    den += wgt
            ref[y, x] = num / den
    errs = [np.max(np.abs(oracle.nlm_direct(img, r, 3, h, rho, n) - ref)) for n in (15, 60, 240)]
    assert errs[0] > errs[1] > errs[2]
    assert 2.5 < errs[0] / errs[1] < 6.0 and 2.5 < errs[1] / errs[2] < 6.0
    assert errs[2] < 0.5
    # the moving-sum algorithm agrees with the definition for p = 3, rho > 0
    assert np.max(np.abs(oracle.nlm_shiftable(img, r, 3, h, rho, 15) - oracle.nlm_direct(img, r, 3, h, rho, 15))) <= 1e-9


# ------------------------------------------ f3: the polynomial range kernel p_N

def test_poly_kernel_converges_to_gaussian_eq5():
    """Eq.(5): p_N(t/sqrt N) -> exp(-t^2/T^2); with
    T = sqrt(2) sigma_r (reading R17) the oracle's phi_p tends to
    exp(-t^2/(2 sigma_r^2)), the sup error over [-255, 255] falling like 1/N
    (log(1 - x) = -x - x^2/2 - ...: N sup|phi_p - g| -> max_x x^2 e^-x/2 at
    x = t^2/(2 sigma^2) = 2, i.e. 2 e^-2 = 0.2707)."""
    sigma = 30.0
    ts = np.linspace(-255, 255, 2041)
    g = np.exp(-ts ** 2 / (2 * sigma ** 2))
    errs = []
    for N in (64, 256, 1024, 4096):
        phi = np.array([oracle.range_kernel_poly(t, sigma, N) for t in ts])
        errs.append(np.max(np.abs(phi - g)))
    for a, b in zip(errs, errs[1:]):
        assert 3.5 < a / b < 4.5                         # ~1/N
    assert abs(4096 * errs[-1] - 2 * math.exp(-2)) < 0.01


def test_poly_nmin_is_the_validity_threshold():
    """phi_p >= 0 and unimodal on [-255, 255] at N = N0 = ceil(255^2/(2 sigma^2)),
    not at N0 - 1 (R17): the base 1 - t^2/(2 N sigma^2) turns negative inside."""
    for sigma in (15.0, 20.0, 30.0, 40.0):
        n0 = oracle.nmin_poly(sigma)
        assert n0 == math.ceil(255 ** 2 / (2 * sigma ** 2) - 1e-12)
        ts = np.arange(0, 256)
        phi = np.array([oracle.range_kernel_poly(t, sigma, n0) for t in ts])
        assert phi.min() >= 0 and np.all(np.diff(phi) <= 1e-15)
        # at N0 - 1 the base (whose N-th power phi_p is) turns negative inside
        # [-255, 255] (phi_p itself underflows there, so the base is the test)
        assert 1 - 255 ** 2 / (2 * n0 * sigma ** 2) >= 0 > 1 - 255 ** 2 / (2 * (n0 - 1) * sigma ** 2)
        assert oracle.range_kernel_poly(255.0, sigma, n0) == pytest.approx(
            (1 - 255 ** 2 / (2 * n0 * sigma ** 2)) ** n0, rel=1e-12, abs=1e-300)
    assert [oracle.nmin_poly(s) for s in (40.0, 30.0, 20.0, 15.0)] == [21, 37, 82, 145]


@pytest.mark.parametrize("N,sigma", [(1, 200.0), (6, 80.0), (21, 40.0), (37, 30.0)])
def test_poly_expansion_identity(N, sigma):
    """Eq.(1) for phi_p in the normalised variable u = (f-128)/128: the
    coefficients d_i(v) reproduce (1 - a (u - v)^2)^N, a = 128^2/(2 N sigma^2),
    at random (u, v) — the binomial theorem twice (pins the signs, the powers
    of v and the C(N,j) C(2j,i) weights)."""
    rng = np.random.default_rng(N)
    a = 128.0 ** 2 / (2 * N * sigma ** 2)
    for _ in range(20):
        u, v = rng.uniform(-1, 1, 2)
        d = oracle.poly_coeffs(N, sigma, v)
        lhs = sum(d[i] * u ** i for i in range(2 * N + 1))
        rhs = (1 - a * (u - v) ** 2) ** N
        assert lhs == pytest.approx(rhs, rel=1e-9, abs=1e-9 * max(1.0, np.abs(d).max()))


def test_poly_algorithm2_equals_bruteforce_and_where_fp64_breaks():
    """Algorithm 2 with the polynomial kernel's monomial basis (O2) equals the
    brute-force Eq.(3) with phi_p (O1) while the basis is well conditioned —
    and, pinned here as a demonstration, breaks down in fp64 at N ~ 80: the
    alternating terms d_i Sum(u^i) grow like (1 + 4a)^N (f3)."""
    img = synth.gen_image(40, 45, 3, 10.0)
    for sigma, N, tol in ((80.0, 6, 1e-9), (40.0, 21, 1e-8), (30.0, 37, 1e-5)):
        o1 = oracle.bilateral_direct(img, 3, 0, sigma, N, range_kind=3)
        o2 = oracle.bilateral_poly_shiftable(img, 3, sigma, N)
        assert np.max(np.abs(o1 - o2)) <= tol, (sigma, N)
    o1 = oracle.bilateral_direct(img, 3, 0, 20.0, 82, range_kind=3)
    o2 = oracle.bilateral_poly_shiftable(img, 3, 20.0, 82)
    assert np.max(np.abs(o1 - o2)) > 1.0


def test_poly_filter_invariants():
    """Constant image unchanged; a 0|255 step preserved (phi_p(255) = 0 at N0
    up to (1 - 255^2/(2 N0 sigma^2))^N0 ~ 0); sigma_r -> infinity with N = 1
    gives the box mean (phi_p -> 1)."""
    c = np.full((20, 23), 91, np.uint8)
    assert np.max(np.abs(oracle.bilateral_direct(c, 4, 0, 30.0, 37, range_kind=3) - 91)) < 1e-12
    step = np.zeros((16, 16), np.uint8)
    step[:, 8:] = 255
    out = oracle.bilateral_direct(step, 3, 0, 30.0, 37, range_kind=3)
    assert np.max(np.abs(out - step)) < 1e-6
    img = synth.gen_image(21, 26, 5, 10.0)
    box = ndimage.uniform_filter(img.astype(np.float64), size=7, mode="mirror")
    assert np.max(np.abs(oracle.bilateral_direct(img, 3, 0, 1e7, 1, range_kind=3) - box)) < 1e-6


# ------------------------- f2: Gaussian-fitted separable spatial kernel (Eq.(7))

def test_spatial_sigma_kernel_converges_to_gaussian_eq7():
    """Eq.(7) (exponent pi^2 by reading R10): q_M(x/sqrt M)
    -> exp(-pi^2 x^2/(8 T^2)) per axis; with T = pi sigma_s/2 (reading R18)
    the oracle's w1(u) = cos(u/(sigma_s sqrt M))^M tends to exp(-u^2/(2 sigma_s^2))
    with a sup error ~1/M (the raised cosine's log-cos series)."""
    r, ss = 12, 3.0
    errs = []
    for M in (16, 64, 256):
        b = oracle.spatial_beta(ss, M)
        w = np.array([oracle.spatial_weight_beta(u, r, 100 + min(M, 16), b) if M <= 16 else
                      math.cos(b * u) ** M for u in range(-r, r + 1)])
        g = np.exp(-np.arange(-r, r + 1) ** 2 / (2 * ss * ss))
        errs.append(np.max(np.abs(w - g)))
    assert errs[0] > errs[1] > errs[2] and 3.0 < errs[0] / errs[1] < 5.0 and 3.0 < errs[1] / errs[2] < 5.0
    # the oracle's weight is the written-out formula for M <= 16
    b = oracle.spatial_beta(ss, 7)
    for u in range(-r, r + 1):
        assert oracle.spatial_weight_beta(u, r, 107, b) == pytest.approx(math.cos(u / (ss * math.sqrt(7))) ** 7,
                                                                          rel=1e-13, abs=1e-300)
    assert oracle.spatial_weight_beta(r + 1, r, 107, b) == 0.0


def test_spatial_sigma_mmin():
    """M0 = ceil((2r/(pi sigma_s))^2): cos(u/(sigma_s sqrt M)) >= 0 on |u| <= r at M0, not at M0 - 1."""
    for r, ss in ((4, 1.0), (10, 3.0), (16, 2.0), (8, 8.0)):
        m0 = oracle.spatial_mmin(r, ss)
        assert r / (ss * math.sqrt(m0)) <= math.pi / 2 + 1e-12
        if m0 > 1:
            assert r / (ss * math.sqrt(m0 - 1)) > math.pi / 2


@pytest.mark.parametrize("r,ss", [(4, 2.0), (6, 2.5), (9, 4.0)])
def test_spatial_sigma_algorithm2_equals_bruteforce_and_algorithm1(r, ss):
    """Algorithm 2 with the sigma_s-fitted spatial expansion (frequencies
    s_m/(sigma_s sqrt M), weights C(M,m)/2^M) equals Eq.(3) brute force with
    w1 = cos(u/(sigma_s sqrt M))^M; with the order-0 range kernel it is the
    normalised correlation with that kernel (scipy.ndimage.correlate)."""
    M = max(oracle.spatial_mmin(r, ss), 2)
    b = oracle.spatial_beta(ss, M)
    img = synth.gen_image(26, 31, 70 + r, 10.0)
    o1 = oracle.bilateral_direct(img, r, 100 + M, 30.0, 30, beta=b)
    o2 = oracle.bilateral_shiftable(img, r, 100 + M, 30.0, 30, beta=b)
    assert np.max(np.abs(o1 - o2)) <= 1e-9
    w1 = np.array([math.cos(u * b) ** M for u in range(-r, r + 1)])
    k2 = np.outer(w1, w1)
    ref = ndimage.correlate(img.astype(np.float64), k2 / k2.sum(), mode="mirror")
    assert np.max(np.abs(oracle.bilateral_shiftable(img, r, 100 + M, 30.0, 0, beta=b) - ref)) <= 1e-9
