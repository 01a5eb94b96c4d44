"""C-ABI host-side checks that need no GPU: the library loads, exports every
symbol include/sf.h declares, and rejects bad arguments synchronously with the
documented status codes (validation runs before any CUDA call, so nothing is
enqueued — these calls never touch a device)."""
import ctypes
import os
import re

import pytest

import paper_1107_4617_b200 as sf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sf.h")

OK, NULL, SHAPE, RADIUS, SIGMA, ORDER, KIND, RANGE, ALIAS, CUDA = range(10)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(sf.lib_path())
    names = declared_functions()
    assert len(names) >= 9
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(sf.EXPORTS) == names


def test_sm100a_cubin_embedded():
    """The library carries sm_100a SASS (built with -gencode arch=compute_100a,code=sm_100a)."""
    import subprocess
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sf.lib_path()],
                         capture_output=True, text=True)
    assert res.returncode == 0 and "sm_100a" in res.stdout


def test_pair_count_and_nmin():
    assert [sf.sf_pair_count(n) for n in (1, 2, 17, 30, 66, 118, 264)] == [1, 2, 9, 16, 34, 60, 133]
    assert [sf.sf_nmin(s) for s in (30.0, 20.0, 40.0, 10.0, 15.0)] == [30, 66, 17, 264, 118]
    assert sf.sf_nmin(-1.0) == -1
    assert sf.sf_status_string(ALIAS) == "output overlaps input"


FAKE_IN = 0x10000000
FAKE_OUT = 0x20000000


def call_filter(img=FAKE_IN, H=64, W=64, r=5, kind=0, s=30.0, N=30, out=FAKE_OUT):
    return sf.load().sf_filter(ctypes.c_void_p(img), H, W, r, kind, s, N, ctypes.c_void_p(out), None)


@pytest.mark.parametrize("kw,code", [
    (dict(img=0), NULL), (dict(out=0), NULL),
    (dict(H=0), SHAPE), (dict(W=-3), SHAPE),
    (dict(kind=2), KIND),
    (dict(s=0.0), SIGMA), (dict(s=float("nan")), SIGMA), (dict(s=float("inf")), SIGMA),
    (dict(r=-1), RADIUS), (dict(r=64, H=64), RADIUS), (dict(r=65, H=500, W=500), RADIUS),
    (dict(N=29), ORDER), (dict(N=4000, s=300.0), ORDER),
    (dict(out=FAKE_IN + 100), ALIAS),
])
def test_filter_validation(kw, code):
    assert call_filter(**kw) == code


def test_rows_accumulate_finalize_validation():
    L = sf.load()
    v = ctypes.c_void_p
    # row ranges
    assert L.sf_filter_rows(v(FAKE_IN), 64, 64, 10, 10, 5, 0, 30.0, 30, v(FAKE_OUT), None) == RANGE
    assert L.sf_filter_rows(v(FAKE_IN), 64, 64, -1, 10, 5, 0, 30.0, 30, v(FAKE_OUT), None) == RANGE
    assert L.sf_filter_rows(v(FAKE_IN), 64, 64, 0, 65, 5, 0, 30.0, 30, v(FAKE_OUT), None) == RANGE
    # pair ranges: 0..pair_count(N)
    assert L.sf_accumulate(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 17, v(FAKE_OUT), v(FAKE_OUT + 10 ** 6),
                           None) == RANGE
    assert L.sf_accumulate(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 5, 4, v(FAKE_OUT), v(FAKE_OUT + 10 ** 6),
                           None) == RANGE
    assert L.sf_accumulate(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 16, v(FAKE_OUT), v(FAKE_OUT + 100),
                           None) == ALIAS
    assert L.sf_accumulate(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 16, None, v(FAKE_OUT), None) == NULL
    assert L.sf_finalize(v(FAKE_OUT), v(FAKE_OUT + 10 ** 6), v(FAKE_IN), 64, 64, v(FAKE_OUT + 8), None) == ALIAS
    assert L.sf_finalize(v(FAKE_OUT), v(FAKE_OUT + 10 ** 6), v(FAKE_IN), 0, 64, v(FAKE_OUT + 10 ** 7), None) == SHAPE
    assert L.sf_filter_host(None, 64, 64, 5, 0, 30.0, 30, v(FAKE_OUT), None) == NULL
    assert sf.sf_last_launch_count() == 0


def test_no_device_fails_loudly():
    """Without a CUDA device a valid compute call must fail (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np
    img = np.zeros((16, 16), np.uint8)
    with pytest.raises(sf.SFError) as ei:
        sf.sf_filter_host(img, 2, 0, 30.0, 30)
    assert ei.value.code == CUDA


def test_truncation_n0_exact_binomials():
    """Host planner of sf_filter_truncated: n0 is the first index whose exact
    binomial weight reaches eps x the largest (independent of the oracle)."""
    import math
    from fractions import Fraction
    for N, eps in [(264, 1e-6), (264, 1e-8), (118, 1e-6), (30, 1e-3), (17, 0.0), (66, 0.5)]:
        cmax = Fraction(math.comb(N, N // 2))
        kept = [n for n in range(N + 1) if Fraction(math.comb(N, n)) >= Fraction(eps) * cmax]
        n0 = sf.sf_truncation_n0(N, eps)
        assert kept == list(range(n0, N - n0 + 1)), (N, eps)
    assert sf.sf_truncation_n0(30, -1.0) == -1 and sf.sf_truncation_n0(30, 1.0) == -1


def test_truncated_validation():
    L = sf.load()
    v = ctypes.c_void_p
    assert L.sf_filter_truncated(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 1.5, v(FAKE_OUT), None) == RANGE
    assert L.sf_filter_truncated(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, float("nan"), v(FAKE_OUT), None) == RANGE
    assert L.sf_filter_truncated(v(FAKE_IN), 64, 64, 5, 0, 30.0, 29, 1e-6, v(FAKE_OUT), None) == ORDER
    assert L.sf_filter_truncated(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 1e-6, v(FAKE_IN + 10), None) == ALIAS
    assert L.sf_filter_truncated(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 1e-6, None, None) == NULL


def test_nlm_validation_and_pair_count():
    L = sf.load()
    v = ctypes.c_void_p
    assert sf.sf_nlm_pair_count(2, 8) == 41 and sf.sf_nlm_pair_count(3, 7) == 256
    assert sf.sf_nlm_pair_count(1, 30) == 16 and sf.sf_nlm_pair_count(4, 3) == -1
    ok = dict(H=64, W=64, r=3, p=2, h=60.0, rho=1.0, n=15)

    def call(img=FAKE_IN, out=FAKE_OUT, **kw):
        a = dict(ok, **kw)
        return L.sf_nlm(v(img), a["H"], a["W"], a["r"], a["p"], a["h"], a["rho"], a["n"], v(out), None)
    assert call(p=0) == KIND and call(p=4) == KIND
    assert call(h=0.0) == SIGMA and call(rho=-1.0) == SIGMA and call(h=float("nan")) == SIGMA
    assert call(n=14) == ORDER                       # below sf_nmin(h / sqrt 2) = 15
    assert call(p=3, n=15) == ORDER                  # 2048 pairs > 512
    assert call(r=64) == RADIUS and call(H=0) == SHAPE
    assert call(img=0) == NULL and call(out=FAKE_IN + 1) == ALIAS


def test_accumulate_add_and_scatter_validation():
    """The adding variants validate like sf_accumulate, before any CUDA call;
    sf_accumulate_scatter also checks the band count and every band pointer."""
    L = sf.load()
    v = ctypes.c_void_p
    num, den = FAKE_OUT, FAKE_OUT + (1 << 20)
    assert L.sf_accumulate_add(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 17, v(num), v(den), None) == RANGE
    assert L.sf_accumulate_add(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 3, 2, v(num), v(den), None) == RANGE
    assert L.sf_accumulate_add(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 16, None, v(den), None) == NULL
    assert L.sf_accumulate_add(v(FAKE_IN), 64, 64, 5, 0, 30.0, 29, 0, 15, v(num), v(den), None) == ORDER
    assert L.sf_accumulate_add(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 16, v(FAKE_IN + 8), v(den), None) == ALIAS

    def scatter(n, ptrs_num, ptrs_den, pe=16):
        a = (ctypes.c_void_p * max(1, len(ptrs_num)))(*ptrs_num)
        b = (ctypes.c_void_p * max(1, len(ptrs_den)))(*ptrs_den)
        return L.sf_accumulate_scatter(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, pe, n,
                                       ctypes.cast(a, v), ctypes.cast(b, v), None)
    assert scatter(0, [num], [den]) == RANGE
    assert scatter(9, [num] * 9, [den] * 9) == RANGE           # more than 8 bands
    assert scatter(2, [num, None], [den, den]) == NULL
    assert scatter(2, [num, num], [den, den], pe=17) == RANGE   # pair range beyond floor(N/2)+1
    assert L.sf_accumulate_scatter(v(FAKE_IN), 64, 64, 5, 0, 30.0, 30, 0, 16, 2, None, None, None) == NULL


def test_binding_validates_buffers_before_the_call():
    """The Python binding checks every caller-supplied buffer (dtype,
    contiguity, shape, device) before passing a raw pointer to the C-ABI, so a
    short or mistyped output cannot be overrun (__init__.py)."""
    import numpy as np
    import torch
    img = np.zeros((8, 9), np.uint8)
    with pytest.raises(TypeError):           # a CPU tensor is not a device image
        sf.sf_filter(torch.zeros((8, 9), dtype=torch.uint8), 2, 0, 30.0, 30)
    with pytest.raises(TypeError):           # float16 output
        sf.sf_filter_host(img, 2, 0, 30.0, 30, out=np.zeros((8, 9), np.float16))
    with pytest.raises(ValueError):          # short output
        sf.sf_filter_host(img, 2, 0, 30.0, 30, out=np.zeros((8, 8), np.float32))
    with pytest.raises(TypeError):           # non-contiguous input
        sf.sf_filter_host(np.zeros((8, 18), np.uint8)[:, ::2], 2, 0, 30.0, 30)
    with pytest.raises(ValueError):          # band must hold rows [max(0,b0-r), min(H,b1+r))
        sf.sf_filter_rows_host(np.zeros((5, 9), np.uint8), 20, 9, 4, 8, 2, 0, 30.0, 30)
    with pytest.raises(ValueError):          # out_band rows = row_end - row_begin
        sf.sf_filter_rows_host(np.zeros((8, 9), np.uint8), 20, 9, 4, 8, 2, 0, 30.0, 30,
                               out_band=np.zeros((5, 9), np.float32))
    with pytest.raises(ValueError):          # bad row range
        sf.sf_filter_rows_host(np.zeros((8, 9), np.uint8), 20, 9, 8, 8, 2, 0, 30.0, 30)


def test_release_scratch_without_device():
    """sf_release_scratch reports SF_ERR_CUDA (not a crash) with no device."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    assert sf.load().sf_release_scratch() == CUDA
