"""fp64 CPU oracle — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and bench.py's `cpu_baseline` /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (`paper_1107_4617_b200/`) and neither imports the other; both read
their inputs from `synth/`.

The arithmetic lives in `sf_oracle.c` (see its header for the paper passages
each function follows).  Pins that tie it to the paper and to mathematics (not
to itself) are in tests/test_oracle_pins.py.  Parity of absolute outputs on
the synthetic configs beyond those pins is "parity unpinned" (the paper prints
no worked example).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile sf_oracle.c with gcc (IEEE fp64, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_expansion.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _dp]
        lib.oracle_range_kernel.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int]
        lib.oracle_range_kernel.restype = ctypes.c_double
        lib.oracle_gaussian_kernel.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.oracle_gaussian_kernel.restype = ctypes.c_double
        lib.oracle_nmin.argtypes = [ctypes.c_double]
        lib.oracle_spatial_weight.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.oracle_spatial_weight.restype = ctypes.c_double
        lib.oracle_moving_sum.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        lib.oracle_range_kernel_truncated.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                                      ctypes.c_int]
        lib.oracle_range_kernel_truncated.restype = ctypes.c_double
        lib.oracle_truncation_n0.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.oracle_bilateral_direct_ex2.argtypes = [
            _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, ctypes.c_int64, _dp, _dp, _dp, ctypes.c_int]
        lib.oracle_bilateral_direct_ex.argtypes = [
            _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, _i64p, ctypes.c_int64, _dp, _dp, _dp, ctypes.c_int]
        lib.oracle_bilateral_shiftable.argtypes = [
            _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _dp, _dp, _dp, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        lib.oracle_nlm_direct.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_int, _dp, ctypes.c_int]
        lib.oracle_nlm_shiftable.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_int, _dp]
        lib.oracle_bilateral_direct_ex3.argtypes = [
            _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, ctypes.c_int64, _dp, _dp, _dp, ctypes.c_int,
            ctypes.c_double]
        lib.oracle_bilateral_shiftable_ex.argtypes = [
            _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _dp, _dp, _dp, ctypes.c_int, ctypes.c_double]
        lib.oracle_spatial_weight_beta.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        lib.oracle_spatial_weight_beta.restype = ctypes.c_double
        lib.oracle_spatial_mmin.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.oracle_range_kernel_poly.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int]
        lib.oracle_range_kernel_poly.restype = ctypes.c_double
        lib.oracle_nmin_poly.argtypes = [ctypes.c_double]
        lib.oracle_poly_coeffs.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp]
        lib.oracle_bilateral_poly_shiftable.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                        ctypes.c_double, ctypes.c_int, _dp]
        _lib = lib
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _check(rc):
    if rc != 0:
        raise ValueError(f"oracle error {rc}")


def max_threads() -> int:
    return _load().oracle_max_threads()


def expansion(N: int, sigma_r: float):
    """(omega_n, c_n), n = 0..N — Eq.(1) coefficients of cos(t/(σ_r√N))^N."""
    om = np.zeros(N + 1)
    c = np.zeros(N + 1)
    _check(_load().oracle_expansion(N, sigma_r, _ptr(om, _dp), _ptr(c, _dp)))
    return om, c


def range_kernel(t: float, sigma_r: float, N: int) -> float:
    return _load().oracle_range_kernel(float(t), float(sigma_r), int(N))


def gaussian_kernel(t: float, sigma_r: float) -> float:
    return _load().oracle_gaussian_kernel(float(t), float(sigma_r))


def nmin(sigma_r: float) -> int:
    return _load().oracle_nmin(float(sigma_r))


def spatial_weight(u: int, radius: int, kind: int) -> float:
    return _load().oracle_spatial_weight(int(u), int(radius), int(kind))


def moving_sum(F: np.ndarray, radius: int) -> np.ndarray:
    F = np.ascontiguousarray(F, dtype=np.float64)
    out = np.empty_like(F)
    _check(_load().oracle_moving_sum(_ptr(F, _dp), F.shape[0], F.shape[1], radius, _ptr(out, _dp)))
    return out


def range_kernel_truncated(t: float, sigma_r: float, N: int, n0: int) -> float:
    """Eq.(1) expansion keeping terms n0..N-n0."""
    return _load().oracle_range_kernel_truncated(float(t), float(sigma_r), int(N), int(n0))


def truncation_n0(N: int, eps: float) -> int:
    """Terms dropped at each end: smallest n0 with c_n0 >= eps * max c_n."""
    return _load().oracle_truncation_n0(int(N), float(eps))


def bilateral_direct(img: np.ndarray, radius: int, kind: int, sigma_r: float, N: int,
                     idx: np.ndarray | None = None, range_kind: int = 0,
                     nthreads: int = 0, return_parts: bool = False, n0: int = 0, beta: float = 0.0):
    """Eq.(3) brute force (O1).  idx: flat pixel indices (None = all pixels).
    range_kind 0: raised cosine; 1: Gaussian; 2: raised cosine truncated to
    terms n0..N-n0; 3: the polynomial kernel (f3).  beta > 0: spatial q_M
    kinds with w1(u) = cos(beta u)^M (f2, spatial_weight_beta)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    if idx is not None:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        n = idx.size
    else:
        n = H * W
    out = np.empty(n)
    num = np.empty(n) if return_parts else None
    den = np.empty(n) if return_parts else None
    _check(_load().oracle_bilateral_direct_ex3(
        _ptr(img, _u8p), H, W, radius, kind, sigma_r, N, range_kind, n0,
        _ptr(idx, _i64p), n, _ptr(out, _dp), _ptr(num, _dp), _ptr(den, _dp), nthreads, float(beta)))
    if idx is None:
        out = out.reshape(H, W)
        if return_parts:
            num, den = num.reshape(H, W), den.reshape(H, W)
    return (out, num, den) if return_parts else out


def bilateral_shiftable(img: np.ndarray, radius: int, kind: int, sigma_r: float, N: int,
                        n_begin: int = 0, n_end: int | None = None,
                        row_begin: int = 0, row_end: int | None = None,
                        nthreads: int = 0, return_parts: bool = False, beta: float = 0.0):
    """Algorithm 2 (O2) over range terms [n_begin, n_end) and rows [row_begin, row_end);
    beta > 0: the spatial q_M frequency (f2, spatial_weight_beta)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    n_end = N + 1 if n_end is None else n_end
    row_end = H if row_end is None else row_end
    rows = row_end - row_begin
    out = np.empty((rows, W))
    num = np.empty((rows, W))
    den = np.empty((rows, W))
    _check(_load().oracle_bilateral_shiftable_ex(
        _ptr(img, _u8p), H, W, radius, kind, sigma_r, N, n_begin, n_end, row_begin, row_end,
        _ptr(num, _dp), _ptr(den, _dp), _ptr(out, _dp), nthreads, float(beta)))
    return (out, num, den) if return_parts else out


def nlm_direct(img: np.ndarray, radius: int, p: int, h: float, rho: float, n: int,
               nthreads: int = 0) -> np.ndarray:
    """Shiftable non-local means by brute force (the definition)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W))
    _check(_load().oracle_nlm_direct(_ptr(img, _u8p), H, W, radius, p, h, rho, n, _ptr(out, _dp), nthreads))
    return out


def nlm_shiftable(img: np.ndarray, radius: int, p: int, h: float, rho: float, n: int) -> np.ndarray:
    """Shiftable non-local means by the paper's moving-sum algorithm."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W))
    _check(_load().oracle_nlm_shiftable(_ptr(img, _u8p), H, W, radius, p, h, rho, n, _ptr(out, _dp)))
    return out


# ------------------------------------------------ f3: polynomial range kernel

def range_kernel_poly(t: float, sigma_r: float, N: int) -> float:
    """phi_p(t) = (1 - t^2/(2 N sigma_r^2))^N: p_N(t/sqrt N) of PAPER.md:202
    in the Eq.(5) scaling with T = sqrt(2) sigma_r (reading R17)."""
    return _load().oracle_range_kernel_poly(float(t), float(sigma_r), int(N))


def nmin_poly(sigma_r: float) -> int:
    """Smallest N with phi_p >= 0 on [-255, 255]: ceil(255^2 / (2 sigma_r^2))."""
    return _load().oracle_nmin_poly(float(sigma_r))


def poly_coeffs(N: int, sigma_r: float, v: float) -> np.ndarray:
    """d_i(v), i = 0..2N: phi_p(128 (u - v)) = sum_i d_i(v) u^i (Eq.(1) for phi_p)."""
    d = np.empty(2 * N + 1)
    _check(_load().oracle_poly_coeffs(int(N), float(sigma_r), float(v), _ptr(d, _dp)))
    return d


def bilateral_poly_shiftable(img: np.ndarray, radius: int, sigma_r: float, N: int) -> np.ndarray:
    """Algorithm 2 with phi_p, monomial basis, box spatial kernel (fp64)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    out = np.empty((H, W))
    _check(_load().oracle_bilateral_poly_shiftable(_ptr(img, _u8p), H, W, int(radius), float(sigma_r), int(N),
                                                   _ptr(out, _dp)))
    return out


# --------------------------------- f2: Gaussian-fitted separable spatial kernel

def spatial_beta(sigma_s: float, M: int) -> float:
    """beta = 1/(sigma_s sqrt M): q_M(u/sqrt M) with T = pi sigma_s/2, whose
    Eq.(7) limit is exp(-u^2/(2 sigma_s^2)) per axis (reading R18)."""
    return 1.0 / (float(sigma_s) * float(M) ** 0.5)


def spatial_weight_beta(u: int, radius: int, kind: int, beta: float) -> float:
    return _load().oracle_spatial_weight_beta(int(u), int(radius), int(kind), float(beta))


def spatial_mmin(radius: int, sigma_s: float) -> int:
    """Smallest M with cos(u/(sigma_s sqrt M)) >= 0 on |u| <= r."""
    return _load().oracle_spatial_mmin(int(radius), float(sigma_s))
