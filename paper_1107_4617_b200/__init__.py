"""B200-native constant-time bilateral filtering with shiftable kernels.

Thin Python binding over the C-ABI library `libsf.so` (include/sf.h).  This
module only marshals arguments (device pointers, sizes, the current CUDA
stream); every step of the filter runs in the CUDA kernels of `csrc/`.  There
is no CPU fallback: if the library is missing or no CUDA device is present the
calls raise.

Names follow the C-ABI: sf_filter, sf_filter_rows, sf_accumulate,
sf_finalize, sf_filter_host, sf_pair_count, sf_nmin, sf_status_string.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["sf_filter", "sf_filter_rows", "sf_accumulate", "sf_finalize", "sf_filter_host",
           "sf_filter_truncated", "sf_truncation_n0", "sf_spatial_filter", "sf_nlm", "sf_nlm_pair_count",
           "sf_filter_rows_host", "sf_filter_rows_host_async", "sf_host_sync", "sf_release_scratch",
           "sf_filter_poly", "sf_nmin_poly", "sf_filter_spatial_sigma", "sf_spatial_filter_sigma",
           "sf_spatial_mmin", "sf_pair_count", "sf_nmin", "sf_status_string", "sf_last_launch_count",
           "SF_SPATIAL_BOX", "SF_SPATIAL_RAISED_COS", "SF_SPATIAL_QM", "SF_CENTER", "SFError", "lib_path", "load"]

SF_SPATIAL_BOX = 0
SF_SPATIAL_RAISED_COS = 1
SF_CENTER = 128.0


def SF_SPATIAL_QM(M: int) -> int:
    """Spatial kind of the separable q_M kernel, M = 1..8 (include/sf.h)."""
    return 100 + int(M)

_HERE = os.path.dirname(os.path.abspath(__file__))
# SF_LIB_OVERRIDE: another build of the same library (tools/ab_build.sh: A/B
# timing of two builds on one box); the default is the in-tree libsf.so
_LIB_PATH = os.environ.get("SF_LIB_OVERRIDE") or os.path.join(_HERE, "libsf.so")
_lib = None

# exported symbols declared in include/sf.h (checked by tests/test_abi.py)
EXPORTS = ["sf_filter", "sf_filter_rows", "sf_accumulate", "sf_accumulate_add", "sf_accumulate_scatter",
           "sf_finalize", "sf_filter_host",
           "sf_filter_truncated", "sf_truncation_n0", "sf_spatial_filter", "sf_nlm", "sf_nlm_pair_count",
           "sf_filter_rows_host", "sf_filter_rows_host_async", "sf_host_sync", "sf_release_scratch",
           "sf_filter_poly", "sf_nmin_poly", "sf_filter_spatial_sigma", "sf_spatial_filter_sigma",
           "sf_spatial_mmin", "sf_pair_count", "sf_nmin", "sf_last_launch_count",
           "sf_status_string"]


class SFError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {sf_status_string(code)} (status {code})")


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load libsf.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(_LIB_PATH)
    u8p, fp, vp = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p
    I, D = ctypes.c_int, ctypes.c_double
    lib.sf_filter.argtypes = [u8p, I, I, I, I, D, I, fp, vp]
    lib.sf_filter_rows.argtypes = [u8p, I, I, I, I, I, I, D, I, fp, vp]
    lib.sf_accumulate.argtypes = [u8p, I, I, I, I, D, I, I, I, fp, fp, vp]
    if hasattr(lib, "sf_accumulate_add"):      # (older builds, SF_LIB_OVERRIDE A/B, lack these)
        lib.sf_accumulate_add.argtypes = [u8p, I, I, I, I, D, I, I, I, fp, fp, vp]
        lib.sf_accumulate_scatter.argtypes = [u8p, I, I, I, I, D, I, I, I, I, vp, vp, vp]
    lib.sf_finalize.argtypes = [fp, fp, u8p, I, I, fp, vp]
    lib.sf_filter_truncated.argtypes = [u8p, I, I, I, I, D, I, D, fp, vp]
    lib.sf_truncation_n0.argtypes = [I, D]
    lib.sf_truncation_n0.restype = I
    lib.sf_spatial_filter.argtypes = [u8p, I, I, I, I, fp, vp]
    lib.sf_nlm.argtypes = [u8p, I, I, I, I, D, D, I, fp, vp]
    lib.sf_nlm_pair_count.argtypes = [I, I]
    lib.sf_nlm_pair_count.restype = I
    lib.sf_filter_host.argtypes = [u8p, I, I, I, I, D, I, fp, vp]
    lib.sf_filter_rows_host.argtypes = [u8p, I, I, I, I, I, I, D, I, fp, vp]
    if hasattr(lib, "sf_filter_rows_host_async"):
        lib.sf_filter_rows_host_async.argtypes = [u8p, I, I, I, I, I, I, D, I, fp, vp]
        lib.sf_filter_rows_host_async.restype = I
        lib.sf_host_sync.argtypes = []
        lib.sf_host_sync.restype = I
    for f in ("sf_filter", "sf_filter_rows", "sf_accumulate", "sf_accumulate_add", "sf_accumulate_scatter",
              "sf_finalize", "sf_filter_host",
              "sf_filter_rows_host", "sf_filter_truncated", "sf_spatial_filter", "sf_nlm"):
        if hasattr(lib, f):
            getattr(lib, f).restype = I
    if hasattr(lib, "sf_filter_spatial_sigma"):
        lib.sf_filter_spatial_sigma.argtypes = [u8p, I, I, I, D, I, D, I, fp, vp]
        lib.sf_filter_spatial_sigma.restype = I
        lib.sf_spatial_filter_sigma.argtypes = [u8p, I, I, I, D, I, fp, vp]
        lib.sf_spatial_filter_sigma.restype = I
        lib.sf_spatial_mmin.argtypes = [I, D]
        lib.sf_spatial_mmin.restype = I
    if hasattr(lib, "sf_filter_poly"):
        lib.sf_filter_poly.argtypes = [u8p, I, I, I, D, I, fp, vp]
        lib.sf_filter_poly.restype = I
        lib.sf_nmin_poly.argtypes = [D]
        lib.sf_nmin_poly.restype = I
    if hasattr(lib, "sf_release_scratch"):
        lib.sf_release_scratch.argtypes = []
        lib.sf_release_scratch.restype = I
    lib.sf_pair_count.argtypes = [I]
    lib.sf_pair_count.restype = I
    lib.sf_nmin.argtypes = [D]
    lib.sf_nmin.restype = I
    lib.sf_last_launch_count.argtypes = []
    lib.sf_last_launch_count.restype = I
    lib.sf_status_string.argtypes = [I]
    lib.sf_status_string.restype = ctypes.c_char_p
    _lib = lib
    return lib


def sf_status_string(code: int) -> str:
    return load().sf_status_string(int(code)).decode()


def sf_pair_count(N: int) -> int:
    return load().sf_pair_count(int(N))


def sf_nmin(sigma_r: float) -> int:
    return load().sf_nmin(float(sigma_r))


def sf_last_launch_count() -> int:
    return load().sf_last_launch_count()


def _check(rc: int, where: str):
    if rc != 0:
        raise SFError(rc, where)


def _stream(stream, device=None):
    """The CUDA stream handle: the given torch stream, else the current stream
    of `device` (the input tensor's device, not the process's current one)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_u8(t, shape=None):
    """A contiguous CUDA uint8 tensor (of the given shape, if any)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.uint8 and t.is_contiguous()):
        raise TypeError("expected a contiguous CUDA uint8 tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected a uint8 tensor of shape {tuple(shape)}, got {tuple(t.shape)}")
    if shape is None and t.dim() != 2:
        raise ValueError(f"expected a 2-D H x W image, got shape {tuple(t.shape)}")
    return t


def _dev_f32(t, shape, device, name="out"):
    """A caller-supplied output / partial buffer: contiguous CUDA float32 of
    exactly `shape` on `device` (the library writes through the raw pointer,
    so anything else would be overrun or misread)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous CUDA float32 tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.device != device:
        raise ValueError(f"{name}: on {t.device}, the image is on {device}")
    return t


def _new_f32(shape, device):
    import torch
    return torch.empty(tuple(shape), dtype=torch.float32, device=device)


def _host_f32(a, shape, name="out"):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous and a.flags.writeable):
        raise TypeError(f"{name}: expected a writeable C-contiguous float32 numpy array")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(a.shape)}")
    return a


def _host_u8(a, shape=None):
    if not (isinstance(a, np.ndarray) and a.dtype == np.uint8 and a.flags.c_contiguous):
        raise TypeError("expected a C-contiguous uint8 numpy array")
    if shape is not None and tuple(a.shape) != tuple(shape):
        raise ValueError(f"expected a uint8 array of shape {tuple(shape)}, got {tuple(a.shape)}")
    return a


def _band_rows(H: int, row_begin: int, row_end: int, radius: int):
    """Input rows a row band needs: [max(0, b0 - r), min(H, b1 + r))."""
    return max(0, row_begin - radius), min(H, row_end + radius)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def sf_filter(img, radius: int, spatial_kind: int, sigma_r: float, N: int, out=None, stream=None):
    """Filter a whole H x W uint8 CUDA tensor; returns (or fills) an H x W float32 tensor."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_filter(_ptr(img), H, W, radius, spatial_kind, sigma_r, N, _ptr(out),
                                _stream(stream, img.device)), "sf_filter")
    return out


def sf_spatial_filter(img, radius: int, spatial_kind: int, out=None, stream=None):
    """Algorithm 1 (constant-time spatial filtering): normalised spatial-kernel
    average of an H x W uint8 CUDA tensor; returns (or fills) H x W float32."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_spatial_filter(_ptr(img), H, W, radius, spatial_kind, _ptr(out),
                                        _stream(stream, img.device)), "sf_spatial_filter")
    return out


def sf_nlm(img, radius: int, p: int, h: float, rho: float, n: int, out=None, stream=None):
    """Shiftable non-local means with a p-pixel patch; H x W float32."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_nlm(_ptr(img), H, W, radius, p, h, rho, n, _ptr(out), _stream(stream, img.device)),
               "sf_nlm")
    return out


def sf_nlm_pair_count(p: int, n: int) -> int:
    return load().sf_nlm_pair_count(int(p), int(n))


def sf_truncation_n0(N: int, eps: float) -> int:
    return load().sf_truncation_n0(int(N), float(eps))


def sf_filter_truncated(img, radius: int, spatial_kind: int, sigma_r: float, N: int, eps: float,
                        out=None, stream=None):
    """Filter with the expansion truncated to terms whose weight is >= eps x the
    largest; returns (or fills) an H x W float32 tensor."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_filter_truncated(_ptr(img), H, W, radius, spatial_kind, sigma_r, N, eps, _ptr(out),
                                          _stream(stream, img.device)), "sf_filter_truncated")
    return out


def sf_filter_rows(img_band, H: int, W: int, row_begin: int, row_end: int, radius: int,
                   spatial_kind: int, sigma_r: float, N: int, out_band=None, stream=None):
    """Output rows [row_begin,row_end); img_band = input rows
    [max(0,row_begin-radius), min(H,row_end+radius)) of the full image."""
    import torch
    if not (0 <= row_begin < row_end <= H):
        raise ValueError(f"bad row range [{row_begin}, {row_end}) for H = {H}")
    in0, in1 = _band_rows(H, row_begin, row_end, radius)
    img_band = _dev_u8(img_band, (in1 - in0, W))
    shape = (row_end - row_begin, W)
    out_band = _new_f32(shape, img_band.device) if out_band is None else \
        _dev_f32(out_band, shape, img_band.device, "out_band")
    with torch.cuda.device(img_band.device):
        _check(load().sf_filter_rows(_ptr(img_band), H, W, row_begin, row_end, radius, spatial_kind,
                                     sigma_r, N, _ptr(out_band), _stream(stream, img_band.device)),
               "sf_filter_rows")
    return out_band


def sf_accumulate(img, radius: int, spatial_kind: int, sigma_r: float, N: int,
                  pair_begin: int, pair_end: int, num=None, den=None, stream=None):
    """Partial (num, den) over conjugate pairs [pair_begin, pair_end) (centred at SF_CENTER)."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    num = _new_f32((H, W), img.device) if num is None else _dev_f32(num, (H, W), img.device, "num")
    den = _new_f32((H, W), img.device) if den is None else _dev_f32(den, (H, W), img.device, "den")
    with torch.cuda.device(img.device):
        _check(load().sf_accumulate(_ptr(img), H, W, radius, spatial_kind, sigma_r, N, pair_begin,
                                    pair_end, _ptr(num), _ptr(den), _stream(stream, img.device)), "sf_accumulate")
    return num, den


def _ptr_any(x, shape=None, name="buffer"):
    """A CUDA float32 tensor's data pointer (checked: contiguous, `shape`), or
    a raw device address (int) — e.g. a peer GPU's buffer mapped by CUDA IPC,
    which the caller vouches for."""
    import torch
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous CUDA float32 tensor or a device address")
    if shape is not None and tuple(x.shape) != tuple(shape) and x.numel() != int(np.prod(shape)):
        raise ValueError(f"{name}: expected {tuple(shape)}, got {tuple(x.shape)}")
    return _ptr(x)


def sf_accumulate_add(img, radius: int, spatial_kind: int, sigma_r: float, N: int,
                      pair_begin: int, pair_end: int, num, den, stream=None):
    """Add the partial (num, den) over pairs [pair_begin, pair_end) into num/den
    (CUDA tensors — possibly views of a peer GPU's buffer mapped by CUDA IPC —
    or raw device addresses)."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    pn, pd = _ptr_any(num, (H, W), "num"), _ptr_any(den, (H, W), "den")
    with torch.cuda.device(img.device):
        _check(load().sf_accumulate_add(_ptr(img), H, W, radius, spatial_kind, sigma_r, N, pair_begin,
                                        pair_end, pn, pd, _stream(stream, img.device)),
               "sf_accumulate_add")


def sf_accumulate_scatter(img, radius: int, spatial_kind: int, sigma_r: float, N: int,
                          pair_begin: int, pair_end: int, band_num, band_den, stream=None):
    """Add the partials of pairs [pair_begin, pair_end) of output band o =
    rows [o H/n, (o+1) H/n) into band_num[o] / band_den[o] (tensors or device
    addresses, typically other ranks' buffers mapped by CUDA IPC)."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    n = len(band_num)
    if n != len(band_den):
        raise ValueError("band_num and band_den differ in length")
    if not 1 <= n <= min(8, H):
        raise ValueError(f"band count {n} outside 1..min(8, H)")
    rows = [(o + 1) * H // n - o * H // n for o in range(n)]
    nums = (ctypes.c_void_p * n)(*[_ptr_any(x, (rows[o], W), f"band_num[{o}]").value
                                   for o, x in enumerate(band_num)])
    dens = (ctypes.c_void_p * n)(*[_ptr_any(x, (rows[o], W), f"band_den[{o}]").value
                                   for o, x in enumerate(band_den)])
    with torch.cuda.device(img.device):
        _check(load().sf_accumulate_scatter(_ptr(img), H, W, radius, spatial_kind, sigma_r, N, pair_begin,
                                            pair_end, n, ctypes.cast(nums, ctypes.c_void_p),
                                            ctypes.cast(dens, ctypes.c_void_p), _stream(stream, img.device)),
               "sf_accumulate_scatter")


def sf_finalize(num, den, img, out=None, stream=None):
    """out = SF_CENTER + num/den (the last line of Algorithm 2)."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    num = _dev_f32(num, (H, W), img.device, "num")
    den = _dev_f32(den, (H, W), img.device, "den")
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_finalize(_ptr(num), _ptr(den), _ptr(img), H, W, _ptr(out), _stream(stream, img.device)),
               "sf_finalize")
    return out


def sf_release_scratch():
    """Return the unused memory of the current device's library scratch pool
    (include/sf.h, Ownership)."""
    _check(load().sf_release_scratch(), "sf_release_scratch")


def sf_filter_host(img: np.ndarray, radius: int, spatial_kind: int, sigma_r: float, N: int,
                   out: np.ndarray | None = None, stream=None) -> np.ndarray:
    """End-to-end: host uint8 array in, host float32 array out (copies inside the call)."""
    img = _host_u8(img)
    if img.ndim != 2:
        raise ValueError(f"expected a 2-D H x W image, got shape {img.shape}")
    H, W = img.shape
    out = np.empty((H, W), dtype=np.float32) if out is None else _host_f32(out, (H, W))
    st = ctypes.c_void_p(0) if stream is None else _stream(stream)
    _check(load().sf_filter_host(ctypes.c_void_p(img.ctypes.data), H, W, radius, spatial_kind,
                                 sigma_r, N, ctypes.c_void_p(out.ctypes.data), st), "sf_filter_host")
    return out


def sf_filter_rows_host(img_band: np.ndarray, H: int, W: int, row_begin: int, row_end: int,
                        radius: int, spatial_kind: int, sigma_r: float, N: int,
                        out_band: np.ndarray | None = None, stream=None) -> np.ndarray:
    """Row band end to end: host uint8 band in, host float32 band out."""
    if not (0 <= row_begin < row_end <= H):
        raise ValueError(f"bad row range [{row_begin}, {row_end}) for H = {H}")
    in0, in1 = _band_rows(H, row_begin, row_end, radius)
    img_band = _host_u8(img_band, (in1 - in0, W))
    shape = (row_end - row_begin, W)
    out_band = np.empty(shape, dtype=np.float32) if out_band is None else _host_f32(out_band, shape, "out_band")
    st = ctypes.c_void_p(0) if stream is None else _stream(stream)
    _check(load().sf_filter_rows_host(ctypes.c_void_p(img_band.ctypes.data), H, W, row_begin, row_end,
                                      radius, spatial_kind, sigma_r, N,
                                      ctypes.c_void_p(out_band.ctypes.data), st), "sf_filter_rows_host")
    return out_band


def sf_filter_rows_host_async(img_band: np.ndarray, H: int, W: int, row_begin: int, row_end: int,
                              radius: int, spatial_kind: int, sigma_r: float, N: int, out_band: np.ndarray,
                              stream=None) -> None:
    """Enqueue a row band end to end (pinned host band in, pinned host float32
    band out) without waiting; successive calls pipeline copies with kernels.
    The buffers must stay alive and untouched until sf_host_sync()."""
    if not (0 <= row_begin < row_end <= H):
        raise ValueError(f"bad row range [{row_begin}, {row_end}) for H = {H}")
    in0, in1 = _band_rows(H, row_begin, row_end, radius)
    img_band = _host_u8(img_band, (in1 - in0, W))
    out_band = _host_f32(out_band, (row_end - row_begin, W), "out_band")
    st = ctypes.c_void_p(0) if stream is None else _stream(stream)
    _check(load().sf_filter_rows_host_async(ctypes.c_void_p(img_band.ctypes.data), H, W, row_begin, row_end,
                                            radius, spatial_kind, sigma_r, N,
                                            ctypes.c_void_p(out_band.ctypes.data), st), "sf_filter_rows_host_async")


def sf_host_sync() -> None:
    """Wait for the copies of every sf_filter_rows_host_async call on the current device."""
    _check(load().sf_host_sync(), "sf_host_sync")


def sf_nmin_poly(sigma_r: float) -> int:
    return load().sf_nmin_poly(float(sigma_r))


def sf_filter_poly(img, radius: int, sigma_r: float, N: int, out=None, stream=None):
    """Bilateral filter with the polynomial range kernel (1 - t^2/(2 N sigma_r^2))^N
    (Eq.(5); include/sf.h), box spatial kernel; H x W float32."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_filter_poly(_ptr(img), H, W, radius, sigma_r, N, _ptr(out), _stream(stream, img.device)),
               "sf_filter_poly")
    return out


def sf_spatial_mmin(radius: int, sigma_s: float) -> int:
    return load().sf_spatial_mmin(int(radius), float(sigma_s))


def sf_filter_spatial_sigma(img, radius: int, sigma_s: float, M: int, sigma_r: float, N: int, out=None,
                            stream=None):
    """Bilateral filter with the Gaussian-fitted separable spatial kernel
    cos(u/(sigma_s sqrt M))^M (Eq.(7); include/sf.h); H x W float32."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_filter_spatial_sigma(_ptr(img), H, W, radius, sigma_s, M, sigma_r, N, _ptr(out),
                                              _stream(stream, img.device)), "sf_filter_spatial_sigma")
    return out


def sf_spatial_filter_sigma(img, radius: int, sigma_s: float, M: int, out=None, stream=None):
    """Algorithm 1 with the Gaussian-fitted separable spatial kernel; H x W float32."""
    import torch
    img = _dev_u8(img)
    H, W = img.shape
    out = _new_f32((H, W), img.device) if out is None else _dev_f32(out, (H, W), img.device)
    with torch.cuda.device(img.device):
        _check(load().sf_spatial_filter_sigma(_ptr(img), H, W, radius, sigma_s, M, _ptr(out),
                                              _stream(stream, img.device)), "sf_spatial_filter_sigma")
    return out
