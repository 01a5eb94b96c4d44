"""Multi-GPU drivers for the constant-time bilateral filter.

One process per GPU, `torch.distributed` for the plumbing.  Two shardings:

* **Row bands** (cfg 5): rank i owns output rows [b0, b1) = [iH/n, (i+1)H/n)
  and holds input rows [b0 - r, b1 + r) (clipped to the image; reflect-101
  beyond).  The filter of a band is independent of every other band — the
  moving sums only reach r rows — so there is no collective on the data path
  (`sf_filter_rows`, include/sf.h).
* **Term split** (cfg 4): the N+1 range terms of Eq.(1) are
  paired by conjugate symmetry into K = floor(N/2)+1 pairs; rank i accumulates
  the partial numerator / denominator of Algorithm 2 step 3
  over pairs [⌊iK/n⌋, ⌊(i+1)K/n⌋) (`sf_accumulate`), the partial images are
  summed over ranks (one collective: `reduce` of the packed [2, H, W] fp32
  buffer to rank 0 — NCCL over NVLink on the GPU box), and rank 0 forms the
  ratio (`sf_finalize`).
* **One-sided term split** (`FusedTermSplit`): the same split without a
  collective library — a reduce-scatter over peer memory.  Every rank owns one
  output band's partial buffer; the buffers are mapped into every rank once
  (CUDA IPC: views of the peer GPUs' memory over NVLink / NVSwitch), and after
  its filter kernel every rank adds each output row's partial sums straight
  into the owner's buffer (`sf_accumulate_scatter`: a scatter-add pass of fp32
  atomics), so each GPU receives only its band; one barrier, then every rank's
  ratio of its band.

The per-rank compute is passed in (default: the CUDA C-ABI binding) so the
host logic — partitioning, halo placement, packing, the collective, the
finalize — is exercised by world-size-2 gloo tests on CPU (tests/test_dist.py)
with a CPU stand-in for the kernels.  The product path has no CPU fallback:
the defaults call the CUDA library and raise if it is missing.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def band_rows(H: int, world: int, rank: int) -> Tuple[int, int]:
    """Output rows [b0, b1) of `rank` (balanced to within one row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * H // world, (rank + 1) * H // world


def band_input_rows(H: int, radius: int, b0: int, b1: int) -> Tuple[int, int]:
    """Input rows a band needs: [max(0, b0 - r), min(H, b1 + r)) (the rest is
    reflect-101 of rows inside the image, include/sf.h sf_filter_rows)."""
    return max(0, b0 - radius), min(H, b1 + radius)


def pair_count(N: int) -> int:
    """Conjugate pairs of the order-N expansion: floor(N/2) + 1."""
    return N // 2 + 1


def pair_range(N: int, world: int, rank: int) -> Tuple[int, int]:
    """Pairs [pb, pe) of `rank`, balanced by pair count."""
    K = pair_count(N)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * K // world, (rank + 1) * K // world


def _default_filter_rows():
    import paper_1107_4617_b200 as sf
    return sf.sf_filter_rows


def _default_accumulate():
    import paper_1107_4617_b200 as sf
    return sf.sf_accumulate


def _default_finalize():
    import paper_1107_4617_b200 as sf
    return sf.sf_finalize


def _default_accumulate_scatter():
    import paper_1107_4617_b200 as sf
    return sf.sf_accumulate_scatter


def _default_share():
    """(export, import) of a CUDA tensor across processes: torch's own CUDA IPC
    reduction (the handle of the allocation + the tensor's offset in it)."""
    from torch.multiprocessing.reductions import reduce_tensor

    def export(t):
        return reduce_tensor(t)

    def import_(shared):
        fn, args = shared
        return fn(*args)
    return export, import_


def rowband_filter(img_band, H: int, W: int, rank: int, world: int, radius: int, kind: int,
                   sigma_r: float, N: int, out_band=None, stream=None,
                   filter_rows: Optional[Callable] = None):
    """Filter this rank's row band.  `img_band` holds input rows
    band_input_rows(H, radius, *band_rows(H, world, rank)).  No collective."""
    b0, b1 = band_rows(H, world, rank)
    i0, i1 = band_input_rows(H, radius, b0, b1)
    if tuple(img_band.shape) != (i1 - i0, W):
        raise ValueError(f"img_band must be rows [{i0},{i1}) x {W}, got {tuple(img_band.shape)}")
    fn = filter_rows or _default_filter_rows()
    return fn(img_band, H, W, b0, b1, radius, kind, sigma_r, N, out_band=out_band, stream=stream)


def termsplit_filter(img, radius: int, kind: int, sigma_r: float, N: int, rank: int, world: int,
                     group=None, buf=None, out=None, stream=None,
                     accumulate: Optional[Callable] = None, finalize: Optional[Callable] = None,
                     dst: int = 0):
    """Term split: partial (num, den) over this rank's pairs, `reduce` of the
    packed [2, H, W] buffer to rank `dst`, ratio on `dst`.  Returns the H x W
    output on `dst` and None elsewhere.  `buf` (optional, [2, H, W] fp32 on
    the rank's device) is reused across calls to keep allocation out of the
    timed region."""
    import torch
    import torch.distributed as dist

    H, W = img.shape
    pb, pe = pair_range(N, world, rank)
    if buf is None:
        buf = torch.empty((2, H, W), dtype=torch.float32, device=img.device)
    acc = accumulate or _default_accumulate()
    acc(img, radius, kind, sigma_r, N, pb, pe, num=buf[0], den=buf[1], stream=stream)
    if world > 1:
        dist.reduce(buf, dst=dst, op=dist.ReduceOp.SUM, group=group)
    if rank != dst:
        return None
    fin = finalize or _default_finalize()
    return fin(buf[0], buf[1], img, out=out, stream=stream)


class FusedTermSplit:
    """Term split over `world` ranks (one process per GPU) with a one-sided
    reduce-scatter over peer memory instead of a collective.

    Rank o owns output band o (band_rows) and a packed [2, rows, W] fp32
    partial buffer for it.  Set-up (once, collective): the buffers' CUDA IPC
    handles are all-gathered and every rank maps every other rank's buffer.
    Each call: every rank zeroes its own buffer, barrier, every rank runs
    sf_accumulate_scatter over its pair range — the filter kernel, then a
    scatter-add pass that adds each output row's partials into the owning
    rank's buffer (fp32 atomics, over NVLink for the peers), so each GPU
    receives only its band — barrier, every rank forms the ratio of its band.  Returns this rank's output band (rows
    band_rows(H, world, rank)).

    `accumulate_scatter`, `finalize`, `alloc`, `share` and `sync` are
    injectable so that the host logic runs in gloo tests on CPU
    (tests/test_dist.py)."""

    def __init__(self, H: int, W: int, rank: int, world: int, device=None, group=None,
                 accumulate_scatter: Optional[Callable] = None, finalize: Optional[Callable] = None,
                 share: Optional[Tuple[Callable, Callable]] = None, sync: Optional[Callable] = None,
                 alloc: Optional[Callable] = None):
        import torch
        import torch.distributed as dist

        self.H, self.W, self.rank, self.world, self.group = H, W, rank, world, group
        self.acc = accumulate_scatter or _default_accumulate_scatter()
        self.fin = finalize or _default_finalize()
        self.sync = sync or (torch.cuda.synchronize if torch.cuda.is_available() else (lambda: None))
        export, import_ = share or _default_share()
        self.b0, self.b1 = band_rows(H, world, rank)
        shape = (2, self.b1 - self.b0, W)
        self.own = alloc(shape) if alloc else torch.zeros(shape, dtype=torch.float32, device=device)
        self._dist = dist
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, export(self.own), group=group)
            self.bands = [self.own if o == rank else import_(handles[o]) for o in range(world)]
        else:
            self.bands = [self.own]

    def _barrier(self):
        self.sync()
        if self.world > 1:
            self._dist.barrier(group=self.group)

    def __call__(self, img, radius: int, kind: int, sigma_r: float, N: int, out=None, stream=None):
        if tuple(img.shape) != (self.H, self.W):
            raise ValueError("image shape differs from the set-up")
        pb, pe = pair_range(N, self.world, self.rank)
        self.own.zero_()
        self._barrier()                             # every band zeroed before any rank adds
        self.acc(img, radius, kind, sigma_r, N, pb, pe, [b[0] for b in self.bands], [b[1] for b in self.bands],
                 stream=stream)
        self._barrier()                             # every rank's adds have landed
        return self.fin(self.own[0], self.own[1], img[self.b0:self.b1], out=out, stream=stream)

    def close(self):
        self.bands = []
        self.own = None
