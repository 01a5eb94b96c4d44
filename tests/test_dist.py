"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in
paper_1107_4617_b200/dist.py: row-band partitioning with r-row halos, the
term split (pair partition, packed [2,H,W] reduce, finalize on rank 0), and
the fused term split (the root's buffer shared with every rank, adds from
every rank, barriers, finalize on the root).

The CUDA kernels cannot run here, so each rank's compute is a CPU stand-in
built from the fp64 oracle (tests only); what is under test is the sharding,
the halo placement and the collective — the parts that run on the host."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1107_4617_b200 import dist as sfd  # noqa: E402

CENTER = 128.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---------------------------------------------------------------- stand-ins
def cpu_filter_rows(img_band, H, W, b0, b1, radius, kind, sigma_r, N, out_band=None, stream=None):
    """CPU stand-in for sf_filter_rows: the band alone must suffice, so the
    rows outside it are filled with garbage before calling the oracle."""
    i0, i1 = sfd.band_input_rows(H, radius, b0, b1)
    full = np.random.default_rng(99).integers(0, 256, (H, W), dtype=np.uint8)
    full[i0:i1] = img_band.numpy()
    res = oracle.bilateral_shiftable(full, radius, kind, sigma_r, N, row_begin=b0, row_end=b1)
    t = torch.from_numpy(res.astype(np.float32))
    if out_band is not None:
        out_band.copy_(t)
        return out_band
    return t


def cpu_accumulate(img, radius, kind, sigma_r, N, pb, pe, num=None, den=None, stream=None):
    """CPU stand-in for sf_accumulate: pairs [pb,pe) = terms {k, N-k}."""
    a = img.numpy()
    tot_n = np.zeros(a.shape)
    tot_d = np.zeros(a.shape)
    ranges = [(pb, pe), (max(N - pe + 1, pe), N - pb + 1)]
    for n0, n1 in ranges:
        if n1 > n0:
            _, nm, dn = oracle.bilateral_shiftable(a, radius, kind, sigma_r, N, n_begin=n0, n_end=n1,
                                                   return_parts=True)
            tot_n += nm
            tot_d += dn
    num.copy_(torch.from_numpy((tot_n - CENTER * tot_d).astype(np.float32)))
    den.copy_(torch.from_numpy(tot_d.astype(np.float32)))
    return num, den


def cpu_accumulate_scatter(img, radius, kind, sigma_r, N, pb, pe, band_num, band_den, stream=None):
    """CPU stand-in for sf_accumulate_scatter into buffers shared by the ranks
    (file mappings): band o of the partials is added into band_num[o] /
    band_den[o]; the adds of concurrent ranks are serialised by a file lock, as
    the GPU's are by atomics."""
    import fcntl
    H, W = img.shape
    n = torch.empty((H, W))
    d = torch.empty((H, W))
    cpu_accumulate(img, radius, kind, sigma_r, N, pb, pe, num=n, den=d)
    with open(os.environ["SF_TEST_LOCK"], "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        for o in range(len(band_num)):
            b0, b1 = sfd.band_rows(H, len(band_num), o)
            band_num[o] += n[b0:b1]
            band_den[o] += d[b0:b1]
        fcntl.flock(lk, fcntl.LOCK_UN)


def cpu_finalize(num, den, img, out=None, stream=None):
    r = CENTER + num / den
    r = torch.where((den > 0) & torch.isfinite(den), r, img.float())
    if out is not None:
        out.copy_(r)
        return out
    return r


# ---------------------------------------------------------------- workers
def _worker(rank, world, port, mode, params, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, W, r, kind, s, N, seed = params
        img = synth.gen_image(H, W, seed, 10.0)
        if mode == "rowband":
            b0, b1 = sfd.band_rows(H, world, rank)
            i0, i1 = sfd.band_input_rows(H, r, b0, b1)
            band = torch.from_numpy(np.ascontiguousarray(img[i0:i1]))
            out = sfd.rowband_filter(band, H, W, rank, world, r, kind, s, N, filter_rows=cpu_filter_rows)
            # gloo all_gather needs equal sizes: pad every band to the largest
            sizes = [sfd.band_rows(H, world, i) for i in range(world)]
            mx = max(e - b for b, e in sizes)
            padded = torch.zeros((mx, W))
            padded[: b1 - b0] = out
            gathered = [torch.empty((mx, W)) for _ in range(world)]
            dist.all_gather(gathered, padded)
            parts = [g[: e - b] for g, (b, e) in zip(gathered, sizes)]
            if rank == 0:
                q.put(("rowband", torch.cat(parts).numpy()))
        elif mode == "fused":
            base = os.environ["SF_TEST_SHARED"]

            def alloc(shape):
                mm = np.memmap(f"{base}.{rank}", dtype=np.float32, mode="w+", shape=shape)
                return torch.from_numpy(mm)

            def export(t):
                return (f"{base}.{rank}", tuple(t.shape))

            def import_(shared):
                pth, shape = shared
                return torch.from_numpy(np.memmap(pth, dtype=np.float32, mode="r+", shape=shape))

            t = torch.from_numpy(img)
            fts = sfd.FusedTermSplit(H, W, rank, world, accumulate_scatter=cpu_accumulate_scatter,
                                     finalize=cpu_finalize, share=(export, import_), alloc=alloc,
                                     sync=lambda: None)
            for _ in range(2):                      # the buffers are re-zeroed per call
                out = fts(t, r, kind, s, N)
            b0, b1 = sfd.band_rows(H, world, rank)
            assert tuple(out.shape) == (b1 - b0, W)
            parts = [None] * world
            dist.all_gather_object(parts, out.numpy().copy())
            fts.close()
            if rank == 0:
                q.put(("fused", np.concatenate(parts)))
        else:
            t = torch.from_numpy(img)
            out = sfd.termsplit_filter(t, r, kind, s, N, rank, world, accumulate=cpu_accumulate,
                                       finalize=cpu_finalize)
            if rank == 0:
                q.put(("termsplit", out.numpy()))
            else:
                assert out is None
    finally:
        dist.destroy_process_group()


def _run(mode, params, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, mode, params, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res[1]


# ---------------------------------------------------------------- host logic
def test_band_rows_cover_image():
    for H in (1, 7, 8192, 1081):
        for n in (1, 2, 3, 4, 8):
            if n > H:
                continue
            spans = [sfd.band_rows(H, n, i) for i in range(n)]
            assert spans[0][0] == 0 and spans[-1][1] == H
            assert all(spans[i][1] == spans[i + 1][0] for i in range(n - 1))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def test_band_input_rows_halo():
    assert sfd.band_input_rows(8192, 16, 0, 1024) == (0, 1040)
    assert sfd.band_input_rows(8192, 16, 1024, 2048) == (1008, 2064)
    assert sfd.band_input_rows(8192, 64, 7168, 8192) == (7104, 8192)


def test_pair_range_partition():
    for N in (17, 30, 118, 264):
        K = sfd.pair_count(N)
        assert K == N // 2 + 1
        for n in (1, 2, 4, 8):
            spans = [sfd.pair_range(N, n, i) for i in range(n)]
            assert spans[0][0] == 0 and spans[-1][1] == K
            assert all(spans[i][1] == spans[i + 1][0] for i in range(n - 1))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def test_rowband_argument_check():
    with pytest.raises(ValueError):
        sfd.rowband_filter(torch.zeros((5, 10), dtype=torch.uint8), 40, 10, 0, 2, 3, 0, 30.0, 30,
                           filter_rows=cpu_filter_rows)


# ---------------------------------------------------------------- gloo, world size 2
@pytest.mark.parametrize("params", [(48, 40, 5, 0, 30.0, 30, 11), (37, 29, 4, 1, 40.0, 17, 12)])
def test_rowband_gloo_ws2(params):
    H, W, r, kind, s, N, seed = params
    got = _run("rowband", params)
    ref = oracle.bilateral_shiftable(synth.gen_image(H, W, seed, 10.0), r, kind, s, N)
    assert np.max(np.abs(got - ref)) < 1e-3


@pytest.mark.parametrize("params", [(32, 28, 4, 0, 10.0, 264, 13), (30, 26, 3, 0, 30.0, 31, 14)])
def test_termsplit_gloo_ws2(params):
    H, W, r, kind, s, N, seed = params
    got = _run("termsplit", params)
    ref = oracle.bilateral_shiftable(synth.gen_image(H, W, seed, 10.0), r, kind, s, N)
    assert np.max(np.abs(got - ref)) < 1e-3


@pytest.mark.parametrize("params", [(32, 28, 4, 0, 10.0, 264, 15), (30, 26, 3, 1, 30.0, 31, 16)])
def test_fused_termsplit_gloo_ws2(params, tmp_path, monkeypatch):
    monkeypatch.setenv("SF_TEST_SHARED", str(tmp_path / "buf.f32"))
    monkeypatch.setenv("SF_TEST_LOCK", str(tmp_path / "buf.lock"))
    H, W, r, kind, s, N, seed = params
    got = _run("fused", params)
    ref = oracle.bilateral_shiftable(synth.gen_image(H, W, seed, 10.0), r, kind, s, N)
    assert np.max(np.abs(got - ref)) < 1e-3
