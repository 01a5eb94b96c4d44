"""GPU tests of the fused term split: sf_accumulate_add and
sf_accumulate_scatter (partials added into num/den, or into per-band buffers,
by a scatter-add pass after the filter kernel) and FusedTermSplit, whose ranks add each row's
partials straight into the owning rank's buffer mapped by CUDA IPC.  Only one GPU is
reachable here, so the two-rank test runs both processes on cuda:0: the IPC
mapping, the cross-process atomics and the barriers are the real ones (the
kernels never wait on one another), only the NVLink hop is missing."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _sf():
    import paper_1107_4617_b200 as sf
    return sf


@pytest.mark.parametrize("r,kind,s,N", [(5, 0, 30.0, 30), (16, 0, 10.0, 264), (4, 1, 40.0, 17), (40, 0, 15.0, 118)])
def test_accumulate_add_matches_oracle(r, kind, s, N):
    """Two adds over the two halves of the pairs into zeroed buffers, then the
    ratio, equal the oracle; a third add of an empty range changes nothing."""
    sf = _sf()
    img = synth.gen_image(90, 300, 40 + r, 10.0)
    t = torch.from_numpy(img).cuda()
    K = sf.sf_pair_count(N)
    num = torch.zeros((90, 300), dtype=torch.float32, device="cuda")
    den = torch.zeros_like(num)
    sf.sf_accumulate_add(t, r, kind, s, N, 0, K // 2, num, den)
    sf.sf_accumulate_add(t, r, kind, s, N, K // 2, K, num, den)
    sf.sf_accumulate_add(t, r, kind, s, N, K, K, num, den)
    out = sf.sf_finalize(num, den, t)
    torch.cuda.synchronize()
    ref = oracle.bilateral_shiftable(img, r, kind, s, N)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    assert err.max() <= 0.05 and err.mean() <= 0.005, (err.max(), err.mean())


@pytest.mark.parametrize("nband", [1, 3])
def test_accumulate_scatter_bands(nband):
    """Three adds over a pair partition into nband band buffers; each band's
    ratio equals the oracle's rows of that band."""
    from paper_1107_4617_b200 import dist as sfd
    sf = _sf()
    H, W, r, kind, s, N = 100, 260, 8, 0, 20.0, 66
    img = synth.gen_image(H, W, 55, 10.0)
    t = torch.from_numpy(img).cuda()
    rows = [sfd.band_rows(H, nband, o) for o in range(nband)]
    bufs = [torch.zeros((2, b1 - b0, W), dtype=torch.float32, device="cuda") for b0, b1 in rows]
    K = sf.sf_pair_count(N)
    for pb, pe in [(0, K // 3), (K // 3, 2 * K // 3), (2 * K // 3, K)]:
        sf.sf_accumulate_scatter(t, r, kind, s, N, pb, pe, [b[0] for b in bufs], [b[1] for b in bufs])
    ref = oracle.bilateral_shiftable(img, r, kind, s, N)
    for (b0, b1), b in zip(rows, bufs):
        out = sf.sf_finalize(b[0], b[1], t[b0:b1]).cpu().numpy().astype(np.float64)
        err = np.abs(out - ref[b0:b1])
        assert err.max() <= 0.05 and err.mean() <= 0.005, (nband, b0, err.max())


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _worker(rank, world, port, params, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1107_4617_b200 import dist as sfd
        H, W, r, kind, s, N, seed = params
        torch.cuda.set_device(0)
        t = torch.from_numpy(synth.gen_image(H, W, seed, 10.0)).cuda()
        fts = sfd.FusedTermSplit(H, W, rank, world, device="cuda")
        for _ in range(2):
            out = fts(t, r, kind, s, N)
        parts = [None] * world
        dist.all_gather_object(parts, out.cpu().numpy())
        if rank == 0:
            q.put(np.concatenate(parts))
        dist.barrier()
        fts.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("params", [(256, 300, 16, 0, 10.0, 264, 21), (120, 200, 5, 1, 40.0, 17, 22)])
def test_fused_termsplit_two_processes(params):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, 2, port, params, q)) for i in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    H, W, r, kind, s, N, seed = params
    ref = oracle.bilateral_shiftable(synth.gen_image(H, W, seed, 10.0), r, kind, s, N)
    err = np.abs(got.astype(np.float64) - ref)
    assert err.max() <= 0.05 and err.mean() <= 0.005, (err.max(), err.mean())
