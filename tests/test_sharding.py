"""Row-sharded NT host logic over world-size-2 gloo (CPU). The local product is
injected (torch CPU matmul) because the product path has no CPU kernels; the
partitioning, the B broadcast and the C all-gather are what is under test."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_03192_b200.sharding import row_range, sharded_gemm_nt, shard_rows


def test_row_range_partitions():
    for m in (1, 7, 8, 65536, 12345):
        for world in (1, 2, 3, 4, 8):
            ranges = [row_range(m, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        row_range(8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, k, gather, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        a = torch.rand(m, k, generator=g) * 2 - 1
        b = torch.rand(n, k, generator=g) * 2 - 1
        a_local = shard_rows(a, rank, world).contiguous()
        c = sharded_gemm_nt(a_local, b if rank == 0 else None, m=m, n=n, k=k, gather=gather,
                            gemm=lambda x, y: x @ y.t())
        want = a.double() @ b.double().t()
        if gather:
            err = float((c.double() - want).norm() / want.norm())
            shape_ok = tuple(c.shape) == (m, n)
        else:
            lo, hi = row_range(m, rank, world)
            err = float((c.double() - want[lo:hi]).norm() / max(want[lo:hi].norm(), 1e-30))
            shape_ok = tuple(c.shape) == (hi - lo, n)
        q.put((rank, err, shape_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,gather", [(64, True), (37, True), (1, True), (64, False)])
def test_sharded_nt_world2_gloo(m, gather):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, 24, 40, gather, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = sorted(q.get(timeout=10) for _ in range(2))
    for rank, err, shape_ok in results:
        assert shape_ok, rank
        assert err < 1e-6, (rank, err)


def _dp_worker(rank, world, port, dout, din, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1702_03192_b200.sharding import dp_weight_grad

        g = torch.Generator().manual_seed(11)
        dz = torch.rand(dout, batch, generator=g) * 2 - 1   # full batch, same on every rank
        x = torch.rand(din, batch, generator=g) * 2 - 1
        lo, hi = row_range(batch, rank, world)               # this rank's batch columns
        dw = dp_weight_grad(dz[:, lo:hi], x[:, lo:hi], gemm=lambda a, b: a @ b.t())
        want = dz.double() @ x.double().t()
        q.put((rank, float((dw.double() - want).norm() / want.norm())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [64, 37])
def test_dp_weight_grad_world2_gloo(batch):
    """Data-parallel FC step: per-rank weight gradients over batch shards,
    summed by the all-reduce, equal the full-batch gradient."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, 24, 40, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err < 1e-6, (rank, err)


# ---------------------------------------------------------------- GPU
def _fused_worker(rank, world, port, m, n, k, q, iters=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1702_03192_b200.sharding import PeerGather

        torch.cuda.set_device(0)  # the ranks share one GPU: IPC maps between processes
        g = torch.Generator().manual_seed(5)
        a = torch.rand(m, k, generator=g) * 2 - 1
        b = torch.rand(n, k, generator=g) * 2 - 1
        lo, hi = row_range(m, rank, world)
        c = torch.full((m, n), float("nan"), device="cuda")
        pg = PeerGather(c)
        bd = b.cuda()
        for it in range(iters):
            # device-side barriers only (sync=False): earlier iterations write
            # scaled results that the last one must fully overwrite on every rank
            scale = float(iters - it)
            a_it = (a[lo:hi] * scale).cuda()
            if it % 2:  # a non-contiguous view: the call's temporary must outlive the launch
                a_it = a_it.t().contiguous().t()
            pg.gemm(a_it, bd, lo, sync=(it == iters - 1))
        pg.check_status()
        got = c.cpu().numpy()
        rows = np.unique(np.r_[0, m - 1, np.arange(0, m, 37)])
        want = oracle.oracle_nt_rows(a.numpy(), b.numpy(), rows, np.arange(n))
        q.put((rank, oracle.rel_frobenius(got[rows], want), bool(np.isfinite(got).all())))
        pg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,iters", [(1024, 768, 512, 1), (600, 300, 264, 1), (2048, 1024, 8192, 1),
                                         (2048, 1024, 1024, 4)])
def test_fused_allgather_two_processes_one_gpu(m, n, k, iters):
    """Two ranks (processes) share the GPU; each computes its row block with
    the all-gather fused into the GEMM epilogue (stores into the other rank's
    IPC-mapped C). Both ranks then hold the full C (no NaN left, oracle match)."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, m, n, k, q, iters))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, err, finite in res:
        assert finite, rank
        assert err < 1e-5, (rank, err)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,row0,mloc", [(2048, 1024, 512, 512, 1024), (256, 300, 64, 100, 64),
                                             (4096, 2048, 8192, 1024, 2048)])
def test_fused_allgather_local_destinations(m, n, k, row0, mloc):
    """The multi-destination epilogue on one process: peers are other local C
    buffers; the row block lands identically in all of them, other rows untouched
    (second case: too small for CTA pairs, so the local-GEMM + peer-copy fallback)."""
    from paper_1702_03192_b200 import _lib
    import ctypes

    g = torch.Generator().manual_seed(2)
    a = (torch.rand(mloc, k, generator=g) * 2 - 1).cuda()
    b = (torch.rand(n, k, generator=g) * 2 - 1).cuda()
    cs = [torch.zeros(m, n, device="cuda") for _ in range(4)]
    peers = (ctypes.c_void_p * 3)(*[c.data_ptr() for c in cs[1:]])
    _lib.check(_lib.lib.mtnn_gemm_nt_allgather(a.data_ptr(), b.data_ptr(), cs[0].data_ptr(), peers, 3,
                                               row0, mloc, n, k, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = (a.double() @ b.double().t())
    for c in cs:
        blk = c[row0:row0 + mloc].double()
        assert float((blk - want).norm() / want.norm()) < 1e-5
        assert torch.equal(c[row0:row0 + mloc], cs[0][row0:row0 + mloc])
        assert float(c[:row0].abs().sum()) == 0.0 and float(c[row0 + mloc:].abs().sum()) == 0.0
