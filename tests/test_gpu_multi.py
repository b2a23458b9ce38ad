"""Multi-GPU intra-column split on one GPU: several in-process
ranks (one context + host thread each) factor the same matrix, each running the
ARA / recompression / TRSM of its round-robin share of every column and
exchanging the new panels.  The factor must be bitwise identical to the
single-rank one (per-tile streams seeded by (root, i, k))."""
import threading

import numpy as np
import pytest

from helpers import covariance_ref, points

pytestmark = pytest.mark.gpu


def _factor_ranks(tg, parts, n, b, eps, cfg, world, mode=0):
    ctxs = [tg.Context(0) for _ in range(world)]
    tg.attach_local(ctxs)
    diag, ranks, U, V = parts
    mats = [tg.TlrMatrix.from_parts(n, b, eps, diag, ranks, U, V, ctx=c) for c in ctxs]
    out, err = [None] * world, [None] * world

    def run(r):
        try:
            f = tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt
            out[r] = f(mats[r], cfg)
        except Exception as e:  # surfaced below
            err[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("world,eps,bs", [(2, 1e-6, 16), (3, 1e-4, 16)])
def test_split_column_factor_is_bitwise_identical(tg, ref, world, eps, bs):
    from paper_2108_11932_b200 import geometry as G
    pts = points(G.GRID2D, 2048, 128)
    A_ref = ref.build(pts, 0, 0.1, 0.0, 128, eps, 0, bs, 5)
    parts = A_ref.to_parts()
    cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=5)
    A1 = tg.TlrMatrix.from_parts(2048, 128, eps, *parts)
    F1 = tg.tlr_cholesky(A1, cfg)
    d1, r1, U1, V1 = F1.L.to_parts()
    Fs = _factor_ranks(tg, parts, 2048, 128, eps, cfg, world)
    for F in Fs:
        d, r, U, V = F.L.to_parts()
        assert (np.asarray(r) == np.asarray(r1)).all()
        for a, b_ in zip(d, d1):
            assert np.array_equal(a, b_)
        for a, b_ in zip(U, U1):
            assert np.array_equal(a, b_)
        for a, b_ in zip(V, V1):
            assert np.array_equal(a, b_)


def test_split_column_ldlt_is_bitwise_identical(tg, ref):
    """LDL^T: D blocks and the intra-tile permutations are computed redundantly
    on every rank, the panels exchanged; factors equal bitwise to 1 rank."""
    from paper_2108_11932_b200 import geometry as G
    pts = points(G.GRID2D, 1024, 128)
    A_ref = ref.build(pts, 1, 0.2, 1e-4, 128, 1e-5, 0, 16, 3)
    parts = A_ref.to_parts()
    cfg = tg.AraConfig(block_samples=16, eps=1e-5, seed=3)
    F1 = tg.tlr_ldlt(tg.TlrMatrix.from_parts(1024, 128, 1e-5, *parts), cfg)
    d1, r1, U1, V1 = F1.L.to_parts()
    for F in _factor_ranks(tg, parts, 1024, 128, 1e-5, cfg, 2, mode=1):
        d, r, U, V = F.L.to_parts()
        assert (np.asarray(r) == np.asarray(r1)).all()
        assert all(np.array_equal(a, b_) for a, b_ in zip(d, d1))
        assert all(np.array_equal(a, b_) for a, b_ in zip(V, V1))
        for k in range(F.L.nb):
            (Da, pa), (Db, pb) = F.dblock(k), F1.dblock(k)
            assert np.array_equal(pa, pb)
            assert np.array_equal(Da.d, Db.d) and np.array_equal(Da.e, Db.e)


def _nccl_worker(rank, world, port, parts, meta, q):
    """One process per GPU: the NCCL transport of the column exchange."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    import paper_2108_11932_b200 as tg
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ctx = tg.Context(rank)
        obj = [tg.tlr.nccl_unique_id(ctx) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.attach_nccl(rank, world, obj[0])
        n, b, eps, bs, seed = meta
        diag, ranks, U, V = parts
        A = tg.TlrMatrix.from_parts(n, b, eps, diag, ranks, U, V, ctx=ctx)
        F = tg.tlr_cholesky(A, tg.AraConfig(block_samples=bs, eps=eps, seed=seed))
        q.put((rank, F.L.ranks().tolist(), F.L.to_parts()[0][-1].tolist()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        q.put((rank, "error", repr(e)))


def test_nccl_two_processes_bitwise_equal_to_one_gpu(tg, ref):
    """Two processes, one GPU each, NCCL panel exchange (comm.cu): the factor
    equals the single-GPU factor bit for bit.  Needs two visible GPUs."""
    import socket

    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs")
    n, b, eps, bs, seed = 2048, 128, 1e-6, 16, 5
    A_ref = covariance_ref(ref, n, b, eps)
    parts = A_ref.to_parts()
    one = tg.tlr_cholesky(tg.TlrMatrix.from_parts(n, b, eps, *parts),
                          tg.AraConfig(block_samples=bs, eps=eps, seed=seed))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, parts, (n, b, eps, bs, seed), q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        item = q.get(timeout=600)
        got[item[0]] = item[1:]
    for p in procs:
        p.join(120)
    for r in (0, 1):
        assert got[r][0] != "error", got[r]
        assert got[r][0] == one.L.ranks().tolist()
        assert np.array_equal(np.array(got[r][1]), one.L.to_parts()[0][-1])
