"""World-size-2 gloo test (CPU) of the row-block decomposition the multi-GPU
path implements (csrc/engine.cu + paper_2111_11148_b200/dist.py): partition
ceil(b*m/p) (parexec.cpp:9-18), Gaussian-sketch partials with GLOBAL Omega
counters, Gram partials, the uniform-sketch zero-row gather, all summed with
an all-reduce; identical small factorizations on every rank; row-local solves.
The per-rank arithmetic here is the CPU oracle (the checker); the partition and
the collectives are the product's host logic."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from oracle import oracle as o
from paper_2111_11148_b200 import dist


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, l, seed = 5003, 12, 24, 77
        a = o.synthesize(m, n, 1e8, 3)
        row0, rows = dist.shard_rows(m, world, rank)
        al = a[row0:row0 + rows]
        # (1) Gaussian sketch partials with global counters sum to the full sketch
        part = torch.from_numpy(o.sketch_gaussian_shard(al, m, row0, l, seed))
        td.all_reduce(part)
        full = o.sketch_gaussian(a, l, seed)
        ok_sketch = np.linalg.norm(part.numpy() - full) <= 1e-13 * np.linalg.norm(full)
        # (2) uniform sketch: owned rows into a zeroed l x n buffer, summed -> exact gather
        a1_full, idx = o.sample_rows_uniform(a, l, seed)
        mine = np.zeros((l, n))
        sel = (idx >= row0) & (idx < row0 + rows)
        mine[sel] = al[idx[sel] - row0]
        g1 = torch.from_numpy(mine)
        td.all_reduce(g1)
        ok_gather = np.array_equal(g1.numpy(), a1_full)
        # (3) identical preconditioner on every rank
        rt = o.qr_r_factor(part.numpy())
        allr = [torch.zeros(n, n, dtype=torch.float64) for _ in range(world)]
        td.all_gather(allr, torch.from_numpy(rt))
        ok_same = all(np.array_equal(x.numpy(), rt) for x in allr)
        # (4) row-local solve + Gram partial all-reduce
        x = o.right_trisolve(al, rt)
        gp = torch.from_numpy(o.gram(x) if rows >= n else x.T @ x)
        td.all_reduce(gp)
        xf = o.right_trisolve(a, rt)
        ok_solve = np.array_equal(x, xf[row0:row0 + rows])
        gf = o.gram(xf)
        ok_gram = np.abs(gp.numpy() - gf).max() <= 1e-13 * np.abs(gf).max()
        out[rank] = int(ok_sketch) + 2 * int(ok_gather) + 4 * int(ok_same) + 8 * int(ok_solve) + 16 * int(ok_gram)
    finally:
        td.destroy_process_group()


def test_row_block_decomposition_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = 29500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    assert dict(out) == {0: 31, 1: 31}, dict(out)


def test_shard_rows_matches_reference_partition():
    for m, p in [(10, 3), (1000003, 8), (4_000_000, 8), (33_554_432, 8)]:
        spans = [dist.shard_rows(m, p, b) for b in range(p)]
        assert spans[0][0] == 0 and sum(r for _, r in spans) == m
        assert all(spans[b][0] + spans[b][1] == spans[b + 1][0] for b in range(p - 1))
        assert [o.block_offset(m, p, b) for b in range(p)] == [s for s, _ in spans]


def _transport_worker(rank, world, port, out):
    """The host transport's C entry points (the function pointers cqr_attach_host_comm
    stores), called as the engine calls them: pinned-like host buffers, blocking."""
    import ctypes as C

    from paper_2111_11148_b200 import _abi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = dist.HostTransport()
        t = tr.table
        pd = C.POINTER(C.c_double)
        ok = 0
        # all-reduce sum of doubles, in place
        x = np.arange(5, dtype=np.float64) + 10 * rank
        assert t.allreduce(None, x.ctypes.data, 5, _abi.COMM_F64_SUM) == 0
        ok += int(np.array_equal(x, sum(np.arange(5.0) + 10 * b for b in range(world))))
        # all-reduce max of int32 (the non-finite / shard flags)
        f = np.array([rank == 1, rank], dtype=np.int32)
        assert t.allreduce(None, f.ctypes.data, 2, _abi.COMM_I32_MAX) == 0
        ok += 2 * int(list(f) == [1, world - 1])
        # send to the next rank, receive from the previous (the Gram chain tail/head), ends have one side
        s = np.full(7, float(rank + 1))
        r = np.zeros(7)
        dst = rank + 1 if rank + 1 < world else -1
        src = rank - 1 if rank > 0 else -1
        assert t.sendrecv(None, s.ctypes.data_as(pd) if dst >= 0 else None, dst,
                          r.ctypes.data_as(pd) if src >= 0 else None, src, 7) == 0
        ok += 4 * int(src < 0 or np.array_equal(r, np.full(7, float(rank))))
        # all-gather in rank order
        g = np.full(3, float(rank))
        allg = np.empty(3 * world)
        assert t.allgather(None, g.ctypes.data_as(pd), allg.ctypes.data_as(pd), 3) == 0
        ok += 8 * int(np.array_equal(allg, np.repeat(np.arange(world, dtype=float), 3)))
        out[rank] = ok if not tr.errors else -1
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_transport_callbacks_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = 30500 + (os.getpid() % 1000) + world
    mp.start_processes(_transport_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    assert dict(out) == {b: 15 for b in range(world)}, dict(out)
