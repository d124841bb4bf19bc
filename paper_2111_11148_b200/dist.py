"""One process per GPU: the row-block data parallelism of the reference's
parexec (parexec.hpp:11-57, simulated there with threads) on real GPUs.

Rank b owns rows [ceil(b*m/p), ceil((b+1)*m/p)) of the global m x n matrix
(parexec.cpp:13-15). The library sums the s x n sketch partials with NCCL
all-reduce (its own communicator, created from a unique id that rank 0
broadcasts through torch.distributed), forms the n x n Gram with the
rank-count-independent protocol of csrc/gram_shard.cu (leaf chains continued
across block boundaries, tree nodes all-gathered: bitwise equal to one GPU for
any p, as the reference's parallel Gram, engine.cpp:24-39), runs the small
factorizations redundantly on every rank (identical inputs give identical R,
so no broadcast and no collective for the retry decision), and leaves Q
row-sharded. torch.distributed is only the plumbing (id exchange, barriers).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from . import cholqr as cq


def shard_rows(m: int, p: int, b: int):
    """(row0, rows) of block b (parexec.cpp:9-18)."""
    lo, hi = cq.block_offset(m, p, b), cq.block_offset(m, p, b + 1)
    return lo, hi - lo


def gram_shard_plan(m: int, p: int, b: int) -> dict:
    """Rank b's part of the rank-count-independent Gram (cqr_gram_shard_plan):
    head/tail/span chains across block boundaries, complete leaves, owned leaves
    and the tree nodes they are combined into."""
    s = _abi.GramShard()
    if cq._lib().cqr_gram_shard_plan(m, p, b, C.byref(s)) != 0:
        raise ValueError("cqr_gram_shard_plan: bad arguments")
    out = {k: getattr(s, k) for k, _ in _abi.GramShard._fields_ if not k.startswith("node_")}
    for k in ("head", "tail", "span"):
        out[k] = bool(out[k])
    out["node_list"] = [(s.node_start[k], s.node_count[k]) for k in range(s.nodes)]
    return out


def gram_tree_program(m: int, p: int):
    """(program, K): postfix ops over gathered slots b*K + k, -1 = left + right."""
    K = C.c_int()
    need = -cq._lib().cqr_gram_tree_program(m, p, None, 0, C.byref(K))
    buf = (C.c_int * max(need, 1))()
    ln = cq._lib().cqr_gram_tree_program(m, p, buf, need, C.byref(K))
    return list(buf[:ln]), K.value


def make_context(device: int, rank: int | None = None, world: int | None = None):
    """Context on `device` with an NCCL communicator over the torch.distributed group."""
    import torch.distributed as td

    ctx = cq.Context(device)
    if world is None:
        world = td.get_world_size() if td.is_initialized() else 1
        rank = td.get_rank() if td.is_initialized() else 0
    if world > 1:
        obj = [cq.make_comm_id() if rank == 0 else None]
        td.broadcast_object_list(obj, src=0)
        ctx.attach_comm(rank, world, obj[0])
    return ctx


class HostTransport:
    """cqr_host_comm over torch.distributed (any backend that takes CPU tensors: gloo).

    The library stages each exchange through pinned host memory and calls back;
    every callback blocks until its exchange is complete, so no GPU kernel ever
    waits on another rank. This runs the multi-rank path of the engine with
    several processes on one GPU (tests/test_gpu_multirank.py) -- the exchange
    steps, their order and the data they move are the NCCL path's."""

    def __init__(self, group=None):
        self.group = group
        self.errors = []
        self.table = _abi.HostComm(None, _abi.ALLREDUCE_FN(self._allreduce), _abi.SENDRECV_FN(self._sendrecv),
                                   _abi.ALLGATHER_FN(self._allgather))

    @staticmethod
    def _view(ptr, count, ctype):
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(int(count),))

    def allreduce(self, arr, dtype):
        import torch
        import torch.distributed as td

        t = torch.from_numpy(arr)
        td.all_reduce(t, op=td.ReduceOp.SUM if dtype == _abi.COMM_F64_SUM else td.ReduceOp.MAX, group=self.group)

    def sendrecv(self, send, dst, recv, src):
        import torch
        import torch.distributed as td

        reqs = []
        if dst >= 0:
            reqs.append(td.isend(torch.from_numpy(send), dst, group=self.group))
        if src >= 0:
            reqs.append(td.irecv(torch.from_numpy(recv), src, group=self.group))
        for r in reqs:
            r.wait()

    def allgather(self, send, recv):
        import torch
        import torch.distributed as td

        world = td.get_world_size(self.group)
        parts = [torch.from_numpy(recv[k * send.size:(k + 1) * send.size]) for k in range(world)]
        td.all_gather(parts, torch.from_numpy(send), group=self.group)

    # ctypes entry points (exceptions must not cross into C)
    def _allreduce(self, user, buf, count, dtype):
        try:
            self.allreduce(self._view(buf, count, C.c_double if dtype == _abi.COMM_F64_SUM else C.c_int32), dtype)
            return 0
        except Exception as e:  # pragma: no cover - surfaced through the status code
            self.errors.append(e)
            return 1

    def _sendrecv(self, user, send, dst, recv, src, count):
        try:
            self.sendrecv(self._view(send, count, C.c_double) if dst >= 0 else None, dst,
                          self._view(recv, count, C.c_double) if src >= 0 else None, src)
            return 0
        except Exception as e:  # pragma: no cover
            self.errors.append(e)
            return 1

    def _allgather(self, user, send, recv, count):
        try:
            import torch.distributed as td

            world = td.get_world_size(self.group)
            self.allgather(self._view(send, count, C.c_double), self._view(recv, count * world, C.c_double))
            return 0
        except Exception as e:  # pragma: no cover
            self.errors.append(e)
            return 1


def attach_host_transport(ctx, group=None):
    """Attach a HostTransport over the torch.distributed group to ctx (kept alive on ctx)."""
    import torch.distributed as td

    tr = HostTransport(group)
    ctx._check(cq._lib().cqr_attach_host_comm(ctx.h, td.get_rank(group), td.get_world_size(group),
                                               C.byref(tr.table)))
    ctx.transport = tr
    return tr


def factor_sharded(ctx, method, a_local, m_global: int, row0: int, cfg: cq.SketchConfig | None = None,
                   opts=None, q_out=None):
    """cqr_factor_dev on this rank's CUDA shard; returns (Q_local, R, report)."""
    import torch

    if opts is None:
        opts = _abi.options()
    cfg_c = (cfg or cq.SketchConfig())._c()
    cq._check_cuda_matrix(a_local, "A", False)
    m_local, n = a_local.shape
    q = q_out if q_out is not None else torch.empty((m_local, n), dtype=torch.float64, device=a_local.device)
    if q.shape != a_local.shape or q.device != a_local.device:
        raise ValueError("q_out must match the shard's shape and device")
    # the library stream waits for torch's pending work on A and Q (stream-ordered, no host sync)
    cq._check_cuda_matrix(q, "q_out", ctx)
    r = np.zeros((n, n))
    rep = _abi.Report()
    st = cq._lib().cqr_factor_dev(ctx.h, method, C.c_void_p(a_local.data_ptr()), m_local, m_global, row0, n,
                                  a_local.stride(0), C.byref(cfg_c), C.byref(opts), C.c_void_p(q.data_ptr()),
                                  q.stride(0), cq._ptr(r), n, C.byref(rep))
    ctx._check(st, rep.index)
    return q, (None if opts.r_less else r), rep


def factor_sharded_host(ctx, method, a_local, m_global: int, row0: int, cfg: cq.SketchConfig | None = None,
                        opts=None, q_out=None):
    """cqr_factor_sharded: this rank's rows as a host (numpy, ideally pinned) buffer; the H2D of the
    shard, the multi-GPU factorization and the D2H of Q_local happen inside. Returns (Q_local, R, report)."""
    if opts is None:
        opts = _abi.options()
    cfg_c = (cfg or cq.SketchConfig())._c()
    a_local = np.ascontiguousarray(a_local, dtype=np.float64)
    m_local, n = a_local.shape
    q = q_out if q_out is not None else np.empty_like(a_local)
    r = np.zeros((n, n))
    rep = _abi.Report()
    st = cq._lib().cqr_factor_sharded(ctx.h, method, cq._ptr(a_local), m_local, m_global, row0, n, n,
                                      C.byref(cfg_c), C.byref(opts), cq._ptr(q), n, cq._ptr(r), n, C.byref(rep))
    ctx._check(st, rep.index)
    return q, (None if opts.r_less else r), rep
