"""The rank-count-independent sharded Gram (csrc/gram_shard.cu, SURVEY 8e
"determinism option"): the product's plan and tree program (read through the
C-ABI, host-only) driven with the oracle's arithmetic must reproduce the
one-process Gram bit for bit for any p, as the reference's parallel Gram does
(test_parexec.cpp:47-56: "the fixed chunk tree actually makes them bitwise
identical"). The oracle is the checker here; the plan is the product."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from oracle import oracle as o
from paper_2111_11148_b200 import dist

LEAF = 1024


def _rank_part(x_local, plan, n, head_in):
    """One rank's arithmetic (oracle): tail chain, head chain, leaves, node values."""
    r0 = plan["row0"]
    tail = None
    if plan["tail"] and not plan["span"]:
        tail = o.gram_chain(x_local[plan["tail_start"] - r0:])
    if plan["span"]:
        return o.gram_chain(x_local, head_in), []
    leaves = []
    if plan["head"]:
        leaves.append(o.gram_chain(x_local[:plan["head_end"] - r0], head_in))
    for s in range(plan["full0"], plan["full1"], LEAF):
        leaves.append(o.gram_chain(x_local[s - r0:min(s + LEAF, plan["full1"]) - r0]))
    assert len(leaves) == plan["hi"] - plan["lo"]
    nodes = []
    for s, c in plan["node_list"]:
        sub = np.stack(leaves[s - plan["lo"]:s - plan["lo"] + c])
        nodes.append(o.tree_combine(sub).reshape(n, n))
    return tail, nodes


def _eval(prog, slots):
    stk = []
    for op in prog:
        if op >= 0:
            stk.append(slots[op])
        else:
            r = stk.pop()
            stk[-1] = stk[-1] + r
    assert len(stk) == 1
    g = np.triu(stk[0])
    return g + np.triu(g, 1).T


def _sim(x, p):
    m, n = x.shape
    prog, K = dist.gram_tree_program(m, p)
    slots = [np.zeros((n, n)) for _ in range(p * K)]
    carry = None
    for b in range(p):
        plan = dist.gram_shard_plan(m, p, b)
        tail, nodes = _rank_part(x[plan["row0"]:plan["row1"]], plan, n, carry if plan["head"] else None)
        for k, v in enumerate(nodes):
            slots[b * K + k] = v
        carry = tail
    return _eval(prog, slots)


def test_plan_covers_rows_and_leaves():
    for m in (1, 1023, 1024, 1025, 3000, 5003, 65536, 1_000_003, 4_000_000):
        L = (m + LEAF - 1) // LEAF
        for p in (1, 2, 3, 4, 7, 8):
            if p > m:
                continue
            owned = []
            prev_out = False
            for b in range(p):
                s = dist.gram_shard_plan(m, p, b)
                assert s["row0"] == dist.shard_rows(m, p, b)[0]
                # a head exists exactly when the previous rank sends a tail or a span
                assert s["head"] == prev_out
                prev_out = s["tail"]
                # rows: head, complete leaves, tail in order, nothing lost
                parts = []
                if s["span"]:
                    parts.append((s["row0"], s["row1"]))
                else:
                    if s["head"]:
                        parts.append((s["row0"], s["head_end"]))
                    if s["full1"] > s["full0"]:
                        parts.append((s["full0"], s["full1"]))
                    if s["tail"]:
                        parts.append((s["tail_start"], s["row1"]))
                assert parts[0][0] == s["row0"] and parts[-1][1] == s["row1"]
                assert all(a[1] == b_[0] for a, b_ in zip(parts, parts[1:]))
                assert s["full1"] == s["full0"] or s["full0"] % LEAF == 0
                # the nodes cover the owned leaves in order, each one aligned
                cur = s["lo"]
                for st, c in s["node_list"]:
                    assert st == cur and c >= 1
                    size = 1 << (c - 1).bit_length()
                    assert st % size == 0 and (c == size or st + c == L)
                    cur += c
                assert cur == s["hi"]
                owned.extend(range(s["lo"], s["hi"]))
            assert prev_out is False
            assert owned == list(range(L))


@pytest.mark.parametrize("m,n,p", [(5003, 12, 3), (4096, 8, 4), (3000, 6, 8), (9000, 5, 7), (2048, 4, 2),
                                   (40_000, 3, 6), (1100, 5, 2), (17 * 1024 + 5, 4, 5)])
def test_sharded_gram_bitwise_for_any_p(m, n, p):
    x = o.gaussian_matrix(m, n, 31 + p)
    ref = o.gram(x)
    assert np.array_equal(_sim(x, p), ref)


def test_tree_program_matches_pairwise_tree_on_random_slots():
    # every node value a random array: evaluating the program over the nodes must
    # equal the level-by-level tree over the leaves when nodes hold their subtree sums
    rng = np.random.default_rng(5)
    for m in (1024 * 37 + 11, 1024 * 64, 1024 * 100 - 3):
        L = (m + LEAF - 1) // LEAF
        leaves = rng.standard_normal((L, 4))
        ref = o.tree_combine(leaves)
        for p in (2, 3, 5, 8):
            prog, K = dist.gram_tree_program(m, p)
            slots = [np.zeros(4) for _ in range(p * K)]
            for b in range(p):
                s = dist.gram_shard_plan(m, p, b)
                for k, (st, c) in enumerate(s["node_list"]):
                    slots[b * K + k] = o.tree_combine(leaves[st:st + c])
            stk = []
            for op in prog:
                if op >= 0:
                    stk.append(slots[op])
                else:
                    r = stk.pop()
                    stk[-1] = stk[-1] + r
            assert np.array_equal(stk[0], ref)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n = 7001, 9
        x = o.gaussian_matrix(m, n, 808)
        plan = dist.gram_shard_plan(m, world, rank)
        xl = x[plan["row0"]:plan["row1"]].copy()
        prog, K = dist.gram_tree_program(m, world)
        head = None
        if not plan["span"]:
            tail, _ = _rank_part(xl, {**plan, "head": False, "full0": 0, "full1": 0, "hi": plan["lo"],
                                      "node_list": []}, n, None)
            reqs = []
            if tail is not None:
                reqs.append(td.isend(torch.from_numpy(tail), rank + 1))
            if plan["head"]:
                buf = torch.zeros(n, n, dtype=torch.float64)
                reqs.append(td.irecv(buf, rank - 1))
            for r in reqs:
                r.wait()
            head = buf.numpy() if plan["head"] else None
            _, nodes = _rank_part(xl, {**plan, "tail": False}, n, head)
        else:
            buf = torch.zeros(n, n, dtype=torch.float64)
            td.recv(buf, rank - 1)
            fwd, nodes = _rank_part(xl, plan, n, buf.numpy())
            td.send(torch.from_numpy(fwd), rank + 1)
        mine = torch.zeros(K, n, n, dtype=torch.float64)
        for k, v in enumerate(nodes):
            mine[k] = torch.from_numpy(v)
        allv = [torch.zeros(K, n, n, dtype=torch.float64) for _ in range(world)]
        td.all_gather(allv, mine)
        slots = [allv[b][k].numpy() for b in range(world) for k in range(K)]
        g = _eval(prog, slots)
        out[rank] = int(np.array_equal(g, o.gram(x)))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gram_gloo(world):
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert [out[r] for r in range(world)] == [1] * world
