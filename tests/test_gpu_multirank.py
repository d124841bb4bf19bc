"""The multi-rank factorization path of the engine, executed: p processes share
cuda:0, each owns its row block ceil(b*m/p) (parexec.cpp:13-15), and the exchange
steps (sketch all-reduce, the rank-count-independent Gram's tail/head send-recv
and node all-gather, the non-finite/shard flag all-reduce, the diagnostics'
sums) run through the library's host transport over gloo (cqr_attach_host_comm).
No kernel waits on another rank -- every exchange is a host call between kernel
launches -- so several ranks on one GPU are safe (B200_PROFILING.md); the NCCL
path makes the same calls on the same buffers in the same order.

Contracts (test_parexec.cpp:41-56, 103-116; acceptance.cpp:293-345):
  * CholeskyQR, CholeskyQR2, sCholeskyQR3 and rLU/rQR with the uniform sketch are
    bitwise equal to the one-GPU result for every p (the Gram is rank-count
    independent, the solves are row-local, the uniform gather is exact);
  * the Gaussian sketch's sum over ranks is order-dependent: ||Q_p - Q_1||_F <= 1e-10
    at kappa <= 1e5 (test_parexec.cpp:113), R within 1e-13;
  * identical status, pivot and retry count on every rank; the comm counters are the
    model at p (parexec.cpp:44-62).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as o
from paper_2111_11148_b200 import _abi
from paper_2111_11148_b200 import cholqr as G

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "helpers", "multirank_worker.py")
U, G_ = _abi.UNIFORM, _abi.GAUSSIAN
FIXED = dict(shift_kind=_abi.SHIFT_FIXED, shift=1e-15)

# acceptance.cpp:298-305: m = 2e5, n = 50, kappa = 1e5, sketch seed 2, fixed shift 1e-15
C8 = [dict(method=_abi.CHOLQR, strategy=U, seed=2, **FIXED), dict(method=_abi.CHOLQR2, strategy=U, seed=2, **FIXED),
      dict(method=_abi.SCHOLQR3, strategy=U, seed=2, **FIXED), dict(method=_abi.RLU, strategy=U, seed=2, **FIXED),
      dict(method=_abi.RQR, strategy=U, seed=2, **FIXED),
      dict(method=_abi.SCHOLQR3, strategy=U, seed=2),  # theory shift
      dict(method=_abi.RQR_GAUSSIAN, strategy=G_, seed=7), dict(method=_abi.RLU, strategy=G_, seed=7),
      dict(method=_abi.RLU, strategy=G_, seed=7, host=True)]  # cqr_factor_sharded (host buffers)
BITWISE = {_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_ranks(tmp, a, cases, p, uneven=False):
    np.save(os.path.join(tmp, "a.npy"), a)
    json.dump({"cases": cases, "uneven": uneven}, open(os.path.join(tmp, "cases.json"), "w"))
    port = _port()
    procs = []
    for b in range(p):
        env = dict(os.environ, RANK=str(b), WORLD_SIZE=str(p), MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="0")
        procs.append(subprocess.Popen([sys.executable, WORKER, tmp], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    logs = [pr.communicate(timeout=600)[0] for pr in procs]
    for pr, lg in zip(procs, logs):
        assert pr.returncode == 0, lg[-3000:]
    return [dict(np.load(os.path.join(tmp, f"rank{b}.npz"))) for b in range(p)]


def one_gpu(a, c):
    cfg = G.SketchConfig(strategy=c["strategy"], size=c.get("size", 0), seed=c["seed"])
    opts = _abi.options(shift_kind=c.get("shift_kind", _abi.SHIFT_THEORY), shift_value=c.get("shift", 0.0))
    f, _, rep = G._factor(c["method"], a, cfg, opts)
    return f, rep


@pytest.fixture(scope="module")
def c8_matrix():
    return o.synthesize(200_000, 50, 1e5, 1)  # acceptance.cpp:296


@pytest.mark.parametrize("p", [2, 3, 8])
def test_c8_ranks_match_one_gpu(p, c8_matrix, tmp_path):
    a = c8_matrix
    n = a.shape[1]
    res = run_ranks(str(tmp_path), a, C8, p)
    l = G.SketchConfig(seed=2).resolved_size(a.shape[0], n)
    for i, c in enumerate(C8):
        f, rep = one_gpu(a, c)
        q = np.concatenate([r[f"q{i}"] for r in res])
        rs = [r[f"r{i}"] for r in res]
        assert all(np.array_equal(rs[0], x) for x in rs), "R identical on every rank"
        st = [r[f"st{i}"] for r in res]
        assert all(s[0] == 0 for s in st) and all(s[2] == rep.stages[0].retries for s in st)
        rmin, rmax, vmin, vmax = G.comm_model(c["method"], p, n, l)
        assert all(s[3] == rmax and s[4] == vmax for s in st)
        tag = (p, _abi.METHOD_NAMES[c["method"]], c.get("strategy"), c.get("shift_kind"))
        if c["method"] in BITWISE or c["strategy"] == U:
            assert np.array_equal(q, f.q) and np.array_equal(rs[0], f.r), tag
        else:
            assert np.linalg.norm(q - f.q) <= 1e-10, tag  # test_parexec.cpp:113
            assert np.linalg.norm(rs[0] - f.r) / np.linalg.norm(f.r) <= 1e-13, tag
        # diagnostics summed over the ranks = the one-GPU diagnostics of the assembled Q
        orth = [r[f"orth{i}"] for r in res]
        assert all(np.array_equal(orth[0], x) for x in orth)
        assert abs(orth[0][0] - o.orthogonality_error(q)) <= 1e-15 + 1e-9 * o.orthogonality_error(q)


def test_breakdown_agrees_on_every_rank(tmp_path):
    a = o.synthesize(50_000, 30, 1e12, 6)
    cases = [dict(method=_abi.CHOLQR2, strategy=U, seed=1), dict(method=_abi.CHOLQR, strategy=U, seed=1)]
    res = run_ranks(str(tmp_path), a, cases, 4)
    for i, c in enumerate(cases):
        with pytest.raises(G.CholeskyBreakdown) as e:
            one_gpu(a, c)
        for r in res:
            assert r[f"st{i}"][0] == _abi.CHOLESKY_BREAKDOWN and r[f"st{i}"][1] == e.value.pivot_index


def test_non_standard_blocks_use_the_plain_sum(tmp_path):
    """Rows not split at ceil(b*m/p): the ranks agree (flag all-reduce) to sum plain Gram
    partials -- tolerance-level p-consistency (test_parexec.cpp:113)."""
    a = o.synthesize(60_000, 40, 1e4, 3)
    cases = [dict(method=_abi.CHOLQR2, strategy=U, seed=1, **FIXED), dict(method=_abi.RLU, strategy=U, seed=4)]
    res = run_ranks(str(tmp_path), a, cases, 3, uneven=True)
    for i, c in enumerate(cases):
        f, _ = one_gpu(a, c)
        q = np.concatenate([r[f"q{i}"] for r in res])
        assert np.linalg.norm(q - f.q) <= 1e-10
