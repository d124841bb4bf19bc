"""The reference's paper-level acceptance criteria (proj/tests/acceptance.cpp) run
on the B200 path.

  C1 (acceptance.cpp:68-94):  m = 1e5, n = 100, l = 2n, kappa = 1e3..1e15, 3 seeds;
      rQR, rLU and sCholeskyQR3 (fixed shift 1e-15) are ok with orth <= 1e-11 and
      res <= 1e-12.
  C2 (acceptance.cpp:97-122): CholeskyQR / CholeskyQR2 break down for kappa >= 1e10,
      are ok for kappa <= 1e6, CholeskyQR's orth at kappa = 1e4 lies in [1e-10, 1e-6].
  C8 (acceptance.cpp:293-345), one-device part: the communication table at
      p = 2, 4, 8 through the factorization report, and the partition independence
      of the triangular solve and (the rank-count-independent) Gram at m = 2e5, n = 50.
      The multi-rank factorization itself is tests/test_gpu_multirank.py.
  C9 (acceptance.cpp:348-368): runtime order rQR <= CholeskyQR2 <= sCholeskyQR3 at
      m = 1e6, n = 100 (device stage clocks, median of 5).

Inputs follow run_accuracy (experiments.cpp:84-96): A = U diag(sigma) V^T from the
matrix seed (generated on the device, matgen.cpp:21-46), sketch seed
derive(seed, 0x5E7C), the bench's fixed shift 1e-15 (experiments.hpp:52).
Orthogonality and residual are the device diagnostics (diagnostics.cpp:10-28;
tests/test_gpu_diagnostics.py pins them against the oracle).
"""
import statistics

import numpy as np
import pytest

from paper_2111_11148_b200 import _abi
from paper_2111_11148_b200 import cholqr as G

pytestmark = pytest.mark.gpu
KAPPAS = [10.0 ** e for e in range(3, 16)]  # acceptance.cpp:60-64
FIXED = G.ShiftMode.fixed(1e-15)


def run(method, a, seed, shift=None, rate=2.0):
    """run_accuracy's measure (experiments.cpp:14-43): status, orth, res."""
    cfg = G.SketchConfig(rate=rate, seed=G.derive(seed, 0x5E7C))
    opts = G._opts(G.Options(), shift or FIXED)
    try:
        f, timing, _ = G._factor(method, a, cfg, opts)
    except G.CholeskyBreakdown:
        return "breakdown", None, None, None
    except G.SingularTriangular:
        return "singular", None, None, None
    return "ok", G.orthogonality_error_dev(f.q), G.residual_error_dev(a, f.q, f.r), timing


@pytest.fixture(scope="module")
def mats():
    cache = {}

    def get(m, n, kappa, seed):
        key = (m, n, kappa, seed)
        if key not in cache:
            cache.clear()
            cache[key] = G.synthesize_dev(m, n, kappa, seed)
        return cache[key]

    return get


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1_randomized_and_shifted_are_stable(seed, mats):
    worst = {}
    for kappa in KAPPAS:
        a = mats(100_000, 100, kappa, seed)
        for method in (_abi.RQR, _abi.RLU, _abi.SCHOLQR3):
            st, orth, res, _ = run(method, a, seed)
            tag = f"{_abi.METHOD_NAMES[method]} kappa={kappa:.0e} seed={seed}"
            assert st == "ok", tag
            assert orth <= 1e-11, (tag, orth)
            assert res <= 1e-12, (tag, res)
            w = worst.setdefault(method, [0.0, 0.0])
            w[0], w[1] = max(w[0], orth), max(w[1], res)
    print({_abi.METHOD_NAMES[k]: v for k, v in worst.items()})


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c2_breakdown_band(seed, mats):
    for kappa in KAPPAS:
        a = mats(100_000, 100, kappa, seed)
        for method in (_abi.CHOLQR, _abi.CHOLQR2):
            st, orth, _, _ = run(method, a, seed, shift=G.ShiftMode.theory())
            tag = f"{_abi.METHOD_NAMES[method]} kappa={kappa:.0e} seed={seed}"
            if kappa >= 1e10:
                assert st == "breakdown", tag
            if kappa <= 1e6:
                assert st == "ok", tag
            if method == _abi.CHOLQR and kappa == 1e4 and st == "ok":
                assert 1e-10 <= orth <= 1e-6, (tag, orth)


def test_c8_comm_table_and_partition_independence():
    import torch

    m, n = 200_000, 50
    a = G.synthesize_dev(m, n, 1e5, 1)
    l = G.SketchConfig(seed=2).resolved_size(m, n)
    for method in (_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3, _abi.RLU, _abi.RQR):
        q1 = None
        for p in (1, 2, 4, 8):
            run_p = G.run_parallel(method, a, p, G.MethodConfig(sketch=G.SketchConfig(seed=2), shift=FIXED))
            qp = run_p.factorization.q
            if q1 is None:
                q1 = qp.clone()
            else:
                assert torch.equal(qp, q1)  # the device result does not depend on the simulated p
            if p > 1:
                pn2 = p * n * n
                lo, hi = {_abi.CHOLQR: (pn2, pn2), _abi.CHOLQR2: (2 * pn2, 2 * pn2),
                          _abi.SCHOLQR3: (3 * pn2, 3 * pn2)}.get(method, (1.5 * pn2, 1.5 * pn2 + n * l))
                assert run_p.timing.comm_volume == hi
                assert G.comm_model(method, p, n, l)[2:] == (lo, hi)
    # the C-ABI report itself carries the model of opts.workers (parexec.cpp:64-75)
    _, _, rep = G._factor(_abi.CHOLQR2, a, None, _abi.options(workers=4))
    assert rep.comm_rounds == 4 and rep.comm_volume == 2 * 4 * n * n
    # parallel_trisolve (acceptance.cpp:329-340): row blocks solved separately are bitwise the whole
    r = torch.as_tensor(np.triu(np.random.default_rng(3).standard_normal((n, n))) + 4 * np.eye(n), device="cuda")
    x1 = G.right_trisolve(a, r)
    for p in (2, 4, 8):
        xp = torch.cat([G.right_trisolve(a[G.block_offset(m, p, b):G.block_offset(m, p, b + 1)].contiguous(), r)
                        for b in range(p)])
        assert torch.equal(xp, x1)
    # the Gram of p ranks (the rank-count-independent protocol) is bitwise the one-device Gram
    g1 = G.gram(a)
    for p in (2, 4, 8):
        assert torch.equal(G.gram_sharded_sim(a, p), g1)


def test_c9_runtime_order():
    m, n = 1_000_000, 100
    a = G.synthesize_dev(m, n, 1e5, 1)
    t = {k: [] for k in (_abi.RQR, _abi.CHOLQR2, _abi.SCHOLQR3)}
    for rnd in range(6):
        for method in t:
            cfg = G.SketchConfig(seed=10 + rnd)
            _, timing, _ = G._factor(method, a, cfg, G._opts(G.Options(), FIXED))
            if rnd:
                t[method].append(timing.total_ms)
    med = {k: statistics.median(v) for k, v in t.items()}
    print({_abi.METHOD_NAMES[k]: round(v, 3) for k, v in med.items()})
    assert med[_abi.RQR] <= med[_abi.CHOLQR2] <= med[_abi.SCHOLQR3]
