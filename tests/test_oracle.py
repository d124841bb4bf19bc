"""Pins the CPU oracle (oracle/) against the reference's own assertions.

Each test names the reference test it replays (proj/tests/*.cpp file:line).
The reference cannot be built here (Eigen/doctest absent), so these
known-answer and property checks, the golden RNG vectors
(tests/golden/rng_golden.json, independent pure-Python restatement) and
numpy/LAPACK cross-checks are what pin the oracle.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as o
from paper_2111_11148_b200 import _abi

U = np.finfo(np.float64).eps


def fma(a, b, c):
    # exactly rounded fused multiply-add (math.fma is Python >= 3.13 only)
    return float(Fraction(a) * Fraction(b) + Fraction(c))


GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")


def spectral_norm(a):
    return o.svd_values(a)[0]


def uniform_cfg(l, seed):
    return _abi.sketch_cfg(size=l, seed=seed)


def check_contract(a, f, res_tol=1e-12):  # test_cholqr.cpp:26-33
    assert f.q.shape == a.shape
    assert f.r.shape == (a.shape[1], a.shape[1])
    assert np.all(np.diag(f.r) > 0)
    assert np.linalg.norm(np.tril(f.r, -1)) == 0.0
    assert o.residual_error(a, f.q, f.r) <= res_tol


# ---------------- rng: golden vectors --------------------------------------
def test_rng_golden_vectors():
    g = json.load(open(GOLDEN))
    for s in g["seeds"]:
        seed = int(s)
        for k, v in g["bits"][s]:
            assert o.bits_at(seed, int(k)) == int(v)
        for k, v in g["gauss"][s]:
            assert o.gaussian_at(seed, int(k)) == float.fromhex(v)
        assert list(o.stream_indices(seed, 1000003, 32)) == g["indices"][s]
    for s, salt, v in g["derive"]:
        assert o.derive(int(s), int(salt)) == int(v)


def test_rng_fill_matches_scalar():
    seed = 77
    b = o.bits_fill(seed, 10, 50)
    assert all(int(b[i]) == o.bits_at(seed, 10 + i) for i in range(50))
    gm = o.gaussian_matrix(7, 9, seed)
    for i in range(7):
        for j in range(9):
            assert gm[i, j] == o.gaussian_at(seed, i * 9 + j)


# ---------------- kernels (test_kernels.cpp) --------------------------------
def test_gram_known_answers():  # :41-50
    assert np.linalg.norm(o.gram(np.eye(3)) - np.eye(3)) == 0.0
    g = o.gram(np.array([[1.0], [2.0], [2.0]]))
    assert g.shape == (1, 1) and g[0, 0] == 9.0


@pytest.mark.parametrize("m,n,seed", [(50, 10, 7), (2500, 6, 11)])
def test_gram_vs_extended_precision(m, n, seed):  # :52-69
    a = o.gaussian_matrix(m, n, seed)
    g = o.gram(a)
    ref = np.array([[math.fsum(a[:, i] * a[:, j]) for j in range(n)] for i in range(n)])
    s = spectral_norm(a)
    assert np.abs(g - ref).max() <= 1e-13 * s * s
    assert np.abs(g - g.T).max() == 0.0


def test_gram_tree_equals_stack_fold():
    # the streaming binary-counter + right-fold form used on the GPU equals the
    # level-by-level pairwise tree of kernels.hpp:42-57, bitwise, for every count
    rng = np.random.default_rng(3)
    for cnt in list(range(1, 70)) + [977, 1024, 1025, 4097]:
        slots = rng.standard_normal((cnt, 5)) * 10.0 ** rng.integers(-8, 8, size=(cnt, 1))
        assert np.array_equal(o.tree_combine(slots), o.stack_combine(slots)), cnt


def test_gram_worker_independent():  # test_parexec.cpp:41-56
    a = o.gaussian_matrix(5000, 10, 3)
    g1 = o.gram(a, 1)
    for p in (2, 4, 7):
        assert np.array_equal(o.gram(a, p), g1)


def test_cholesky_known_answers():  # :71-80
    assert np.linalg.norm(o.cholesky_upper(np.eye(4)) - np.eye(4)) == 0.0
    r = o.cholesky_upper(np.array([[4.0, 2.0], [2.0, 2.0]]))
    assert np.array_equal(r, np.array([[2.0, 1.0], [0.0, 1.0]]))


def test_cholesky_residual():  # :82-88
    a = o.gaussian_matrix(200, 30, 3)
    g = o.gram(a)
    r = o.cholesky_upper(g)
    assert np.linalg.norm(r.T @ r - g) <= 50.0 * 30 * U * np.linalg.norm(g)
    assert np.all(np.diag(r) > 0)
    assert np.allclose(r, np.linalg.cholesky(g).T, rtol=1e-12, atol=1e-12 * np.abs(r).max())


def test_cholesky_breakdown():  # :90-93
    a = o.synthesize(1000, 20, 1e10, 42)
    with pytest.raises(o.OracleError) as e:
        o.cholesky_upper(o.gram(a))
    assert e.value.status == _abi.CHOLESKY_BREAKDOWN and e.value.index >= 0


def test_trisolve_known_answers():  # :95-110
    a = o.gaussian_matrix(30, 5, 1)
    assert np.linalg.norm(o.right_trisolve(a, np.eye(5)) - a) == 0.0
    x = o.right_trisolve(np.array([[2.0, 3.0]]), np.array([[2.0, 1.0], [0.0, 1.0]]))
    assert abs(x[0, 0] - 1.0) <= 1e-15 and abs(x[0, 1] - 2.0) <= 1e-15
    big = o.gaussian_matrix(100, 8, 5)
    rr = o.qr_r_factor(o.gaussian_matrix(40, 8, 6))
    xx = o.right_trisolve(big, rr)
    assert np.linalg.norm(xx @ rr - big) <= 1e-13 * np.linalg.norm(big)


def test_trisolve_round_trip_bound():  # :112-119
    a = o.gaussian_matrix(300, 12, 9)
    r = o.qr_r_factor(o.gaussian_matrix(60, 12, 10))
    x = o.right_trisolve(a, r)
    sv = o.svd_values(r)
    assert np.linalg.norm(x @ r - a) <= 100.0 * 12 * U * (sv[0] / sv[-1]) * np.linalg.norm(a)


def test_trisolve_zero_diagonal():  # :121-126
    r = np.eye(3)
    r[1, 1] = 0.0
    with pytest.raises(o.OracleError) as e:
        o.right_trisolve(o.gaussian_matrix(4, 3, 2), r)
    assert e.value.status == _abi.SINGULAR_TRIANGULAR and e.value.index == 1


def test_trisolve_partition_independent():  # test_parexec.cpp:67-89
    a = o.gaussian_matrix(2000, 9, 5)
    r = o.qr_r_factor(o.gaussian_matrix(50, 9, 6))
    x1 = o.right_trisolve(a, r, 1)
    for p in (2, 8):
        assert np.array_equal(o.right_trisolve(a, r, p), x1)
    # the exact recurrence equals a plain per-row fma loop
    n = 9
    xr = a[:3].copy()
    for i in range(3):
        for j in range(n):
            y = xr[i, j]
            for k in range(j):
                if r[k, j] != 0.0:
                    y = fma(-r[k, j], xr[i, k], y)
            xr[i, j] = y / r[j, j]
    assert np.array_equal(xr, x1[:3])


def test_qr_r_factor():  # :128-152
    q = o.random_orthogonal(6, 6, 3)
    assert np.linalg.norm(o.qr_r_factor(q) - np.eye(6)) <= 1e-14 * 6
    assert abs(o.qr_r_factor(np.array([[3.0], [4.0]]))[0, 0] - 5.0) <= 5e-15
    a1 = o.gaussian_matrix(40, 10, 8)
    r = o.qr_r_factor(a1)
    s = spectral_norm(a1)
    assert np.abs(r.T @ r - a1.T @ a1).max() <= 1e-12 * s * s
    assert np.all(np.diag(r) >= 0) and np.linalg.norm(np.tril(r, -1)) == 0.0
    # LAPACK cross-check (same unique positive-diagonal factor)
    rl = np.linalg.qr(a1, mode="r")
    rl = rl * np.sign(np.diag(rl))[:, None]
    assert np.abs(r - rl).max() <= 1e-13 * s
    a2 = o.synthesize(80, 12, 1e3, 17)
    assert np.abs(o.qr_r_factor(a2) - o.cholesky_upper(o.gram(a2))).max() <= 1e-8


def test_lu_known_answers():  # :154-163, :179-183
    assert np.linalg.norm(o.lu_u_factor(np.eye(4)) - np.eye(4)) == 0.0
    u = o.lu_u_factor(np.array([[2.0, 1.0], [4.0, 3.0]]))
    assert np.array_equal(u, np.array([[4.0, 3.0], [0.0, -0.5]]))
    z = np.zeros((4, 2))
    z[:, 0] = 1.0
    with pytest.raises(o.OracleError) as e:
        o.lu_u_factor(z)
    assert e.value.status == _abi.SINGULAR_TRIANGULAR


def test_lu_reconstruction():  # :165-177
    a1 = o.gaussian_matrix(30, 10, 12)
    packed, perm = o.lu_decompose(a1)
    l, n = a1.shape
    low = np.tril(packed, -1)[:, :n].copy()
    low[:n] += np.eye(n)
    u = np.triu(packed[:n])
    assert np.linalg.norm(a1[perm] - low @ u) <= 1e-12 * np.linalg.norm(a1)
    # same pivots as LAPACK's partial pivoting on this input
    import scipy.linalg as sl
    p_, l_, u_ = sl.lu(a1)
    assert np.abs(np.abs(u) - np.abs(u_[:n])).max() <= 1e-12 * np.abs(u).max()


def test_svd_values():  # :185-219
    sv = o.svd_values(np.diag([3.0, 1.0]))
    assert abs(sv[0] - 3) <= 1e-15 * 3 and abs(sv[1] - 1) <= 1e-15
    a = o.synthesize(1000, 20, 1e5, 4)
    sv = o.svd_values(a)
    assert abs(sv[0] / sv[19] / 1e5 - 1) <= 1e-8
    tall = o.gaussian_matrix(9, 4, 30)
    assert np.abs(o.svd_values(tall) - o.svd_values(tall.T)).max() <= 1e-13 * o.svd_values(tall)[0]


# ---------------- sketch (test_sketch.cpp) ----------------------------------
def test_uniform_replay():  # :18-33
    a = o.gaussian_matrix(5, 2, 1)
    a1, idx = o.sample_rows_uniform(a, 5, 42)
    assert list(idx) == list(o.stream_indices(42, 5, 5))
    assert np.all((idx >= 0) & (idx < 5))
    assert np.array_equal(a1, a[idx])


def test_uniform_deterministic_and_without_replacement():  # :35-45, :66-76
    a = o.gaussian_matrix(1000, 10, 2)
    a1, i1 = o.sample_rows_uniform(a, 20, 7)
    a2, i2 = o.sample_rows_uniform(a, 20, 7)
    assert np.array_equal(i1, i2) and np.array_equal(a1, a2)
    _, idx = o.sample_rows_uniform(o.gaussian_matrix(30, 3, 5), 30, 9, without_replacement=True)
    assert sorted(idx) == list(range(30))


def test_uniform_chi2():  # :47-64
    counts = np.bincount(o.stream_indices(11, 50, 50000), minlength=50)
    exp = 50000 / 50
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 <= 49.0 + 3.0 * math.sqrt(98.0)


def test_gaussian_sketch_zero_and_repro():  # :118-132
    assert np.abs(o.sketch_gaussian(np.zeros((60, 4)), 8, 21)).max() == 0.0
    a = o.gaussian_matrix(60, 4, 22)
    assert np.array_equal(o.sketch_gaussian(a, 8, 21), o.sketch_gaussian(a, 8, 21))


def test_gaussian_sketch_is_omega_times_a():
    # Omega(i, j) = gaussian_at(seed, i*m + j) (sketch.cpp:112); 2048-column chunks
    m, n, l, seed = 5000, 7, 9, 1234
    a = o.gaussian_matrix(m, n, 5)
    om = o.gaussian_fill(seed, 0, l * m).reshape(l, m)
    ref = om @ a
    got = o.sketch_gaussian(a, l, seed)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_gaussian_sketch_expectation():  # :134-148
    a = o.gaussian_matrix(50, 5, 30)
    target = 10.0 * (a.T @ a)
    mean = np.zeros((5, 5))
    for t in range(2000):
        a1 = o.sketch_gaussian(a, 10, o.derive(100, t))
        mean += a1.T @ a1
    mean /= 2000
    assert np.linalg.norm(mean - target) <= 0.05 * np.linalg.norm(target)


def test_resolved_size():  # :170-177
    c = _abi.sketch_cfg(rate=0.5)
    assert o.resolved_size(c, 100, 10) == 10
    c.rate = 50.0
    assert o.resolved_size(c, 100, 10) == 100
    c.size = 20
    assert o.resolved_size(c, 100, 10) == 20


# ---------------- algorithms (test_cholqr.cpp) -------------------------------
def test_cholqr_fixed_point():  # :37-43
    a = o.random_orthogonal(200, 12, 1)
    f = o.factor(_abi.CHOLQR, a)
    assert np.linalg.norm(f.q - a) <= 1e-13 and np.linalg.norm(f.r - np.eye(12)) <= 1e-13
    check_contract(a, f)


def test_cholqr_kappa2u_and_breakdown():  # :45-55
    a = o.synthesize(10000, 50, 1e3, 2)
    f = o.factor(_abi.CHOLQR, a)
    assert o.orthogonality_error(f.q) <= 1e-9
    check_contract(a, f)
    with pytest.raises(o.OracleError) as e:
        o.factor(_abi.CHOLQR, o.synthesize(2000, 20, 1e10, 3))
    assert e.value.status == _abi.CHOLESKY_BREAKDOWN


def test_cholqr2():  # :57-74
    q0 = o.random_orthogonal(300, 10, 4)
    f0 = o.factor(_abi.CHOLQR2, q0)
    assert np.linalg.norm(f0.q - q0) <= 1e-13 and np.linalg.norm(f0.r - np.eye(10)) <= 1e-12
    m, n = 20000, 50
    a = o.synthesize(m, n, 1e5, 5)
    f = o.factor(_abi.CHOLQR2, a)
    assert o.orthogonality_error(f.q) <= 6.0 * (m + n + 1) * n * U
    check_contract(a, f)
    with pytest.raises(o.OracleError) as e:
        o.factor(_abi.CHOLQR2, o.synthesize(2000, 20, 1e12, 6))
    assert e.value.status == _abi.CHOLESKY_BREAKDOWN


def test_scholqr3():  # :76-101
    fixed = _abi.options(shift_kind=_abi.SHIFT_FIXED, shift_value=1e-15)
    q0 = o.random_orthogonal(300, 10, 7)
    assert o.orthogonality_error(o.factor(_abi.SCHOLQR3, q0, opts=fixed).q) <= 1e-13
    a = o.synthesize(20000, 50, 1e12, 8)
    f = o.factor(_abi.SCHOLQR3, a, opts=fixed)
    assert o.orthogonality_error(f.q) <= 1e-12
    check_contract(a, f)
    shifts = [s for s in f.stages if s.has_shift]
    assert shifts and shifts[0].shift == 1e-15
    a = o.synthesize(10000, 50, 1e5, 9)
    ef = o.orthogonality_error(o.factor(_abi.SCHOLQR3, a, opts=fixed).q)
    et = o.orthogonality_error(o.factor(_abi.SCHOLQR3, a, opts=_abi.options()).q)
    assert et <= 10 * ef and ef <= 10 * et


def test_precond_exact_and_identity():  # :103-121
    a = o.synthesize(500, 20, 1e4, 10)
    cfg = _abi.sketch_cfg(size=500, seed=11, without_replacement=True)
    f = o.precond_factor(a, o.qr_r_factor, cfg)
    assert o.orthogonality_error(f.q) <= 1e-13
    check_contract(a, f)
    a = o.synthesize(400, 10, 1e2, 12)
    base = o.factor(_abi.CHOLQR, a)
    f = o.precond_factor(a, lambda a1: np.eye(a1.shape[1]), uniform_cfg(20, 13))
    assert np.array_equal(f.q, base.q) and np.array_equal(f.r, base.r)


def test_rqr_rlu_orthogonal_inputs():  # :123-134
    a = o.random_orthogonal(400, 16, 14)
    assert np.linalg.norm(o.factor(_abi.RQR, a, uniform_cfg(32, 15)).q - a) <= 1e-13
    a = o.random_orthogonal(400, 16, 16)
    f = o.factor(_abi.RLU, a, uniform_cfg(32, 17))
    assert o.orthogonality_error(f.q) <= 1e-12
    check_contract(a, f, 1e-13)


@pytest.mark.parametrize("kappa,seed", [(1e12, 18), (1e15, 21)])
def test_randomized_ill_conditioned(kappa, seed):  # :136-152
    a = o.synthesize(20000, 50, kappa, seed)
    if kappa == 1e12:
        with pytest.raises(o.OracleError):
            o.factor(_abi.CHOLQR2, a)
    for meth, s in ((_abi.RQR, seed + 1), (_abi.RLU, seed + 2)):
        f = o.factor(meth, a, uniform_cfg(100, s))
        assert o.orthogonality_error(f.q) <= 1e-11
        check_contract(a, f)


def test_rqr_cond_x_modest():  # :154-171
    small = 0
    for t in range(100):
        a = o.synthesize(2000, 40, 1e5, 3000 + t)
        f = o.factor(_abi.RQR, a, uniform_cfg(80, 4000 + t), _abi.options(diagnostics=True))
        conds = [s.cond_x for s in f.stages if s.has_cond_x]
        assert conds
        small += conds[0] <= 100.0
    assert small >= 95


def test_scale_invariance_and_determinism():  # :191-209
    a = o.synthesize(600, 12, 1e6, 23)
    f1 = o.factor(_abi.RQR, a, uniform_cfg(24, 24))
    f2 = o.factor(_abi.RQR, 1024.0 * a, uniform_cfg(24, 24))
    assert np.array_equal(f1.q, f2.q) and np.array_equal(f2.r, 1024.0 * f1.r)
    a = o.synthesize(500, 15, 1e8, 25)
    g1 = o.factor(_abi.RLU, a, uniform_cfg(30, 26))
    g2 = o.factor(_abi.RLU, a, uniform_cfg(30, 26))
    assert np.array_equal(g1.q, g2.q) and np.array_equal(g1.r, g2.r)


def test_retry_on_degenerate_draw():  # :211-234
    a = np.eye(2)
    exercised = False
    for seed in range(256):
        _, idx = o.sample_rows_uniform(a, 2, seed)
        if idx[0] != idx[1]:
            continue
        try:
            f = o.factor(_abi.RQR, a, uniform_cfg(2, seed))
        except o.OracleError:
            continue
        assert f.stages[0].retries >= 1
        assert o.orthogonality_error(f.q) <= 1e-12
        exercised = True
        break
    assert exercised


def test_r_less():  # :236-244
    a = o.synthesize(300, 10, 1e4, 27)
    f = o.factor(_abi.RQR, a, uniform_cfg(20, 28), _abi.options(r_less=True))
    assert f.r is None and f.report.r_less == 1
    assert o.orthogonality_error(f.q) <= 1e-12


def test_gaussian_variant():  # :246-256
    a = o.synthesize(800, 16, 1e10, 29)
    cfg = _abi.sketch_cfg(strategy=_abi.GAUSSIAN, size=48, seed=30)
    f = o.precond_factor(a, o.qr_r_factor, cfg)
    assert o.orthogonality_error(f.q) <= 1e-11
    check_contract(a, f)
    g = o.factor(_abi.RQR_GAUSSIAN, a, cfg)
    assert np.array_equal(g.q, f.q)


def test_non_finite_rejected():  # :258-262
    a = np.ones((8, 2))
    a[3, 1] = np.nan
    with pytest.raises(o.OracleError) as e:
        o.factor(_abi.CHOLQR, a)
    assert e.value.status == _abi.INVALID_ARGUMENT


# ---------------- parexec (test_parexec.cpp) --------------------------------
def test_partition_offsets():  # :14-39
    assert [o.block_offset(10, 3, b) for b in range(4)] == [0, 4, 7, 10]
    for t in range(20):
        m, p = 3 + (t * 37) % 200, 1 + t % 7
        if p > m:
            continue
        sizes = [o.block_offset(m, p, b + 1) - o.block_offset(m, p, b) for b in range(p)]
        assert sum(sizes) == m and max(sizes) - min(sizes) <= 1


def test_run_parallel_p_consistent():  # :91-126
    a = o.synthesize(4000, 24, 1e5, 9)
    fixed = _abi.options(shift_kind=_abi.SHIFT_FIXED, shift_value=1e-15)
    for meth in (_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3, _abi.RLU, _abi.RQR):
        q1 = o.factor(meth, a, _abi.sketch_cfg(seed=10), fixed, workers=1).q
        for p in (2, 4, 8):
            qp = o.factor(meth, a, _abi.sketch_cfg(seed=10), fixed, workers=p).q
            assert np.array_equal(qp, q1)


def test_comm_model():  # :128-154
    p, n, l = 16, 100, 200
    pn2 = 16.0 * 100 * 100
    assert o.comm_model(_abi.CHOLQR, p, n, l) == (2, 2, pn2, pn2)
    assert o.comm_model(_abi.CHOLQR2, p, n, l)[1::2] == (4, 2 * pn2)
    assert o.comm_model(_abi.SCHOLQR3, p, n, l)[1::2] == (6, 3 * pn2)
    for m in (_abi.RLU, _abi.RQR):
        assert o.comm_model(m, p, n, l) == (3, 4, 1.5 * pn2, 1.5 * pn2 + 100.0 * 200.0)


def test_diagnostics_known_answer():  # test_diagnostics.cpp:28-31
    assert abs(o.orthogonality_error(2.0 * np.eye(3)) - 3.0 * math.sqrt(3.0)) <= 1e-14


def test_matgen():  # test_matgen.cpp:17-51
    assert abs(abs(o.random_orthogonal(1, 1, 5)[0, 0]) - 1.0) <= 1e-15
    q = o.random_orthogonal(100, 10, 3)
    assert o.orthogonality_error(q) <= 1e-13
    assert np.linalg.norm(q - o.random_orthogonal(100, 10, 4)) > 1e-3
    a = o.synthesize(1000, 20, 1e5, 11)
    sv = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(sv, 1e5 ** (-np.arange(20) / 19.0), rtol=1e-8)
    assert np.array_equal(o.synthesize(200, 10, 1e3, 77), o.synthesize(200, 10, 1e3, 77))
    assert np.linalg.norm(o.embedded_identity(6, 6) - np.eye(6)) == 0.0
