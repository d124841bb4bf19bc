"""Parity of the B200 path (through the C-ABI, libcqr.so) against the CPU oracle.

Bitwise where the oracle pins the operation order and the device follows it:
RNG integers, uniform row extraction, Gram (leaf tree), Cholesky, trisolve,
LU, triangular product -> CholeskyQR/CholeskyQR2/sCholeskyQR3 and rLU with the
uniform sketch are bit-identical to the oracle end to end (up to the sign of
zero, which numpy's == ignores). Tolerance where it cannot be: the Box-Muller
transcendentals (CUDA libm vs glibc, <= a few ulp), and therefore the Gaussian
sketch and everything downstream of it, and the Householder R of rQR (tree
reductions). Tolerances are written next to each assertion.
"""
import json
import math
import os

import ctypes as C
import numpy as np
import pytest

from oracle import oracle as o
from paper_2111_11148_b200 import _abi
from paper_2111_11148_b200 import cholqr as G
from paper_2111_11148_b200 import dist

pytestmark = pytest.mark.gpu
U = np.finfo(np.float64).eps
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert os.path.exists(G.LIB_PATH), "libcqr.so not built"
    yield


def uni(l, seed):
    return G.SketchConfig(size=l, seed=seed)


def relf(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------- rng ---------------------------------------------------------------
def test_rng_bits_bitwise_golden():
    g = json.load(open(GOLDEN))
    for s in g["seeds"]:
        seed = int(s)
        ks = [int(k) for k, _ in g["bits"][s]]
        for k, v in g["bits"][s]:
            assert int(G.rng_bits(seed, int(k), 1)[0]) == int(v)
        b = G.rng_bits(seed, 0, 4096)
        assert np.array_equal(b, o.bits_fill(seed, 0, 4096))
        del ks


def test_rng_gaussian_within_ulps():
    for seed in (0, 1, 42, o.derive(1, 0x5E7C)):
        n = 200000
        gd = G.rng_gaussian(seed, 12345, n)
        go = o.gaussian_fill(seed, 12345, n)
        # table Box-Muller vs glibc: |diff| <= 16 ulp of max(|g|, 1) (1e7 draws: max 12.5, the
        # absolute error of cos/sin near their zeros times r <= 8.6; tools/gpu/bm_acc.py)
        tol = 16 * U * np.maximum(np.abs(go), 1.0)
        assert np.all(np.abs(gd - go) <= tol)
        assert np.mean(gd == go) > 0.5  # most draws are bit-identical


def _box_muller_edge_bits():
    """Counter bits that put u1 and u2 on the edges of the draw's table reduction."""
    rng = np.random.default_rng(5)
    n1 = [2**53 - j for j in range(256)] + list(range(1, 257))
    for k in range(1, 54):  # exponent boundaries of u1
        n1 += [2**k - 1, 2**k, min(2**k + 1, 2**53)]
    for e in (0, 1, 5, 30, 52):  # table rounding points and the sqrt(2) split, mantissa-relative
        base = 2**e
        for t in list(range(0, 257, 7)) + [212, 213, 214]:
            c = base + (t * base) // 512
            n1 += [max(1, c - 1), c, c + 1]
    n1 += [int(v) for v in rng.integers(1, 2**53, 4000, dtype=np.int64)]
    n2 = [0, 1, 2, 2**53 - 1, 2**53 - 2]
    for k in range(0, 257):  # table points of a, incl. the quadrant boundaries
        c = k * 2**45
        n2 += [v for v in (c - 2**44, c - 1, c, c + 1, c + 2**44 - 1) if 0 <= v < 2**53]
    n2 = np.array(n2 + [int(v) for v in rng.integers(0, 2**53, 4000 - len(n2) % 4000, dtype=np.int64)], dtype=np.uint64)
    n1 = np.array([min(max(v, 1), 2**53) for v in n1], dtype=np.uint64)
    npairs = max(len(n1), len(n2))
    n1 = np.resize(n1, npairs)
    n2 = np.resize(rng.permutation(n2), npairs)
    low = rng.integers(0, 2**11, (2, npairs), dtype=np.uint64)
    bits = np.empty(2 * npairs, dtype=np.uint64)
    bits[0::2] = ((n1 - np.uint64(1)) << np.uint64(11)) | low[0]
    bits[1::2] = (n2 << np.uint64(11)) | low[1]
    return bits


def test_box_muller_edge_bits():
    import math
    bits = _box_muller_edge_bits()
    got = G.box_muller_bits(bits)
    worst_abs = worst_rad = 0.0
    for i in range(bits.size // 2):
        u1 = float((int(bits[2 * i]) >> 11) + 1) * 2.0**-53
        u2 = float(int(bits[2 * i + 1]) >> 11) * 2.0**-53
        r = math.sqrt(-2.0 * math.log(u1))
        a = 2.0 * math.pi * u2
        ref = (r * math.cos(a), r * math.sin(a))  # rng.hpp:52-54 with glibc, as the oracle
        for g, gr in zip(got[2 * i:2 * i + 2], ref):
            worst_abs = max(worst_abs, abs(g - gr) / (U * max(abs(gr), 1.0)))
        if r > 0:  # the radius keeps full relative accuracy, also for u1 -> 1 (tiny r)
            worst_rad = max(worst_rad, abs(math.hypot(*got[2 * i:2 * i + 2]) - r) / (U * r))
        else:
            assert got[2 * i] == 0.0 and got[2 * i + 1] == 0.0
    assert worst_abs <= 16, worst_abs
    assert worst_rad <= 8, worst_rad


# ---------------- kernels -------------------------------------------------------------
@pytest.mark.parametrize("m,n,seed", [(3, 3, 0), (50, 10, 7), (2500, 6, 11), (3000, 12, 2), (5000, 64, 3),
                                      (4113, 128, 4), (2048, 1, 5), (20000, 33, 6), (9000, 200, 7),
                                      (3000, 300, 8), (33 * 1024 + 5, 16, 9), (70000, 64, 10), (16 * 1024, 24, 11),
                                      # n in (64, 128] past one wave of leaves: the last wave split over 3 CTAs
                                      (200_000, 128, 12), (1_000_003, 72, 13)])
def test_gram_bitwise(m, n, seed):
    a = o.gaussian_matrix(m, n, seed)
    g = G.gram(a)
    assert np.array_equal(g, o.gram(a))
    assert np.array_equal(g, g.T)


@pytest.mark.parametrize("m,n,p,ld", [(5003, 12, 3, 12), (3000, 6, 8, 6), (100_000, 128, 8, 128),
                                      (1_000_003, 64, 7, 64), (50_000, 256, 5, 256), (20000, 33, 4, 40),
                                      (9000, 200, 2, 200), (2048, 16, 2, 16), (300_000, 128, 3, 130)])
def test_sharded_gram_sim_bitwise_for_any_p(m, n, p, ld):
    # the multi-rank Gram protocol (head/tail chains across block boundaries, owned
    # tree nodes, all-gathered top of the tree) run rank by rank on this device:
    # bit-identical to the one-GPU Gram and to the oracle for every p, as the
    # reference's parallel Gram is (test_parexec.cpp:47-56)
    import torch

    full = torch.as_tensor(o.gaussian_matrix(m, ld, 40 + p), device="cuda")
    x = full[:, :n]
    one = G.gram(x)
    for q in sorted({1, 2, p}):
        assert torch.equal(G.gram_sharded_sim(x, q), one), q
    # the hand-offs through NCCL itself (send/recv to self, all-gather) on a one-rank communicator
    coll = G.Context(0)
    coll.attach_comm(0, 1, G.make_comm_id())
    assert torch.equal(G.gram_sharded_sim(x, p, ctx=coll), one)
    if m * n <= 2e7:
        assert np.array_equal(one.cpu().numpy(), o.gram(x.cpu().numpy()))


def test_gram_known_answers():
    assert np.array_equal(G.gram(np.eye(3)), np.eye(3))
    assert G.gram(np.array([[1.0], [2.0], [2.0]]))[0, 0] == 9.0


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (30, 3), (64, 4), (128, 5), (129, 6), (256, 7), (300, 8), (512, 9),
                                    (7, 10), (16, 11), (17, 12), (33, 13), (95, 14), (100, 15), (112, 16), (127, 17)])
def test_cholesky_bitwise(n, seed):
    a = o.gaussian_matrix(3 * n + 5, n, seed)
    g = o.gram(a)
    assert np.array_equal(G.cholesky_upper(g), o.cholesky_upper(g))


def test_cholesky_known_and_breakdown():
    assert np.array_equal(G.cholesky_upper(np.array([[4.0, 2.0], [2.0, 2.0]])), np.array([[2.0, 1.0], [0.0, 1.0]]))
    g = o.gram(o.synthesize(1000, 20, 1e10, 42))
    with pytest.raises(o.OracleError) as eo:
        o.cholesky_upper(g)
    with pytest.raises(G.CholeskyBreakdown) as eg:
        G.cholesky_upper(g)
    assert eg.value.pivot_index == eo.value.index
    # a deep breakdown index in the register-resident kernel (n <= 128) and in the blocked one
    for n in (120, 200):
        g = o.gram(o.synthesize(4000, n, 1e12, 43))
        with pytest.raises(o.OracleError) as eo:
            o.cholesky_upper(g)
        with pytest.raises(G.CholeskyBreakdown) as eg:
            G.cholesky_upper(g)
        assert eg.value.pivot_index == eo.value.index > 10


@pytest.mark.parametrize("m,n,seed", [(1, 2, 1), (30, 5, 2), (100, 8, 3), (2000, 9, 4), (3001, 24, 5),
                                      (10000, 64, 6), (4099, 128, 7), (1000, 100, 8), (700, 256, 9),
                                      (300, 300, 10), (200, 512, 11),
                                      # the 128-column panel path (GEMM update + n = 128 panel solves)
                                      (20003, 256, 12), (5003, 512, 13), (1, 384, 14), (3000, 384, 15)])
def test_trisolve_bitwise(m, n, seed):
    a = o.gaussian_matrix(m, n, seed)
    r = o.qr_r_factor(o.gaussian_matrix(2 * n + 3, n, seed + 100))
    assert np.array_equal(G.right_trisolve(a, r), o.right_trisolve(a, r))


def test_trisolve_division_is_correctly_rounded():
    # diagonal R: x = a / d elementwise, so the device's reciprocal + Markstein
    # division must equal numpy's IEEE division bit for bit
    rng = np.random.default_rng(5)
    for n in (8, 64, 128):
        a = rng.standard_normal((4096, n)) * 10.0 ** rng.integers(-30, 30, size=(4096, n))
        a[::17, 0] = 0.0
        a[::19, 1] = -0.0
        d = rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, size=n)
        d[0] = 3.0
        d[1] = -1e-310  # subnormal divisor: IEEE fallback path
        a[:, 1] *= 1e-290  # keep that column's quotients finite (inf * 0 in a DMMA tile would give NaN)
        x = G.right_trisolve(a, np.diag(d))
        ref = a / d
        assert np.array_equal(x.view(np.int64), ref.view(np.int64))


def test_trisolve_division_extreme_operands():
    # operands across the whole exponent range: the fast division's window
    # (|y| in [2^-400, 2^400], |d| in [2^-500, 2^500]) and the IEEE fallback
    # outside it, including subnormal quotients; all must match IEEE bit for bit
    rng = np.random.default_rng(11)
    for n in (16, 128):
        a = rng.standard_normal((2048, n)) * 10.0 ** rng.integers(-300, 300, size=(2048, n))
        d = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 6, size=n)
        x = G.right_trisolve(a, np.diag(d))
        ref = a / d
        assert np.isfinite(ref).all()
        assert np.array_equal(x.view(np.int64), ref.view(np.int64))
        d2 = rng.standard_normal(n) * 10.0 ** rng.integers(-160, 160, size=n)
        a2 = rng.standard_normal((2048, n)) * 10.0 ** rng.integers(-140, 140, size=(2048, n))
        ref2 = a2 / d2
        assert np.isfinite(ref2).all()
        assert np.array_equal(G.right_trisolve(a2, np.diag(d2)).view(np.int64), ref2.view(np.int64))


def test_trisolve_identity_and_singular():
    a = o.gaussian_matrix(30, 5, 1)
    assert np.array_equal(G.right_trisolve(a, np.eye(5)), a)
    r = np.eye(3)
    r[1, 1] = 0.0
    with pytest.raises(G.SingularTriangular) as e:
        G.right_trisolve(o.gaussian_matrix(4, 3, 2), r)
    assert e.value.index == 1


@pytest.mark.parametrize("l,n,seed", [(2, 2, 1), (30, 10, 2), (128, 64, 3), (256, 128, 4), (300, 150, 5),
                                      (512, 256, 6), (768, 512, 7), (1100, 40, 8),
                                      # l in (512, 1024]: panel launches + trailing launches over many SMs
                                      (600, 100, 9), (1000, 333, 10), (700, 500, 11), (513, 17, 12)])
def test_lu_bitwise(l, n, seed):
    a1 = o.gaussian_matrix(l, n, seed)
    assert np.array_equal(G.lu_u_factor(a1), o.lu_u_factor(a1))


@pytest.mark.parametrize("l,n,seed", [(64, 32, 1), (300, 100, 2), (1100, 40, 3), (96, 96, 4), (800, 200, 5),
                                      (640, 64, 6)])
def test_lu_pivot_ties(l, n, seed):
    # small integers: many equal |pivot| candidates, so the "first maximum in the
    # reference's swapped row order" rule decides; also exact zero pivots
    a1 = np.random.default_rng(seed).integers(-2, 3, size=(l, n)).astype(np.float64)
    try:
        ref = o.lu_u_factor(a1)
    except o.OracleError as e:
        with pytest.raises(G.SingularTriangular) as eg:
            G.lu_u_factor(a1)
        assert eg.value.index == e.index
        return
    assert np.array_equal(G.lu_u_factor(a1), ref)


def test_lu_known_and_singular():
    assert np.array_equal(G.lu_u_factor(np.array([[2.0, 1.0], [4.0, 3.0]])), np.array([[4.0, 3.0], [0.0, -0.5]]))
    z = np.zeros((4, 2))
    z[:, 0] = 1.0
    with pytest.raises(G.SingularTriangular):
        G.lu_u_factor(z)


@pytest.mark.parametrize("l,n,seed", [(2, 1, 1), (40, 10, 2), (128, 64, 3), (256, 128, 4), (512, 256, 5),
                                      (700, 300, 6), (1000, 100, 7), (310, 290, 8)])
def test_qr_r_tolerance(l, n, seed):
    a1 = o.gaussian_matrix(l, n, seed)
    # different reduction trees: R agrees to a small multiple of u*cond
    assert relf(G.qr_r_factor(a1), o.qr_r_factor(a1)) <= 1e-13
    assert abs(G.qr_r_factor(np.array([[3.0], [4.0]]))[0, 0] - 5.0) <= 5e-15


@pytest.mark.parametrize("m,n,l,seed", [(60, 4, 8, 21), (5000, 7, 9, 1234), (20001, 64, 128, 5),
                                        (30000, 128, 256, 6), (4000, 200, 300, 7)])
def test_sketch_gaussian_tolerance(m, n, l, seed):
    a = o.gaussian_matrix(m, n, seed + 1)
    ref = o.sketch_gaussian(a, l, seed)
    got = G.sketch_gaussian(a, G.SketchConfig(strategy=G.Strategy.Gaussian, size=l), seed).a1
    # Omega within a few ulp and a different summation tree: relative 1e-13
    assert relf(got, ref) <= 1e-13
    assert np.array_equal(got, G.sketch_gaussian(a, G.SketchConfig(strategy=G.Strategy.Gaussian, size=l),
                                                 seed).a1)  # deterministic


def test_sketch_gaussian_long_subchunks():
    """A k-chunk long enough for every sub-chunk size of the int8 kernel (16, 64, 256, then 512-step sub-chunks
    at the exactness cap, and a short last one): 4.2e6 rows over 148 one-CTA chunks, ~28k rows each."""
    m, n, l, seed = 4_200_000, 40, 80, 17
    a = o.gaussian_matrix(m, n, seed + 1)
    a[123_457, 7] = 1e3   # one large entry deep inside a chunk: its sub-chunk's exponent bound, not the others'
    ref = o.sketch_gaussian(a, l, seed)
    got = G.sketch_gaussian(a, G.SketchConfig(strategy=G.Strategy.Gaussian, size=l), seed).a1
    assert relf(got, ref) <= 1e-13


def test_uniform_gather_bitwise():
    a = o.gaussian_matrix(1000, 10, 2)
    for wr in (False, True):
        s = G.sample_rows_uniform(a, G.SketchConfig(size=20, without_replacement=wr), 7)
        a1, idx = o.sample_rows_uniform(a, 20, 7, wr)
        assert np.array_equal(s.indices, idx) and np.array_equal(s.a1, a1)


# ---------------- algorithms: bitwise families -----------------------------------------
FIXED = _abi.options(shift_kind=_abi.SHIFT_FIXED, shift_value=1e-15)


@pytest.mark.parametrize("method", [_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3])
@pytest.mark.parametrize("m,n,kappa,seed", [(400, 10, 1e2, 12), (5000, 24, 1e5, 9), (20000, 50, 1e6, 5),
                                            (10000, 128, 1e4, 3)])
def test_cholqr_family_bitwise(method, m, n, kappa, seed):
    a = o.synthesize(m, n, kappa, seed)
    ref = o.factor(method, a, opts=FIXED)
    f, _, rep = G._factor(method, a, None, FIXED)
    assert np.array_equal(f.q, ref.q) and np.array_equal(f.r, ref.r)
    assert [s.stage for s in f.report.stages] == [_abi.STAGE_NAMES[s.stage] for s in ref.stages]


@pytest.mark.parametrize("m,n,kappa,seed", [(10000, 50, 1e5, 9), (100_000, 100, 1e12, 4)])
def test_scholqr3_theory_shift_tolerance(m, n, kappa, seed):
    # The oracle resolves the theory shift from a.squaredNorm() (engine.cpp:270, cholqr.cpp:21-26);
    # the device from trace(G1) of its first Gram -- equal in exact arithmetic, so the shift agrees
    # to a few ulp and (Q, R) to rounding: a tolerance test.
    a = o.synthesize(m, n, kappa, seed)
    th = _abi.options()
    ref = o.factor(_abi.SCHOLQR3, a, opts=th)
    f, _, _ = G._factor(_abi.SCHOLQR3, a, None, th)
    sh_g = [s.shift for s in f.report.stages if s.shift is not None][0]
    sh_o = [s.shift for s in ref.stages if s.has_shift][0]
    assert abs(sh_g - sh_o) <= 1e-13 * sh_o
    assert relf(f.r, ref.r) <= 1e-12
    assert np.linalg.norm(f.q - ref.q) / math.sqrt(n) <= q_tol(kappa)
    assert o.orthogonality_error(f.q) <= max(2 * o.orthogonality_error(ref.q), 1e-11)
    assert o.residual_error(a, f.q, f.r) <= max(2 * o.residual_error(a, ref.q, ref.r), 1e-12)


def test_breakdowns_match():
    for method, kappa, seed in ((_abi.CHOLQR, 1e10, 3), (_abi.CHOLQR2, 1e12, 6)):
        a = o.synthesize(2000, 20, kappa, seed)
        with pytest.raises(o.OracleError) as eo:
            o.factor(method, a)
        with pytest.raises(G.CholeskyBreakdown) as eg:
            G._factor(method, a, None, _abi.options())
        assert eg.value.pivot_index == eo.value.index


@pytest.mark.parametrize("m,n,kappa,l,seed", [(400, 16, 1.0, 32, 17), (500, 15, 1e8, 30, 26),
                                              (20000, 50, 1e12, 100, 20), (20000, 50, 1e15, 100, 21),
                                              (100000, 64, 1e10, 128, 1),
                                              # n in (64, 128]: the solve fused with the Gram leaves
                                              (200_000, 128, 1e12, 256, 2), (5000, 100, 1e8, 200, 3),
                                              (3000, 65, 1e6, 130, 4), (160_000 + 37, 96, 1e14, 192, 5)])
def test_rlu_uniform_bitwise(m, n, kappa, l, seed):
    a = o.synthesize(m, n, kappa, seed) if kappa > 1 else o.random_orthogonal(m, n, seed)
    ref = o.factor(_abi.RLU, a, _abi.sketch_cfg(size=l, seed=seed + 1))
    f = G.rlu_cholesky_qr(a, uni(l, seed + 1))
    assert np.array_equal(f.q, ref.q) and np.array_equal(f.r, ref.r)


def test_identity_preconditioner_is_cholesky_qr():  # test_cholqr.cpp:113-121
    a = o.synthesize(400, 10, 1e2, 12)
    base = G.cholesky_qr(a)
    f = G.precond_cholesky_qr(a, lambda a1: np.eye(a1.shape[1]), uni(20, 13))
    assert np.array_equal(f.q, base.q) and np.array_equal(f.r, base.r)


# ---------------- algorithms: tolerance families -----------------------------------------
def q_tol(kappa):
    # Q is determined to O(kappa*u): 10x the oracle's seed-to-seed spread, floor 1e-10
    return max(1e-10, 0.5 * kappa * U)


@pytest.mark.parametrize("m,n,kappa,l,seed", [(400, 16, 1.0, 32, 14), (20000, 50, 1e12, 100, 18),
                                              (20000, 50, 1e15, 100, 21), (100000, 64, 1e10, 128, 2)])
def test_rqr_uniform_tolerance(m, n, kappa, l, seed):
    a = o.synthesize(m, n, kappa, seed) if kappa > 1 else o.random_orthogonal(m, n, seed)
    ref = o.factor(_abi.RQR, a, _abi.sketch_cfg(size=l, seed=seed + 1))
    f = G.rqr_cholesky_qr(a, uni(l, seed + 1))
    assert relf(f.r, ref.r) <= 1e-13
    assert np.linalg.norm(f.q - ref.q) / math.sqrt(n) <= q_tol(kappa)
    assert o.orthogonality_error(f.q) <= max(2 * o.orthogonality_error(ref.q), 1e-11)
    assert o.residual_error(a, f.q, f.r) <= max(2 * o.residual_error(a, ref.q, ref.r), 1e-12)


@pytest.mark.parametrize("method", [_abi.RQR_GAUSSIAN, _abi.RLU])
@pytest.mark.parametrize("m,n,kappa,seed", [(800, 16, 1e10, 29), (100000, 64, 1e10, 1), (50000, 128, 1e14, 2)])
def test_gaussian_sketch_methods_tolerance(method, m, n, kappa, seed):
    a = o.synthesize(m, n, kappa, seed)
    cfg = _abi.sketch_cfg(strategy=_abi.GAUSSIAN, rate=2.0, seed=o.derive(seed, 0x5E7C))
    ref = o.factor(method, a, cfg)
    f, _, _ = G._factor(method, a, G.SketchConfig(strategy=G.Strategy.Gaussian, seed=o.derive(seed, 0x5E7C)),
                        _abi.options())
    assert relf(f.r, ref.r) <= 1e-12
    assert np.linalg.norm(f.q - ref.q) / math.sqrt(n) <= q_tol(kappa)
    assert o.orthogonality_error(f.q) <= max(2 * o.orthogonality_error(ref.q), 1e-11)
    assert o.residual_error(a, f.q, f.r) <= max(2 * o.residual_error(a, ref.q, ref.r), 1e-12)


# ---------------- behaviour -------------------------------------------------------------------
def test_retry_on_degenerate_draw():  # test_cholqr.cpp:211-234
    a = np.eye(2)
    exercised = False
    for seed in range(256):
        _, idx = o.sample_rows_uniform(a, 2, seed)
        if idx[0] != idx[1]:
            continue
        try:
            ref = o.factor(_abi.RQR, a, _abi.sketch_cfg(size=2, seed=seed))
        except o.OracleError:
            with pytest.raises(G.Error):
                G.rqr_cholesky_qr(a, uni(2, seed))
            continue
        f = G.rqr_cholesky_qr(a, uni(2, seed))
        assert f.report.stages[0].retries == ref.stages[0].retries >= 1
        assert np.allclose(f.q, ref.q, atol=1e-15)
        exercised = True
        break
    assert exercised


def test_r_less_and_non_finite():
    a = o.synthesize(300, 10, 1e4, 27)
    f = G.rqr_cholesky_qr(a, uni(20, 28), G.Options(r_less=True))
    assert f.r is None and f.report.r_less
    assert o.orthogonality_error(f.q) <= 1e-12
    b = np.ones((8, 2))
    b[3, 1] = np.nan
    with pytest.raises(ValueError):
        G.cholesky_qr(b)
    # every path rejects non-finite input up front, before any breakdown (engine.cpp:222)
    c = o.synthesize(5000, 16, 1e14, 3)
    c[4321, 7] = np.inf
    for meth in (_abi.CHOLQR2, _abi.SCHOLQR3, _abi.RQR_GAUSSIAN, _abi.RLU, _abi.RQR):
        with pytest.raises(ValueError):
            G._factor(meth, c, G.SketchConfig(seed=3), _abi.options())
    # the int8 sketch's scanner warps check every sub-chunk: a NaN late in a long k-chunk
    d = o.gaussian_matrix(900_000, 24, 5)
    d[899_000, 20] = np.nan
    with pytest.raises(ValueError):
        G._factor(_abi.RQR_GAUSSIAN, d, G.SketchConfig(seed=3), _abi.options())


def test_invalid_arguments_match_reference():
    """engine.cpp:215-224 / errors.hpp:86-93: m < n, empty, p out of range and non-finite input are
    invalid arguments on every method; ragged leading dimensions are rejected at the C-ABI."""
    for shape in ((3, 5), (0, 4), (4, 0)):
        a = np.ones(shape)
        for meth in (_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3, _abi.RQR, _abi.RLU, _abi.RQR_GAUSSIAN):
            with pytest.raises(ValueError):
                G._factor(meth, a, G.SketchConfig(seed=1), _abi.options())
    a = o.synthesize(500, 8, 1e3, 5)
    for p in (0, 501):
        with pytest.raises(ValueError):
            G.run_parallel(_abi.CHOLQR2, a, p)
    # lda < n, ldq < n through the C entry point itself
    ctx = G.context()
    q = np.empty_like(a)
    r = np.empty((8, 8))
    rep = _abi.Report()
    lib = G._lib()
    cfg, opt = _abi.sketch_cfg(seed=1), _abi.options()
    for lda, ldq in ((7, 8), (8, 7)):
        st = lib.cqr_factor(ctx.h, _abi.CHOLQR, G._ptr(a), 500, 8, lda, C.byref(cfg), C.byref(opt), G._ptr(q), ldq,
                            G._ptr(r), 8, C.byref(rep))
        assert st == 3 and rep.status == 3  # CQR_INVALID_ARGUMENT
    # a valid call on the same context still works afterwards
    f = G.cholesky_qr2(a)
    assert o.orthogonality_error(f.q) <= 1e-13


def test_diagnostics_cond_x():  # test_cholqr.cpp:154-171 (20 of the 100 trials)
    small = 0
    for t in range(20):
        a = o.synthesize(2000, 40, 1e5, 3000 + t)
        f = G.rqr_cholesky_qr(a, uni(80, 4000 + t), G.Options(diagnostics=True))
        ref = o.factor(_abi.RQR, a, _abi.sketch_cfg(size=80, seed=4000 + t), _abi.options(diagnostics=True))
        c = [s.cond_x for s in f.report.stages if s.cond_x is not None][0]
        cr = [s.cond_x for s in ref.stages if s.has_cond_x][0]
        assert abs(c - cr) <= 1e-8 * cr
        small += c <= 100.0
    assert small >= 19


def test_device_tensors_match_host():
    import torch

    a = o.synthesize(20000, 64, 1e12, 3)
    cfg = G.SketchConfig(strategy=G.Strategy.Gaussian, seed=77)
    fh = G.rqr_cholesky_qr(a, cfg)
    ad = torch.as_tensor(a, device="cuda")
    fd = G.rqr_cholesky_qr(ad, cfg)
    assert np.array_equal(fd.q.cpu().numpy(), fh.q) and np.array_equal(fd.r, fh.r)
    assert G.orthogonality_error_dev(fd.q) <= 1e-12
    assert G.residual_error_dev(ad, fd.q, fd.r) <= 1e-14


def test_run_parallel_counters():
    a = o.synthesize(1000, 10, 1e3, 13)
    run = G.run_parallel(G.Method.CholeskyQr, a, 4)
    assert run.timing.comm_rounds == 2 and run.timing.comm_volume == 4.0 * 10 * 10
    assert run.timing.total_ms > 0.0


def test_launch_count_and_determinism():
    a = o.synthesize(50000, 64, 1e8, 25)
    ctx = G.context()
    before = ctx.launches
    f1 = G.rlu_cholesky_qr(a, G.SketchConfig(strategy=G.Strategy.Gaussian, seed=5))
    f2 = G.rlu_cholesky_qr(a, G.SketchConfig(strategy=G.Strategy.Gaussian, seed=5))
    assert ctx.launches - before >= 2 * 8
    assert np.array_equal(f1.q, f2.q) and np.array_equal(f1.r, f2.r)


@pytest.mark.parametrize("orth", [G.Orth.RqrCholeskyQr, G.Orth.CholeskyQr2])
def test_orthonormalize_matches_reference_caller(orth):  # apps.cpp:166-196
    y = o.synthesize(3000, 20, 1e6, 9)
    seed, calls = 77, [0, 1, 5]
    for call in calls:
        q = G.orthonormalize(y, orth, seed, call)
        if orth == G.Orth.RqrCholeskyQr:
            cfg = _abi.sketch_cfg(strategy=_abi.UNIFORM, rate=2.0, seed=o.derive(seed, 0xA110 + call))
            ref = o.factor(_abi.RQR, y, cfg, _abi.options(r_less=True)).q
            assert np.linalg.norm(q - ref) / math.sqrt(20) <= 1e-10
        else:
            ref = o.factor(_abi.CHOLQR2, y, None, _abi.options(r_less=True)).q
            assert np.array_equal(q, ref)
    # apps.cpp:171-172: householder_qr_thin(y).q, on the device
    qh = G.orthonormalize(y, G.Orth.HouseholderQr, seed, 0)
    refq = o.householder_qr_thin(y)[0]
    assert np.linalg.norm(qh - refq) / math.sqrt(20) <= 4 * 1e6 * U  # Q to O(kappa u), test_gpu_householder.py


def test_one_rank_nccl_collective_path_is_bit_identical():
    # an attached communicator runs the multi-GPU exchange steps (NCCL all-reduce of the
    # sketch and Gram partials, the agreement on non-finite input); with one rank every
    # all-reduce is the identity, so the results equal the single-GPU path bit for bit
    import torch

    plain = G.Context(0)
    coll = G.Context(0)
    coll.attach_comm(0, 1, G.make_comm_id())
    a = torch.as_tensor(o.synthesize(20000, 48, 1e6, 3), device="cuda")
    for meth, cfg in [(_abi.RLU, G.SketchConfig(strategy=G.Strategy.Gaussian, seed=5)),
                      (_abi.RQR, G.SketchConfig(seed=6)), (_abi.CHOLQR2, None)]:
        res = []
        for ctx in (plain, coll):
            q, r, rep = dist.factor_sharded(ctx, meth, a, a.shape[0], 0, cfg)
            res.append((q.cpu().numpy(), np.asarray(r)))
        assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    bad = a.clone()
    bad[7, 3] = float("nan")
    with pytest.raises(ValueError):
        dist.factor_sharded(coll, _abi.RLU, bad, bad.shape[0], 0, G.SketchConfig(strategy=G.Strategy.Gaussian))


@pytest.mark.slow
def test_more_than_2_31_rows():
    # 64-bit row indexing end to end (the TMA paths step aside above 2^31 rows):
    # m = 2^31 + 1000 rows, n = 2, checked through the device diagnostics
    import torch

    free, _ = torch.cuda.mem_get_info()
    m, n = (1 << 31) + 1000, 2
    if free < 8 * m * n * 3 + (8 << 30):
        pytest.skip("needs ~110 GB of free device memory")
    ctx = G.Context(0)
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    a[:, 1] += 0.5 * a[:, 0]
    q = torch.empty_like(a)
    for meth, cfg in [(_abi.CHOLQR2, None), (_abi.RQR_GAUSSIAN, G.SketchConfig(strategy=G.Strategy.Gaussian))]:
        _, r, _ = dist.factor_sharded(ctx, meth, a, m, 0, cfg, q_out=q)
        assert G.orthogonality_error_dev(q, ctx) < 1e-12
        assert G.residual_error_dev(a, q, r, ctx) < 1e-14
    del a, q
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [128, 256])
def test_strided_odd_inputs_use_the_fallback_kernels(n):
    # an odd leading dimension and an odd row count: no TMA path applies (sketch, Gram and
    # trisolve fall back to the cp.async / register kernels); Gram, Cholesky, LU and the
    # trisolves are order-identical, so CholeskyQR2 and uniform-sketch rLU match the
    # contiguous run and the oracle bit for bit; the Gaussian sketch only differs in its
    # k-chunking (tolerance)
    import torch

    m = 30001
    a = o.synthesize(m, n, 1e6, 4)
    base = torch.zeros((m, n + 1), dtype=torch.float64, device="cuda")
    base[:, :n] = torch.as_tensor(a, device="cuda")
    a_s = base[:, :n]  # stride n + 1 (odd)
    a_c = torch.as_tensor(a, device="cuda")
    ctx = G.Context(0)
    for meth, cfg in [(_abi.CHOLQR2, None), (_abi.RLU, G.SketchConfig(seed=3))]:
        qs, rs, _ = dist.factor_sharded(ctx, meth, a_s, m, 0, cfg)
        qc, rc, _ = dist.factor_sharded(ctx, meth, a_c, m, 0, cfg)
        assert np.array_equal(qs.cpu().numpy(), qc.cpu().numpy()) and np.array_equal(rs, rc)
        ref = o.factor(meth, a, None if cfg is None else cfg._c())
        assert np.array_equal(qs.cpu().numpy(), ref.q) and np.array_equal(rs, ref.r)
    cfg = G.SketchConfig(strategy=G.Strategy.Gaussian, seed=9)
    qs, rs, _ = dist.factor_sharded(ctx, _abi.RQR_GAUSSIAN, a_s, m, 0, cfg)
    ref = o.factor(_abi.RQR_GAUSSIAN, a, cfg._c())
    assert relf(rs, ref.r) <= 1e-12
    assert G.orthogonality_error_dev(qs, ctx) <= 1e-12


def test_sharded_host_api_one_rank():
    # cqr_factor_sharded (host buffers, one rank of a multi-GPU job) with a one-rank
    # communicator equals cqr_factor bit for bit; without a communicator a real shard
    # (m_local < m_global) is refused, as is the unsharded call on a multi-rank context
    a = o.synthesize(12000, 40, 1e8, 8)
    cfg = G.SketchConfig(strategy=G.Strategy.Gaussian, seed=11)
    ref = G.rlu_cholesky_qr(a, cfg)
    coll = G.Context(0)
    coll.attach_comm(0, 1, G.make_comm_id())
    q, r, _ = dist.factor_sharded_host(coll, _abi.RLU, a, a.shape[0], 0, cfg)
    assert np.array_equal(q, ref.q) and np.array_equal(r, ref.r)
    with pytest.raises(ValueError):
        dist.factor_sharded_host(G.Context(0), _abi.RLU, a[:6000], a.shape[0], 0, cfg)


def test_randomized_parity_sweep():
    # 96 random shapes across every method and both sketch strategies, host buffers and
    # strided device views; status (ok / breakdown / singular, with index) must match the
    # oracle; bit-identical Q and R for the order-pinned methods, tolerances otherwise
    import torch

    rng = np.random.default_rng(2024)
    exact = {_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3}
    for case in range(96):
        meth = int(rng.choice([_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3, _abi.RLU, _abi.RQR, _abi.RQR_GAUSSIAN]))
        n = int(rng.integers(1, 131))
        m = int(rng.integers(n, max(n + 1, 6000)))
        kappa = float(10.0 ** rng.uniform(0, 9))
        gauss = meth == _abi.RQR_GAUSSIAN or (meth == _abi.RLU and rng.random() < 0.5)
        l = int(rng.integers(n, min(m, 3 * n) + 1))
        seed = int(rng.integers(1, 1 << 30))
        a = o.synthesize(m, n, kappa, seed)
        cfg_c = _abi.sketch_cfg(strategy=_abi.GAUSSIAN if gauss else _abi.UNIFORM, size=l, seed=seed + 7)
        cfg = G.SketchConfig(strategy=G.Strategy.Gaussian if gauss else G.Strategy.Uniform, size=l, seed=seed + 7)
        try:
            ref = o.factor(meth, a, cfg_c)
            ref_err = None
        except o.OracleError as e:
            ref, ref_err = None, e
        use_dev = rng.random() < 0.4
        try:
            if use_dev:  # strided device view (leading dimension n + 3)
                base = torch.zeros((m, n + 3), dtype=torch.float64, device="cuda")
                base[:, :n] = torch.as_tensor(a, device="cuda")
                qd, r, _ = dist.factor_sharded(G.context(0), meth, base[:, :n], m, 0, cfg)
                q = qd.cpu().numpy()
            else:
                f, _, _ = G._factor(meth, a, cfg, _abi.options())
                q, r = f.q, f.r
            err = None
        except (G.CholeskyBreakdown, G.SingularTriangular) as e:
            err = e
        ctx_msg = f"case {case}: method {meth} m={m} n={n} l={l} kappa={kappa:.1e} gauss={gauss} dev={use_dev}"
        if ref_err is not None:
            assert err is not None, ctx_msg
            idx = getattr(err, "pivot_index", getattr(err, "index", None))
            assert idx == ref_err.index, ctx_msg
            continue
        if meth in exact or (meth == _abi.RLU and not gauss):
            assert err is None and np.array_equal(q, ref.q) and np.array_equal(r, ref.r), ctx_msg
        else:
            assert err is None, ctx_msg
            assert relf(r, ref.r) <= 1e-11, ctx_msg
            assert o.orthogonality_error(q) <= max(2 * o.orthogonality_error(ref.q), 1e-11), ctx_msg


def test_randomized_kernel_sweep():
    # the kernel-level entry points at random shapes around every padding boundary
    rng = np.random.default_rng(77)
    widths = [1, 2, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 200, 255, 256, 257, 384, 511, 512]
    for case in range(40):
        n = int(rng.choice(widths))
        m = int(rng.integers(n, n + 3000))
        seed = int(rng.integers(1, 1 << 30))
        x = o.gaussian_matrix(m, n, seed)
        g = o.gram(x)
        assert np.array_equal(G.gram(x), g), (case, m, n)
        rr = o.cholesky_upper(g)
        assert np.array_equal(G.cholesky_upper(g), rr), (case, n)
        assert np.array_equal(G.right_trisolve(x, rr), o.right_trisolve(x, rr)), (case, m, n)
        l = int(rng.integers(n, 2 * n + 2))
        a1 = o.gaussian_matrix(l, n, seed + 1)
        assert np.array_equal(G.lu_u_factor(a1), o.lu_u_factor(a1)), (case, l, n)
        assert relf(G.qr_r_factor(a1), o.qr_r_factor(a1)) <= 1e-12, (case, l, n)


def test_concurrent_threads_get_their_own_contexts():
    """concurrent calls on distinct inputs are safe. Each host thread gets its own
    default context (stream, status word, workspace); results equal the sequential ones bitwise."""
    import threading

    mats = [o.synthesize(20000 + 1000 * i, 24 + 8 * i, 1e8, 40 + i) for i in range(4)]
    cfgs = [G.SketchConfig(strategy=G.Strategy.Gaussian, seed=70 + i) for i in range(4)]
    seq = [G.rlu_cholesky_qr(a, c) for a, c in zip(mats, cfgs)]
    out = [None] * 4
    errs = []

    def work(i):
        try:
            for _ in range(3):
                out[i] = G.rlu_cholesky_qr(mats[i], cfgs[i])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for s, f in zip(seq, out):
        assert np.array_equal(s.q, f.q) and np.array_equal(s.r, f.r)


def test_stream_ordered_inputs():
    """A written on a torch side stream behind a long-running kernel: the device-buffer calls order the
    library stream after torch's current stream (cqr_order_after, no host sync) and see the final A."""
    import torch

    m, n = 50_000, 64
    ah = o.synthesize(m, n, 1e8, 4)
    src = torch.as_tensor(ah, device="cuda")
    ref = G.cholesky_qr2(src.clone())
    ctx = dist.make_context(0, 0, 1)
    side = torch.cuda.Stream()
    for trial in range(3):
        a = torch.zeros_like(src)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            torch.cuda._sleep(20_000_000)  # ~10 ms of device time ahead of the copy
            a.copy_(src)
            q, r, _ = dist.factor_sharded(ctx, _abi.CHOLQR2, a, m, 0)
            f = G.cholesky_qr2(a)
        assert np.array_equal(r, ref.r), trial
        assert torch.equal(q, ref.q), trial
        assert np.array_equal(f.r, ref.r) and torch.equal(f.q, ref.q), trial
