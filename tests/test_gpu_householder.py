"""The HouseholderQr baseline method (engine.cpp:227-239, kernels.hpp:192-209) and
the reference's matrix generator (matgen.cpp:12-46: random_orthogonal = the thin
Householder Q of a Gaussian counter matrix, signs as Householder leaves them) on
the device, against the oracle's restatement of the same Householder algorithm.
Reduction orders differ (block partials vs sequential fma chains): tolerances.
"""
import math

import numpy as np
import pytest

from oracle import oracle as o
from paper_2111_11148_b200 import _abi
from paper_2111_11148_b200 import cholqr as G

pytestmark = pytest.mark.gpu
U = 2.0 ** -52


def relf(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("m,n,kappa,seed", [(1, 1, 1.0, 1), (7, 3, 1e3, 2), (3000, 17, 1e8, 3), (20000, 64, 1e12, 4),
                                            (50_000, 100, 1e15, 5), (4096, 256, 1e6, 6)])
def test_householder_method_matches_oracle(m, n, kappa, seed):
    a = o.synthesize(m, n, kappa, seed) if n > 1 else np.array([[3.0]] * m)
    ref = o.factor(_abi.HOUSEHOLDER, a)
    f, _, rep = G._factor(_abi.HOUSEHOLDER, a, None, _abi.options())
    assert [s.stage for s in f.report.stages] == ["householder"]
    assert np.all(np.diag(f.r) >= 0) and np.allclose(np.tril(f.r, -1), 0)
    assert relf(f.r, ref.r) <= 1e-12
    # Q's trailing columns are determined only to O(kappa u): two Householder runs with different
    # reduction orders differ by ~0.65 kappa u at kappa = 1e8 (measured); bound 4 kappa u
    assert np.linalg.norm(f.q - ref.q) / math.sqrt(n) <= max(1e-10, 4 * kappa * U)
    # unconditionally stable: orthogonality at the rounding floor even at kappa = 1e15
    assert o.orthogonality_error(f.q) <= max(2 * o.orthogonality_error(ref.q), 50 * n * U)
    assert o.residual_error(a, f.q, f.r) <= max(2 * o.residual_error(a, ref.q, ref.r), 10 * U)


def test_householder_known_answer_and_thin_api():
    # kernels.hpp:132-134 style: [[3],[4]] -> R = [5], Q = [[0.6],[0.8]]
    q, r = G.householder_qr_thin(np.array([[3.0], [4.0]]))
    assert np.allclose(r, [[5.0]], atol=1e-15) and np.allclose(q, [[0.6], [0.8]], atol=1e-15)
    # device tensors and host buffers give the same bits; r_less leaves R out
    import torch

    a = o.synthesize(5000, 24, 1e6, 9)
    fh = G._factor(_abi.HOUSEHOLDER, a, None, _abi.options())[0]
    fd = G._factor(_abi.HOUSEHOLDER, torch.as_tensor(a, device="cuda"), None, _abi.options())[0]
    assert np.array_equal(fh.q, fd.q.cpu().numpy()) and np.array_equal(fh.r, fd.r)
    fr = G._factor(_abi.HOUSEHOLDER, a, None, _abi.options(r_less=True))[0]
    assert fr.r is None and np.array_equal(fr.q, fh.q)


@pytest.mark.parametrize("rows,cols,seed", [(5, 5, 1), (300, 7, 2), (4096, 64, 3), (10_000, 128, 4)])
def test_random_orthogonal_matches_reference_signs(rows, cols, seed):
    """matgen.cpp:12-19: the device U is the Householder Q itself (not sign-normalised)."""
    sig = np.ones(cols)
    a = G.synthesize_dev(rows, cols, seed=seed, sigma=sig).cpu().numpy()  # = U V^T with sigma = 1
    ref = o.synthesize(rows, cols, 1.0, seed, sigma=sig)
    assert relf(a, ref) <= 1e-13


@pytest.mark.parametrize("m,n,kappa,seed", [(20_000, 50, 1e10, 1), (60_000, 128, 1e14, 2), (8192, 512, 1e8, 3)])
def test_synthesize_matches_oracle(m, n, kappa, seed):
    """matgen.cpp:21-46: A = U diag(sigma) V^T, the reference's A up to rounding."""
    a = G.synthesize_dev(m, n, kappa, seed).cpu().numpy()
    ref = o.synthesize(m, n, kappa, seed)
    assert relf(a, ref) <= 1e-13
    sv = np.linalg.svd(a, compute_uv=False)
    assert abs(sv[0] - 1.0) <= 1e-12 and abs(sv[-1] / kappa ** -1 - 1.0) <= 1e-3 * max(1.0, kappa * 1e-13)


def test_device_diagnostics_match_oracle():
    """diagnostics.cpp:10-28 on the device against the oracle on the same Q, R, A."""
    import torch

    for m, n, kappa, meth in ((20_000, 50, 1e8, _abi.CHOLQR2), (100_000, 128, 1e14, _abi.RLU), (3000, 7, 1e3, _abi.RQR)):
        a = o.synthesize(m, n, kappa, 7)
        cfg = G.SketchConfig(strategy=G.Strategy.Gaussian, seed=11) if meth == _abi.RLU else G.SketchConfig(seed=11)
        f = G._factor(meth, a, cfg, _abi.options(shift_kind=_abi.SHIFT_FIXED, shift_value=1e-15))[0]
        qd, ad = torch.as_tensor(f.q, device="cuda"), torch.as_tensor(a, device="cuda")
        og, oo = G.orthogonality_error_dev(qd), o.orthogonality_error(f.q)
        rg, ro = G.residual_error_dev(ad, qd, f.r), o.residual_error(a, f.q, f.r)
        assert abs(og - oo) <= 1e-12 * oo + 1e-300, (og, oo)
        assert abs(rg - ro) <= 1e-12 * ro + 1e-300, (rg, ro)


@pytest.mark.parametrize("m,n,l,kappa,seed", [(20_000, 128, 256, 1e10, 5), (8_000, 256, 300, 1e10, 6),
                                                (20_000, 128, 256, 10.0, 7), (6_000, 200, 400, 1e3, 8)])
def test_device_cond_x_matches_oracle(m, n, l, kappa, seed):
    """engine.cpp:94-100: cond(X) of the preconditioned X on the device (a Jacobi sweep over R^, no host math)
    against the oracle's qr_r_factor(X) + one-sided Jacobi. X = A R~^{-1} with R~ the Householder R of the
    sampled rows (a tolerance-class kernel: its reduction order differs from the oracle's), so cond(X) carries
    an O(kappa(A) u) relative difference (measured 4e-8 at kappa = 1e10); at small kappa the bound is tight."""
    a = o.synthesize(m, n, kappa, seed)
    f = G.rqr_cholesky_qr(a, G.SketchConfig(size=l, seed=seed + 1), G.Options(diagnostics=True))
    ref = o.factor(_abi.RQR, a, _abi.sketch_cfg(size=l, seed=seed + 1), _abi.options(diagnostics=True))
    c = [s.cond_x for s in f.report.stages if s.cond_x is not None][0]
    cr = [s.cond_x for s in ref.stages if s.has_cond_x][0]
    assert abs(c - cr) <= max(1e-12, 10 * kappa * U) * cr, (c, cr)
