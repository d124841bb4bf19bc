"""numpy-facing bindings of the CPU oracle (oracle/build/libcqr_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg. The product
package never imports this module.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2111_11148_b200 import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libcqr_oracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        d, i64, u64, i32 = C.c_double, C.c_int64, C.c_uint64, C.c_int
        P = C.POINTER
        pd, pi64, pu64 = P(d), P(i64), P(u64)
        sig = {
            "orc_mix64": (u64, [u64]),
            "orc_bits_at": (u64, [u64, u64]),
            "orc_derive": (u64, [u64, u64]),
            "orc_unit_at": (d, [u64, u64]),
            "orc_gaussian_at": (d, [u64, u64]),
            "orc_bits_fill": (None, [u64, u64, i64, pu64]),
            "orc_gaussian_fill": (None, [u64, u64, i64, pd]),
            "orc_gaussian_matrix": (None, [i64, i64, u64, pd]),
            "orc_stream_indices": (None, [u64, u64, i64, i64, pi64]),
            "orc_resolved_size": (i64, [P(_abi.SketchCfg), i64, i64]),
            "orc_sample_rows_uniform": (i32, [pd, i64, i64, i64, i64, u64, i32, pd, pi64]),
            "orc_set_test_threads": (None, [i32]),
            "orc_sketch_gaussian": (i32, [pd, i64, i64, i64, i64, u64, pd]),
            "orc_sketch_gaussian_shard": (i32, [pd, i64, i64, i64, i64, i64, u64, pd]),
            "orc_gram": (i32, [pd, i64, i64, i64, i32, pd]),
            "orc_gram_tree_combine": (None, [pd, i64, i64, pd]),
            "orc_gram_chain": (None, [pd, i64, i64, i64, pd, pd]),
            "orc_gram_stack_combine": (None, [pd, i64, i64, pd]),
            "orc_cholesky_upper": (i32, [pd, i64, pd, pi64]),
            "orc_trisolve_inplace": (i32, [pd, i64, i64, i64, pd, i32, pi64]),
            "orc_qr_r_factor": (i32, [pd, i64, i64, pd]),
            "orc_lu_decompose": (i32, [pd, i64, i64, pd, pi64, pi64]),
            "orc_lu_u_factor": (i32, [pd, i64, i64, pd, pi64]),
            "orc_householder_qr_thin": (i32, [pd, i64, i64, pd, pd]),
            "orc_svd_values": (i32, [pd, i64, i64, pd]),
            "orc_triangular_product": (None, [pd, pd, i64, pd]),
            "orc_factor": (i32, [i32, pd, i64, i64, i64, P(_abi.SketchCfg), P(_abi.Options), i32, pd, pd,
                                 P(_abi.Report)]),
            "orc_precond_factor": (i32, [pd, i64, i64, i64, _abi.PRECOND_FN, C.c_void_p, P(_abi.SketchCfg),
                                         P(_abi.Options), i32, pd, pd, P(_abi.Report)]),
            "orc_orthogonality_error": (d, [pd, i64, i64]),
            "orc_residual_error": (d, [pd, pd, pd, i64, i64]),
            "orc_random_orthogonal": (i32, [i64, i64, u64, pd]),
            "orc_synthesize": (i32, [i64, i64, d, u64, pd]),
            "orc_synthesize_sigma": (i32, [i64, i64, pd, u64, pd]),
            "orc_embedded_identity": (i32, [i64, i64, u64, pd]),
            "orc_block_offset": (i64, [i64, i32, i32]),
            "orc_comm_model": (None, [i32, i32, i64, i64, P(C.c_int), P(C.c_int), pd, pd]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# ---------------------------------------------------------------------------
class OracleError(Exception):
    def __init__(self, status, index=-1):
        self.status, self.index = status, index
        super().__init__(f"oracle status {status} index {index}")


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pi64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(st, index=-1):
    if st != 0:
        raise OracleError(st, index)


def set_test_threads(w):
    """Test-harness knob: split the Gaussian sketch's rows and the diagnostics over
    w threads (bitwise the same results; the reference's sketch, and the bench's
    CPU arm, are serial)."""
    lib().orc_set_test_threads(int(w))


# rng (rng.hpp)
def mix64(z):
    return lib().orc_mix64(z)


def bits_at(seed, k):
    return lib().orc_bits_at(seed, k)


def derive(seed, salt):
    return lib().orc_derive(seed & (2**64 - 1), salt & (2**64 - 1))


def unit_at(seed, k):
    return lib().orc_unit_at(seed, k)


def gaussian_at(seed, k):
    return lib().orc_gaussian_at(seed, k)


def bits_fill(seed, k0, count):
    out = np.empty(count, dtype=np.uint64)
    lib().orc_bits_fill(seed, k0, count, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def gaussian_fill(seed, k0, count):
    out = np.empty(count, dtype=np.float64)
    lib().orc_gaussian_fill(seed, k0, count, _pd(out))
    return out


def gaussian_matrix(rows, cols, seed):
    out = np.empty((rows, cols), dtype=np.float64)
    lib().orc_gaussian_matrix(rows, cols, seed, _pd(out))
    return out


def stream_indices(seed, bound, count, start=0):
    out = np.empty(count, dtype=np.int64)
    lib().orc_stream_indices(seed, start, bound, count, _pi64(out))
    return out


# sketch
def resolved_size(cfg, m, n):
    return lib().orc_resolved_size(C.byref(cfg), m, n)


def sample_rows_uniform(a, l, seed, without_replacement=False):
    a = _f64(a)
    m, n = a.shape
    a1 = np.empty((l, n))
    idx = np.empty(l, dtype=np.int64)
    _check(lib().orc_sample_rows_uniform(_pd(a), m, n, n, l, seed, int(without_replacement), _pd(a1), _pi64(idx)))
    return a1, idx


def sketch_gaussian(a, l, seed):
    a = _f64(a)
    m, n = a.shape
    a1 = np.empty((l, n))
    _check(lib().orc_sketch_gaussian(_pd(a), m, n, n, l, seed, _pd(a1)))
    return a1


def sketch_gaussian_shard(a_local, m_global, row0, l, seed):
    a = _f64(a_local)
    m, n = a.shape
    a1 = np.empty((l, n))
    _check(lib().orc_sketch_gaussian_shard(_pd(a), m, m_global, row0, n, l, seed, _pd(a1)))
    return a1


# kernels
def gram(x, workers=1):
    x = _f64(x)
    m, n = x.shape
    g = np.empty((n, n))
    _check(lib().orc_gram(_pd(x), m, n, n, workers, _pd(g)))
    return g


def gram_chain(x, init=None):
    """fma chain over the rows of x continued from init (upper triangle, +0 if None)."""
    x = _f64(x)
    rows, n = x.shape
    out = np.zeros((n, n))
    ip = _pd(_f64(init)) if init is not None else None
    lib().orc_gram_chain(_pd(x), n, rows, n, ip, _pd(out))
    return out


def tree_combine(slots):
    s = _f64(slots)
    cnt = s.shape[0]
    length = s[0].size
    out = np.empty(length)
    lib().orc_gram_tree_combine(_pd(s), cnt, length, _pd(out))
    return out


def stack_combine(slots):
    s = _f64(slots)
    cnt = s.shape[0]
    length = s[0].size
    out = np.empty(length)
    lib().orc_gram_stack_combine(_pd(s), cnt, length, _pd(out))
    return out


def cholesky_upper(g):
    g = _f64(g)
    n = g.shape[0]
    r = np.empty((n, n))
    piv = C.c_int64(-1)
    st = lib().orc_cholesky_upper(_pd(g), n, _pd(r), C.byref(piv))
    _check(st, piv.value)
    return r


def right_trisolve(a, r, workers=1):
    x = _f64(a).copy()
    m, n = x.shape
    r = _f64(r)
    idx = C.c_int64(-1)
    st = lib().orc_trisolve_inplace(_pd(x), m, n, n, _pd(r), workers, C.byref(idx))
    _check(st, idx.value)
    return x


def qr_r_factor(a1):
    a1 = _f64(a1)
    l, n = a1.shape
    r = np.empty((n, n))
    _check(lib().orc_qr_r_factor(_pd(a1), l, n, _pd(r)))
    return r


def lu_decompose(a1):
    a1 = _f64(a1)
    l, n = a1.shape
    packed = np.empty((l, n))
    perm = np.empty(l, dtype=np.int64)
    idx = C.c_int64(-1)
    st = lib().orc_lu_decompose(_pd(a1), l, n, _pd(packed), _pi64(perm), C.byref(idx))
    _check(st, idx.value)
    return packed, perm


def lu_u_factor(a1):
    a1 = _f64(a1)
    l, n = a1.shape
    u = np.empty((n, n))
    idx = C.c_int64(-1)
    st = lib().orc_lu_u_factor(_pd(a1), l, n, _pd(u), C.byref(idx))
    _check(st, idx.value)
    return u


def householder_qr_thin(a):
    a = _f64(a)
    m, n = a.shape
    q = np.empty((m, n))
    r = np.empty((n, n))
    _check(lib().orc_householder_qr_thin(_pd(a), m, n, _pd(q), _pd(r)))
    return q, r


def svd_values(a):
    a = _f64(a)
    rows, cols = a.shape
    sv = np.empty(min(rows, cols))
    _check(lib().orc_svd_values(_pd(a), rows, cols, _pd(sv)))
    return sv


def triangular_product(left, right):
    left, right = _f64(left), _f64(right)
    n = left.shape[0]
    out = np.empty((n, n))
    lib().orc_triangular_product(_pd(left), _pd(right), n, _pd(out))
    return out


# engine / algorithm API
class Result:
    def __init__(self, q, r, report):
        self.q, self.r, self.report = q, r, report

    @property
    def stages(self):
        rep = self.report
        return [rep.stages[i] for i in range(rep.n_stages)]


def factor(method, a, cfg=None, opts=None, workers=1):
    """run_method / parexec::run_parallel (engine.cpp:221-305, parexec.cpp:64-75)."""
    a = _f64(a)
    m, n = a.shape
    q = np.empty((m, n))
    r = np.zeros((n, n))
    rep = _abi.Report()
    cfg = cfg if cfg is not None else _abi.sketch_cfg()
    opts = opts if opts is not None else _abi.options()
    st = lib().orc_factor(method, _pd(a), m, n, n, C.byref(cfg), C.byref(opts), workers, _pd(q), _pd(r),
                          C.byref(rep))
    _check(st, rep.index)
    return Result(q, None if opts.r_less else r, rep)


def precond_factor(a, precond, cfg=None, opts=None, workers=1):
    """precond_cholesky_qr with a python preconditioner (cholqr.hpp:100)."""
    a = _f64(a)
    m, n = a.shape

    def cb(user, a1p, l, nn, rp, idxp):
        a1 = np.ctypeslib.as_array(a1p, shape=(l, nn)).copy()
        try:
            rr = np.ascontiguousarray(precond(a1), dtype=np.float64)
        except OracleError as e:
            idxp[0] = e.index
            return e.status
        np.ctypeslib.as_array(rp, shape=(nn, nn))[:] = rr
        return 0

    fn = _abi.PRECOND_FN(cb)
    q = np.empty((m, n))
    r = np.zeros((n, n))
    rep = _abi.Report()
    cfg = cfg if cfg is not None else _abi.sketch_cfg()
    opts = opts if opts is not None else _abi.options()
    st = lib().orc_precond_factor(_pd(a), m, n, n, fn, None, C.byref(cfg), C.byref(opts), workers, _pd(q),
                                  _pd(r), C.byref(rep))
    _check(st, rep.index)
    return Result(q, None if opts.r_less else r, rep)


# diagnostics / matgen / parexec
def orthogonality_error(q):
    q = _f64(q)
    return lib().orc_orthogonality_error(_pd(q), q.shape[0], q.shape[1])


def residual_error(a, q, r):
    a, q, r = _f64(a), _f64(q), _f64(r)
    return lib().orc_residual_error(_pd(a), _pd(q), _pd(r), a.shape[0], a.shape[1])


def random_orthogonal(rows, cols, seed):
    out = np.empty((rows, cols))
    _check(lib().orc_random_orthogonal(rows, cols, seed, _pd(out)))
    return out


def synthesize(m, n, kappa, seed, sigma=None):
    out = np.empty((m, n))
    if sigma is None:
        _check(lib().orc_synthesize(m, n, float(kappa), seed, _pd(out)))
    else:
        s = _f64(sigma)
        _check(lib().orc_synthesize_sigma(m, n, _pd(s), seed, _pd(out)))
    return out


def embedded_identity(m, n, seed=0):
    out = np.empty((m, n))
    _check(lib().orc_embedded_identity(m, n, seed, _pd(out)))
    return out


def block_offset(m, p, b):
    return lib().orc_block_offset(m, p, b)


def comm_model(method, p, n, l):
    a, b = C.c_int(), C.c_int()
    c, d = C.c_double(), C.c_double()
    lib().orc_comm_model(method, p, n, l, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
    return a.value, b.value, c.value, d.value
