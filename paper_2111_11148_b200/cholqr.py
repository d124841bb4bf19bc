"""Host-side mirror of the reference's public API over the C-ABI (include/cqr.h).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/cholqr/{cholqr,parexec,kernels,sketch}.hpp:

    cholesky_qr(a, opts)                      cholqr.hpp:82
    cholesky_qr2(a, opts)                     cholqr.hpp:85
    shifted_cholesky_qr3(a, shift, opts)      cholqr.hpp:89-91
    precond_cholesky_qr(a, precond, cfg, opts) cholqr.hpp:100
    rqr_cholesky_qr(a, cfg, opts)             cholqr.hpp:104
    rlu_cholesky_qr(a, cfg, opts)             cholqr.hpp:108
    run_parallel(method, a, p, cfg)           parexec.hpp:89
    gram / cholesky_upper / right_trisolve(_in_place) / qr_r_factor / lu_u_factor   kernels.hpp
    sketch_gaussian / sample_rows_uniform / make_sketch                              sketch.hpp

Errors are the reference's exception types (errors.hpp): CholeskyBreakdown
(.pivot_index), SingularTriangular (.index), ValueError for invalid arguments.

Inputs may be numpy arrays (host buffers: the call includes the copies to and
from HBM) or CUDA torch tensors (device buffers, no copies; the result Q is a
CUDA tensor). Every computation runs in the sm_100a kernels of libcqr.so;
there is no CPU fallback — without the library or a GPU the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import threading

import numpy as np

from . import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CQR_LIB") or os.path.join(_HERE, "libcqr.so")

# ---- errors (errors.hpp) ------------------------------------------------------------


class Error(RuntimeError):
    """cholqr::Error"""


class CholeskyBreakdown(Error):
    def __init__(self, pivot_index):
        super().__init__(f"cholesky breakdown at pivot {pivot_index}")
        self.pivot_index = pivot_index


class SingularTriangular(Error):
    def __init__(self, index):
        super().__init__(f"singular triangular factor, zero diagonal at {index}")
        self.index = index


class DeviceError(Error):
    pass


# ---- configuration (sketch.hpp:16-33, cholqr.hpp:48-78) ----------------------------
class Strategy:
    Uniform, Leverage, Gaussian = _abi.UNIFORM, _abi.LEVERAGE, _abi.GAUSSIAN


class Method:
    HouseholderQr = _abi.HOUSEHOLDER
    CholeskyQr = _abi.CHOLQR
    CholeskyQr2 = _abi.CHOLQR2
    ShiftedCholeskyQr3 = _abi.SCHOLQR3
    RluCholeskyQr = _abi.RLU
    RqrCholeskyQr = _abi.RQR
    RqrCholeskyQrGaussian = _abi.RQR_GAUSSIAN


def method_name(m):
    return _abi.METHOD_NAMES[m]


@dataclasses.dataclass
class SketchConfig:
    strategy: int = Strategy.Uniform
    size: int = 0
    rate: float = 2.0
    seed: int = 0
    max_retries: int = 2
    retry_growth: float = 2.0
    without_replacement: bool = False

    def resolved_size(self, m, n):
        return _lib().cqr_resolved_size(C.byref(self._c()), m, n)

    def _c(self):
        return _abi.sketch_cfg(self.strategy, self.size, self.rate, self.seed, self.max_retries,
                               self.retry_growth, self.without_replacement)


@dataclasses.dataclass
class ShiftMode:
    kind: int = _abi.SHIFT_THEORY
    value: float = 0.0

    @staticmethod
    def theory():
        return ShiftMode(_abi.SHIFT_THEORY, 0.0)

    @staticmethod
    def fixed(eps):
        return ShiftMode(_abi.SHIFT_FIXED, float(eps))


@dataclasses.dataclass
class Options:
    diagnostics: bool = False
    r_less: bool = False
    workers: int = 1


@dataclasses.dataclass
class MethodConfig:
    sketch: SketchConfig = dataclasses.field(default_factory=SketchConfig)
    shift: ShiftMode = dataclasses.field(default_factory=ShiftMode.theory)
    diagnostics: bool = False
    r_less: bool = False


@dataclasses.dataclass
class StageInfo:
    stage: str
    cond_x: float | None
    shift: float | None
    retries: int


@dataclasses.dataclass
class StageReport:
    stages: list
    r_less: bool


@dataclasses.dataclass
class QRFactorization:
    q: object
    r: object
    report: StageReport


@dataclasses.dataclass
class TimingBreakdown:
    stage_ms: list
    total_ms: float
    comm_rounds: int
    comm_volume: float


@dataclasses.dataclass
class ParallelRun:
    factorization: QRFactorization
    timing: TimingBreakdown


# ---- library / context ------------------------------------------------------------------
_LIB = None
_LOCK = threading.Lock()
_TLS = threading.local()  # per-thread default contexts (cqr.h: a context is not shared across threads)


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        d, i64, u64, i32, vp = C.c_double, C.c_int64, C.c_uint64, C.c_int, C.c_void_p
        P = C.POINTER
        pd, pi64 = P(d), P(i64)
        sig = {
            "cqr_abi_version": (i32, []),
            "cqr_resolved_size": (i64, [P(_abi.SketchCfg), i64, i64]),
            "cqr_create": (i32, [P(vp), i32]),
            "cqr_destroy": (i32, [vp]),
            "cqr_last_error": (C.c_char_p, [vp]),
            "cqr_comm_id_size": (i32, []),
            "cqr_comm_make_id": (i32, [vp]),
            "cqr_attach_comm": (i32, [vp, i32, i32, vp]),
            "cqr_attach_host_comm": (i32, [vp, i32, i32, P(_abi.HostComm)]),
            "cqr_stream_handle": (i32, [vp, P(vp)]),
            "cqr_order_after": (i32, [vp, vp]),
            "cqr_launch_count": (i64, [vp]),
            "cqr_factor": (i32, [vp, i32, vp, i64, i64, i64, P(_abi.SketchCfg), P(_abi.Options), vp, i64, vp,
                                 i64, P(_abi.Report)]),
            "cqr_factor_dev": (i32, [vp, i32, vp, i64, i64, i64, i64, i64, P(_abi.SketchCfg), P(_abi.Options),
                                     vp, i64, vp, i64, P(_abi.Report)]),
            "cqr_factor_sharded": (i32, [vp, i32, vp, i64, i64, i64, i64, i64, P(_abi.SketchCfg), P(_abi.Options),
                                         vp, i64, vp, i64, P(_abi.Report)]),
            "cqr_precond_factor": (i32, [vp, vp, i64, i64, i64, _abi.PRECOND_FN, vp, P(_abi.SketchCfg),
                                         P(_abi.Options), vp, i64, vp, i64, P(_abi.Report)]),
            "cqr_gram": (i32, [vp, vp, i64, i64, i64, vp]),
            "cqr_gram_dev": (i32, [vp, vp, i64, i64, i64, vp]),
            "cqr_gram_sharded_sim": (i32, [vp, vp, i64, i64, i64, i32, vp]),
            "cqr_gram_shard_plan": (i32, [i64, i32, i32, P(_abi.GramShard)]),
            "cqr_gram_tree_program": (i32, [i64, i32, P(C.c_int), i32, P(C.c_int)]),
            "cqr_cholesky_upper": (i32, [vp, vp, i64, vp, pi64]),
            "cqr_trisolve_inplace": (i32, [vp, vp, i64, i64, i64, vp, pi64]),
            "cqr_trisolve_inplace_dev": (i32, [vp, vp, i64, i64, i64, vp, pi64]),
            "cqr_qr_r_factor": (i32, [vp, vp, i64, i64, vp]),
            "cqr_lu_u_factor": (i32, [vp, vp, i64, i64, vp, pi64]),
            "cqr_sketch_gaussian": (i32, [vp, vp, i64, i64, i64, i64, u64, vp]),
            "cqr_sketch_gaussian_dev": (i32, [vp, vp, i64, i64, i64, i64, i64, i64, u64, vp]),
            "cqr_sample_rows_uniform": (i32, [vp, vp, i64, i64, i64, i64, u64, i32, vp, vp]),
            "cqr_rng_bits": (i32, [vp, u64, u64, i64, vp]),
            "cqr_rng_gaussian": (i32, [vp, u64, u64, i64, vp]),
            "cqr_box_muller_bits": (i32, [vp, vp, i64, vp]),
            "cqr_orthogonality_error_dev": (i32, [vp, vp, i64, i64, i64, pd]),
            "cqr_residual_error_dev": (i32, [vp, vp, i64, vp, i64, vp, i64, i64, pd]),
            "cqr_synthesize_dev": (i32, [vp, i64, i64, i64, i64, vp, u64, vp, i64]),
            "cqr_block_offset": (i64, [i64, i32, i32]),
            "cqr_comm_model": (i32, [i32, i32, i64, i64, P(C.c_int), P(C.c_int), pd, pd]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


class Context:
    """cqr_ctx: device, stream, workspace and (optionally) an NCCL communicator."""

    def __init__(self, device=0):
        self.device = device
        h = C.c_void_p()
        st = _lib().cqr_create(C.byref(h), device)
        if st != 0:
            raise DeviceError(f"cqr_create(device={device}) failed with status {st}")
        self.h = h

    def close(self):
        if self.h:
            _lib().cqr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self):
        s = C.c_void_p()
        _lib().cqr_stream_handle(self.h, C.byref(s))
        return s.value

    @property
    def launches(self):
        return _lib().cqr_launch_count(self.h)

    def attach_comm(self, rank, world, comm_id: bytes):
        buf = C.create_string_buffer(comm_id, len(comm_id))
        self._check(_lib().cqr_attach_comm(self.h, rank, world, buf))

    def last_error(self):
        return (_lib().cqr_last_error(self.h) or b"").decode(errors="replace")

    def _check(self, st, index=-1):
        _raise(st, index, self.last_error())


def make_comm_id():
    n = _lib().cqr_comm_id_size()
    buf = C.create_string_buffer(n)
    st = _lib().cqr_comm_make_id(buf)
    if st != 0:
        raise DeviceError("ncclGetUniqueId failed")
    return buf.raw


def context(device=None):
    """Default context of (this thread, device). The reference is pure and
    reentrant on distinct inputs, while a cqr_ctx owns one stream,
    status word and workspace and must not be shared across host threads
    (cqr.h), so every thread gets its own -- as the C++ shim's thread_local
    Context does."""
    if device is None:
        device = _current_device()
    cache = getattr(_TLS, "ctx", None)
    if cache is None:
        cache = _TLS.ctx = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = Context(device)
    return ctx


def _current_device():
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


def _raise(st, index, msg=""):
    if st == _abi.OK:
        return
    if st == _abi.CHOLESKY_BREAKDOWN:
        raise CholeskyBreakdown(index)
    if st == _abi.SINGULAR_TRIANGULAR:
        raise SingularTriangular(index)
    if st == _abi.INVALID_ARGUMENT:
        raise ValueError(msg or "invalid argument")
    if st == _abi.UNSUPPORTED:
        raise NotImplementedError(msg or "unsupported")
    raise DeviceError(f"status {st}: {msg}")


# ---- buffers --------------------------------------------------------------------------------
def _is_torch_cuda(x):
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _host(a):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    return a


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def _stages(rep):
    out = []
    for i in range(rep.n_stages):
        s = rep.stages[i]
        out.append(StageInfo(_abi.STAGE_NAMES[s.stage], s.cond_x if s.has_cond_x else None,
                             s.shift if s.has_shift else None, s.retries))
    return out


def _check_cuda_matrix(a, what="A", ctx=None):
    """A CUDA tensor the library may read as a row-major float64 matrix with
    leading dimension stride(0); waits for the producer's pending work (the
    library runs on its own non-blocking stream, which is not ordered after
    torch's streams). With `ctx` the wait is stream-ordered (cqr_order_after on
    torch's current stream) instead of a host synchronisation; ctx=False only
    validates (the caller has ordered the producer already)."""
    import torch

    if a.dtype != torch.float64 or a.dim() != 2 or a.stride(1) != 1 or a.stride(0) < a.shape[1]:
        raise ValueError(f"{what}: expected a CUDA float64 row-major matrix (stride(1) == 1, stride(0) >= cols)")
    if ctx is False:
        return
    if ctx is not None:
        ctx._check(_lib().cqr_order_after(ctx.h, C.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)), -1)
    else:
        torch.cuda.current_stream(a.device).synchronize()


def _factor(method, a, cfg: SketchConfig | None, opts_c, ctx=None, precond=None):
    cfg_c = (cfg or SketchConfig())._c()
    rep = _abi.Report()
    r_less = bool(opts_c.r_less)
    if _is_torch_cuda(a):
        import torch

        _check_cuda_matrix(a, "A", False)
        if precond is not None:
            raise ValueError("a custom preconditioner needs host buffers")
        ctx = ctx or context(a.device.index)
        m, n = a.shape
        q = torch.empty((m, n), dtype=torch.float64, device=a.device)
        _check_cuda_matrix(q, "Q", ctx)  # stream-ordered after torch's pending work on A (and Q's memory)
        r = np.zeros((n, n))
        st = _lib().cqr_factor_dev(ctx.h, method, C.c_void_p(a.data_ptr()), m, m, 0, n, a.stride(0),
                                   C.byref(cfg_c), C.byref(opts_c), C.c_void_p(q.data_ptr()), n, _ptr(r), n,
                                   C.byref(rep))
    else:
        a = _host(a)
        ctx = ctx or context()
        m, n = a.shape
        q = np.empty((m, n))
        r = np.zeros((n, n))
        if precond is None:
            st = _lib().cqr_factor(ctx.h, method, _ptr(a), m, n, n, C.byref(cfg_c), C.byref(opts_c), _ptr(q), n,
                                   _ptr(r), n, C.byref(rep))
        else:
            def cb(user, a1p, l, nn, rp, idxp):
                a1 = np.ctypeslib.as_array(a1p, shape=(l, nn)).copy()
                try:
                    rr = np.ascontiguousarray(precond(a1), dtype=np.float64)
                except SingularTriangular as e:
                    idxp[0] = e.index
                    return _abi.SINGULAR_TRIANGULAR
                np.ctypeslib.as_array(rp, shape=(nn, nn))[:] = rr
                return 0

            fn = _abi.PRECOND_FN(cb)
            st = _lib().cqr_precond_factor(ctx.h, _ptr(a), m, n, n, fn, None, C.byref(cfg_c), C.byref(opts_c),
                                           _ptr(q), n, _ptr(r), n, C.byref(rep))
    ctx._check(st, rep.index)
    fact = QRFactorization(q, None if r_less else r, StageReport(_stages(rep), bool(rep.r_less)))
    timing = TimingBreakdown(list(rep.stage_ms), rep.total_ms, rep.comm_rounds, rep.comm_volume)
    return fact, timing, rep


def _opts(opts: Options | None, shift: ShiftMode | None = None, diagnostics=None, r_less=None):
    o = opts or Options()
    sh = shift or ShiftMode.theory()
    return _abi.options(o.diagnostics if diagnostics is None else diagnostics,
                        o.r_less if r_less is None else r_less, sh.kind, sh.value, o.workers)


# ---- algorithm API (cholqr.hpp:82-109) -----------------------------------------------------
def cholesky_qr(a, opts: Options | None = None):
    return _factor(Method.CholeskyQr, a, None, _opts(opts))[0]


def cholesky_qr2(a, opts: Options | None = None):
    return _factor(Method.CholeskyQr2, a, None, _opts(opts))[0]


def shifted_cholesky_qr3(a, shift: ShiftMode | Options | None = None, opts: Options | None = None):
    if isinstance(shift, Options):
        shift, opts = None, shift
    return _factor(Method.ShiftedCholeskyQr3, a, None, _opts(opts, shift))[0]


def precond_cholesky_qr(a, precond, cfg: SketchConfig, opts: Options | None = None):
    return _factor(Method.RqrCholeskyQr, a, cfg, _opts(opts), precond=precond)[0]


def rqr_cholesky_qr(a, cfg: SketchConfig, opts: Options | None = None):
    return _factor(Method.RqrCholeskyQr, a, cfg, _opts(opts))[0]


def rlu_cholesky_qr(a, cfg: SketchConfig, opts: Options | None = None):
    return _factor(Method.RluCholeskyQr, a, cfg, _opts(opts))[0]


# ---- the RSVD caller's orthogonalizer (apps.cpp:166-196) ----------------------
_M64 = (1 << 64) - 1


def _mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive(seed, salt):
    """rng::derive (rng.hpp:36-38): mix64(seed ^ mix64(salt + 0x51ED270B8A5EC473))."""
    return _mix64((seed & _M64) ^ _mix64((salt + 0x51ED270B8A5EC473) & _M64))


class Orth:
    HouseholderQr, RqrCholeskyQr, CholeskyQr2 = 0, 1, 2


def orth_name(o):
    return {Orth.HouseholderQr: "qr", Orth.RqrCholeskyQr: "rqr", Orth.CholeskyQr2: "cholqr2"}[o]


def orthonormalize(y, orth, seed, call_counter, workers=1, ctx=None):
    """apps.cpp:166-196 orthonormalize: Q of Y with R discarded (r_less). rQR
    draws fresh rows every call: uniform sketch, rate 2, seed
    derive(seed, 0xA110 + call_counter); HouseholderQr is householder_qr_thin
    (kernels.hpp:192-209) on the device (csrc/householder.cu)."""
    opts = Options(diagnostics=False, r_less=True, workers=workers)
    if orth == Orth.RqrCholeskyQr:
        cfg = SketchConfig(rate=2.0, seed=derive(seed, 0xA110 + int(call_counter)))
        return _factor(Method.RqrCholeskyQr, y, cfg, _opts(opts), ctx=ctx)[0].q
    if orth == Orth.CholeskyQr2:
        return _factor(Method.CholeskyQr2, y, None, _opts(opts), ctx=ctx)[0].q
    if orth == Orth.HouseholderQr:
        return _factor(Method.HouseholderQr, y, None, _opts(opts), ctx=ctx)[0].q
    raise ValueError(f"unknown orthogonalizer {orth}")


def run_parallel(method, a, p=1, cfg: MethodConfig | None = None, ctx=None):
    """parexec::run_parallel (parexec.hpp:89-90). On one process `p` only sets
    the communication-model counters (the device does not split work by it);
    multi-GPU runs shard A over ranks with paper_2111_11148_b200.dist."""
    cfg = cfg or MethodConfig()
    if p < 1 or p > np.shape(a)[0]:
        raise ValueError("worker count must be in [1, m]")
    o = _abi.options(cfg.diagnostics, cfg.r_less, cfg.shift.kind, cfg.shift.value, p)
    fact, timing, rep = _factor(method, a, cfg.sketch, o, ctx=ctx)
    n = np.shape(a)[1]
    l = cfg.sketch.resolved_size(np.shape(a)[0], n)
    rmin, rmax, vmin, vmax = comm_model(method, p, n, l)
    timing.comm_rounds, timing.comm_volume = rmax, vmax
    return ParallelRun(fact, timing)


# ---- parexec helpers (parexec.cpp:9-62) -------------------------------------------------------
def block_offset(m, p, b):
    return _lib().cqr_block_offset(m, p, b)


def comm_model(method, p, n, l):
    a, b = C.c_int(), C.c_int()
    c, d = C.c_double(), C.c_double()
    st = _lib().cqr_comm_model(method, p, n, l, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
    _raise(st, -1, "unknown method")
    return a.value, b.value, c.value, d.value


# ---- kernel-level API (kernels.hpp, sketch.hpp) ------------------------------------------------
def gram(x, ctx=None):
    """kernels::gram (kernels.hpp:64): G = X^T X, symmetric to the bit."""
    if _is_torch_cuda(x):
        import torch

        _check_cuda_matrix(x, "gram")
        ctx = ctx or context(x.device.index)
        m, n = x.shape
        g = torch.empty((n, n), dtype=torch.float64, device=x.device)
        ctx._check(_lib().cqr_gram_dev(ctx.h, C.c_void_p(x.data_ptr()), m, n, x.stride(0), C.c_void_p(g.data_ptr())))
        return g
    x = _host(x)
    ctx = ctx or context()
    m, n = x.shape
    if m < n:
        raise ValueError("gram: matrix must have rows >= cols")
    g = np.empty((n, n))
    ctx._check(_lib().cqr_gram(ctx.h, _ptr(x), m, n, n, _ptr(g)))
    return g


def gram_sharded_sim(x, p, ctx=None):
    """G of a CUDA matrix as p ranks of the rank-count-independent sharded Gram
    compute it (cqr_gram_sharded_sim: the multi-rank protocol on one device)."""
    import torch

    _check_cuda_matrix(x, "gram_sharded_sim")
    ctx = ctx or context(x.device.index)
    m, n = x.shape
    g = torch.empty((n, n), dtype=torch.float64, device=x.device)
    ctx._check(_lib().cqr_gram_sharded_sim(ctx.h, C.c_void_p(x.data_ptr()), m, n, x.stride(0), p,
                                            C.c_void_p(g.data_ptr())))
    return g


def cholesky_upper(g, ctx=None):
    """kernels::cholesky_upper (kernels.hpp:77); raises CholeskyBreakdown."""
    g = _host(g)
    if g.shape[0] != g.shape[1]:
        raise ValueError("cholesky_upper: matrix must be square")
    ctx = ctx or context()
    n = g.shape[0]
    r = np.empty((n, n))
    piv = C.c_int64(-1)
    st = _lib().cqr_cholesky_upper(ctx.h, _ptr(g), n, _ptr(r), C.byref(piv))
    ctx._check(st, piv.value)
    return r


def right_trisolve_in_place(x, r, ctx=None):
    """kernels::right_trisolve_in_place (kernels.hpp:102): X R = A, X overwrites A."""
    if _is_torch_cuda(x):
        import torch

        _check_cuda_matrix(x, "right_trisolve_in_place")
        ctx = ctx or context(x.device.index)
        m, n = x.shape
        rd = r if _is_torch_cuda(r) else torch.as_tensor(np.ascontiguousarray(r, dtype=np.float64), device=x.device)
        rd = rd.to(torch.float64).contiguous()
        if tuple(rd.shape) != (n, n):
            raise ValueError("right_trisolve: dimension mismatch")
        idx = C.c_int64(-1)
        torch.cuda.current_stream(x.device).synchronize()
        st = _lib().cqr_trisolve_inplace_dev(ctx.h, C.c_void_p(x.data_ptr()), m, n, x.stride(0),
                                             C.c_void_p(rd.data_ptr()), C.byref(idx))
        ctx._check(st, idx.value)
        return x
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
        raise ValueError("right_trisolve_in_place needs a C-contiguous float64 array")
    r = _host(r)
    m, n = x.shape
    if r.shape != (n, n):
        raise ValueError("right_trisolve: dimension mismatch")
    ctx = ctx or context()
    idx = C.c_int64(-1)
    st = _lib().cqr_trisolve_inplace(ctx.h, _ptr(x), m, n, n, _ptr(r), C.byref(idx))
    ctx._check(st, idx.value)
    return x


def right_trisolve(a, r, ctx=None):
    """kernels::right_trisolve (kernels.hpp:130)."""
    if _is_torch_cuda(a):
        return right_trisolve_in_place(a.clone(), r, ctx)
    return right_trisolve_in_place(np.array(a, dtype=np.float64, order="C"), r, ctx)


def householder_qr_thin(a, ctx=None):
    """kernels::householder_qr_thin (kernels.hpp:192-209): (Q, R) with R's diagonal
    non-negative, by the device's tall Householder QR (csrc/householder.cu)."""
    f, _, _ = _factor(Method.HouseholderQr, a, None, _opts(None), ctx=ctx)
    return f.q, f.r


def qr_r_factor(a1, ctx=None):
    """kernels::qr_r_factor (kernels.hpp:175)."""
    a1 = _host(a1)
    l, n = a1.shape
    if l < n:
        raise ValueError("qr_r_factor: need rows >= cols")
    ctx = ctx or context()
    r = np.empty((n, n))
    ctx._check(_lib().cqr_qr_r_factor(ctx.h, _ptr(a1), l, n, _ptr(r)))
    return r


def lu_u_factor(a1, ctx=None):
    """kernels::lu_u_factor (kernels.hpp:251); raises SingularTriangular."""
    a1 = _host(a1)
    l, n = a1.shape
    if l < n:
        raise ValueError("lu_decompose: need rows >= cols")
    ctx = ctx or context()
    u = np.empty((n, n))
    idx = C.c_int64(-1)
    st = _lib().cqr_lu_u_factor(ctx.h, _ptr(a1), l, n, _ptr(u), C.byref(idx))
    ctx._check(st, idx.value)
    return u


@dataclasses.dataclass
class Sketch:
    """sketch::Sketch (sketch.hpp:36-45)."""
    a1: np.ndarray
    strategy: int
    indices: np.ndarray | None = None
    projection_seed: int = 0


def sketch_gaussian(a, cfg: SketchConfig, seed=None, ctx=None):
    """sketch::sketch_gaussian (sketch.cpp:94-116); Omega generated in-kernel."""
    a = _host(a)
    m, n = a.shape
    l = cfg.resolved_size(m, n)
    seed = cfg.seed if seed is None else seed
    ctx = ctx or context()
    a1 = np.empty((l, n))
    ctx._check(_lib().cqr_sketch_gaussian(ctx.h, _ptr(a), m, n, n, l, seed & (2**64 - 1), _ptr(a1)))
    return Sketch(a1, Strategy.Gaussian, None, seed)


def sample_rows_uniform(a, cfg: SketchConfig, seed=None, ctx=None):
    """sketch::sample_rows_uniform (sketch.cpp:45-55)."""
    a = _host(a)
    m, n = a.shape
    l = cfg.resolved_size(m, n)
    seed = cfg.seed if seed is None else seed
    ctx = ctx or context()
    a1 = np.empty((l, n))
    idx = np.empty(l, dtype=np.int64)
    ctx._check(_lib().cqr_sample_rows_uniform(ctx.h, _ptr(a), m, n, n, l, seed & (2**64 - 1),
                                              int(cfg.without_replacement), _ptr(a1), _ptr(idx)))
    return Sketch(a1, Strategy.Uniform, idx, 0)


def make_sketch(a, cfg: SketchConfig, seed=None, ctx=None):
    """sketch::make_sketch (sketch.cpp:118-127)."""
    if cfg.strategy == Strategy.Uniform:
        return sample_rows_uniform(a, cfg, seed, ctx)
    if cfg.strategy == Strategy.Gaussian:
        return sketch_gaussian(a, cfg, seed, ctx)
    raise ValueError("leverage sampling needs an oracle Q; call sample_rows_leverage directly")


def rng_bits(seed, k0, count, ctx=None):
    ctx = ctx or context()
    out = np.empty(count, dtype=np.uint64)
    ctx._check(_lib().cqr_rng_bits(ctx.h, seed & (2**64 - 1), k0, count, _ptr(out)))
    return out


def rng_gaussian(seed, k0, count, ctx=None):
    ctx = ctx or context()
    out = np.empty(count)
    ctx._check(_lib().cqr_rng_gaussian(ctx.h, seed & (2**64 - 1), k0, count, _ptr(out)))
    return out


def box_muller_bits(bits, ctx=None):
    """Box-Muller step (rng.hpp:47-55) of the device draws on given counter bits:
    bits[2i] -> u1, bits[2i+1] -> u2; returns [r cos a, r sin a] per pair."""
    ctx = ctx or context()
    bits = np.ascontiguousarray(bits, dtype=np.uint64)
    assert bits.size % 2 == 0
    out = np.empty(bits.size)
    ctx._check(_lib().cqr_box_muller_bits(ctx.h, _ptr(bits), bits.size // 2, _ptr(out)))
    return out


def geometric_sigma(n, kappa):
    """sigma_i = exp(-ln(kappa) i/(n-1)) (matgen.cpp:27-31)."""
    sig = np.ones(n)
    if n > 1:
        sig[1:] = np.exp(-np.log(kappa) * np.arange(1, n) / (n - 1))
    return sig


def synthesize_dev(m, n, kappa=None, seed=0, sigma=None, device=0, m_global=None, row0=0, ctx=None):
    """matgen::synthesize on the device (matgen.cpp:21-46): rows [row0, row0+m) of
    an m_global x n matrix U diag(sigma) V^T, returned as a CUDA tensor. U and V
    are random_orthogonal (matgen.cpp:12-19): the thin Householder Q (signs as
    Householder leaves them) of the reference's Gaussian counter matrices, formed
    by the device Householder QR -- the reference's A up to rounding."""
    import torch

    ctx = ctx or context(device)
    sig = np.ascontiguousarray(sigma if sigma is not None else geometric_sigma(n, kappa), dtype=np.float64)
    a = torch.empty((m, n), dtype=torch.float64, device=f"cuda:{ctx.device}")
    mg = m if m_global is None else m_global
    ctx._check(_lib().cqr_synthesize_dev(ctx.h, m, mg, row0, n, _ptr(sig), seed & (2**64 - 1),
                                         C.c_void_p(a.data_ptr()), n))
    return a


def orthogonality_error_dev(q, ctx=None):
    """diagnostics::orthogonality_error (diagnostics.cpp:10-14) on a CUDA tensor."""
    import torch

    _check_cuda_matrix(q, "Q")
    ctx = ctx or context(q.device.index)
    out = C.c_double()
    m, n = q.shape
    ctx._check(_lib().cqr_orthogonality_error_dev(ctx.h, C.c_void_p(q.data_ptr()), m, n, q.stride(0), C.byref(out)))
    return out.value


def residual_error_dev(a, q, r, ctx=None):
    """diagnostics::residual_error (diagnostics.cpp:16-28) on CUDA tensors (r host)."""
    import torch

    _check_cuda_matrix(a, "A")
    _check_cuda_matrix(q, "Q")
    if q.shape != a.shape:
        raise ValueError("residual_error: A and Q shapes differ")
    ctx = ctx or context(a.device.index)
    out = C.c_double()
    m, n = a.shape
    rh = np.ascontiguousarray(r, dtype=np.float64)
    if rh.shape != (n, n):
        raise ValueError("residual_error: R must be n x n")
    ctx._check(_lib().cqr_residual_error_dev(ctx.h, C.c_void_p(a.data_ptr()), a.stride(0), C.c_void_p(q.data_ptr()),
                                             q.stride(0), _ptr(rh), m, n, C.byref(out)))
    return out.value
