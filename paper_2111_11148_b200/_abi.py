"""ctypes mirror of include/cqr.h (POD structs and enums, no behaviour).

Shared by the product bindings (paper_2111_11148_b200/cholqr.py) and by the
test-side oracle bindings (oracle/oracle.py), so both speak the same structs.
"""
import ctypes as C

# cqr_status (errors.hpp:11-93)
OK, CHOLESKY_BREAKDOWN, SINGULAR_TRIANGULAR, INVALID_ARGUMENT = 0, 1, 2, 3
CUDA_ERROR, NCCL_ERROR, UNSUPPORTED, OUT_OF_MEMORY, NO_CONVERGENCE = 4, 5, 6, 7, 8

# cholqr::Method (types.hpp:35-43)
HOUSEHOLDER, CHOLQR, CHOLQR2, SCHOLQR3, RLU, RQR, RQR_GAUSSIAN = range(7)
METHOD_NAMES = {
    HOUSEHOLDER: "householder", CHOLQR: "cholqr", CHOLQR2: "cholqr2",
    SCHOLQR3: "scholqr3", RLU: "rlu", RQR: "rqr", RQR_GAUSSIAN: "rqr-gaussian",
}

# sketch::Strategy (sketch.hpp:14)
UNIFORM, LEVERAGE, GAUSSIAN = 0, 1, 2

# Stage (cholqr.hpp:12-21)
STAGE_NAMES = ["sketch", "precondition", "gram", "cholesky", "trisolve", "recover", "householder"]
STAGE_COUNT = 7
MAX_STAGE_INFOS = 16

SHIFT_THEORY, SHIFT_FIXED = 0, 1


class SketchCfg(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32),
        ("size", C.c_int64),
        ("rate", C.c_double),
        ("seed", C.c_uint64),
        ("max_retries", C.c_int32),
        ("retry_growth", C.c_double),
        ("without_replacement", C.c_int32),
    ]


class Options(C.Structure):
    _fields_ = [
        ("diagnostics", C.c_int32),
        ("r_less", C.c_int32),
        ("shift_kind", C.c_int32),
        ("shift_value", C.c_double),
        ("workers", C.c_int32),
    ]


class StageInfo(C.Structure):
    _fields_ = [
        ("stage", C.c_int32),
        ("has_cond_x", C.c_int32),
        ("cond_x", C.c_double),
        ("has_shift", C.c_int32),
        ("shift", C.c_double),
        ("retries", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("index", C.c_int64),
        ("r_less", C.c_int32),
        ("n_stages", C.c_int32),
        ("stages", StageInfo * MAX_STAGE_INFOS),
        ("stage_ms", C.c_double * STAGE_COUNT),
        ("total_ms", C.c_double),
        ("comm_rounds", C.c_int32),
        ("comm_volume", C.c_double),
        ("sketch_rows", C.c_int64),
    ]


class GramShard(C.Structure):
    """cqr_gram_shard: rank b's part of the rank-count-independent Gram."""
    _fields_ = [
        ("row0", C.c_int64), ("row1", C.c_int64),
        ("head", C.c_int32), ("tail", C.c_int32), ("span", C.c_int32),
        ("head_end", C.c_int64), ("tail_start", C.c_int64),
        ("full0", C.c_int64), ("full1", C.c_int64),
        ("lo", C.c_int64), ("hi", C.c_int64),
        ("nodes", C.c_int32),
        ("node_start", C.c_int64 * 64), ("node_count", C.c_int64 * 64),
    ]


# cqr_host_comm (cqr.h): a caller-owned transport for the rank exchanges, on host buffers
COMM_F64_SUM, COMM_I32_MAX = 0, 1
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int)
SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double), C.c_int,
                          C.c_int64)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)


class HostComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce", ALLREDUCE_FN), ("sendrecv", SENDRECV_FN),
                ("allgather", ALLGATHER_FN)]


PRECOND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_int64,
                         C.POINTER(C.c_double), C.POINTER(C.c_int64))


def sketch_cfg(strategy=UNIFORM, size=0, rate=2.0, seed=0, max_retries=2, retry_growth=2.0,
               without_replacement=False):
    """sketch::SketchConfig defaults (sketch.hpp:16-33)."""
    return SketchCfg(int(strategy), int(size), float(rate), int(seed) & (2**64 - 1),
                     int(max_retries), float(retry_growth), int(bool(without_replacement)))


def options(diagnostics=False, r_less=False, shift_kind=SHIFT_THEORY, shift_value=0.0, workers=1):
    """Options (cholqr.hpp:61-70) + the ShiftMode of MethodConfig (cholqr.hpp:73-78)."""
    return Options(int(bool(diagnostics)), int(bool(r_less)), int(shift_kind), float(shift_value),
                   int(workers))
