/*
 * cqr.h — C-ABI of the B200-native randomized preconditioned CholeskyQR path.
 *
 * This is the drop-in boundary for the reference library's hot path
 * (`/root/reference/proj/include/cholqr/` headers). Every entry point below names
 * the reference interface it replaces. Conventions:
 *   - all tall matrices are row-major binary64 with an explicit leading
 *     dimension (row stride, in elements) >= n, as Eigen::Ref<RowMajor> with an
 *     outer stride (reference types.hpp:18-19);
 *   - calls block until the result is available (reference semantics);
 *   - failures are returned as a cqr_status code; the index that the
 *     reference's exception carries (CholeskyBreakdown::pivot_index,
 *     SingularTriangular::index, errors.hpp:18-33) is written to `*index` /
 *     `report->index`; the message of the last error of a context is
 *     available from cqr_last_error();
 *   - `_dev` entry points take device pointers on the context's device; the
 *     others take host pointers and include the host<->device copies.
 * No torch types appear here: plain pointers, sizes and POD structs only.
 */
#ifndef CQR_H_
#define CQR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CQR_ABI_VERSION 1

/* Status codes (the reference's exception hierarchy, errors.hpp:11-93). */
typedef enum {
  CQR_OK = 0,
  CQR_CHOLESKY_BREAKDOWN = 1, /* cholqr::CholeskyBreakdown, errors.hpp:18-24 */
  CQR_SINGULAR_TRIANGULAR = 2, /* cholqr::SingularTriangular, errors.hpp:27-33 */
  CQR_INVALID_ARGUMENT = 3,    /* std::invalid_argument, errors.hpp:84-93 */
  CQR_CUDA_ERROR = 4,
  CQR_NCCL_ERROR = 5,
  CQR_UNSUPPORTED = 6,         /* e.g. leverage sketch (sketch.cpp:118-127) */
  CQR_OUT_OF_MEMORY = 7
} cqr_status;

/* cholqr::Method, types.hpp:35-43 (same order, same values). */
typedef enum {
  CQR_HOUSEHOLDER = 0,
  CQR_CHOLQR = 1,
  CQR_CHOLQR2 = 2,
  CQR_SCHOLQR3 = 3,
  CQR_RLU = 4,
  CQR_RQR = 5,
  CQR_RQR_GAUSSIAN = 6
} cqr_method;

/* cholqr::sketch::Strategy, sketch.hpp:14. */
typedef enum { CQR_UNIFORM = 0, CQR_LEVERAGE = 1, CQR_GAUSSIAN = 2 } cqr_strategy;

/* cholqr::Stage, cholqr.hpp:12-21. */
typedef enum {
  CQR_STAGE_SKETCH = 0,
  CQR_STAGE_PRECONDITION = 1,
  CQR_STAGE_GRAM = 2,
  CQR_STAGE_CHOLESKY = 3,
  CQR_STAGE_TRISOLVE = 4,
  CQR_STAGE_RECOVER = 5,
  CQR_STAGE_HOUSEHOLDER = 6
} cqr_stage;
#define CQR_STAGE_COUNT 7

/* cholqr::sketch::SketchConfig, sketch.hpp:16-33. */
typedef struct {
  int32_t strategy;            /* cqr_strategy; default CQR_UNIFORM */
  int64_t size;                /* explicit l; 0 = use rate */
  double rate;                 /* default 2.0 */
  uint64_t seed;
  int32_t max_retries;         /* default 2 */
  double retry_growth;         /* default 2.0 */
  int32_t without_replacement; /* default 0 */
} cqr_sketch_cfg;

/* cholqr::ShiftMode::Kind, cholqr.hpp:48-59. */
typedef enum { CQR_SHIFT_THEORY = 0, CQR_SHIFT_FIXED = 1 } cqr_shift_kind;

/* cholqr::Options (cholqr.hpp:61-70) + MethodConfig (cholqr.hpp:73-78). */
typedef struct {
  int32_t diagnostics; /* record cond(X) on the Precondition stage */
  int32_t r_less;      /* skip R */
  int32_t shift_kind;  /* cqr_shift_kind; default CQR_SHIFT_THEORY */
  double shift_value;  /* used when shift_kind == CQR_SHIFT_FIXED */
  int32_t workers;     /* p of parexec::run_parallel: must be in [0, m] (0 = 1); sets the comm-model
                          counters of a one-process call; device work is not split by it */
} cqr_options;

/* cholqr::StageInfo, cholqr.hpp:25-34 (optionals carried as has_* flags). */
typedef struct {
  int32_t stage;
  int32_t has_cond_x;
  double cond_x;
  int32_t has_shift;
  double shift;
  int32_t retries;
} cqr_stage_info;

#define CQR_MAX_STAGE_INFOS 16

/* StageReport (cholqr.hpp:36-39) + parexec::TimingBreakdown (parexec.hpp:73-79). */
typedef struct {
  int32_t status;       /* cqr_status of the call */
  int64_t index;        /* pivot / diagonal index for statuses 1 and 2, else -1 */
  int32_t r_less;
  int32_t n_stages;
  cqr_stage_info stages[CQR_MAX_STAGE_INFOS];
  double stage_ms[CQR_STAGE_COUNT]; /* CUDA-event time per stage, summed over retries */
  double total_ms;
  int32_t comm_rounds;  /* parexec::comm_model rounds_max (parexec.cpp:44-62) */
  double comm_volume;   /* parexec::comm_model volume_max, values */
  int64_t sketch_rows;  /* l actually used by the successful attempt (0 if unsketched) */
} cqr_report;

/* Preconditioner callback (cholqr::Preconditioner, cholqr.hpp:94): given the
 * l x n sketch a1 (host, row-major, ld = n) write the n x n upper-triangular
 * factor to r (host, row-major, ld = n). Return CQR_OK, or
 * CQR_SINGULAR_TRIANGULAR with *index set to make the engine re-sketch. */
typedef int (*cqr_precond_fn)(void* user, const double* a1, int64_t l, int64_t n, double* r,
                              int64_t* index);

typedef struct cqr_ctx cqr_ctx;

/* ---- defaults ------------------------------------------------------------ */
void cqr_sketch_cfg_default(cqr_sketch_cfg* cfg);
void cqr_options_default(cqr_options* opts);
/* sketch::SketchConfig::resolved_size, sketch.cpp:20-23 */
int64_t cqr_resolved_size(const cqr_sketch_cfg* cfg, int64_t m, int64_t n);
int cqr_abi_version(void);

/* ---- context --------------------------------------------------------------- */
/* Owns the device, a stream, device workspace and (optionally) an NCCL
 * communicator. Not shared across host threads (reference: one call per
 * thread). */
int cqr_create(cqr_ctx** ctx, int device);
int cqr_destroy(cqr_ctx* ctx);
const char* cqr_last_error(const cqr_ctx* ctx);
/* Size of an NCCL unique id (opaque bytes exchanged by the caller, e.g. via
 * torch.distributed or MPI). */
int cqr_comm_id_size(void);
/* Rank 0 fills `id` (cqr_comm_id_size() bytes); every rank then passes the
 * same bytes to cqr_attach_comm. This replaces the reference's simulated
 * workers (parexec.cpp:64-75, engine.cpp:12-22) with one process per GPU. */
int cqr_comm_make_id(void* id);
/* An attached communicator switches the exchange steps on (sketch and Gram
 * all-reduce, agreement on non-finite input), also for world == 1 (a one-rank
 * NCCL communicator). */
int cqr_attach_comm(cqr_ctx* ctx, int rank, int world, const void* id);

/* A caller-owned transport for the same exchange steps, on HOST buffers (the
 * library stages device data through pinned memory around each call; every call
 * blocks until the exchange is complete). This is how the multi-rank path runs
 * with fewer GPUs than ranks -- several processes on one GPU whose kernels never
 * wait on one another, the exchanges going through e.g. torch.distributed/gloo --
 * and how a host that already owns an MPI communicator plugs it in. Callbacks
 * return 0 on success. dtype: CQR_COMM_F64_SUM (double, sum) or CQR_COMM_I32_MAX
 * (int32, max). sendrecv: send `count` doubles to rank dst (dst < 0: none) and
 * receive `count` doubles from rank src (src < 0: none), concurrently. allgather:
 * every rank contributes `count` doubles; recv holds world * count in rank order.
 * world == 1 with a NULL table detaches. */
enum { CQR_COMM_F64_SUM = 0, CQR_COMM_I32_MAX = 1 };
typedef struct {
  void* user;
  int (*allreduce)(void* user, void* buf, int64_t count, int dtype);
  int (*sendrecv)(void* user, const double* send, int dst, double* recv, int src, int64_t count);
  int (*allgather)(void* user, const double* send, double* recv, int64_t count);
} cqr_host_comm;
int cqr_attach_host_comm(cqr_ctx* ctx, int rank, int world, const cqr_host_comm* comm);
int cqr_stream_handle(cqr_ctx* ctx, void** stream); /* cudaStream_t the context launches on */
/* Order the context's next launches after all work queued so far on `stream` (a cudaStream_t of the
 * context's device; NULL = the legacy default stream): an event recorded there and waited on by the
 * context stream, no host synchronisation. Device-buffer callers whose inputs come from another stream
 * use this instead of synchronising the producer; every call returns with its own work complete. */
int cqr_order_after(cqr_ctx* ctx, void* stream);

/* ---- whole factorizations (cholqr.hpp:82-109, parexec.hpp:89-90) ----------- */
/* Host buffers. Q is m x n (ldq >= n); R is n x n (ldr >= n), untouched when
 * opts->r_less. `cfg` may be NULL for unsketched methods. Replaces
 * cholesky_qr (cholqr.hpp:82), cholesky_qr2 (:85), shifted_cholesky_qr3
 * (:89-91), rqr_cholesky_qr (:104), rlu_cholesky_qr (:108) and
 * parexec::run_parallel (parexec.hpp:89). */
int cqr_factor(cqr_ctx* ctx, int method, const double* a, int64_t m, int64_t n, int64_t lda,
               const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q, int64_t ldq,
               double* r, int64_t ldr, cqr_report* report);

/* Host buffers, one rank of a multi-GPU job: rows [row0, row0 + m_local) of the
 * m_global-row matrix (blocks ceil(b*m/p), cqr_block_offset); Q is this rank's
 * rows, R the full factor (identical on every rank). Needs cqr_attach_comm;
 * host-buffer counterpart of cqr_factor_dev (parexec::run_parallel,
 * parexec.hpp:89-90). */
int cqr_factor_sharded(cqr_ctx* ctx, int method, const double* a, int64_t m_local, int64_t m_global, int64_t row0,
                       int64_t n, int64_t lda, const cqr_sketch_cfg* cfg, const cqr_options* opts, double* q,
                       int64_t ldq, double* r, int64_t ldr, cqr_report* report);
/* Device buffers, row-block sharded when a communicator is attached: this
 * rank owns global rows [row0, row0 + m_local) of an m_global x n matrix
 * (blocks ceil(b*m/p), parexec.cpp:9-18). q may alias a (in-place, like the
 * reference Engine, engine.cpp:45-74). r is a HOST buffer (every rank gets
 * the same R). */
int cqr_factor_dev(cqr_ctx* ctx, int method, const double* a, int64_t m_local, int64_t m_global,
                   int64_t row0, int64_t n, int64_t lda, const cqr_sketch_cfg* cfg,
                   const cqr_options* opts, double* q, int64_t ldq, double* r, int64_t ldr,
                   cqr_report* report);

/* precond_cholesky_qr with a user preconditioner (cholqr.hpp:100). */
int cqr_precond_factor(cqr_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                       cqr_precond_fn precond, void* user, const cqr_sketch_cfg* cfg,
                       const cqr_options* opts, double* q, int64_t ldq, double* r, int64_t ldr,
                       cqr_report* report);

/* ---- kernel-level entry points (kernels.hpp, sketch.hpp) ---------------- */
/* kernels::gram, kernels.hpp:64 — G = X^T X, n x n, symmetric to the bit. */
int cqr_gram(cqr_ctx* ctx, const double* x, int64_t m, int64_t n, int64_t ldx, double* g);
int cqr_gram_dev(cqr_ctx* ctx, const double* x, int64_t m, int64_t n, int64_t ldx, double* g);
/* kernels::cholesky_upper, kernels.hpp:77 — *pivot = breakdown index. */
int cqr_cholesky_upper(cqr_ctx* ctx, const double* g, int64_t n, double* r, int64_t* pivot);
/* kernels::right_trisolve_in_place, kernels.hpp:102 — X R = A, X overwrites A. */
int cqr_trisolve_inplace(cqr_ctx* ctx, double* x, int64_t m, int64_t n, int64_t ldx,
                         const double* r, int64_t* index);
int cqr_trisolve_inplace_dev(cqr_ctx* ctx, double* x, int64_t m, int64_t n, int64_t ldx,
                             const double* r_dev, int64_t* index);
/* kernels::qr_r_factor, kernels.hpp:175 (sign-normalized R of a Householder QR). */
int cqr_qr_r_factor(cqr_ctx* ctx, const double* a1, int64_t l, int64_t n, double* r);
/* kernels::lu_u_factor, kernels.hpp:251 (row-partially-pivoted LU, U only). */
int cqr_lu_u_factor(cqr_ctx* ctx, const double* a1, int64_t l, int64_t n, double* u,
                    int64_t* index);
/* sketch::sketch_gaussian, sketch.cpp:94-116 — a1 = Omega A, Omega(i,j) =
 * gaussian_at(seed, i*m + j) generated in-kernel, never stored. l rows. */
int cqr_sketch_gaussian(cqr_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                        int64_t l, uint64_t seed, double* a1);
int cqr_sketch_gaussian_dev(cqr_ctx* ctx, const double* a, int64_t m_local, int64_t m_global,
                            int64_t row0, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                            double* a1_dev);
/* sketch::sample_rows_uniform, sketch.cpp:45-55 — indices drawn from
 * Stream(seed) (rng.hpp:69-71); idx may be NULL. */
int cqr_sample_rows_uniform(cqr_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                            int64_t l, uint64_t seed, int without_replacement, double* a1,
                            int64_t* idx);
/* rng::gaussian_matrix / bits_at on the device (rng.hpp:29-92), for checks. */
int cqr_rng_bits(cqr_ctx* ctx, uint64_t seed, uint64_t k0, int64_t count, uint64_t* out);
int cqr_rng_gaussian(cqr_ctx* ctx, uint64_t seed, uint64_t k0, int64_t count, double* out);
/* The Box-Muller step of rng.hpp:47-55 on given counter bits (host arrays):
 * bits[2i] -> u1 = ((bits[2i] >> 11) + 1) 2^-53, bits[2i+1] -> u2 = (bits[2i+1] >> 11) 2^-53;
 * out[2i] = sqrt(-2 ln u1) cos(2 pi u2), out[2i+1] = ... sin(2 pi u2). For edge-case checks. */
int cqr_box_muller_bits(cqr_ctx* ctx, const uint64_t* bits, int64_t pairs, double* out);

/* ---- diagnostics on the device (diagnostics.cpp:10-28) ------------------ */
int cqr_orthogonality_error_dev(cqr_ctx* ctx, const double* q, int64_t m, int64_t n, int64_t ldq,
                                double* out);
int cqr_residual_error_dev(cqr_ctx* ctx, const double* a, int64_t lda, const double* q,
                           int64_t ldq, const double* r_host, int64_t m, int64_t n, double* out);

/* ---- input synthesis on the device (matgen.cpp:21-46) ----------- */
/* A = U diag(sigma) V^T for rows [row0, row0+m_local) of an m_global x n matrix
 * (sigma: host array of n values). U, V: orthonormalised counter-RNG Gaussians
 * (seeds derive(seed,0), derive(seed,1)); same spectrum as the reference's
 * synthesize, not bit-identical (column signs). Sharded over an attached comm. */
int cqr_synthesize_dev(cqr_ctx* ctx, int64_t m_local, int64_t m_global, int64_t row0, int64_t n,
                       const double* sigma, uint64_t seed, double* a, int64_t lda);

/* ---- parexec helpers (parexec.cpp:9-62) ----------------------------------- */
/* offset(b) = ceil(b*m/p) */
int64_t cqr_block_offset(int64_t m, int p, int b);
/* comm_model(method, p, n, l) -> rounds/volumes (values, not bytes). */
int cqr_comm_model(int method, int p, int64_t n, int64_t l, int* rounds_min, int* rounds_max,
                   double* volume_min, double* volume_max);

/* Sharded Gram whose result does not depend on the rank count (the reference's
 * parallel_gram splits global 1024-row leaves over workers and combines them in one
 * fixed tree, engine.cpp:24-39; test_parexec.cpp:47-56 asserts bitwise identity
 * across p). Rank b of p owns rows [row0, row1) = parexec.cpp:13-15; a leaf
 * straddling a block boundary is one fma chain continued across ranks (head: from
 * rank b-1, tail: to rank b+1, span: both, inside one leaf); owned leaves [lo, hi)
 * are combined into the pairwise-tree nodes listed; every rank all-gathers the nodes
 * and evaluates the rest of the tree. Used by every multi-rank factorization whose
 * shards are the standard partition. Host-only (no GPU needed). */
typedef struct {
  int64_t row0, row1;
  int head, tail, span;
  int64_t head_end, tail_start; /* head rows [row0, head_end), tail rows [tail_start, row1) */
  int64_t full0, full1;         /* rows of the leaves complete on this rank */
  int64_t lo, hi;               /* owned global leaves */
  int nodes;
  int64_t node_start[64], node_count[64];
} cqr_gram_shard;
int cqr_gram_shard_plan(int64_t m, int p, int b, cqr_gram_shard* out);
/* Postfix program of the tree top over gathered slots b*K + k (op -1 = left + right).
 * Returns its length (negative: -length when cap is too small); *slots_per_rank = K. */
int cqr_gram_tree_program(int64_t m, int p, int* prog, int cap, int* slots_per_rank);
/* The p-rank protocol run rank by rank on this one device (the exchanges become
 * device copies): G of the device matrix x (m x n) as p ranks would compute it.
 * Test entry for the multi-rank arithmetic on a one-GPU box. */
int cqr_gram_sharded_sim(cqr_ctx* ctx, const double* x, int64_t m, int64_t n, int64_t ldx, int p,
                         double* g_dev);

/* Number of kernels this library launched since the context was created
 * (evidence for the bench's gpu_launches count). */
int64_t cqr_launch_count(const cqr_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* CQR_H_ */
