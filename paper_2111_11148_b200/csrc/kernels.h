// kernels.h — internal launch interface between the host engine and the
// sm_100a kernels (not part of the C-ABI; see include/cqr.h for that).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace cqr {

struct DevStatus;

// ---- trisolve.cu --------------------------------------------------------------
int trisolve_np(int n);                 // padded width bucket of the trisolve kernel
size_t trisolve_pack_doubles(int n);    // workspace for the packed R
cudaError_t launch_pack_r(const double* r, int ldr, int n, double* pack, int degenerate, DevStatus* st,
                          cudaStream_t s, const double* sgn = nullptr);  // sgn: pack diag(sgn) R
struct TrisolveArgs {
  const double* in;
  long long ldi;
  double* out;  // may alias in
  long long ldo;
  long long m;
  int n;
  const double* pack;  // from launch_pack_r
  const double* bpack;
  const double* dpack;
  int vec16;
  int num_sms;
  const DevStatus* status;
  int variant = 0;  // 0: the TMA kernel when eligible, else the register kernel; nonzero: the register kernel
};
cudaError_t launch_trisolve(TrisolveArgs a, cudaStream_t s);
// panel.cu: X[:, c0:c0+128] <- A[:, c0:c0+128] - X[:, 0:c0] R[0:c0, c0:c0+128] (k-ordered DMMA chains)
cudaError_t launch_panel_update(const TrisolveArgs& a, int c0, cudaStream_t s);
// trisolve_tma.cu: the TMA-staged kernel (16-byte aligned bases, even leading dimensions, np >= 32)
bool trisolve_tma_eligible(const TrisolveArgs& a, int np);
cudaError_t launch_trisolve_tma(const TrisolveArgs& a, int np, cudaStream_t s);
// trisolve_rr.cu: register-resident right-looking kernel (np <= 128; same eligibility as the TMA kernel)
cudaError_t launch_trisolve_rr(const TrisolveArgs& a, int np, cudaStream_t s);

// ---- gram.cu ---------------------------------------------------------------------
struct GramPlan {
  int n = 0, np = 0, leaves = 0, parts = 0, maxt = 0, wpc = 0, ch = 0, persistent = 0, tma = 0;
  long long m = 0;
  size_t partial_doubles = 0;    // leaves * np * np
  size_t workspace_doubles = 0;  // partials + the per-group sums of the combine
  size_t tiles_bytes = 0;
};
GramPlan gram_plan(long long m, int n, bool tma_ok = false);
// X is TMA-addressable for the TMA-fed leaf kernel (16-byte aligned base, even leading dimension)
bool gram_tma_ok(const double* x, long long ldx, long long m, int n);
// Host-side tile table for the plan (parts * wpc * maxt entries, packed I2 | J2<<16, -1 = none).
void gram_tiles(const GramPlan& p, int32_t* out);
// Leaf partials (1024-row leaves, kernels.hpp:20-38) -> partial[leaf][np*np] (upper tiles).
// check=1: also flag non-finite input (status INVALID_ARGUMENT, outranks others).
// [leaf0, leaf1): the leaves this launch computes (default all); results are per leaf.
cudaError_t launch_gram_leaves(const GramPlan& p, const double* x, long long ldx, const int32_t* tiles_dev,
                               double* partial, int vec16, int check, const DevStatus* st, cudaStream_t s,
                               int leaf0 = 0, int leaf1 = -1, int num_sms = 148);
// Pairwise tree over leaves (kernels.hpp:42-57, streaming form) -> g upper (ld = n);
// mirror=1 also writes the lower triangle (kernels.hpp:69).
cudaError_t launch_gram_combine(const GramPlan& p, double* partial, double* g, int mirror,
                                const DevStatus* st, cudaStream_t s);
cudaError_t launch_mirror_upper(double* g, int n, const DevStatus* st, cudaStream_t s);

// ---- sketch.cu ---------------------------------------------------------------------
struct SketchPlan {
  int n = 0, np = 0, l = 0, lp = 0, s_tiles = 0, kchunks = 0, ws = 0;  // ws: warp-specialised kernel
  int i8 = 0;            // the integer tensor-core kernel (sketch_i8.cu)
  int st = 64, npc = 128;  // Omega rows and A columns per CTA
  long long m_local = 0, rows_per_chunk = 0;
  size_t partial_doubles = 0;
};
// ws_ok: the caller's A qualifies for the warp-specialised kernel (sketch_ws_ok);
// splits: the k-chunks will be launched in this many row ranges as A arrives (host pipeline),
// so each range still fills the GPU
SketchPlan sketch_plan(long long m_local, int n, int l, int num_sms, bool ws_ok = false, int splits = 1);
bool sketch_ws_ok(const double* a, long long lda, long long m_global, long long row0, int n);
// [y0, y1): the k-chunks (rows_per_chunk rows each) this launch covers (default all).
cudaError_t launch_sketch_gaussian(const SketchPlan& p, const double* a, long long lda, long long m_global,
                                   long long row0, uint64_t seed, double* partial, int vec16, int check,
                                   const DevStatus* st, cudaStream_t s, int y0 = 0, int y1 = -1);
// sketch_i8.cu: the sketch as an exact integer product on tcgen05 (kind::i8) -- A needs the TMA
// alignment of the warp-specialised kernel; sketch_i8_plan turns a plan into the i8 kernel's
bool sketch_i8_ok(const double* a, long long lda, long long m_global, long long row0, int n);
void sketch_i8_plan(SketchPlan& p, long long m_local, int n, int l, int num_sms, int splits = 1);
cudaError_t launch_sketch_i8(const SketchPlan& p, const double* a, long long lda, long long m_global, long long row0,
                             uint64_t seed, double* partial, const DevStatus* st, cudaStream_t s,
                             int y0 = 0, int y1 = -1);
// a1[i][c] = sum over k-chunks (ascending) of partial -> l x n (ld = n)
cudaError_t launch_sketch_reduce(const SketchPlan& p, const double* partial, double* a1, const DevStatus* st,
                                 cudaStream_t s);
// Uniform row extraction (sketch.cpp:45-55). idx_host == nullptr: indices
// drawn on the device as floor(unit_at(seed, k) * m_global) (rng.hpp:69-71);
// rows outside [row0, row0+m_local) are written as zeros (the caller sums
// the shards). idx_out (device, optional) receives the indices.
cudaError_t launch_gather_rows(const double* a, long long lda, long long m_local, long long m_global,
                               long long row0, int n, int l, uint64_t seed, const long long* idx_dev,
                               double* a1, long long* idx_out, const DevStatus* st, cudaStream_t s);
cudaError_t launch_rng_bits(uint64_t seed, uint64_t k0, long long count, uint64_t* out, cudaStream_t s);
cudaError_t launch_rng_gaussian(uint64_t seed, uint64_t k0, long long count, double* out, cudaStream_t s);
cudaError_t launch_box_muller_bits(const uint64_t* bits, long long pairs, double* out, cudaStream_t s);

// ---- small.cu (single-CTA factorizations, all on device) ------------------------------
// kernels.hpp:76-90 (+ G += shift*I, engine.cpp:85; theory shift from trace(G)).
// shift_mode 0 none, 1 fixed (value), 2 theory (coef * trace(G)); shift_out optional.
size_t small_work_doubles(int rows, int n);
size_t qr_work_doubles(int l, int n);  // workspace of launch_qr_r / launch_lu_u
cudaError_t launch_cholesky(const double* g, int n, double* r, double* work, int shift_mode, double shift_value,
                            double theory_coef, double* shift_out, DevStatus* st, cudaStream_t s);
// kernels.hpp:211-257 (U only; status SingularTriangular(j) on a zero pivot).
cudaError_t launch_lu_u(const double* a1, int l, int n, double* u, double* work, DevStatus* st, cudaStream_t s);
// kernels.hpp:165-184 (sign-normalised R of a Householder QR).
cudaError_t launch_qr_r(const double* a1, int l, int n, double* r, double* work, DevStatus* st, cudaStream_t s);
// engine.cpp:103-107 dense L*R with the strict lower part zeroed.
cudaError_t launch_triangular_product(const double* left, const double* right, int n, double* out,
                                      const DevStatus* st, cudaStream_t s);
// engine.cpp:109-116 on R (rows with a negative diagonal flipped); sgn[i] = +-1
// is then applied to Q's columns by the final trisolve.
cudaError_t launch_normalize_sign(double* r, int n, double* sgn, const DevStatus* st, cudaStream_t s);

// diag.cu: cond(R) by a one-sided Jacobi sweep on the device (out[0]; work holds n x n doubles)
cudaError_t launch_jacobi_cond(const double* r, int n, double* work, double* out, cudaStream_t s);

// ---- householder.cu: tall Householder QR (HouseholderQr method, matgen's random_orthogonal) ----
int hh_blocks(long long m_local, int num_sms);
// red[0..w) = block-ordered sums of X(i,c) Y(i,c+t) over rows with global index > c, red[w..2w) = Y(c, c+t)
// on the rank holding row c (0 elsewhere); partial holds blocks * w doubles, w = n - c
cudaError_t launch_hh_reduce(const double* X, long long ldx, const double* Y, long long ldy, long long m_local,
                             long long row0, int c, int n, int blocks, double* partial, double* red, cudaStream_t s);
// the reflector of column c from the (rank-summed) red, R(c, c..), tau[c]; v stored below the diagonal
cudaError_t launch_hh_reflect_update(double* W, long long ldw, long long m_local, long long row0, int c, int n,
                                     double* red, double* coef, double* R, double* tau, int num_sms, cudaStream_t s);
cudaError_t launch_hh_qinit(double* Q, long long ldq, long long m_local, long long row0, int n, int num_sms,
                            cudaStream_t s);
cudaError_t launch_hh_qstep(const double* W, long long ldw, double* Q, long long ldq, long long m_local,
                            long long row0, int c, int n, const double* red, const double* tau, double* coef,
                            int num_sms, cudaStream_t s);
cudaError_t launch_col_sign(double* Q, long long ldq, long long m, int n, const double* sgn, int num_sms,
                            cudaStream_t s);

// ---- matgen.cu ---------------------------------------------------------------------------
// C = X * B, X m x n (ldx), B n x n row-major, C m x n (ldc), C != X.
cudaError_t launch_gemm_tall(const double* x, long long ldx, const double* b, double* c, long long ldc, long long m,
                             int n, int num_sms, cudaStream_t s);

// ---- diag.cu ------------------------------------------------------------------------------
// sum over rows of ||a_i - q_i R||^2 and ||a_i||^2 into out[0], out[1] (fixed order).
cudaError_t launch_residual(const double* a, long long lda, const double* q, long long ldq, const double* r,
                            long long m, int n, double* partial, int nblocks, double* out, cudaStream_t s);
cudaError_t launch_orth_from_gram(const double* g, int n, double* out, cudaStream_t s);

}  // namespace cqr
