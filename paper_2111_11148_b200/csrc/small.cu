// small.cu — the small s x n and n x n factorizations, on device, one CTA each
// (latency-bound: n <= 512 steps of O(n) parallel work). The working matrix
// lives in shared memory when it fits (<= ~200 KB) and otherwise in an
// L2-resident global workspace; the same kernel body serves both through a
// generic pointer.
//
//  cholesky_kernel  kernels.hpp:76-90 (+ G += shift*I, engine.cpp:85): right-looking,
//                   every element an fma chain in k order from g(i,j) (the
//                   oracle's pinned order) -> bitwise equal to the oracle.
//  lu_kernel        kernels.hpp:211-257: partial pivoting with the first maximum,
//                   fma trailing update skipped for zero multipliers -> bitwise.
//  qr_kernel        kernels.hpp:165-184: Householder (beta = -sign(c0)*norm),
//                   sign-normalised R; reductions in a fixed tree order
//                   (deterministic; tolerance parity with the oracle).
//  triangular_product_kernel  engine.cpp:103-107 (fma chain over all k) -> bitwise.
//  normalize_sign_kernel      engine.cpp:109-116 (R rows; Q columns via sgn).

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "trisolve_common.cuh"

namespace cqr {

namespace {

constexpr int kT = 1024;
constexpr size_t kSmemCap = 200 * 1024;

// Deterministic block sum (fixed xor tree in each warp, then warp 0 over the
// warp sums in index order through the same tree). All threads get the result.
__device__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0) scratch[32] = w;
  }
  __syncthreads();
  return scratch[32];
}

__global__ void __launch_bounds__(kT) cholesky_kernel(const double* __restrict__ g, int n, double* __restrict__ r,
                                                      double* work, int use_smem, int shift_mode, double shift_value,
                                                      double theory_coef, double* shift_out, DevStatus* st) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_d;
  __shared__ int s_bad;
  if (failed(st)) return;
  double* S = use_smem ? smem : work;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < n * n; e += nt) S[e] = g[e];
  __syncthreads();
  if (shift_mode != 0 && tid == 0) {
    double sh = shift_value;
    if (shift_mode == 2) {  // theory shift from trace(G) == ||A||_F^2 (cholqr.cpp:21-26)
      double tr = 0.0;
      for (int j = 0; j < n; ++j) tr += g[(long long)j * n + j];
      sh = theory_coef * tr;
    }
    for (int j = 0; j < n; ++j) S[(long long)j * n + j] += sh;
    if (shift_out) *shift_out = sh;
  }
  __syncthreads();
  for (int i = 0; i < n; ++i) {
    if (tid == 0) {
      const double sii = S[(long long)i * n + i];
      if (!(sii > 0.0)) {
        s_bad = 1;
        set_status(st, 1 /*CQR_CHOLESKY_BREAKDOWN*/, i);
      } else {
        s_bad = 0;
        s_d = sqrt(sii);
        S[(long long)i * n + i] = s_d;
      }
    }
    __syncthreads();
    if (s_bad) return;
    const double d = s_d;
    double* Si = S + (long long)i * n;
    for (int j = i + 1 + tid; j < n; j += nt) Si[j] = Si[j] / d;
    __syncthreads();
    // trailing update of the upper triangle: warps over rows, lanes over columns
    for (int a = i + 1 + (tid >> 5); a < n; a += nt >> 5) {
      const double ra = Si[a];
      double* Sa = S + (long long)a * n;
      for (int b = a + (tid & 31); b < n; b += 32) Sa[b] = fma(-ra, Si[b], Sa[b]);
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, j = e % n;
    r[e] = j >= i ? S[e] : 0.0;
  }
}

// Rows [0, rs) of the working matrix live in shared memory, rows [rs, l) in the
// L1-cached global workspace (c1: 200 of 256 rows in smem, the rest fits L1).
__global__ void __launch_bounds__(kT) lu_kernel(const double* __restrict__ a1, int l, int n, double* __restrict__ u,
                                                double* work, int rs, DevStatus* st) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double wb[32];
  __shared__ int wi[32];
  __shared__ int s_piv;
  if (failed(st)) return;
  auto row = [&](int i) -> double* { return i < rs ? smem + (long long)i * n : work + (long long)i * n; };
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int i = warp; i < l; i += nw) {
    double* ri = row(i);
    for (int c = lane; c < n; c += 32) ri[c] = a1[(long long)i * n + c];
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    // first maximum of |W(i, j)| over i >= j (kernels.hpp:226-234)
    double best = -1.0;
    int idx = 0x7fffffff;
    for (int i = j + tid; i < l; i += nt) {
      const double v = fabs(row(i)[j]);
      if (v > best) {
        best = v;
        idx = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ob > best || (ob == best && oi < idx)) {
        best = ob;
        idx = oi;
      }
    }
    if (lane == 0) {
      wb[warp] = best;
      wi[warp] = idx;
    }
    __syncthreads();
    if (warp == 0) {
      best = lane < nw ? wb[lane] : -1.0;
      idx = lane < nw ? wi[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ob > best || (ob == best && oi < idx)) {
          best = ob;
          idx = oi;
        }
      }
      if (lane == 0) s_piv = idx;
    }
    __syncthreads();
    const int piv = s_piv;
    if (piv >= l || row(piv)[j] == 0.0) {
      if (tid == 0) set_status(st, 2 /*CQR_SINGULAR_TRIANGULAR*/, j);
      return;
    }
    double* pj = row(j);
    if (piv != j) {
      double* pp = row(piv);
      for (int c = tid; c < n; c += nt) {
        const double t = pj[c];
        pj[c] = pp[c];
        pp[c] = t;
      }
      __syncthreads();
    }
    const double d = pj[j];
    for (int i = j + 1 + tid; i < l; i += nt) {
      double* ri = row(i);
      ri[j] = ri[j] / d;
    }
    __syncthreads();
    // trailing update: one warp per row, lanes over columns
    for (int i = j + 1 + warp; i < l; i += nw) {
      double* ri = row(i);
      const double mult = ri[j];
      if (mult != 0.0)
        for (int c = j + 1 + lane; c < n; c += 32) ri[c] = fma(-mult, pj[c], ri[c]);
    }
    __syncthreads();
  }
  for (int i = warp; i < n; i += nw) {
    const double* ri = row(i);
    for (int c = lane; c < n; c += 32) u[(long long)i * n + c] = c >= i ? ri[c] : 0.0;
  }
}

// Blocked right-looking LU (kernels.hpp:211-257), bitwise equal to the unblocked
// fma form: 32-column panels are factored in shared memory exactly as the
// unblocked loop (first maximum, zero-pivot check, multipliers, fma updates
// skipped for zero multipliers); the trailing columns then get the panel's
// row swaps, the unit-lower solve U12 = L11^-1 A12 (per column, fma chain over
// the pivots in order, zero multipliers skipped) and A22 += (-L21) U12 on DMMA
// (k = the panel's pivots in ascending order). Every trailing element thus sees
// the same fma sequence as in the unblocked algorithm. Only U is returned, so
// the L part left of a panel is never permuted.
constexpr int kLuPanel = 32;
constexpr int kLuLdp = kLuPanel + 1;

template <bool PSMEM>
__global__ void __launch_bounds__(512) lu_blocked_kernel(const double* __restrict__ a1, int l, int n,
                                                        double* __restrict__ u, double* W, double* Pg,
                                                        DevStatus* st) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double wb[32];
  __shared__ int wi[32];
  __shared__ int s_piv[kLuPanel];
  __shared__ int s_bad;
  if (failed(st)) return;
  double* P = PSMEM ? smem : Pg;  // (l - j0) x kLuPanel panel, stride kLuLdp (smem, or global when too tall)
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int i = warp; i < l; i += nw)
    for (int c = lane; c < n; c += 32) W[(long long)i * n + c] = a1[(long long)i * n + c];
  if (tid == 0) s_bad = -1;
  __syncthreads();
  for (int j0 = 0; j0 < n; j0 += kLuPanel) {
    const int w = min(kLuPanel, n - j0);
    const int pr = l - j0;  // panel rows
    for (int r = warp; r < pr; r += nw)
      if (lane < w) P[r * kLuLdp + lane] = W[(long long)(j0 + r) * n + j0 + lane];
    __syncthreads();
    // ---- panel factorization (unblocked, shared memory)
    for (int jj = 0; jj < w; ++jj) {
      double best = -1.0;
      int idx = 0x7fffffff;
      for (int r = jj + tid; r < pr; r += nt) {
        const double v = fabs(P[r * kLuLdp + jj]);
        if (v > best) {
          best = v;
          idx = r;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ob > best || (ob == best && oi < idx)) {
          best = ob;
          idx = oi;
        }
      }
      if (lane == 0) {
        wb[warp] = best;
        wi[warp] = idx;
      }
      __syncthreads();
      if (warp == 0) {
        best = lane < nw ? wb[lane] : -1.0;
        idx = lane < nw ? wi[lane] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
          if (ob > best || (ob == best && oi < idx)) {
            best = ob;
            idx = oi;
          }
        }
        if (lane == 0) {
          s_piv[jj] = idx;
          if (idx >= pr || P[idx * kLuLdp + jj] == 0.0) s_bad = j0 + jj;
        }
      }
      __syncthreads();
      if (s_bad >= 0) {
        if (tid == 0) set_status(st, 2 /*CQR_SINGULAR_TRIANGULAR*/, s_bad);
        return;
      }
      const int piv = s_piv[jj];
      if (piv != jj && tid < w) {
        const double t = P[jj * kLuLdp + tid];
        P[jj * kLuLdp + tid] = P[piv * kLuLdp + tid];
        P[piv * kLuLdp + tid] = t;
      }
      __syncthreads();
      const double d = P[jj * kLuLdp + jj];
      for (int r = jj + 1 + tid; r < pr; r += nt) P[r * kLuLdp + jj] = P[r * kLuLdp + jj] / d;
      __syncthreads();
      // rank-1 update of the panel: warps over rows (four per pass, every load issued before
      // the stores so the passes are not serialised on possible aliasing), lanes over columns
      {
        const int c = lane;
        const double pc = (c > jj && c < w) ? P[jj * kLuLdp + c] : 0.0;
        for (int rb = jj + 1 + warp; rb < pr; rb += 4 * nw) {
          double mv[4], xv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = rb + k * nw;
            mv[k] = r < pr ? P[r * kLuLdp + jj] : 0.0;
            xv[k] = (r < pr && c > jj && c < w) ? P[r * kLuLdp + c] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = rb + k * nw;
            if (r < pr && mv[k] != 0.0 && c > jj && c < w) P[r * kLuLdp + c] = fma(-mv[k], pc, xv[k]);
          }
        }
      }
      __syncthreads();
    }
    // U rows of the panel (the L part stays in P for the trailing update)
    for (int r = warp; r < w; r += nw)
      if (lane < w) W[(long long)(j0 + r) * n + j0 + lane] = P[r * kLuLdp + lane];
    const int c1 = j0 + w;
    if (c1 < n) {
      // row swaps on the trailing columns, in pivot order
      for (int jj = 0; jj < w; ++jj) {
        const int piv = s_piv[jj];
        if (piv != jj) {
          double* ra = W + (long long)(j0 + jj) * n;
          double* rb = W + (long long)(j0 + piv) * n;
          for (int c = c1 + tid; c < n; c += nt) {
            const double t = ra[c];
            ra[c] = rb[c];
            rb[c] = t;
          }
        }
        __syncthreads();
      }
      // U12 = L11^-1 A12: one thread per trailing column, fma chain over the pivots
      for (int c = c1 + tid; c < n; c += nt) {
        double x[kLuPanel];
#pragma unroll
        for (int jj = 0; jj < kLuPanel; ++jj) x[jj] = jj < w ? W[(long long)(j0 + jj) * n + c] : 0.0;
#pragma unroll
        for (int jj = 1; jj < kLuPanel; ++jj) {
          if (jj < w) {
#pragma unroll
            for (int k = 0; k < jj; ++k) {
              const double mult = P[jj * kLuLdp + k];
              if (mult != 0.0) x[jj] = fma(-mult, x[k], x[jj]);
            }
          }
        }
#pragma unroll
        for (int jj = 1; jj < kLuPanel; ++jj)
          if (jj < w) W[(long long)(j0 + jj) * n + c] = x[jj];
      }
      __syncthreads();
      // A22 += (-L21) U12 on DMMA: 8x8 tiles over rows [j0+w, l) x cols [c1, n)
      const int q = lane & 3, gr = lane >> 2;
      const int tr = (l - c1 + 7) / 8, tc = (n - c1 + 7) / 8;
      for (int t = warp; t < tr * tc; t += nw) {
        const int rt = t / tc, ct = t - (t / tc) * tc;
        const int r0 = c1 + rt * 8, cc0 = c1 + ct * 8;  // absolute row / column of the tile
        const int row = r0 + gr, col = cc0 + 2 * q;
        double c0v = 0.0, c1v = 0.0;
        if (row < l && col < n) c0v = W[(long long)row * n + col];
        if (row < l && col + 1 < n) c1v = W[(long long)row * n + col + 1];
        for (int k4 = 0; k4 < (w + 3) / 4; ++k4) {
          const int kk = 4 * k4 + q;                 // A: row gr, k = q
          const double av = (row < l && kk < w) ? -P[(row - j0) * kLuLdp + kk] : 0.0;
          const int bk = 4 * k4 + q, bc = cc0 + gr;  // B: k = q, col = gr
          const double bv = (bk < w && bc < n) ? W[(long long)(j0 + bk) * n + bc] : 0.0;
          dmma(c0v, c1v, av, bv);
        }
        if (row < l && col < n) W[(long long)row * n + col] = c0v;
        if (row < l && col + 1 < n) W[(long long)row * n + col + 1] = c1v;
      }
    }
    __syncthreads();
  }
  for (int i = warp; i < n; i += nw)
    for (int c = lane; c < n; c += 32) u[(long long)i * n + c] = c >= i ? W[(long long)i * n + c] : 0.0;
}

__device__ __forceinline__ double div_rn(double y, double d, double inv) {
  // correctly rounded y / d from inv = RN(1/d), one Markstein correction (see trisolve_common.cuh)
  const double ay = fabs(y);
  if (!(ay >= 0x1p-400 && ay <= 0x1p+400) || !(fabs(d) >= 0x1p-500 && fabs(d) <= 0x1p+500)) return y / d;
  const double q0 = y * inv;
  const double r = fma(-q0, d, y);
  return fma(r, inv, q0);
}

// Arg-max of (|x| as its bit pattern (hi, lo), then the smallest logical position) over a warp's
// lanes; lanes with cand false take no part. Fast path: one redux.sync on the high word when it
// is unique and non-zero; otherwise the full key. Returns the winning lane (-1 if no candidate).
__device__ __forceinline__ int warp_argmax_key(bool cand, unsigned hi, unsigned lo, unsigned pos) {
  constexpr unsigned kFull = 0xffffffffu;
  const unsigned mhi = __reduce_max_sync(kFull, cand ? hi : 0u);
  const unsigned top = __ballot_sync(kFull, cand && hi == mhi);
  if (mhi != 0u && __popc(top) == 1) return __ffs(top) - 1;
  const bool c1 = cand && hi == mhi;
  const unsigned mlo = __reduce_max_sync(kFull, c1 ? lo : 0u);
  const bool c2 = c1 && lo == mlo;
  const unsigned mpos = __reduce_min_sync(kFull, c2 ? pos : 0xffffffffu);
  return __ffs(__ballot_sync(kFull, c2 && pos == mpos)) - 1;
}

#ifdef CQR_LU_TRACE  // probe: clock64 marks of thread 0 (read with cqr_debug_lu_trace, tools/gpu/lu_trace.py)
__device__ long long g_lu_trace[1024];
#define LU_MARK(i) \
  {                                          \
    if (threadIdx.x == 0) g_lu_trace[i] = clock64(); \
  }
// the clock read issues only after v is available (in-order issue behind the compare that reads v)
__device__ __forceinline__ long long clock_after(double v) {
  long long t;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.f64 p, %1, 0d7FF1234500000000;\n\tmov.u64 %0, %%clock64;\n\t@p add.s64 %0, %0, 1;\n\t}"
      : "=l"(t)
      : "d"(v)
      : "memory");
  return t;
}
#else
#define LU_MARK(i) \
  {}
#endif
#ifndef CQR_LU_UNROLL
#define CQR_LU_UNROLL 16
#endif
constexpr int kLuUnroll = CQR_LU_UNROLL;
#ifndef CQR_LU_ROWTILES
#define CQR_LU_ROWTILES 8
#endif
constexpr int kLuRowTilesMax = CQR_LU_ROWTILES;
#ifndef CQR_LU_ROT_PANEL
#define CQR_LU_ROT_PANEL 16
#endif
constexpr int kLuRotPanel = CQR_LU_ROT_PANEL;  // panel width of lu_rot_kernel

// l <= 512: one thread per physical row, the panel's 32 columns of that row in
// registers. Rows never move: partial pivoting is tracked with logical
// positions (ties go to the smallest one: the reference's "first maximum" in its
// swapped order), each thread updating its own position from the arg-max. The
// current column is always x[0] (the row is shifted one place per step, so the
// step loop stays rolled: no dynamic register indexing, a small I-cache
// footprint). Per pivot step: one arg-max barrier, one barrier to publish the
// pivot row, register fma updates; U rows go straight to the output.
// SPLIT (l in (512, 1024], c4: 768 x 512): one launch per panel (columns [j0, j0 + PW)) that only
// takes the pivot steps; the multipliers (Pg, l x PW), logical positions (LPg) and pivot rows (PVg)
// go to global memory and lu_trail_kernel applies U12 and the A22 update over many SMs.
template <int NW, int PW, bool SPLIT = false>
__global__ void __launch_bounds__(NW * 32) lu_rot_kernel(const double* __restrict__ a1, int l, int n,
                                                        double* __restrict__ u, double* W, DevStatus* st,
                                                        int j0s = 0, double* Pg = nullptr, int* LPg = nullptr,
                                                        int* PVg = nullptr) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(16) double cv[2][NW][PW];  // each warp winner's panel row, double-buffered
  __shared__ double cinv[2][NW];                  // and RN(1 / its current element)
  __shared__ unsigned chi[2][NW], clo[2][NW], clp[2][NW];
  __shared__ int crow[2][NW];
  __shared__ int pv[PW];
  if (failed(st)) return;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  double* P = smem;                                                    // multipliers: l x kLuLdp
  int* lpS = reinterpret_cast<int*>(smem + (size_t)l * kLuLdp);        // logical positions after a panel
  const bool mine = tid < l;
  if constexpr (!SPLIT) {  // W = A1, eight independent loads in flight per thread
    const long long total = (long long)l * n;
    for (long long e0 = tid; e0 < total; e0 += 8LL * nt) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = e0 + k * nt < total ? __ldg(a1 + e0 + k * nt) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (e0 + k * nt < total) W[e0 + k * nt] = v[k];
    }
    for (int i = warp; i < n; i += NW)
      for (int c = lane; c < i; c += 32) u[(long long)i * n + c] = 0.0;
  }
  int my_lp = SPLIT ? (j0s == 0 || !mine ? tid : LPg[tid]) : tid, buf = 0;
  __syncthreads();
  LU_MARK(0)
  for (int j0 = SPLIT ? j0s : 0; j0 < (SPLIT ? min(n, j0s + PW) : n); j0 += PW) {
    const int w = min(PW, n - j0);
    LU_MARK(1 + 4 * (j0 / PW))
    double x[PW];
#pragma unroll
    for (int c = 0; c < PW; ++c) x[c] = (mine && c < w) ? W[(long long)tid * n + j0 + c] : 0.0;
    // kLuUnroll pivot steps per iteration with the current column x[o] (compile-time u), then
    // one rotation by kLuUnroll: the rolled loop keeps the code small, the unroll divides the
    // register moves of the rotation
#pragma unroll 1
    for (int jb = 0; jb < w; jb += kLuUnroll) {
#pragma unroll
      for (int o = 0; o < kLuUnroll; ++o) {
        const int jj = jb + o;
        if (jj >= w) break;
        const int j = j0 + jj;
        LU_MARK(100 + j)
        const bool act = mine && my_lp >= j;
        {  // this warp's arg-max; its winner publishes key, row (from x[o] on) and RN(1/x[o])
          const double ax = fabs(x[o]);
          const unsigned khi = (unsigned)__double2hiint(ax), klo = (unsigned)__double2loint(ax);
          const int wl = warp_argmax_key(act, khi, klo, (unsigned)my_lp);
          if (lane == (wl < 0 ? 0 : wl)) {
#pragma unroll
            for (int c = o; c < PW; c += 2)
              *reinterpret_cast<double2*>(&cv[buf][warp][c - o]) = make_double2(x[c], c + 1 < PW ? x[c + 1] : 0.0);
            cinv[buf][warp] = wl < 0 ? 0.0 : __drcp_rn(x[o]);
            chi[buf][warp] = wl < 0 ? 0u : khi;
            clo[buf][warp] = wl < 0 ? 0u : klo;
            clp[buf][warp] = wl < 0 ? 0xffffffffu : (unsigned)my_lp;
            crow[buf][warp] = tid;
          }
        }
        if (j < 32) LU_MARK(300 + 8 * j)
        __syncthreads();
        if (j < 32) LU_MARK(301 + 8 * j)
        // the NW slots, reduced the same way in every warp (all take the same decision)
        const bool in = lane < NW;
        const unsigned ghi = in ? chi[buf][lane] : 0u, glo = in ? clo[buf][lane] : 0u;
        const unsigned glp = in ? clp[buf][lane] : 0xffffffffu;
        const int ww = warp_argmax_key(in && glp != 0xffffffffu, ghi, glo, glp);
        if (ww < 0 || (chi[buf][ww] | clo[buf][ww]) == 0u) {  // exact zero pivot (kernels.hpp:235)
          if (tid == 0) set_status(st, 2 /*CQR_SINGULAR_TRIANGULAR*/, j);
          return;
        }
        const double* prow = cv[buf][ww];
        const int ps = crow[buf][ww], blp = (int)clp[buf][ww];
        const double pinv = cinv[buf][ww];
        buf ^= 1;
        if (j < 32) LU_MARK(302 + 8 * j)
        if (warp == 0) {  // U row j, panel part
          if (lane < w - jj) u[(long long)j * n + j + lane] = prow[lane];
          if (lane == 0) {
            pv[jj] = ps;
            if constexpr (SPLIT) PVg[jj] = ps;
          }
        }
        if (act && tid != ps) {
          const double mult = div_rn(x[o], prow[0], pinv);
          if constexpr (SPLIT)
            Pg[tid * PW + jj] = mult;
          else
            P[tid * kLuLdp + jj] = mult;
          if (mult != 0.0) {
#pragma unroll
            for (int c = o + 1; c < PW; ++c) x[c] = fma(-mult, prow[c - o], x[c]);
          }
        }
        if (j < 32) LU_MARK(303 + 8 * j)
        if (tid == ps)
          my_lp = j;
        else if (my_lp == j)
          my_lp = blp;  // the row at position j takes the pivot's old position
      }
#pragma unroll
      for (int c = 0; c < PW; ++c) x[c] = c + kLuUnroll < PW ? x[c + kLuUnroll] : 0.0;
    }
    if constexpr (SPLIT) {
      if (mine) LPg[tid] = my_lp;
      return;
    }
    if (mine) lpS[tid] = my_lp;
    __syncthreads();
    LU_MARK(2 + 4 * (j0 / PW))
    const int c1 = j0 + w;
    if (c1 < n) {
      // U12 = L11^-1 A12 on the pivot rows: one thread per trailing column, fma chain over
      // the panel's pivots in order, zero multipliers skipped
      for (int c = c1 + tid; c < n; c += nt) {
        double y[PW];
#pragma unroll
        for (int jj = 0; jj < PW; ++jj) y[jj] = jj < w ? W[(long long)pv[jj] * n + c] : 0.0;
#pragma unroll
        for (int jj = 1; jj < PW; ++jj) {
          if (jj < w) {
            const double* pr = P + pv[jj] * kLuLdp;
#pragma unroll
            for (int k = 0; k < jj; ++k) {
              const double mult = pr[k];
              if (mult != 0.0) y[jj] = fma(-mult, y[k], y[jj]);
            }
          }
        }
#pragma unroll
        for (int jj = 0; jj < PW; ++jj)
          if (jj < w) u[(long long)(j0 + jj) * n + c] = y[jj];
      }
      __syncthreads();
      LU_MARK(4 + 4 * (j0 / PW))
      // A22 += (-L21) U12 on DMMA for the rows still unpivoted (k = pivots in order). A work item
      // is one 8-column strip x kLuRowTiles row tiles: the strip's B fragments (U12) are loaded
      // once, then every tile's loads are issued before the interleaved DMMA chains.
      const int q = lane & 3, gr = lane >> 2;
      constexpr int kLuRowTiles = NW >= 16 ? 1 : kLuRowTilesMax;  // 512 threads: 128 registers
      const int tr = (l + 7) / 8, tc = (n - c1 + 7) / 8, nrc = (tr + kLuRowTiles - 1) / kLuRowTiles;
      for (int it = warp; it < tc * nrc; it += NW) {
        const int ct = it % tc, rc = it / tc;
        const int cc0 = c1 + ct * 8, col = cc0 + 2 * q, bc = cc0 + gr;
        double bv[PW / 4];
#pragma unroll
        for (int k4 = 0; k4 < PW / 4; ++k4) {
          const int kk = 4 * k4 + q;
          bv[k4] = (kk < w && bc < n) ? u[(long long)(j0 + kk) * n + bc] : 0.0;  // B: k = q, col = gr
        }
        double c0v[kLuRowTiles], c1v[kLuRowTiles], av[kLuRowTiles][PW / 4];
        bool live[kLuRowTiles];
        int row[kLuRowTiles];
#pragma unroll
        for (int r = 0; r < kLuRowTiles; ++r) {
          row[r] = (rc * kLuRowTiles + r) * 8 + gr;
          live[r] = row[r] < l && lpS[row[r]] >= c1;
          c0v[r] = (live[r] && col < n) ? W[(long long)row[r] * n + col] : 0.0;
          c1v[r] = (live[r] && col + 1 < n) ? W[(long long)row[r] * n + col + 1] : 0.0;
#pragma unroll
          for (int k4 = 0; k4 < PW / 4; ++k4) {
            const int kk = 4 * k4 + q;
            av[r][k4] = (row[r] < l && kk < w) ? -P[row[r] * kLuLdp + kk] : 0.0;  // A: row gr, k = q
          }
        }
#pragma unroll
        for (int k4 = 0; k4 < PW / 4; ++k4)
#pragma unroll
          for (int r = 0; r < kLuRowTiles; ++r) dmma(c0v[r], c1v[r], av[r][k4], bv[k4]);
#pragma unroll
        for (int r = 0; r < kLuRowTiles; ++r) {
          if (live[r] && col < n) W[(long long)row[r] * n + col] = c0v[r];
          if (live[r] && col + 1 < n) W[(long long)row[r] * n + col + 1] = c1v[r];
        }
      }
    }
    __syncthreads();
    LU_MARK(3 + 4 * (j0 / PW))
  }
}

// The trailing part of panel [j0, j0 + w) for lu_rot_kernel<..., SPLIT>: one CTA per 8-column strip of
// [j0 + w, n). U12 of the strip (one thread per column, fma chain over the panel's pivots in order,
// zero multipliers skipped), then A22 += (-L21) U12 on DMMA for the rows still unpivoted (k = the
// pivots in order): the same operations, in the same order, as the one-CTA kernel.
template <int PW>
__global__ void __launch_bounds__(256) lu_trail_kernel(double* W, int l, int n, int j0, int w, double* __restrict__ u,
                                                       const double* __restrict__ Pg, const int* __restrict__ LPg,
                                                       const int* __restrict__ PVg, const DevStatus* st) {
  __shared__ double sU[PW][8];
  if (failed(st)) return;
  const int c1 = j0 + w, cc0 = c1 + 8 * blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 8) {  // every row chunk of the strip recomputes the strip's U12; chunk 0 writes it
    const int c = cc0 + tid;
    double y[PW];
#pragma unroll
    for (int jj = 0; jj < PW; ++jj) y[jj] = (jj < w && c < n) ? W[(long long)PVg[jj] * n + c] : 0.0;
#pragma unroll
    for (int jj = 1; jj < PW; ++jj) {
      if (jj < w) {
        const double* pr = Pg + (long long)PVg[jj] * PW;
#pragma unroll
        for (int k = 0; k < jj; ++k) {
          const double mult = pr[k];
          if (mult != 0.0) y[jj] = fma(-mult, y[k], y[jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < PW; ++jj) {
      if (jj < w && c < n && blockIdx.y == 0) u[(long long)(j0 + jj) * n + c] = y[jj];
      sU[jj][tid] = (jj < w && c < n) ? y[jj] : 0.0;
    }
  }
  __syncthreads();
  const int q = lane & 3, gr = lane >> 2, col = cc0 + 2 * q;
  double bv[PW / 4];
#pragma unroll
  for (int k4 = 0; k4 < PW / 4; ++k4) bv[k4] = sU[4 * k4 + q][gr];  // B: k = q, col = gr
  // this CTA's row chunk: tiles [blockIdx.y * 32, +32), at most 4 per warp, all loads issued before the DMMAs
  constexpr int TPW = 4;
  double c0v[TPW], c1v[TPW], av[TPW][PW / 4];
  bool live[TPW];
  int row[TPW];
#pragma unroll
  for (int h = 0; h < TPW; ++h) {
    const int rt = blockIdx.y * 32 + warp + 8 * h;
    row[h] = rt * 8 + gr;
    live[h] = row[h] < l && LPg[row[h]] >= c1;
    c0v[h] = (live[h] && col < n) ? W[(long long)row[h] * n + col] : 0.0;
    c1v[h] = (live[h] && col + 1 < n) ? W[(long long)row[h] * n + col + 1] : 0.0;
#pragma unroll
    for (int k4 = 0; k4 < PW / 4; ++k4) {
      const int kk = 4 * k4 + q;
      av[h][k4] = (row[h] < l && kk < w) ? -Pg[(long long)row[h] * PW + kk] : 0.0;  // A: row gr, k = q
    }
  }
#pragma unroll
  for (int k4 = 0; k4 < PW / 4; ++k4)
#pragma unroll
    for (int h = 0; h < TPW; ++h) dmma(c0v[h], c1v[h], av[h][k4], bv[k4]);
#pragma unroll
  for (int h = 0; h < TPW; ++h) {
    if (live[h] && col < n) W[(long long)row[h] * n + col] = c0v[h];
    if (live[h] && col + 1 < n) W[(long long)row[h] * n + col + 1] = c1v[h];
  }
}

// l in (512, 1024]: panel launches on one CTA (one thread per row) + trailing launches over many SMs.
// work: W (l x n), then Pg (l x PW), LPg (l ints), PVg (PW ints) -- within l * (n + 33) doubles.
template <int NW, int PW>
cudaError_t launch_lu_split(const double* a1, int l, int n, double* u, double* work, DevStatus* st, cudaStream_t s) {
  double* W = work;
  double* Pg = work + (size_t)l * n;
  int* LPg = reinterpret_cast<int*>(Pg + (size_t)l * PW);
  int* PVg = LPg + l;
  cudaError_t e = cudaMemcpyAsync(W, a1, sizeof(double) * l * n, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(u, 0, sizeof(double) * n * n, s);
  if (e != cudaSuccess) return e;
  for (int j0 = 0; j0 < n; j0 += PW) {
    lu_rot_kernel<NW, PW, true><<<1, NW * 32, 0, s>>>(a1, l, n, u, W, st, j0, Pg, LPg, PVg);
    const int w = min(PW, n - j0), c1 = j0 + w;
    if (c1 < n)  // one CTA per 8-column strip and 32 row tiles (256 rows)
      lu_trail_kernel<PW><<<dim3((n - c1 + 7) / 8, (l + 255) / 256), 256, 0, s>>>(W, l, n, j0, w, u, Pg, LPg, PVg, st);
  }
  return cudaGetLastError();
}

template <int NW, int PW>
cudaError_t launch_lu_rot(const double* a1, int l, int n, double* u, double* work, DevStatus* st, cudaStream_t s) {
  const size_t smem = (size_t)l * kLuLdp * sizeof(double) + (size_t)l * sizeof(int);
  cudaError_t e = allow_max_smem(lu_rot_kernel<NW, PW>);
  if (e != cudaSuccess) return e;
  lu_rot_kernel<NW, PW><<<1, NW * 32, smem, s>>>(a1, l, n, u, work, st);
  return cudaGetLastError();
}

// Blocked right-looking Cholesky (kernels.hpp:76-90 in the oracle's pinned
// right-looking order), bitwise equal to cholesky_kernel: for each 32-row
// panel the panel rows are factored exactly as the unblocked loop (rows of R
// divided by the pivot, updates inside the panel rows), then the trailing
// upper triangle gets s(a,b) += sum_i (-r(i,a)) r(i,b) over the panel's i in
// ascending order on DMMA. S lives in the L2-resident global workspace, the
// panel rows in shared memory.
#ifndef CQR_CH_PANEL
#define CQR_CH_PANEL 16
#endif
constexpr int kChPanel = CQR_CH_PANEL;
#ifndef CQR_CH_THREADS
#define CQR_CH_THREADS 512
#endif
constexpr int kChThreads = CQR_CH_THREADS;

// SPLIT (n >= 256): one launch per panel for the panel rows (S = G copied by the launcher, the shift
// added by the first launch); chol_trail_kernel applies the trailing update over many SMs and
// chol_out_kernel writes R.
template <bool SPLIT = false>
__global__ void __launch_bounds__(kChThreads) cholesky_blocked_kernel(const double* __restrict__ g, int n,
                                                               double* __restrict__ r, double* S, int shift_mode,
                                                               double shift_value, double theory_coef,
                                                               double* shift_out, DevStatus* st, int j0s = 0) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_pd[kChPanel];  // the panel's pivots, stored after the panel
  if (failed(st)) return;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int ldp = n + 1;
  double* Pn = smem;  // kChPanel x n panel rows (stride ldp), absolute column index
  if constexpr (!SPLIT) {
    for (int i = warp; i < n; i += nw)
      for (int c = lane; c < n; c += 32) S[(long long)i * n + c] = g[(long long)i * n + c];
    __syncthreads();
  }
  if (shift_mode != 0 && tid == 0 && (!SPLIT || j0s == 0)) {
    double sh = shift_value;
    if (shift_mode == 2) {
      double tr = 0.0;
      for (int j = 0; j < n; ++j) tr += g[(long long)j * n + j];
      sh = theory_coef * tr;
    }
    for (int j = 0; j < n; ++j) S[(long long)j * n + j] += sh;
    if (shift_out) *shift_out = sh;
  }
  __syncthreads();
  for (int j0 = SPLIT ? j0s : 0; j0 < (SPLIT ? min(n, j0s + kChPanel) : n); j0 += kChPanel) {
    const int w = min(kChPanel, n - j0);
    for (int rr = warp; rr < w; rr += nw)
      for (int c = j0 + rr + lane; c < n; c += 32) Pn[rr * ldp + c] = S[(long long)(j0 + rr) * n + c];
    __syncthreads();
    // Two barriers per step: every thread takes the pivot square root and RN(1/d) itself (no
    // single-thread section and no barrier to publish them), divides its entry of row i, then
    // the remaining panel rows are updated with the divided row. The pivots go to the diagonal
    // once the panel is done.
    for (int ii = 0; ii < w; ++ii) {
      const int i = j0 + ii;
      double* Pi = Pn + ii * ldp;
      const double sii = Pi[i];
      if (!(sii > 0.0)) {  // kernels.hpp:84 (NaN included); every thread sees the same sii
        if (tid == 0) set_status(st, 1 /*CQR_CHOLESKY_BREAKDOWN*/, i);
        return;
      }
      const double d = sqrt(sii), inv = __drcp_rn(d);
      if (tid == 0) s_pd[ii] = d;  // the diagonal entry is stored after the panel (Pi[i] is still being read)
      for (int c = i + 1 + tid; c < n; c += nt) Pi[c] = div_rn(Pi[c], d, inv);
      __syncthreads();
      // update the remaining panel rows a in (i, j0+w), columns b >= a
      for (int aa = ii + 1 + warp; aa < w; aa += nw) {
        const int a = j0 + aa;
        const double ra = Pi[a];
        double* Pa = Pn + aa * ldp;
        for (int b = a + lane; b < n; b += 32) Pa[b] = fma(-ra, Pi[b], Pa[b]);
      }
      __syncthreads();
    }
    if (tid < w) Pn[tid * ldp + j0 + tid] = s_pd[tid];
    __syncthreads();
    // panel rows of R back to S
    for (int rr = warp; rr < w; rr += nw)
      for (int c = j0 + rr + lane; c < n; c += 32) S[(long long)(j0 + rr) * n + c] = Pn[rr * ldp + c];
    if constexpr (SPLIT) return;
    // trailing upper triangle: S22 += (-R12^T) R12, 8x8 tiles, k = panel rows ascending
    const int c1 = j0 + w;
    if (c1 < n) {
      const int q = lane & 3, gr = lane >> 2;
      const int T = (n - c1 + 7) / 8;
      for (int t = warp; t < T * T; t += nw) {
        const int ti = t / T, tj = t - (t / T) * T;
        if (tj < ti) continue;  // upper tiles only (diagonal tiles include a harmless lower part)
        const int a0 = c1 + 8 * ti, b0 = c1 + 8 * tj;
        const int row = a0 + gr, col = b0 + 2 * q;
        double c0v = 0.0, c1v = 0.0;
        if (row < n && col < n) c0v = S[(long long)row * n + col];
        if (row < n && col + 1 < n) c1v = S[(long long)row * n + col + 1];
#pragma unroll
        for (int k4 = 0; k4 < kChPanel / 4; ++k4) {
          const int k = 4 * k4 + q;
          const double av = (k < w && row < n) ? -Pn[k * ldp + row] : 0.0;          // A[row][k] = -R(j0+k, row)
          const double bv = (k < w && b0 + gr < n) ? Pn[k * ldp + b0 + gr] : 0.0;  // B[k][col] = R(j0+k, col)
          dmma(c0v, c1v, av, bv);
        }
        if (row < n && col < n) S[(long long)row * n + col] = c0v;
        if (row < n && col + 1 < n) S[(long long)row * n + col + 1] = c1v;
      }
    }
    __syncthreads();
  }
  for (int i = warp; i < n; i += nw)
    for (int c = lane; c < n; c += 32) r[(long long)i * n + c] = c >= i ? S[(long long)i * n + c] : 0.0;
}

__global__ void __launch_bounds__(kT) qr_kernel(const double* __restrict__ a1, int l, int n, double* __restrict__ r,
                                                double* work, int use_smem, DevStatus* st) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double scratch[33];
  __shared__ double ts[512];
  __shared__ double s_tau, s_beta, s_denom;
  __shared__ int s_zero;
  if (failed(st)) return;
  double* W = use_smem ? smem : work;  // column-major l x n
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (long long e = tid; e < (long long)l * n; e += nt) {
    const int i = (int)(e / n), c = (int)(e % n);
    W[(long long)c * l + i] = a1[e];
  }
  __syncthreads();
  const double tol = 2.2250738585072014e-308 * 2.2250738585072014e-308;  // (smallest normal)^2
  for (int j = 0; j < n; ++j) {
    double* col = W + (long long)j * l;
    double part = 0.0;
    for (int i = j + 1 + tid; i < l; i += nt) part = fma(col[i], col[i], part);
    const double tail = block_sum(part, scratch);
    if (tid == 0) {
      const double c0 = col[j];
      if (tail <= tol) {
        s_zero = 1;
        s_tau = 0.0;
        s_beta = c0;
        s_denom = 1.0;
      } else {
        s_zero = 0;
        double beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        s_beta = beta;
        s_denom = c0 - beta;
        s_tau = (beta - c0) / beta;
      }
    }
    __syncthreads();
    const double denom = s_denom, tau = s_tau;
    const int zero = s_zero;
    for (int i = j + 1 + tid; i < l; i += nt) col[i] = zero ? 0.0 : col[i] / denom;
    __syncthreads();
    if (tid == 0) col[j] = s_beta;
    if (tau != 0.0) {
      for (int c = j + 1 + warp; c < n; c += nw) {
        const double* cc = W + (long long)c * l;
        double s = 0.0;
        for (int i = j + 1 + lane; i < l; i += 32) s = fma(col[i], cc[i], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) ts[c] = tau * (cc[j] + s);
      }
      __syncthreads();
      for (int c = j + 1 + warp; c < n; c += nw) {
        double* cc = W + (long long)c * l;
        const double t = ts[c];
        for (int i = j + lane; i < l; i += 32) {
          if (i == j)
            cc[j] -= t;
          else
            cc[i] = fma(-t, col[i], cc[i]);
        }
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, c = e % n;
    r[e] = c >= i ? W[(long long)c * l + i] : 0.0;
  }
  __syncthreads();
  // normalize_r_sign (kernels.hpp:165-168)
  for (int i = tid; i < n; i += nt)
    if (r[(long long)i * n + i] < 0.0)
      for (int c = i; c < n; ++c) r[(long long)i * n + c] = -r[(long long)i * n + c];
}

// 32x32 output tile per CTA (32x8 threads, 4 rows each); k chunks of 32 staged
// in shared memory, ascending, so every element is the fma chain over k = 0..n-1.
// Blocked Householder QR (compact WY) for sketches too large for shared memory
// (e.g. c2: 512 x 256): the working matrix W (column-major) stays in the
// L2-resident workspace; each 32-column panel is copied to shared memory and
// factored there with the reflectors of qr_kernel (same beta / tau / v formulas,
// fixed reduction trees), T of Q_panel = I - V T V^T is built from V^T V, and the
// trailing columns get A2 -= V (T^T (V^T A2)) as two DMMA products. The result
// differs from the column-by-column kernel only by rounding (tolerance parity,
// like qr_kernel itself against the oracle).
constexpr int kQrB = 32;
constexpr int kQrT = 512;

// SPLIT (c2: 512 x 256): one launch per panel (the panel's reflectors, its R rows and T), V and T to
// global memory (Vg: kQrB columns of ld l, Tg: kQrB x kQrB); qr_trail_kernel applies A2 -= V (T^T
// (V^T A2)) with one CTA per 8-column strip and qr_out_kernel writes the sign-normalised R. Same
// operations in the same order per element as the one-CTA kernel.
// W (column-major, ld l) = A1 (l x n, row-major), 32 x 32 tiles through shared memory over many CTAs
__global__ void transpose_kernel(const double* __restrict__ a, int l, int n, double* __restrict__ w,
                                 const DevStatus* st) {
  __shared__ double t[32][33];
  if (failed(st)) return;
  const int i0 = blockIdx.y * 32, c0 = blockIdx.x * 32, tx = threadIdx.x, ty = threadIdx.y;
  for (int u = ty; u < 32; u += 8)
    if (i0 + u < l && c0 + tx < n) t[u][tx] = a[(long long)(i0 + u) * n + c0 + tx];
  __syncthreads();
  for (int u = ty; u < 32; u += 8)
    if (c0 + u < n && i0 + tx < l) w[(long long)(c0 + u) * l + i0 + tx] = t[tx][u];
}

template <bool SPLIT = false>
__global__ void __launch_bounds__(kQrT) qr_blocked_kernel(const double* __restrict__ a1, int l, int n,
                                                         double* __restrict__ r, double* W, DevStatus* st,
                                                         int j0s = 0, double* Vg = nullptr, double* Tg = nullptr) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double scratch[33];
  __shared__ double taus[kQrB];
  __shared__ double T[kQrB][kQrB + 1];
  __shared__ double s_tau, s_beta, s_denom;
  __shared__ int s_zero;
  if (failed(st)) return;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int ldr = l + 4;             // panel column stride (bank spread for the DMMA fragments)
  double* Pn = smem;                 // kQrB columns of (l - j0) rows
  double* Ys = smem + kQrB * ldr;    // kQrB x n (row stride n + 4): V^T A2, then T^T V^T A2
  const int ldy = n + 4;
  if (!SPLIT) {  // (SPLIT: transpose_kernel has written W)
    for (long long e = tid; e < (long long)l * n; e += nt) {
      const int i = (int)(e / n), c = (int)(e % n);
      W[(long long)c * l + i] = a1[e];
    }
    __syncthreads();
  }
  const double tol = 2.2250738585072014e-308 * 2.2250738585072014e-308;  // (smallest normal)^2
  for (int j0 = SPLIT ? j0s : 0; j0 < (SPLIT ? min(n, j0s + kQrB) : n); j0 += kQrB) {
    const int b = min(kQrB, n - j0), rp = l - j0;  // panel width, panel rows
    for (int e = tid; e < b * rp; e += nt) {
      const int c = e / rp, i = e - (e / rp) * rp;
      Pn[c * ldr + i] = W[(long long)(j0 + c) * l + j0 + i];
    }
    __syncthreads();
    // ---- panel: Householder reflectors column by column (qr_kernel's arithmetic)
    for (int jj = 0; jj < b; ++jj) {
      double* col = Pn + jj * ldr;
      double part = 0.0;
      for (int i = jj + 1 + tid; i < rp; i += nt) part = fma(col[i], col[i], part);
      const double tail = block_sum(part, scratch);
      if (tid == 0) {
        const double c0 = col[jj];
        if (tail <= tol) {
          s_zero = 1;
          s_tau = 0.0;
          s_beta = c0;
          s_denom = 1.0;
        } else {
          s_zero = 0;
          double beta = sqrt(c0 * c0 + tail);
          if (c0 >= 0.0) beta = -beta;
          s_beta = beta;
          s_denom = c0 - beta;
          s_tau = (beta - c0) / beta;
        }
        taus[jj] = s_tau;
      }
      __syncthreads();
      const double denom = s_denom, tau = s_tau;
      const int zero = s_zero;
      for (int i = jj + 1 + tid; i < rp; i += nt) col[i] = zero ? 0.0 : col[i] / denom;
      __syncthreads();
      if (tid == 0) col[jj] = s_beta;
      if (tau != 0.0) {  // warps own the remaining panel columns: dot, then axpy
        for (int c = jj + 1 + warp; c < b; c += nw) {
          double* cc = Pn + c * ldr;
          double sdot = 0.0;
          for (int i = jj + 1 + lane; i < rp; i += 32) sdot = fma(col[i], cc[i], sdot);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
          const double t = tau * (cc[jj] + sdot);
          __syncwarp();
          for (int i0 = jj; i0 < rp; i0 += 128) {  // four rows per lane and pass, loads ahead of the stores
            double cv[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + lane + 32 * u;
              cv[u] = (i > jj && i < rp) ? col[i] : 0.0;
              xv[u] = i < rp ? cc[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < rp) cc[i] = (i == jj) ? xv[u] - t : fma(-t, cv[u], xv[u]);
            }
          }
        }
      }
      __syncthreads();
    }
    // R rows of the panel back to W; V (unit diagonal, zeros above) stays in Pn
    for (int e = tid; e < b * b; e += nt) {
      const int c = e / b, i = e - (e / b) * b;
      if (i <= c) W[(long long)(j0 + c) * l + j0 + i] = Pn[c * ldr + i];
    }
    __syncthreads();
    for (int e = tid; e < b * rp; e += nt) {
      const int c = e / rp, i = e - (e / rp) * rp;
      if (i <= c) Pn[c * ldr + i] = i == c ? 1.0 : 0.0;
    }
    for (int e = tid; e < (kQrB - b) * rp; e += nt) Pn[(b + e / rp) * ldr + e % rp] = 0.0;  // short last panel
    __syncthreads();
    const int c1 = j0 + b;
    if (c1 < n) {
      // ---- T (upper triangular, kQrB x kQrB): T[k][k] = tau_k, T[0:k][k] = -tau_k T[0:k][0:k] (V^T v_k)[0:k]
      for (int e = warp; e < kQrB * kQrB; e += nw) {  // G[i][k] = v_i . v_k for i < k (in T's lower half)
        const int i = e / kQrB, k = e - (e / kQrB) * kQrB;
        if (i >= k || k >= b) continue;
        double sdot = 0.0;
        for (int rr = k + lane; rr < rp; rr += 32) sdot = fma(Pn[i * ldr + rr], Pn[k * ldr + rr], sdot);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
        if (lane == 0) T[k][i] = sdot;
      }
      __syncthreads();
      if (warp == 0) {
        for (int k = 0; k < kQrB; ++k) {
          double v = 0.0;
          if (k < b && lane < k) {
            for (int jx = lane; jx < k; ++jx) v = fma(T[lane][jx], T[k][jx], v);
            v *= -taus[k];
          }
          __syncwarp();
          if (lane < k) T[lane][k] = k < b ? v : 0.0;
          if (lane == k) T[k][k] = k < b ? taus[k] : 0.0;
          __syncwarp();
        }
      }
      __syncthreads();
      if constexpr (SPLIT) {  // V (rows [0, rp) of the panel, unit diagonal) and T for qr_trail_kernel
        for (int e = tid; e < kQrB * rp; e += nt) {
          const int c = e / rp, i = e - (e / rp) * rp;
          Vg[(long long)c * l + i] = Pn[c * ldr + i];
        }
        for (int e = tid; e < kQrB * kQrB; e += nt) Tg[e] = T[e / kQrB][e % kQrB];
        return;
      }
      // ---- Y = V^T A2 (kQrB x n2, k over the panel rows) on DMMA
      const int q = lane & 3, gr = lane >> 2;
      const int n2 = n - c1, tcn = (n2 + 7) / 8;
      for (int t = warp; t < (kQrB / 8) * tcn; t += nw) {
        const int kt = t / tcn, ct = t - (t / tcn) * tcn;
        const int cbase = c1 + ct * 8;
        double y0 = 0.0, y1 = 0.0;
        const int cb = cbase + gr;
        for (int r0 = 0; r0 < rp; r0 += 32) {  // 8 k-steps per pass, every load issued before the chain
          double av[8], bv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rr = r0 + 4 * u + q;
            av[u] = rr < rp ? Pn[(kt * 8 + gr) * ldr + rr] : 0.0;             // A = V^T: row k, col r
            bv[u] = (rr < rp && cb < n) ? W[(long long)cb * l + j0 + rr] : 0.0;  // B = A2: row r, col c
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) dmma(y0, y1, av[u], bv[u]);
        }
        const int cc = ct * 8 + 2 * q;
        Ys[(kt * 8 + gr) * ldy + cc] = y0;
        Ys[(kt * 8 + gr) * ldy + cc + 1] = y1;
      }
      __syncthreads();
      // ---- Y <- T^T Y (in place, column by column of Y)
      for (int c = tid; c < n2; c += nt) {  // k descending: z_k needs y_0..y_k, all still unwritten
        for (int k = kQrB - 1; k >= 0; --k) {
          double z = 0.0;
          for (int i = 0; i <= k; ++i) z = fma(T[i][k], Ys[i * ldy + c], z);
          Ys[k * ldy + c] = z;
        }
      }
      __syncthreads();
      // ---- A2 -= V Z on DMMA (rows of the panel range, trailing columns)
      const int trt = (rp + 7) / 8, ntile = trt * tcn;
      for (int t0 = warp; t0 < ntile; t0 += 2 * nw) {  // two tiles per pass: their global loads overlap
        double c0v[2], c1v[2], av[2][kQrB / 4], bv[2][kQrB / 4];
        int rowl[2], col[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = t0 + h * nw;
          const bool live = t < ntile;
          const int rt = live ? t / tcn : 0, ct = live ? t - (t / tcn) * tcn : 0;
          rowl[h] = live ? rt * 8 + gr : rp;
          col[h] = c1 + ct * 8 + 2 * q;
          c0v[h] = (rowl[h] < rp && col[h] < n) ? W[(long long)col[h] * l + j0 + rowl[h]] : 0.0;
          c1v[h] = (rowl[h] < rp && col[h] + 1 < n) ? W[(long long)(col[h] + 1) * l + j0 + rowl[h]] : 0.0;
#pragma unroll
          for (int k4 = 0; k4 < kQrB / 4; ++k4) {
            const int kk = 4 * k4 + q;
            av[h][k4] = rowl[h] < rp ? -Pn[kk * ldr + rowl[h]] : 0.0;  // A = -V: row r, col k
            const int cz = ct * 8 + gr;
            bv[h][k4] = cz < n2 ? Ys[kk * ldy + cz] : 0.0;          // B = Z: row k, col c
          }
        }
#pragma unroll
        for (int k4 = 0; k4 < kQrB / 4; ++k4)
#pragma unroll
          for (int h = 0; h < 2; ++h) dmma(c0v[h], c1v[h], av[h][k4], bv[h][k4]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (rowl[h] < rp && col[h] < n) W[(long long)col[h] * l + j0 + rowl[h]] = c0v[h];
          if (rowl[h] < rp && col[h] + 1 < n) W[(long long)(col[h] + 1) * l + j0 + rowl[h]] = c1v[h];
        }
      }
    }
    __syncthreads();
  }
  if constexpr (SPLIT) return;
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, c = e % n;
    r[e] = c >= i ? W[(long long)c * l + i] : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += nt)  // normalize_r_sign (kernels.hpp:165-168)
    if (r[(long long)i * n + i] < 0.0)
      for (int c = i; c < n; ++c) r[(long long)i * n + c] = -r[(long long)i * n + c];
}

__global__ void triangular_product_kernel(const double* __restrict__ left, const double* __restrict__ right, int n,
                                          double* __restrict__ out, const DevStatus* st) {
  __shared__ double sl[32][33], sr[32][33];
  if (failed(st)) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const bool any = j0 + 31 >= i0;  // tile touches the upper triangle
  for (int k0 = 0; any && k0 < n; k0 += 32) {
    for (int u = 0; u < 4; ++u) {
      const int r = ty + 8 * u;
      sl[r][tx] = (i0 + r < n && k0 + tx < n) ? left[(long long)(i0 + r) * n + k0 + tx] : 0.0;
      sr[r][tx] = (k0 + r < n && j0 + tx < n) ? right[(long long)(k0 + r) * n + j0 + tx] : 0.0;
    }
    __syncthreads();
    const int kk = min(32, n - k0);
    for (int k = 0; k < kk; ++k)
      for (int u = 0; u < 4; ++u) acc[u] = fma(sl[ty + 8 * u][k], sr[k][tx], acc[u]);
    __syncthreads();
  }
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + ty + 8 * u, j = j0 + tx;
    if (i < n && j < n) out[(long long)i * n + j] = (j >= i) ? acc[u] : 0.0;
  }
}

__global__ void normalize_sign_kernel(double* r, int n, double* sgn, const DevStatus* st) {
  __shared__ double s[512];
  if (failed(st)) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = r[(long long)i * n + i] < 0.0 ? -1.0 : 1.0;
    s[i] = v;
    sgn[i] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < n; i += nw)
    if (s[i] < 0.0)
      for (int c = i + lane; c < n; c += 32) r[(long long)i * n + c] = -r[(long long)i * n + c];
}

template <typename K, typename... Args>
cudaError_t launch_small(K kernel, size_t bytes, cudaStream_t s, Args... args) {
  const int use_smem = bytes <= kSmemCap ? 1 : 0;
  const size_t smem = use_smem ? bytes : 0;
  cudaError_t e = allow_max_smem(kernel);
  if (e != cudaSuccess) return e;
  (void)use_smem;
  kernel<<<1, kT, smem, s>>>(args...);
  return cudaGetLastError();
}

}  // namespace

size_t small_work_doubles(int rows, int n) { return (size_t)rows * n; }
// workspace of launch_qr_r / launch_lu_u: W (l x n) + panel buffers (the split QR: V, kQrB x l, and T)
size_t qr_work_doubles(int l, int n) { return (size_t)l * (n + 33) + (size_t)kQrB * kQrB; }

// Trailing update of cholesky_blocked_kernel<true>'s panel [j0, j0 + w): one warp per upper 8x8 tile of
// [c1, n)^2, S(a,b) += sum over the panel rows i ascending of (-R(i,a)) R(i,b) on DMMA (the blocked
// kernel's tile loop, with the panel rows read from S).
__global__ void __launch_bounds__(256) chol_trail_kernel(double* S, int n, int j0, int w, const DevStatus* st) {
  if (failed(st)) return;
  const int lane = threadIdx.x & 31;
  const int c1 = j0 + w;
  const int T = (n - c1 + 7) / 8;
  int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T * (T + 1) / 2) return;
  int ti = 0;  // upper tile t in row-major order: row ti has T - ti tiles
  while (t >= T - ti) {
    t -= T - ti;
    ++ti;
  }
  const int tj = ti + t;
  const int q = lane & 3, gr = lane >> 2;
  const int a0 = c1 + 8 * ti, b0 = c1 + 8 * tj;
  const int row = a0 + gr, col = b0 + 2 * q;
  double c0v = 0.0, c1v = 0.0;
  if (row < n && col < n) c0v = S[(long long)row * n + col];
  if (row < n && col + 1 < n) c1v = S[(long long)row * n + col + 1];
#pragma unroll
  for (int k4 = 0; k4 < kChPanel / 4; ++k4) {
    const int k = 4 * k4 + q;
    const double av = (k < w && row < n) ? -S[(long long)(j0 + k) * n + row] : 0.0;
    const double bv = (k < w && b0 + gr < n) ? S[(long long)(j0 + k) * n + b0 + gr] : 0.0;
    dmma(c0v, c1v, av, bv);
  }
  if (row < n && col < n) S[(long long)row * n + col] = c0v;
  if (row < n && col + 1 < n) S[(long long)row * n + col + 1] = c1v;
}

// Register-resident Cholesky for n <= 128 (c1: 128, c3: 64), two barriers per step and a short critical
// path. S's upper triangle is cut into SEG-column segments of each row; one thread holds one segment in
// registers (rows packed greedily into warps). Step i: thread t < n - i reads s(i,i) (left in shared
// memory by row i's lanes), takes d = sqrt(s(i,i)) (kernels.hpp:84-86) and RN(1/d), and divides s(i,i+t)
// (correctly rounded, as `/`; t = 0 writes d) into the shared row R(i,:); barrier; every row a > i applies
// s(a,b) = fma(-r(i,a), r(i,b), s(a,b)) to its segment, and row i+1's lanes leave their updated entries in
// shared memory; barrier. Each entry thus sees the fma chain over i = 0..a-1 in order and one division:
// the same operations as cholesky_kernel (bitwise). (A dataflow variant -- one pivot warp, mbarriers per
// row instead of block barriers -- measured slower: 111 vs 89 us at n = 128.)
template <int SEG>
__host__ __device__ inline int chol_reg_warps(int n, int warp = -1, int lane = 0, int* my_a = nullptr,
                                              int* my_sb = nullptr) {
  const int nseg = (n + SEG - 1) / SEG;
  int w = 0, pos = 0;
  for (int a = 0; a < n; ++a) {
    const int s = nseg - a / SEG;
    if (pos + s > 32) {
      ++w;
      pos = 0;
    }
    if (w == warp && lane >= pos && lane < pos + s) {
      *my_a = a;
      *my_sb = a / SEG + (lane - pos);
    }
    pos += s;
  }
  return w + 1;
}
constexpr int kChRegMaxN = 128;
template <int SEG>
__device__ __forceinline__ int chol_rb(int b) {  // shared slot of column b: segments 2 doubles apart (no bank conflicts)
  return (b / SEG) * (SEG + 2) + b % SEG;
}
template <int SEG>
__global__ void __launch_bounds__(608) chol_reg_kernel(const double* __restrict__ g, int n, double* __restrict__ r,
                                                       int shift_mode, double shift_value, double theory_coef,
                                                       double* shift_out, DevStatus* st) {
  constexpr int RB = (kChRegMaxN / SEG) * (SEG + 2);
  __shared__ __align__(16) double rowbuf[2][RB];  // R(i, :), double-buffered
  __shared__ __align__(16) double und[RB];        // s(i, :) before the division
  __shared__ double s_sh;
  if (failed(st)) return;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  int my_a = -1, my_sb = 0;
  chol_reg_warps<SEG>(n, warp, lane, &my_a, &my_sb);
  const int c0 = SEG * my_sb, s0 = (SEG + 2) * my_sb;
  double x[SEG];
#pragma unroll
  for (int k = 0; k < SEG; ++k) x[k] = (my_a >= 0 && c0 + k < n) ? g[(long long)my_a * n + c0 + k] : 0.0;
  for (int i = warp; i < n; i += nt >> 5)  // R's strict lower triangle
    for (int c = lane; c < i; c += 32) r[(long long)i * n + c] = 0.0;
  if (tid == 0) {
    double sh = shift_value;
    if (shift_mode == 2) {  // theory shift from trace(G) (cholqr.cpp:21-26), as cholesky_kernel
      double tr = 0.0;
      for (int j = 0; j < n; ++j) tr += g[(long long)j * n + j];
      sh = theory_coef * tr;
    }
    s_sh = sh;
    if (shift_mode != 0 && shift_out) *shift_out = sh;
  }
  __syncthreads();
  if (shift_mode != 0 && my_a >= 0 && my_sb == my_a / SEG) {
    const int o = my_a % SEG;
#pragma unroll
    for (int k = 0; k < SEG; ++k)
      if (k == o) x[k] += s_sh;
  }
  if (my_a == 0) {
#pragma unroll
    for (int k = 0; k < SEG; k += 2) *reinterpret_cast<double2*>(und + s0 + k) = make_double2(x[k], x[k + 1]);
  }
  const int ra_slot = my_a >= 0 ? chol_rb<SEG>(my_a) : 0;
  for (int i = 0; i < n; ++i) {
    double* rb = rowbuf[i & 1];
    __syncthreads();
    const double sii = und[chol_rb<SEG>(i)];
    if (!(sii > 0.0)) {  // kernels.hpp:84 (NaN included); every thread sees the same value
      if (tid == 0) set_status(st, 1 /*CQR_CHOLESKY_BREAKDOWN*/, i);
      return;
    }
    if (tid < n - i) {  // the pivot and the divisions of row i, one entry per thread
      const double d = sqrt(sii), inv = __drcp_rn(d);
      const bool safe = fabs(d) >= 0x1p-500 && fabs(d) <= 0x1p+500;
      const int b = i + tid, slot = chol_rb<SEG>(b);
      const double q = tid == 0 ? d : tri::fast_div(und[slot], d, inv, safe);
      rb[slot] = q;
      r[(long long)i * n + b] = q;
    }
    __syncthreads();
    if (my_a > i) {
      const double ra = rb[ra_slot];
#pragma unroll
      for (int k = 0; k < SEG; k += 2) {
        const double2 rv = *reinterpret_cast<const double2*>(rb + s0 + k);
        x[k] = fma(-ra, rv.x, x[k]);
        x[k + 1] = fma(-ra, rv.y, x[k + 1]);
      }
      if (my_a == i + 1) {
#pragma unroll
        for (int k = 0; k < SEG; k += 2) *reinterpret_cast<double2*>(und + s0 + k) = make_double2(x[k], x[k + 1]);
      }
    }
  }
}

__global__ void chol_out_kernel(const double* __restrict__ S, int n, double* __restrict__ r, const DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) r[(long long)i * n + c] = c >= i ? S[(long long)i * n + c] : 0.0;
}

cudaError_t launch_cholesky(const double* g, int n, double* r, double* work, int shift_mode, double shift_value,
                            double theory_coef, double* shift_out, DevStatus* st, cudaStream_t s) {
  static const int split_min = [] {  // A/B runs: CQR_CHOL_SPLIT_MIN=n0 splits from n0 columns on
    const char* v = std::getenv("CQR_CHOL_SPLIT_MIN");
    return v ? std::atoi(v) : 256;
  }();
  static const bool reg_off = std::getenv("CQR_CHOL_LEGACY") != nullptr;  // A/B runs: the blocked kernels
  if (!reg_off && n <= 128) {
    chol_reg_kernel<16><<<1, 32 * chol_reg_warps<16>(n), 0, s>>>(g, n, r, shift_mode, shift_value, theory_coef,
                                                                 shift_out, st);
    return cudaGetLastError();
  }
  if (n >= split_min && n > 64) {
    const size_t smem = (size_t)kChPanel * (n + 1) * sizeof(double);
    cudaError_t e =
        allow_max_smem(cholesky_blocked_kernel<true>);
    if (e == cudaSuccess) e = cudaMemcpyAsync(work, g, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    for (int j0 = 0; j0 < n; j0 += kChPanel) {
      cholesky_blocked_kernel<true><<<1, kChThreads, smem, s>>>(g, n, r, work, shift_mode, shift_value, theory_coef,
                                                                shift_out, st, j0);
      const int w = min(kChPanel, n - j0), c1 = j0 + w;
      if (c1 < n) {
        const int T = (n - c1 + 7) / 8;
        chol_trail_kernel<<<(T * (T + 1) / 2 + 7) / 8, 256, 0, s>>>(work, n, j0, w, st);
      }
    }
    chol_out_kernel<<<dim3((n + 127) / 128, n), 128, 0, s>>>(work, n, r, st);
    return cudaGetLastError();
  }
  if (n > 64) {
    const size_t smem = (size_t)kChPanel * (n + 1) * sizeof(double);
    cudaError_t e =
        allow_max_smem(cholesky_blocked_kernel<false>);
    if (e != cudaSuccess) return e;
    cholesky_blocked_kernel<false><<<1, kChThreads, smem, s>>>(g, n, r, work, shift_mode, shift_value, theory_coef, shift_out, st);
    return cudaGetLastError();
  }
  const size_t bytes = (size_t)n * n * sizeof(double);
  const int use_smem = bytes <= kSmemCap;
  return launch_small(cholesky_kernel, bytes, s, g, n, r, work, use_smem, shift_mode, shift_value, theory_coef,
                      shift_out, st);
}

cudaError_t launch_lu_u(const double* a1, int l, int n, double* u, double* work, DevStatus* st, cudaStream_t s) {
  static const bool legacy = std::getenv("CQR_LU_LEGACY") != nullptr;  // tuning: the swapping blocked kernel
  static const bool split_all = std::getenv("CQR_LU_SPLIT_ALL") != nullptr;  // A/B runs: split launches for l <= 512
  if (!legacy && split_all && l <= 256) return launch_lu_split<8, kLuRotPanel>(a1, l, n, u, work, st, s);
  if (!legacy && split_all && l <= 512) return launch_lu_split<16, kLuRotPanel>(a1, l, n, u, work, st, s);
  if (!legacy && l <= 512 && (size_t)l * kLuLdp * sizeof(double) + (size_t)l * sizeof(int) <= 220 * 1024) {
    // as few warps as rows need: the per-step barriers and arg-max dominate (8 vs 16 warps at
    // l = 256: 276 vs 332 us)
    if (l <= 128) return launch_lu_rot<4, kLuRotPanel>(a1, l, n, u, work, st, s);
    if (l <= 256) return launch_lu_rot<8, kLuRotPanel>(a1, l, n, u, work, st, s);
    return launch_lu_rot<16, kLuRotPanel>(a1, l, n, u, work, st, s);
  }
  // taller sketches (c4: 768 x 512): panel launches + trailing launches over many SMs (the one-CTA
  // swapping kernel did the 768-row trailing updates on one SM: 4.97 ms)
  static const bool no_split = std::getenv("CQR_LU_NO_SPLIT") != nullptr;  // A/B runs
  if (!legacy && !no_split && l <= 768) return launch_lu_split<24, kLuRotPanel>(a1, l, n, u, work, st, s);
  if (!legacy && !no_split && l <= 1024) return launch_lu_split<32, kLuRotPanel>(a1, l, n, u, work, st, s);
  {
    const bool fits = (size_t)l * kLuLdp * sizeof(double) <= 220 * 1024;
    const size_t smem = fits ? (size_t)l * kLuLdp * sizeof(double) : 0;
    // work holds l*n doubles for W, followed by the tall panel when it does not fit
    if (fits) {
      cudaError_t e =
          allow_max_smem(lu_blocked_kernel<true>);
      if (e != cudaSuccess) return e;
      lu_blocked_kernel<true><<<1, 512, smem, s>>>(a1, l, n, u, work, nullptr, st);
    } else {
      lu_blocked_kernel<false><<<1, 512, 0, s>>>(a1, l, n, u, work, work + (size_t)l * n, st);
    }
    return cudaGetLastError();
  }
  const int rs = (int)std::min<size_t>((size_t)l, kSmemCap / ((size_t)n * sizeof(double)));
  const size_t smem = (size_t)rs * n * sizeof(double);
  cudaError_t e = allow_max_smem(lu_kernel);
  if (e != cudaSuccess) return e;
  lu_kernel<<<1, kT, smem, s>>>(a1, l, n, u, work, rs, st);
  return cudaGetLastError();
}

// The trailing update of qr_blocked_kernel<true>'s panel [j0, j0 + kQrB): one CTA (8 warps) per
// 8-column strip of [j0 + b, n); the blocked kernel's Y / T^T Y / A2 -= V Z steps for that strip.
__global__ void __launch_bounds__(256) qr_trail_kernel(double* W, int l, int n, int j0, int b,
                                                       const double* __restrict__ Vg, const double* __restrict__ Tg,
                                                       const DevStatus* st) {
  __shared__ double Ys[kQrB][9];
  __shared__ double Ts[kQrB][kQrB + 1];
  if (failed(st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, gr = lane >> 2;
  const int rp = l - j0, c1 = j0 + b, cbase = c1 + 8 * blockIdx.x;
  for (int e = tid; e < kQrB * kQrB; e += 256) Ts[e / kQrB][e % kQrB] = Tg[e];
  if (warp < kQrB / 8) {  // Y tile kt = warp: rows k of V^T, the strip's 8 columns
    const int kt = warp, cb = cbase + gr;
    double y0 = 0.0, y1 = 0.0;
    for (int r0 = 0; r0 < rp; r0 += 32) {
      double av[8], bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int rr = r0 + 4 * u + q;
        av[u] = rr < rp ? Vg[(long long)(kt * 8 + gr) * l + rr] : 0.0;
        bv[u] = (rr < rp && cb < n) ? W[(long long)cb * l + j0 + rr] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma(y0, y1, av[u], bv[u]);
    }
    Ys[kt * 8 + gr][2 * q] = y0;
    Ys[kt * 8 + gr][2 * q + 1] = y1;
  }
  __syncthreads();
  if (tid < 8) {  // Y <- T^T Y, column tid, k descending
    for (int k = kQrB - 1; k >= 0; --k) {
      double z = 0.0;
      for (int i = 0; i <= k; ++i) z = fma(Ts[i][k], Ys[i][tid], z);
      Ys[k][tid] = z;
    }
  }
  __syncthreads();
  double bv[kQrB / 4];
#pragma unroll
  for (int k4 = 0; k4 < kQrB / 4; ++k4) bv[k4] = cbase + gr < n ? Ys[4 * k4 + q][gr] : 0.0;  // B = Z: row k, col c
  const int col = cbase + 2 * q;
  for (int rt = warp; rt * 8 < rp; rt += 8) {
    const int rowl = rt * 8 + gr;
    double c0v = (rowl < rp && col < n) ? W[(long long)col * l + j0 + rowl] : 0.0;
    double c1v = (rowl < rp && col + 1 < n) ? W[(long long)(col + 1) * l + j0 + rowl] : 0.0;
#pragma unroll
    for (int k4 = 0; k4 < kQrB / 4; ++k4) {
      const int kk = 4 * k4 + q;
      const double av = rowl < rp ? -Vg[(long long)kk * l + rowl] : 0.0;  // A = -V: row r, col k
      dmma(c0v, c1v, av, bv[k4]);
    }
    if (rowl < rp && col < n) W[(long long)col * l + j0 + rowl] = c0v;
    if (rowl < rp && col + 1 < n) W[(long long)(col + 1) * l + j0 + rowl] = c1v;
  }
}

__global__ void qr_out_kernel(const double* __restrict__ W, int l, int n, double* __restrict__ r,
                              const DevStatus* st) {  // R = upper part of W, rows sign-normalised (kernels.hpp:165-168)
  if (failed(st)) return;
  const int i = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double sg = W[(long long)i * l + i] < 0.0 ? -1.0 : 1.0;
  r[(long long)i * n + c] = c >= i ? sg * W[(long long)c * l + i] : 0.0;
}

// Householder R of a sketch that fits in shared memory, one barrier per column: warp w owns the columns
// c = w (mod NW). The owner of column j has applied reflectors 0 .. j-1 to it by itself, so it forms
// reflector j (tail norm by a lane-strided sum and shuffles, beta / tau / v as qr_kernel) right after its
// own update of column j in step j-1 -- before its other columns -- and one barrier publishes v_j; every
// warp then applies it to its own columns (dot product over the rows, rank-1 update). Same reflector
// formulas as qr_kernel and the oracle; the reductions are trees (tolerance parity, R <= 1e-13).
template <int NW>
__global__ void __launch_bounds__(NW * 32) qr_warp_kernel(const double* __restrict__ a1, int l, int n,
                                                          double* __restrict__ r, DevStatus* st) {
  extern __shared__ __align__(16) double W[];  // column-major, leading dimension ld = l | 1 (odd: no bank conflicts)
  __shared__ double s_tau[2];
  if (failed(st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ld = l | 1;
  for (long long e = tid; e < (long long)l * n; e += NW * 32) {
    const int i = (int)(e / n), c = (int)(e % n);
    W[(long long)c * ld + i] = __ldg(a1 + e);
  }
  __syncthreads();
  const double tol = 2.2250738585072014e-308 * 2.2250738585072014e-308;  // (smallest normal)^2
  // reflector j by the owner warp (column j up to date): v below the diagonal, beta on it, tau published
  auto reflect = [&](int j) {
    double* col = W + (long long)j * ld;
    double part = 0.0;
    for (int i = j + 1 + lane; i < l; i += 32) part = fma(col[i], col[i], part);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double c0 = col[j];
    double tau, beta, denom;
    bool zero;
    if (part <= tol) {
      zero = true;
      tau = 0.0;
      beta = c0;
      denom = 1.0;
    } else {
      zero = false;
      beta = sqrt(c0 * c0 + part);
      if (c0 >= 0.0) beta = -beta;
      denom = c0 - beta;
      tau = (beta - c0) / beta;
    }
    const double rden = 1.0 / denom;  // v = x / (c0 - beta) as x * RN(1 / (c0 - beta)): within an ulp
    for (int i = j + 1 + lane; i < l; i += 32) col[i] = zero ? 0.0 : col[i] * rden;
    __syncwarp();  // every lane has read c0
    if (lane == 0) {
      col[j] = beta;
      s_tau[j & 1] = tau;
    }
    __syncwarp();
  };
  // H_j applied to column c (c > j): t = tau (W(j, c) + v^T W(j+1.., c)), W(.., c) -= t v
  auto apply = [&](int j, int c, double tau) {
    const double* v = W + (long long)j * ld;
    double* cc = W + (long long)c * ld;
    double sacc = 0.0;
    for (int i = j + 1 + lane; i < l; i += 32) sacc = fma(v[i], cc[i], sacc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    const double t = tau * (cc[j] + sacc);
    __syncwarp();
    if (lane == 0) cc[j] -= t;
    for (int i = j + 1 + lane; i < l; i += 32) cc[i] = fma(-t, v[i], cc[i]);
    __syncwarp();
  };
  // the same for columns c, c + S, ..., c + (cnt - 1) S at once (independent chains: ILP), cnt <= 4
  auto apply4 = [&](int j, int c, int S, int cnt, double tau) {
    const double* v = W + (long long)j * ld;
    double sacc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = j + 1 + lane; i < l; i += 32) {
      const double vi = v[i];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < cnt) sacc[k] = fma(vi, W[(long long)(c + S * k) * ld + i], sacc[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int k = 0; k < 4; ++k) sacc[k] += __shfl_xor_sync(0xffffffffu, sacc[k], o);
    double t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = k < cnt ? tau * (W[(long long)(c + S * k) * ld + j] + sacc[k]) : 0.0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < cnt && lane == k) W[(long long)(c + S * k) * ld + j] -= t[k];
    for (int i = j + 1 + lane; i < l; i += 32) {
      const double vi = v[i];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < cnt) {
          double* p = W + (long long)(c + S * k) * ld + i;
          *p = fma(-t[k], vi, *p);
        }
    }
    __syncwarp();
  };
  if (warp == 0) reflect(0);
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double tau = s_tau[j & 1];
    // step j: warp (j + 1) % NW brings column j + 1 up to date and forms reflector j + 1; the other
    // NW - 1 warps share the columns j + 2 .. n - 1 (W lives in shared memory: any warp may take any column)
    const int owner = (j + 1) % NW;
    if (warp == owner) {
      if (j + 1 < n) {
        if (tau != 0.0) apply(j, j + 1, tau);
        reflect(j + 1);
      }
    } else if (tau != 0.0) {
      const int rank = (warp - owner + NW) % NW - 1;  // 0 .. NW - 2
      for (int c = j + 2 + rank; c < n; c += 4 * (NW - 1))
        apply4(j, c, NW - 1, min(4, (n - c + NW - 2) / (NW - 1)), tau);
    }
    __syncthreads();
  }
  // R: the upper triangle, rows with a negative diagonal negated (normalize_r_sign, kernels.hpp:165-168)
  for (int e = tid; e < n * n; e += NW * 32) {
    const int i = e / n, c = e % n;
    const double sg = W[(long long)i * ld + i] < 0.0 ? -1.0 : 1.0;
    r[e] = c >= i ? sg * W[(long long)c * ld + i] : 0.0;
  }
}

cudaError_t launch_qr_r(const double* a1, int l, int n, double* r, double* work, DevStatus* st, cudaStream_t s) {
  if (n > 512) return cudaErrorInvalidValue;
  const size_t bytes = (size_t)l * n * sizeof(double);
  const int use_smem = bytes <= kSmemCap;
  const size_t bsmem = ((size_t)kQrB * (l + 4) + (size_t)kQrB * (n + 4)) * sizeof(double);
  static const bool no_split = std::getenv("CQR_QR_NO_SPLIT") != nullptr;  // A/B runs: the one-CTA kernel
  if (!use_smem && bsmem <= 200 * 1024 && !no_split) {  // per-panel launches, trailing update over many SMs
    cudaError_t e =
        allow_max_smem(qr_blocked_kernel<true>);
    if (e != cudaSuccess) return e;
    double* Vg = work + (size_t)l * n;  // kQrB x l, then Tg (kQrB x kQrB): qr_work_doubles
    double* Tg = Vg + (size_t)kQrB * l;
    transpose_kernel<<<dim3((n + 31) / 32, (l + 31) / 32), dim3(32, 8), 0, s>>>(a1, l, n, work, st);
    for (int j0 = 0; j0 < n; j0 += kQrB) {
      qr_blocked_kernel<true><<<1, kQrT, bsmem, s>>>(a1, l, n, r, work, st, j0, Vg, Tg);
      const int b = min(kQrB, n - j0), c1 = j0 + b;
      if (c1 < n) qr_trail_kernel<<<(n - c1 + 7) / 8, 256, 0, s>>>(work, l, n, j0, b, Vg, Tg, st);
    }
    qr_out_kernel<<<dim3((n + 127) / 128, n), 128, 0, s>>>(work, l, n, r, st);
    return cudaGetLastError();
  }
  if (!use_smem && bsmem <= 200 * 1024) {  // blocked: the panel and V^T A2 in shared memory
    cudaError_t e =
        allow_max_smem(qr_blocked_kernel<false>);
    if (e != cudaSuccess) return e;
    qr_blocked_kernel<false><<<1, kQrT, bsmem, s>>>(a1, l, n, r, work, st);
    return cudaGetLastError();
  }
  static const bool legacy_qr = std::getenv("CQR_QR_LEGACY") != nullptr;  // A/B runs: the one-barrier-per-step kernel off
  const size_t wbytes = (size_t)(l | 1) * n * sizeof(double);
  if (!legacy_qr && wbytes <= kSmemCap) {
#ifndef CQR_QR_WARPS
#define CQR_QR_WARPS 16
#endif
    cudaError_t e =
        allow_max_smem(qr_warp_kernel<CQR_QR_WARPS>);
    if (e != cudaSuccess) return e;
    qr_warp_kernel<CQR_QR_WARPS><<<1, CQR_QR_WARPS * 32, wbytes, s>>>(a1, l, n, r, st);
    return cudaGetLastError();
  }
  return launch_small(qr_kernel, bytes, s, a1, l, n, r, work, use_smem, st);
}

cudaError_t launch_triangular_product(const double* left, const double* right, int n, double* out,
                                      const DevStatus* st, cudaStream_t s) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  triangular_product_kernel<<<grid, dim3(32, 8), 0, s>>>(left, right, n, out, st);
  return cudaGetLastError();
}

cudaError_t launch_normalize_sign(double* r, int n, double* sgn, const DevStatus* st, cudaStream_t s) {
  normalize_sign_kernel<<<1, 1024, 0, s>>>(r, n, sgn, st);
  return cudaGetLastError();
}

}  // namespace cqr

#ifdef CQR_LU_TRACE
extern "C" int cqr_debug_lu_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, cqr::g_lu_trace, sizeof(cqr::g_lu_trace));
}
#endif
