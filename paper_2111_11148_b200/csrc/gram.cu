// gram.cu — G = X^T X over fixed 1024-row leaves combined by the pairwise tree
// (kernels.hpp:17-71, engine.cpp:24-39).
//
// Per leaf, every upper element is an fma chain over the leaf's rows in
// ascending order from +0 (the oracle's pinned order). One CTA owns a leaf (or
// a part of its output when n is large); each warp owns up to MAXT 16x16
// macro tiles of the upper triangle and marches over the leaf's rows with
// DMMA m8n8k4 (k = 4 rows per step; DMMA's internal order is the sequential
// chain), so each leaf partial is bit-identical to the oracle's. Rows are
// streamed through a cp.async double buffer. The leaf partials are then
// combined per element with the streaming form of the pairwise tree
// (binary counter + right fold, proven equal to the level-by-level tree in
// tests/test_oracle.py::test_gram_tree_equals_stack_fold) and mirrored.
//
// HBM bytes per row: 8n; flops: n(n+1) per row (upper triangle incl. diagonal).

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace cqr {

namespace {

constexpr int kLeafRows = 1024;  // kernels.hpp:20
constexpr int kWpc = 8;

int gram_np(int n) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (n <= 256) return 256;
  return 512;
}

template <int NP, int MAXT, int CH>
__global__ void __launch_bounds__(kWpc * 32) gram_leaf_kernel(const double* __restrict__ x, long long ldx,
                                                               long long m, int n, int parts,
                                                               const int32_t* __restrict__ tiles,
                                                               double* __restrict__ partial, int vec16, int check,
                                                               int leaf0, DevStatus* st) {
  constexpr int LDX = NP + 4;
  extern __shared__ __align__(16) double smem[];
  if (failed(st)) return;
  const int leaf = blockIdx.x / parts + leaf0, part = blockIdx.x - (blockIdx.x / parts) * parts;
  const long long r0 = (long long)leaf * kLeafRows;
  const int rows = (int)min((long long)kLeafRows, m - r0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, gr = lane >> 2;
  int mt[MAXT];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) mt[t] = tiles[(part * kWpc + warp) * MAXT + t];
  double acc[MAXT][4][2];
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

  const double* xg = x + r0 * ldx;
  const int nch = (rows + CH - 1) / CH;
  // the two chunk buffers as offsets into smem[] (keeps the loads in the shared window)
  bool bad = false;  // the union of the warps' fragments covers every column of the leaf
  stage_rows(smem, LDX, xg, ldx, min(CH, rows), CH, n, NP, tid, kWpc * 32, vec16 != 0);
  cp_async_commit();
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      const int rr = min(CH, rows - (c + 1) * CH);
      stage_rows(smem + ((c + 1) & 1) * CH * LDX, LDX, xg + (long long)(c + 1) * CH * ldx, ldx, rr, CH, n, NP, tid,
                 kWpc * 32, vec16 != 0);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int boff = (c & 1) * CH * LDX;
#pragma unroll 2
    for (int k4 = 0; k4 < CH / 4; ++k4) {
      const int xo = boff + (4 * k4 + q) * LDX + gr;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (mt[t] < 0) continue;
        const int I2 = mt[t] & 0xffff, J2 = mt[t] >> 16;
        const double a0 = smem[xo + 16 * I2], a1 = smem[xo + 16 * I2 + 8];
        const double b0 = smem[xo + 16 * J2], b1 = smem[xo + 16 * J2 + 8];
        bad |= nonfinite(a0) | nonfinite(a1) | nonfinite(b0) | nonfinite(b1);
        dmma(acc[t][0][0], acc[t][0][1], a0, b0);
        dmma(acc[t][1][0], acc[t][1][1], a0, b1);
        if (I2 != J2) dmma(acc[t][2][0], acc[t][2][1], a1, b0);
        dmma(acc[t][3][0], acc[t][3][1], a1, b1);
      }
    }
    __syncthreads();
  }
  if (check && __any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  double* out = partial + (long long)leaf * NP * NP;
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    if (mt[t] < 0) continue;
    const int I2 = mt[t] & 0xffff, J2 = mt[t] >> 16;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int si = u >> 1, sj = u & 1;
      if (I2 == J2 && si == 1 && sj == 0) continue;
      const int i = 16 * I2 + 8 * si + gr, j = 16 * J2 + 8 * sj + 2 * q;
      *reinterpret_cast<double2*>(out + i * NP + j) = make_double2(acc[t][u][0], acc[t][u][1]);
    }
  }
}

// n in (32, 64] (c3): 32 x 32 macro tiles, four warps per leaf -- warp 0 the diagonal tile of columns
// 0..31 (10 upper 8 x 8 blocks), warp 1 that of 32..63, warps 2 and 3 the two 32 x 16 halves of the
// off-diagonal tile (8 blocks each): 36 DMMAs per k4 step against 20 fragment loads (the 16 x 16 tiling
// needs 40 loads for the same 36 DMMAs, and its 10 tiles spread unevenly over 8 warps). Same k order per
// element as gram_leaf_kernel: bit-identical partials.
template <int CH>
__global__ void __launch_bounds__(128) gram_leaf64_kernel(const double* __restrict__ x, long long ldx, long long m,
                                                          int n, double* __restrict__ partial, int vec16, int check,
                                                          int leaf0, DevStatus* st) {
  constexpr int NP = 64, LDX = NP + 4;
  extern __shared__ __align__(16) double smem[];
  if (failed(st)) return;
  const int leaf = blockIdx.x + leaf0;
  const long long r0 = (long long)leaf * kLeafRows;
  const int rows = (int)min((long long)kLeafRows, m - r0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, gr = lane >> 2;
  // this warp's row blocks I in [i0, i0 + 4) and column blocks J in [j0, j0 + nj); diagonal tiles keep I <= J
  const int i0 = warp == 1 ? 4 : 0;
  const int j0 = warp == 0 ? 0 : warp == 1 ? 4 : warp == 2 ? 4 : 6;
  const bool diag = warp < 2;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* xg = x + r0 * ldx;
  const int nch = (rows + CH - 1) / CH;
  bool bad = false;
  stage_rows(smem, LDX, xg, ldx, min(CH, rows), CH, n, NP, tid, 128, vec16 != 0);
  cp_async_commit();
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      const int rr = min(CH, rows - (c + 1) * CH);
      stage_rows(smem + ((c + 1) & 1) * CH * LDX, LDX, xg + (long long)(c + 1) * CH * ldx, ldx, rr, CH, n, NP, tid,
                 128, vec16 != 0);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* xb = smem + (c & 1) * CH * LDX;
#pragma unroll 2
    for (int k4 = 0; k4 < CH / 4; ++k4) {
      const double* xr = xb + (4 * k4 + q) * LDX + gr;
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = xr[8 * (i0 + a)];
      if (diag) {
#pragma unroll
        for (int a = 0; a < 4; ++a) bad |= nonfinite(av[a]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = a; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], av[a], av[b]);
      } else {
#pragma unroll
        for (int b = 0; b < 2; ++b) bv[b] = xr[8 * (j0 + b)];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
      }
    }
    __syncthreads();
  }
  if (check && __any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  double* out = partial + (long long)leaf * NP * NP;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (diag ? b < a : b >= 2) continue;
      const int i = 8 * (i0 + a) + gr, j = 8 * (diag ? i0 + b : j0 + b) + 2 * q;
      *reinterpret_cast<double2*>(out + i * NP + j) = make_double2(acc[a][b][0], acc[a][b][1]);
    }
}

template <int CH>
cudaError_t launch_leaves_64(const GramPlan& p, const double* x, long long ldx, double* partial, int vec16, int check,
                             const DevStatus* st, cudaStream_t s, int leaf0, int leaf1) {
  if (leaf1 < 0) leaf1 = p.leaves;
  if (leaf1 <= leaf0) return cudaSuccess;
  const size_t smem = (size_t)2 * CH * (64 + 4) * sizeof(double);
  auto k = gram_leaf64_kernel<CH>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)(leaf1 - leaf0), 128, smem, s>>>(x, ldx, p.m, p.n, partial, vec16, check, leaf0,
                                                 const_cast<DevStatus*>(st));
  return cudaGetLastError();
}

// Persistent variant (the default where the tile count divides evenly over the
// warps): one CTA per SM walks the leaves blockIdx.x, +gridDim.x, ...; the row
// chunks of consecutive leaves form one cp.async stream, so the next leaf's
// first chunk loads during the current leaf's last. Same per-leaf arithmetic as
// gram_leaf_kernel (the partials are identical); balanced waves: 977 leaves
// (c1) over 148 CTAs is 6.6 per CTA instead of 3.3 per slot over 2 per SM.
template <int NP, int WPC, int MAXT, int CH, bool CHECK>
__global__ void __launch_bounds__(WPC * 32, 1)
    gram_leaf_p_kernel(const double* __restrict__ x, long long ldx, long long m, int n,
                       const int32_t* __restrict__ tiles, double* __restrict__ partial, int vec16, int leaf0,
                       int leaf1, DevStatus* st) {
  constexpr int LDX = NP + 4;
  constexpr int NTH = WPC * 32;
  extern __shared__ __align__(16) double smem[];
  if (failed(st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, gr = lane >> 2;
  int leaf = leaf0 + blockIdx.x;
  if (leaf >= leaf1) return;
  int mt[MAXT];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) mt[t] = tiles[warp * MAXT + t];
  double acc[MAXT][4][2];
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  auto leaf_rows = [&](int lf) { return (int)min((long long)kLeafRows, m - (long long)lf * kLeafRows); };
  auto stage = [&](int lf, int c, int buf) {
    const int rows = leaf_rows(lf);
    stage_rows(smem + buf * CH * LDX, LDX, x + ((long long)lf * kLeafRows + (long long)c * CH) * ldx, ldx,
               min(CH, rows - c * CH), CH, n, NP, tid, NTH, vec16 != 0);
    cp_async_commit();
  };
  bool bad = false;
  int c = 0, buf = 0;
  stage(leaf, 0, 0);
  while (true) {
    const int nch = (leaf_rows(leaf) + CH - 1) / CH;
    int nleaf = leaf, nc = c + 1;
    if (nc == nch) {
      nleaf = leaf + gridDim.x;
      nc = 0;
    }
    if (nleaf < leaf1) {
      stage(nleaf, nc, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int boff = buf * CH * LDX;
#pragma unroll 2
    for (int k4 = 0; k4 < CH / 4; ++k4) {
      const int xo = boff + (4 * k4 + q) * LDX + gr;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (mt[t] < 0) continue;
        const int I2 = mt[t] & 0xffff, J2 = mt[t] >> 16;
        const double a0 = smem[xo + 16 * I2], a1 = smem[xo + 16 * I2 + 8];
        const double b0 = smem[xo + 16 * J2], b1 = smem[xo + 16 * J2 + 8];
        if constexpr (CHECK) bad |= nonfinite(a0) | nonfinite(a1) | nonfinite(b0) | nonfinite(b1);
        dmma(acc[t][0][0], acc[t][0][1], a0, b0);
        dmma(acc[t][1][0], acc[t][1][1], a0, b1);
        if (I2 != J2) dmma(acc[t][2][0], acc[t][2][1], a1, b0);
        dmma(acc[t][3][0], acc[t][3][1], a1, b1);
      }
    }
    __syncthreads();
    if (nc == 0) {  // leaf done: write its partial, restart the chains
      double* out = partial + (long long)leaf * NP * NP;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (mt[t] < 0) continue;
        const int I2 = mt[t] & 0xffff, J2 = mt[t] >> 16;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int si = u >> 1, sj = u & 1;
          if (I2 == J2 && si == 1 && sj == 0) continue;
          const int i = 16 * I2 + 8 * si + gr, j = 16 * J2 + 8 * sj + 2 * q;
          *reinterpret_cast<double2*>(out + i * NP + j) = make_double2(acc[t][u][0], acc[t][u][1]);
          acc[t][u][0] = acc[t][u][1] = 0.0;
        }
      }
    }
    leaf = nleaf;
    c = nc;
    buf ^= 1;
    if (leaf >= leaf1) break;
  }
  if constexpr (CHECK) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  }
}

// TMA-fed persistent variant (the default for n in (64, 128] when X is
// TMA-addressable): one producer warp streams the 32-row chunks of this CTA's
// leaves through a 4-stage ring (SWIZZLE_128B boxes of 16 columns) and 12 MMA
// warps consume them behind full/empty mbarriers: no block barrier and no
// cp.async issue work per chunk. Same tiles, same k order as gram_leaf_p_kernel:
// bit-identical partials.
constexpr int kGtMma = 12;
#ifndef CQR_GRAM_CH256
#define CQR_GRAM_CH256 32  // rows per ring stage at n in (128, 256] (16 rows: 2.32 vs 2.30 ms)
#endif
#ifndef CQR_GRAM256_PARTS
#define CQR_GRAM256_PARTS 3
#define CQR_GRAM256_MAXT 4
#endif
#ifndef CQR_GRAM512_PARTS
#define CQR_GRAM512_PARTS 11
#define CQR_GRAM512_MAXT 4
#endif
#ifndef CQR_GRAM_CH64
#define CQR_GRAM_CH64 32
#endif
#ifndef CQR_GRAM_CH128
#define CQR_GRAM_CH128 64  // rows per ring stage at n in (64, 128] (16/32/64: 0.677/0.636/0.628 ms at c1)
#endif
constexpr int kGtThreads = (kGtMma + 1) * 32;

// Stage layout (NP <= 256): NP/8 boxes of ROWS x 8 columns (64-byte rows, no swizzle). A fragment load reads
// 8 consecutive columns of 4 consecutive rows (k = 4 rows per DMMA step); with 64-byte rows, rows
// q and q + 1 sit in opposite bank halves, so the 256 bytes take the minimum two wavefronts (the
// earlier 16-column SWIZZLE_128B boxes kept all four rows in one half: four wavefronts, LSU 83%).
// NP = 512 keeps 16-column SWIZZLE_128B boxes: 64 narrow boxes per 16-row stage from one producer lane
// cost more than the conflicts they remove (9.31 vs 11.44 ms at m = 1e6).
template <int NP, int ROWS, int BW_ = (NP <= 256 ? 8 : 16)>
struct GtShape {
  static constexpr int BW = BW_;
  static constexpr int CHUNK = ROWS * NP;  // doubles per stage (NP/BW boxes of ROWS x BW)
  static constexpr int BOX = ROWS * BW;
  static constexpr int STAGES = CHUNK * 8 * 4 <= 200 * 1024 ? 4 : 3;
  static constexpr size_t SMEM = (size_t)STAGES * CHUNK * sizeof(double) + 1024;
};

// Work item w = blockIdx.x + k * gridDim.x (gridDim.x a multiple of parts): part
// w % parts (fixed per CTA: its warps' macro-tile lists), leaf leaf0 + w / parts.
template <int NP, int MAXT, int ROWS, bool CHECK, int BW = (NP <= 256 ? 8 : 16)>
__global__ void __launch_bounds__(kGtThreads, 1)
    gram_leaf_tma_kernel(const __grid_constant__ CUtensorMap tmx, int tma3, long long m, int parts,
                         const int32_t* __restrict__ tiles, double* __restrict__ partial, int leaf0, int leaf1,
                         DevStatus* st) {
  using S = GtShape<NP, ROWS, BW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[S::STAGES], empty[S::STAGES];
  if (failed(st)) return;
  double* sm = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int part = blockIdx.x % parts;
  if (tid == 0) {
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGtMma);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  __syncthreads();
  auto leaf_chunks = [&](int lf) {
    const long long rows = min((long long)kLeafRows, m - (long long)lf * kLeafRows);
    return (int)((rows + ROWS - 1) / ROWS);
  };
  if (warp == kGtMma) {  // ---- producer
    if (lane == 0) {
      int it = 0;
      for (int w = blockIdx.x;; w += gridDim.x) {
        const int lf = leaf0 + w / parts;
        if (lf >= leaf1) break;
        const int nch = leaf_chunks(lf);
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % S::STAGES;
          mbar_wait(&empty[s], ((it / S::STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], S::CHUNK * 8);
          const int row = lf * kLeafRows + c * ROWS;
          if (tma3) {  // all NP/BW column boxes of the stage in one 3-D load
            tma_load_3d(sm + s * S::CHUNK, &tmx, 0, row, 0, &full[s]);
          } else {
#pragma unroll
            for (int b = 0; b < NP / S::BW; ++b)
              tma_load_2d(sm + s * S::CHUNK + b * S::BOX, &tmx, S::BW * b, row, &full[s]);
          }
        }
      }
    }
    return;
  }
  // ---- MMA warps: MAXT 16x16 macro tiles each
  const int q = lane & 3, gr = lane >> 2;
  int mt[MAXT];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) mt[t] = tiles[(part * kGtMma + warp) * MAXT + t];
  double acc[MAXT][4][2];
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  bool bad = false;
  // column group h (8 columns) of row r inside a stage: box h (64-byte rows), or box h/2 with
  // 128B-swizzled 16-byte chunks (16-column boxes)
  auto at = [&](const double* base, int r, int h) {
    if constexpr (S::BW == 8) {
      return base[h * S::BOX + r * 8 + gr];
    } else {
      return base[(h >> 1) * S::BOX + r * 16 + 2 * ((4 * (h & 1) + (gr >> 1)) ^ (r & 7)) + (gr & 1)];
    }
  };
  int it = 0;
  for (int w = blockIdx.x;; w += gridDim.x) {
    const int lf = leaf0 + w / parts;
    if (lf >= leaf1) break;
    const int nch = leaf_chunks(lf);
    for (int c = 0; c < nch; ++c, ++it) {
      const int s = it % S::STAGES;
      mbar_wait(&full[s], (it / S::STAGES) & 1);
      const double* base = sm + s * S::CHUNK;
#pragma unroll 2
      for (int k4 = 0; k4 < ROWS / 4; ++k4) {
        const int r = 4 * k4 + q;
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          if (mt[t] < 0) continue;
          const int I2 = mt[t] & 0xffff, J2 = mt[t] >> 16;
          const double a0 = at(base, r, 2 * I2), a1 = at(base, r, 2 * I2 + 1);
          const double b0 = at(base, r, 2 * J2), b1 = at(base, r, 2 * J2 + 1);
          if constexpr (CHECK) bad |= nonfinite(a0) | nonfinite(a1) | nonfinite(b0) | nonfinite(b1);
          dmma(acc[t][0][0], acc[t][0][1], a0, b0);
          dmma(acc[t][1][0], acc[t][1][1], a0, b1);
          if (I2 != J2) dmma(acc[t][2][0], acc[t][2][1], a1, b0);
          dmma(acc[t][3][0], acc[t][3][1], a1, b1);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    double* out = partial + (long long)lf * NP * NP;  // leaf done: its partial, then restart the chains
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      if (mt[t] < 0) continue;
      const int I2 = mt[t] & 0xffff, J2 = mt[t] >> 16;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int si = u >> 1, sj = u & 1;
        if (!(I2 == J2 && si == 1 && sj == 0)) {
          const int i = 16 * I2 + 8 * si + gr, j = 16 * J2 + 8 * sj + 2 * q;
          *reinterpret_cast<double2*>(out + i * NP + j) = make_double2(acc[t][u][0], acc[t][u][1]);
        }
        acc[t][u][0] = acc[t][u][1] = 0.0;
      }
    }
  }
  if constexpr (CHECK) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  }
}

// x is encoded here: 8-column boxes (conflict-free fragment loads), one 3-D load per stage when n % 8 == 0
// (NP = 512 needs it: 64 separate narrow boxes per stage are TMA-issue bound), else 2-D boxes
// (16-column SWIZZLE_128B ones at NP = 512).
template <int NP, int MAXT, int ROWS>
cudaError_t launch_leaves_tma(const GramPlan& p, const double* x, long long ldx, const int32_t* tiles,
                              double* partial, int check, const DevStatus* st, cudaStream_t s, int leaf0, int leaf1,
                              int num_sms) {
  if (leaf1 < 0) leaf1 = p.leaves;
  if (leaf1 <= leaf0) return cudaSuccess;
  CUtensorMap tm;
  static const bool no3d = std::getenv("CQR_GRAM_TMA2D") != nullptr;  // A/B runs
  const bool tma3 = !no3d && p.n % 8 == 0 &&
                    make_tmap_colblocks(&tm, x, p.n, p.m, ldx, ROWS, NP / 8, CU_TENSOR_MAP_SWIZZLE_NONE, 8);
  const long long items = (long long)(leaf1 - leaf0) * p.parts;
  const int slots = std::max(1, num_sms / p.parts) * p.parts;
  const int grid = (int)std::min<long long>(items, slots);
  auto run = [&](auto kfn, size_t smem) -> cudaError_t {
    cudaError_t e = allow_max_smem(kfn);
    if (e != cudaSuccess) return e;
    kfn<<<(unsigned)grid, kGtThreads, smem, s>>>(tm, tma3 ? 1 : 0, p.m, p.parts, tiles, partial, leaf0, leaf1,
                                                const_cast<DevStatus*>(st));
    return cudaGetLastError();
  };
  if (tma3 || NP <= 256) {
    if (!tma3 && !make_tmap_2d(&tm, x, p.n, p.m, ldx, 8, ROWS, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    using S = GtShape<NP, ROWS, 8>;
    return check ? run(gram_leaf_tma_kernel<NP, MAXT, ROWS, true, 8>, S::SMEM)
                 : run(gram_leaf_tma_kernel<NP, MAXT, ROWS, false, 8>, S::SMEM);
  }
  if (!make_tmap_2d(&tm, x, p.n, p.m, ldx, 16, ROWS, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  using S = GtShape<NP, ROWS, 16>;
  return check ? run(gram_leaf_tma_kernel<NP, MAXT, ROWS, true, 16>, S::SMEM)
               : run(gram_leaf_tma_kernel<NP, MAXT, ROWS, false, 16>, S::SMEM);
}

// The pairwise tree of kernels.hpp:42-57 in streaming form: after pushing leaf
// i, merge (top-1) + top once per trailing zero of (i+1); at the end fold the
// stack right to left. Two levels for parallelism: level A folds each aligned
// group of kGroup leaves (a complete group is a perfect subtree; the last,
// partial group is folded by the same rule), level B runs the counter over the
// complete groups and appends the partial group last. Equal to the one-level
// form because subtrees of different sizes never merge.
constexpr int kGroup = 16;

__device__ __forceinline__ void push_merge(double* stk, int& top, double v, unsigned count_after) {
  while ((count_after & 1u) == 0u) {
    v = stk[--top] + v;
    count_after >>= 1;
  }
  stk[top++] = v;
}

// Level A over the upper triangle laid out linearly (thread e -> (i, j >= i), every lane busy; a
// row-per-block grid left half of each block idle): 16 leaf loads in flight per element.
__global__ void gram_combine_a_kernel(const double* __restrict__ partial, int leaves, int np, int n,
                                      double* __restrict__ gsum, const DevStatus* st) {
  if (failed(st)) return;
  const int tri = n * (n + 1) / 2;
  const int per = (tri + blockDim.x - 1) / blockDim.x;  // blocks per group
  const int grp = blockIdx.x / per;
  const int e = (blockIdx.x - grp * per) * blockDim.x + threadIdx.x;
  if (e >= tri) return;
  // row i: elements [i n - i (i - 1) / 2, ...) of the packed upper triangle
  const double tn = 2.0 * n + 1.0;
  int i = (int)((tn - sqrt(tn * tn - 8.0 * e)) * 0.5);
  while (i > 0 && i * n - i * (i - 1) / 2 > e) --i;
  while ((i + 1) * n - (i + 1) * i / 2 <= e) ++i;
  const int j = i + (e - (i * n - i * (i - 1) / 2));
  const long long stride = (long long)np * np;
  const int l0 = grp * kGroup, l1 = min(leaves, l0 + kGroup);
  const double* p = partial + (long long)i * np + j;
  double v[kGroup];
#pragma unroll
  for (int u = 0; u < kGroup; ++u) v[u] = (l0 + u < l1) ? __ldg(p + (long long)(l0 + u) * stride) : 0.0;
  double stk[8];
  int top = 0;
#pragma unroll
  for (int u = 0; u < kGroup; ++u)
    if (l0 + u < l1) push_merge(stk, top, v[u], (unsigned)(u + 1));
  double acc = stk[top - 1];
  for (int k = top - 2; k >= 0; --k) acc = stk[k] + acc;
  gsum[(long long)grp * np * np + (long long)i * np + j] = acc;
}

__global__ void gram_combine_b_kernel(const double* __restrict__ gsum, int leaves, int np, int n,
                                      double* __restrict__ g, int mirror, const DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y;
  const int j = i + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int full = leaves / kGroup, groups = (leaves + kGroup - 1) / kGroup;
  const long long stride = (long long)np * np;
  const double* p = gsum + (long long)i * np + j;
  double stk[40];
  int top = 0;
  for (int k0 = 0; k0 < full; k0 += 8) {  // eight loads in flight, merged in order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = k0 + u < full ? __ldg(p + (long long)(k0 + u) * stride) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < full) push_merge(stk, top, v[u], (unsigned)(k0 + u + 1));
  }
  if (groups > full) stk[top++] = __ldg(p + (long long)full * stride);
  double acc = stk[top - 1];
  for (int k = top - 2; k >= 0; --k) acc = stk[k] + acc;
  g[(long long)i * n + j] = acc;
  if (mirror) g[(long long)j * n + i] = acc;
}

__global__ void mirror_kernel(double* g, int n, const DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < i) g[(long long)i * n + j] = g[(long long)j * n + i];
}

template <int NP, int MAXT, int CH>
cudaError_t launch_leaves_t(const GramPlan& p, const double* x, long long ldx, const int32_t* tiles,
                            double* partial, int vec16, int check, const DevStatus* st, cudaStream_t s, int leaf0,
                            int leaf1) {
  if (leaf1 < 0) leaf1 = p.leaves;
  if (leaf1 <= leaf0) return cudaSuccess;
  const size_t smem = (size_t)2 * CH * (NP + 4) * sizeof(double);
  auto k = gram_leaf_kernel<NP, MAXT, CH>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)((leaf1 - leaf0) * p.parts), kWpc * 32, smem, s>>>(x, ldx, p.m, p.n, p.parts, tiles, partial, vec16,
                                                                     check, leaf0, const_cast<DevStatus*>(st));
  return cudaGetLastError();
}

template <int NP, int WPC, int MAXT, int CH>
cudaError_t launch_leaves_p(const GramPlan& p, const double* x, long long ldx, const int32_t* tiles,
                            double* partial, int vec16, int check, const DevStatus* st, cudaStream_t s, int leaf0,
                            int leaf1, int num_sms) {
  if (leaf1 < 0) leaf1 = p.leaves;
  if (leaf1 <= leaf0) return cudaSuccess;
  const size_t smem = (size_t)2 * CH * (NP + 4) * sizeof(double);
  auto k = check ? gram_leaf_p_kernel<NP, WPC, MAXT, CH, true> : gram_leaf_p_kernel<NP, WPC, MAXT, CH, false>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  const int grid = std::min(leaf1 - leaf0, num_sms);
  k<<<(unsigned)grid, WPC * 32, smem, s>>>(x, ldx, p.m, p.n, tiles, partial, vec16, leaf0, leaf1,
                                           const_cast<DevStatus*>(st));
  return cudaGetLastError();
}

}  // namespace

bool gram_tma_ok(const double* x, long long ldx, long long m, int n) {
  static const bool off = std::getenv("CQR_GRAM_NO_TMA") != nullptr;  // tuning: the cp.async kernels
  CUtensorMap probe;
  return !off && n > 64 && m > 0 && m < (1LL << 31) - 1024 && make_tmap_2d(&probe, x, n, m, ldx, 8, 16, CU_TENSOR_MAP_SWIZZLE_NONE);
}

GramPlan gram_plan(long long m, int n, bool tma_ok) {
  GramPlan p;
  p.n = n;
  p.m = m;
  p.np = gram_np(n);
  p.leaves = (int)((m + kLeafRows - 1) / kLeafRows);
  const int nm = p.np / 16;
  const int macros = nm * (nm + 1) / 2;
  static const bool legacy = std::getenv("CQR_GRAM_LEGACY") != nullptr;  // tuning: the per-leaf kernel
  if (tma_ok && p.np >= 128) {  // TMA-fed: 12 DMMA warps, the macro tiles over `parts` CTAs per leaf (n = 64: the
                                // cp.async kernel is faster, 0.97 vs 1.02 ms at c3)
    p.tma = 1;
    p.persistent = 1;
    p.wpc = kGtMma;
    p.parts = p.np == 128 ? 1 : p.np == 256 ? CQR_GRAM256_PARTS : CQR_GRAM512_PARTS;  // 36 / 136 / 528 macros: 3, 4, 4 per warp (13 warps: 128 regs)
    p.maxt = (macros + p.wpc * p.parts - 1) / (p.wpc * p.parts);
    p.ch = p.np == 512 ? 16 : p.np == 128 ? CQR_GRAM_CH128 : CQR_GRAM_CH256;
  } else if (p.np == 128 && !legacy) {  // persistent: the 36 macro tiles divide evenly over 12 warps (measured: n = 64 is faster per leaf)
    p.persistent = 1;
    p.wpc = p.np == 64 ? 10 : 12;
    p.parts = 1;
    p.maxt = macros / p.wpc;
    p.ch = 32;
  } else {
    p.wpc = kWpc;
    const int cap = 9;
    p.parts = (macros + kWpc * cap - 1) / (kWpc * cap);
    int maxt = (macros + kWpc * p.parts - 1) / (kWpc * p.parts);
    p.maxt = maxt <= 1 ? 1 : maxt <= 2 ? 2 : maxt <= 5 ? 5 : 9;
    p.ch = p.np <= 128 ? 32 : 16;
  }
  p.partial_doubles = (size_t)p.leaves * p.np * p.np;
  p.workspace_doubles = p.partial_doubles + (size_t)((p.leaves + kGroup - 1) / kGroup) * p.np * p.np;
  p.tiles_bytes = (size_t)p.parts * p.wpc * p.maxt * sizeof(int32_t);
  return p;
}

void gram_tiles(const GramPlan& p, int32_t* out) {
  const int nm = p.np / 16;
  const int slots = p.parts * p.wpc;
  for (int e = 0; e < slots * p.maxt; ++e) out[e] = -1;
  // round-robin the upper macro tiles over (part, warp) slots, filling each slot's list
  int idx = 0;
  for (int I = 0; I < nm; ++I)
    for (int J = I; J < nm; ++J) {
      const int slot = idx % slots, t = idx / slots;
      out[slot * p.maxt + t] = I | (J << 16);
      ++idx;
    }
}

cudaError_t launch_gram_leaves(const GramPlan& p, const double* x, long long ldx, const int32_t* tiles,
                               double* partial, int vec16, int check, const DevStatus* st, cudaStream_t s, int leaf0,
                               int leaf1, int num_sms) {
  if (p.tma) {
    if (p.np == 128 && p.maxt == 1)  // the split last wave (engine gram_dev)
      return launch_leaves_tma<128, 1, CQR_GRAM_CH128>(p, x, ldx, tiles, partial, check, st, s, leaf0, leaf1, num_sms);
    if (p.np == 128)
      return launch_leaves_tma<128, 3, CQR_GRAM_CH128>(p, x, ldx, tiles, partial, check, st, s, leaf0, leaf1, num_sms);
    if (p.np == 256) return launch_leaves_tma<256, CQR_GRAM256_MAXT, CQR_GRAM_CH256>(p, x, ldx, tiles, partial, check, st, s, leaf0, leaf1, num_sms);
    if (p.np == 512) return launch_leaves_tma<512, CQR_GRAM512_MAXT, 16>(p, x, ldx, tiles, partial, check, st, s, leaf0, leaf1, num_sms);
    return cudaErrorInvalidValue;
  }
  static const bool no64 = std::getenv("CQR_GRAM_NO64") != nullptr;  // A/B: the 16 x 16 tiling at n <= 64
  if (p.np == 64 && !p.persistent && !no64)
    return launch_leaves_64<CQR_GRAM_CH64>(p, x, ldx, partial, vec16, check, st, s, leaf0, leaf1);
  if (p.persistent) {
    if (p.np == 128 && p.maxt == 3)
      return launch_leaves_p<128, 12, 3, 32>(p, x, ldx, tiles, partial, vec16, check, st, s, leaf0, leaf1, num_sms);
    if (p.np == 64 && p.maxt == 1)
      return launch_leaves_p<64, 10, 1, 32>(p, x, ldx, tiles, partial, vec16, check, st, s, leaf0, leaf1, num_sms);
    return cudaErrorInvalidValue;
  }
#define CQR_GRAM_CASE(NP_, CH_)                                                                     \
  case NP_:                                                                                          \
    switch (p.maxt) {                                                                                \
      case 1: return launch_leaves_t<NP_, 1, CH_>(p, x, ldx, tiles, partial, vec16, check, st, s, leaf0, leaf1);         \
      case 2: return launch_leaves_t<NP_, 2, CH_>(p, x, ldx, tiles, partial, vec16, check, st, s, leaf0, leaf1);         \
      case 5: return launch_leaves_t<NP_, 5, CH_>(p, x, ldx, tiles, partial, vec16, check, st, s, leaf0, leaf1);         \
      default: return launch_leaves_t<NP_, 9, CH_>(p, x, ldx, tiles, partial, vec16, check, st, s, leaf0, leaf1);        \
    }
  switch (p.np) {
    CQR_GRAM_CASE(16, 32)
    CQR_GRAM_CASE(32, 32)
    CQR_GRAM_CASE(64, 32)
    CQR_GRAM_CASE(128, 32)
    CQR_GRAM_CASE(256, 16)
    CQR_GRAM_CASE(512, 16)
  }
#undef CQR_GRAM_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_gram_combine(const GramPlan& p, double* partial, double* g, int mirror,
                                const DevStatus* st, cudaStream_t s) {
  const int groups = (p.leaves + kGroup - 1) / kGroup;
  double* gsum = partial + p.partial_doubles;  // workspace after the leaf partials (gram_plan reserves it)
  const int tri = p.n * (p.n + 1) / 2;
  gram_combine_a_kernel<<<(unsigned)(((tri + 255) / 256) * groups), 256, 0, s>>>(partial, p.leaves, p.np, p.n, gsum,
                                                                                   st);
  dim3 gb((unsigned)((p.n + 127) / 128), (unsigned)p.n);
  gram_combine_b_kernel<<<gb, 128, 0, s>>>(gsum, p.leaves, p.np, p.n, g, mirror, st);
  return cudaGetLastError();
}

cudaError_t launch_mirror_upper(double* g, int n, const DevStatus* st, cudaStream_t s) {
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)n);
  mirror_kernel<<<grid, 128, 0, s>>>(g, n, st);
  return cudaGetLastError();
}

}  // namespace cqr
