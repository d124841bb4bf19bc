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

#include "common.cuh"
#include "kernels.h"

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

__global__ void gram_combine_a_kernel(const double* __restrict__ partial, int leaves, int np, int n,
                                      double* __restrict__ gsum, const DevStatus* st) {
  if (failed(st)) return;
  const int i = blockIdx.y;
  const int j = i + blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = blockIdx.z;
  if (j >= n) return;
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
  for (int k = 0; k < full; ++k) push_merge(stk, top, __ldg(p + (long long)k * stride), (unsigned)(k + 1));
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
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)((leaf1 - leaf0) * p.parts), kWpc * 32, smem, s>>>(x, ldx, p.m, p.n, p.parts, tiles, partial, vec16,
                                                                     check, leaf0, const_cast<DevStatus*>(st));
  return cudaGetLastError();
}

}  // namespace

GramPlan gram_plan(long long m, int n) {
  GramPlan p;
  p.n = n;
  p.m = m;
  p.np = gram_np(n);
  p.leaves = (int)((m + kLeafRows - 1) / kLeafRows);
  p.wpc = kWpc;
  const int nm = p.np / 16;
  const int macros = nm * (nm + 1) / 2;
  const int cap = 9;
  p.parts = (macros + kWpc * cap - 1) / (kWpc * cap);
  int maxt = (macros + kWpc * p.parts - 1) / (kWpc * p.parts);
  p.maxt = maxt <= 1 ? 1 : maxt <= 2 ? 2 : maxt <= 5 ? 5 : 9;
  p.ch = p.np <= 128 ? 32 : 16;
  p.partial_doubles = (size_t)p.leaves * p.np * p.np;
  p.workspace_doubles = p.partial_doubles + (size_t)((p.leaves + kGroup - 1) / kGroup) * p.np * p.np;
  p.tiles_bytes = (size_t)p.parts * kWpc * p.maxt * sizeof(int32_t);
  return p;
}

void gram_tiles(const GramPlan& p, int32_t* out) {
  const int nm = p.np / 16;
  const int slots = p.parts * kWpc;
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
                               int leaf1) {
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
  dim3 ga((unsigned)((p.n + 127) / 128), (unsigned)p.n, (unsigned)groups);
  gram_combine_a_kernel<<<ga, 128, 0, s>>>(partial, p.leaves, p.np, p.n, gsum, st);
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
