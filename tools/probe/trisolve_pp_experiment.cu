// trisolve_pp.cu — the n = 128 right trisolve X R = A with the left-looking work of the next pass
// pipelined under the current pass's diagonal recurrences (c1, and every 128-column panel of c4).
//
// Same arithmetic as trisolve_tma_kernel (per element: k = 0 .. j-1 ascending, off-block terms on DMMA chains,
// in-block terms as scalar fma, then the correctly rounded division: kernels.hpp:116-123 bit for bit). What
// changes is the schedule. In trisolve_tma_kernel a warp runs, per 32-column pass, a left-looking DMMA phase
// and then the pass's four diagonal recurrences; a recurrence is a ~31-deep dependent FP64 chain that waits
// behind the other warps' DMMAs on the shared pipe, so the warp idles through it. Here every warp holds TWO
// passes' accumulators: while pass P's blocks are solved, the accumulators of pass P+1 receive their
// left-looking terms from tensor memory, 16 columns (a chunk) at a time, in k order -- chunks [0, 2P] spread
// over pass P's four blocks, each block's DMMAs in the same basic block as its recurrence so they fill the
// chain's stalls; chunk 2P+1 (the pass's own last two blocks) once the pass is done. Pass P+1 then starts with
// complete accumulators: there is no separate left-looking phase.
//
// A warp owns 32 rows; all its solved blocks of passes 0..2 stay in its TMEM lane quarter (A-fragment order,
// 8 columns per k4 step: 192 columns per warp, two warps per quarter: 8 warps). Input tiles arrive by TMA one
// pass ahead; solved blocks leave by TMA tensor stores from the swizzled staging tiles.

#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"
#include "trisolve_common.cuh"

namespace cqr {

namespace {
using namespace tri;

__device__ __forceinline__ int swz64p(int r, int u) { return r * 8 + 2 * (u ^ ((r >> 1) & 3)); }

constexpr int kPpRW = 32;                 // rows per warp
constexpr int kPpTile = kPpRW * 8;        // doubles per 8-column tile
constexpr int kPpWarp = 6 * kPpTile;      // 2 staging tiles + 4 input tiles
constexpr int kPpNT = 16, kPpW = 4, kPpPasses = 4;
constexpr int kPpTmCols = 192;            // TMEM columns per warp (blocks 0..11, 16 columns each)
constexpr int kPpHead = (kPpNT * kDiagStride + kPpNT * (kPpNT - 1) * 32 + 127) / 128 * 128;

__device__ __forceinline__ void pp_tm_ld32(uint32_t taddr, double (&v)[16]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void pp_tm_st16(uint32_t taddr, const double (&v)[8]) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r[2 * i] = (uint32_t)__double2loint(v[i]);
    r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// DMMA without `volatile`: the compiler may interleave it with the diagonal recurrence
__device__ __forceinline__ void dmma_pp(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int WPC>
__global__ void __launch_bounds__(WPC * 32, 1)
    trisolve_pp_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_st,
                       long long m, const double* __restrict__ bpack, const double* __restrict__ dpack,
                       const DevStatus* st) {
  static_assert(WPC <= 8, "TMEM holds two warps' solved blocks per lane quarter");
  constexpr int NT = kPpNT, W = kPpW;
  constexpr int NB = NT * (NT - 1) * 32, ND = NT * kDiagStride;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t tmem_base;
  if (failed(st)) return;
  double* smem = reinterpret_cast<double*>(smem_raw + ((512u - (smem_u32(smem_raw) & 511u)) & 511u));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  double* sD = smem;
  double* sB = smem + ND;
  double* sT = smem + kPpHead + warp * kPpWarp;  // two staging tiles
  double* sIn = sT + 2 * kPpTile;                 // the next pass's four input tiles
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kPpHead + WPC * kPpWarp) + warp;
  for (int e = threadIdx.x; e < ND; e += WPC * 32) sD[e] = dpack[e];
  for (int e = threadIdx.x; e < NB; e += WPC * 32) sB[e] = bpack[e];
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmw = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kPpTmCols);

  const uint64_t pol_in = l2_policy_evict_first();
  auto issue_in = [&](int P, long long grp) {
    mbar_expect_tx(bar, W * kPpTile * 8);
#pragma unroll
    for (int t = 0; t < W; ++t)
      tma_load_2d_hint(sIn + t * kPpTile, &tm_in, 8 * W * P + 8 * t, (int)(grp * kPpRW), bar, pol_in);
  };
  auto load_in = [&](double (&a)[4][4][2]) {
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const double2 v = *reinterpret_cast<const double2*>(sIn + t * kPpTile + (8 * g + gr) * 8 + 2 * q);
        a[g][t][0] = v.x;
        a[g][t][1] = v.y;
      }
  };
  // pass-P+1 accumulators += chunk c (columns 16c .. 16c+15, k4 = 4c .. 4c+3) of this warp's solved rows
  auto apply_chunk = [&](double (&a2)[4][4][2], int P, int c) {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    double af16[16];
    pp_tm_ld32(tmw + 32u * c, af16);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int k4 = 4 * c + s;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const int JJ = W * (P + 1) + t;
        const double bv = sB[(JJ * (JJ - 1) + k4) * 32 + lane];
#pragma unroll
        for (int g = 0; g < 4; ++g) dmma_pp(a2[g][t][0], a2[g][t][1], af16[4 * s + g], bv);
      }
    }
  };

  uint32_t ph = 0;
  const long long groups = (m + kPpRW - 1) / kPpRW;
  const long long gstride = (long long)gridDim.x * WPC;
  const long long rounds = groups / gstride;
  auto next_grp = [&](long long g) -> long long {  // as trisolve_tma.cu: the last partial round dealt CTA-major
    const long long k = g < rounds * gstride ? g / gstride : rounds;
    if (k + 1 < rounds) return g + gstride;
    if (k + 1 == rounds) return rounds * gstride + (long long)warp * gridDim.x + blockIdx.x;
    return groups;
  };
  long long grp = rounds > 0 ? (long long)blockIdx.x * WPC + warp : (long long)warp * gridDim.x + blockIdx.x;
  double acc[4][4][2], acc2[4][4][2];
  if (grp < groups) {
    if (lane == 0) issue_in(0, grp);
    mbar_wait(bar, ph);
    ph ^= 1;
    load_in(acc);
    fence_async_shared();
    __syncwarp();
    if (lane == 0) issue_in(1, grp);
  }
  for (; grp < groups; grp = next_grp(grp)) {
    const int row0 = (int)(grp * kPpRW);
    const long long ng = next_grp(grp);
#pragma unroll 1
    for (int P = 0; P < kPpPasses; ++P) {
      // the next pass's input (pass P+1, or pass 0 of the next group) -> acc2, then the one after into sIn
      const bool has_next = P + 1 < kPpPasses || ng < groups;
      if (has_next) {
        mbar_wait(bar, ph);
        ph ^= 1;
        load_in(acc2);
        const int P2 = P + 2;
        const bool more = P2 < kPpPasses || ng < groups;
        if (more) {
          fence_async_shared();
          __syncwarp();
          if (lane == 0) issue_in(P2 < kPpPasses ? P2 : P2 - kPpPasses, P2 < kPpPasses ? grp : ng);
        }
      }
      const int C = P + 1 < kPpPasses ? 2 * P + 1 : 0;  // chunks of pass P+1 applied during this pass
#pragma unroll 1
      for (int Jl = 0; Jl < W; ++Jl) {
        const int J = W * P + Jl;
        double* tile = sT + (J & 1) * kPpTile;
        if (lane == 0) bulk_wait_read<1>();  // the store that last used this tile has read it
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 4; ++g)
          *reinterpret_cast<double2*>(tile + swz64p(8 * g + gr, q)) = make_double2(acc[g][0][0], acc[g][0][1]);
        __syncwarp();
        const double* D = sD + J * kDiagStride;
        double y[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 v = *reinterpret_cast<const double2*>(tile + swz64p(lane, u));
          y[2 * u] = v.x;
          y[2 * u + 1] = v.y;
        }
        // this block's share of pass P+1's left-looking chunks, all but the last in their own step, the last
        // one in the recurrence's basic block
        const int c_lo = Jl * C / 4, c_hi = (Jl + 1) * C / 4;
        for (int c = c_lo; c + 1 < c_hi; ++c) apply_chunk(acc2, P, c);
        const bool last_chunk = c_hi > c_lo;
        double af16[16];
        if (last_chunk) {
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          pp_tm_ld32(tmw + 32u * (c_hi - 1), af16);
        }
        bool good = D[80] != 0.0;  // uniform: no zero in the strict upper block, safe divisors
        if (good) {
          if (last_chunk) {  // the chunk's DMMAs, free to interleave with the recurrence below
            const int c = c_hi - 1;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int k4 = 4 * c + s;
#pragma unroll
              for (int t = 0; t < W; ++t) {
                const int JJ = W * (P + 1) + t;
                const double bv = sB[(JJ * (JJ - 1) + k4) * 32 + lane];
#pragma unroll
                for (int g = 0; g < 4; ++g) dmma_pp(acc2[g][t][0], acc2[g][t][1], af16[4 * s + g], bv);
              }
            }
          }
          bool ok = true;
          const double* Dc = D + kColBase;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            double v[10];
#pragma unroll
            for (int h = 0; h < (j + 3) / 2; ++h) {
              const double2 t2 = *reinterpret_cast<const double2*>(Dc + col_start(j) + 2 * h);
              v[2 * h] = t2.x;
              v[2 * h + 1] = t2.y;
            }
#pragma unroll
            for (int kk = 0; kk < j; ++kk) y[j] = fma(-v[kk], y[kk], y[j]);
            bool okj;
            y[j] = div_fast(y[j], v[j], v[j + 1], okj);
            ok &= okj;
          }
          good = __all_sync(0xffffffffu, ok);
        } else if (last_chunk) {
          const int c = c_hi - 1;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const int k4 = 4 * c + s;
#pragma unroll
            for (int t = 0; t < W; ++t) {
              const int JJ = W * (P + 1) + t;
              const double bv = sB[(JJ * (JJ - 1) + k4) * 32 + lane];
#pragma unroll
              for (int g = 0; g < 4; ++g) dmma_pp(acc2[g][t][0], acc2[g][t][1], af16[4 * s + g], bv);
            }
          }
        }
        if (!good) {  // rare: zeros in the block, extreme exponents or exact zeros
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = tile[swz64p(lane, j >> 1) + (j & 1)];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int kk = 0; kk < j; ++kk) {
              const double rv = D[kk * 8 + j];
              if (rv != 0.0) y[j] = fma(-rv, y[kk], y[j]);
            }
            y[j] = fast_div(y[j], D[j * 8 + j], D[64 + j], D[72 + j] != 0.0);
          }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<double2*>(tile + swz64p(lane, u)) = make_double2(y[2 * u], y[2 * u + 1]);
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tm_st, 8 * J, row0, tile);
          bulk_commit();
        }
        double af[4][2];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int kk4 = 0; kk4 < 2; ++kk4) af[g][kk4] = tile[swz64p(8 * g + gr, 2 * kk4 + (q >> 1)) + (q & 1)];
        if (J < NT - W) {
          const double v8[8] = {af[0][0], af[1][0], af[2][0], af[3][0], af[0][1], af[1][1], af[2][1], af[3][1]};
          pp_tm_st16(tmw + 16u * J, v8);
        }
        // right-looking inside the pass (k = this block's 8 columns, after everything before them)
        const double* bcol = sB + (2 * J) * 32 + lane;
#pragma unroll
        for (int t = 1; t < W; ++t) {
          if (Jl + t < W) {
            const int JJ = J + t;
            const double* bp = bcol + (JJ * (JJ - 1)) * 32;
#pragma unroll
            for (int kk4 = 0; kk4 < 2; ++kk4) {
              const double bv = bp[kk4 * 32];
#pragma unroll
              for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g][kk4], bv);
            }
          }
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            acc[g][t - 1][0] = acc[g][t][0];
            acc[g][t - 1][1] = acc[g][t][1];
          }
        }
      }
      // the pass's own last chunk (its blocks 2 and 3), then pass P+1 starts from complete accumulators
      if (P + 1 < kPpPasses) apply_chunk(acc2, P, 2 * P + 1);
      if (has_next) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int t = 0; t < W; ++t) {
            acc[g][t][0] = acc2[g][t][0];
            acc[g][t][1] = acc2[g][t][1];
          }
      }
    }
  }
  if (lane == 0) bulk_wait<0>();
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

}  // namespace

#ifndef CQR_TRI_PP_WPC
#define CQR_TRI_PP_WPC 8
#endif
cudaError_t launch_trisolve_pp(const TrisolveArgs& a, cudaStream_t s) {
  if (trisolve_np(a.n) != 128) return cudaErrorNotSupported;
  CUtensorMap tin, tst;
  if (!make_tmap_2d(&tin, a.in, a.n, a.m, a.ldi, 8, kPpRW, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_tmap_2d(&tst, a.out, a.n, a.m, a.ldo, 8, kPpRW, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorNotSupported;
  constexpr int WPC = CQR_TRI_PP_WPC;
  const size_t smem = (size_t)(kPpHead + WPC * kPpWarp) * 8 + WPC * 8 + 512;
  auto k = trisolve_pp_kernel<WPC>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  const long long groups = (a.m + kPpRW - 1) / kPpRW;
  long long grid = (groups + WPC - 1) / WPC;
  if (grid > (long long)a.num_sms) grid = a.num_sms;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, WPC * 32, smem, s>>>(tin, tst, a.m, a.bpack, a.dpack, a.status);
  return cudaGetLastError();
}

}  // namespace cqr
