// trisolve_tma.cu — the super-block right trisolve X R = A with TMA-staged
// tiles (the default when A and X are TMA-addressable: 16-byte aligned bases,
// even leading dimensions).
//
// Same arithmetic as trisolve_sb_kernel (trisolve.cu) — per element k = 0..j-1
// ascending through DMMA chains, the in-block terms as scalar fma, then the
// correctly rounded division: the reference recurrence (kernels.hpp:116-123)
// bit for bit. What changes is how the tall data moves, because the register
// kernel is bound by the L1 data pipe (profiles/r01_trisolve_tma.md):
//  * a pass's input columns arrive by TMA as 8-column x 32-row tiles and are read
//    into the DMMA accumulators with conflict-free 16-byte shared loads;
//  * the left-looking operand (this warp's already-solved columns) streams
//    back by TMA as 4-column x 32-row slabs, double buffered, so each DMMA A
//    fragment is one conflict-free 8-byte shared load instead of an 8-line
//    global load;
//  * each solved 8-column block leaves through a TMA tensor store from the
//    64-byte-swizzled staging tile that the diagonal recurrence already uses.
// A warp owns 32 rows; its TMA traffic is issued by lane 0 and tracked with
// two mbarriers (loads) and bulk async-groups (stores).
//  * TMW of the warps (n = 128: 8 of 12, n = 256: 4 of 16; as many as the 512 TMEM
//    columns hold) keep the left-looking operand in tensor memory instead: each
//    solved block's A fragments go to the thread's own TMEM lane (tcgen05.st) and
//    come back with one tcgen05.ld per 16 columns -- no store/read-back round trip
//    through L2 for those warps. Same values, same DMMA order: bit-identical.
// Probe builds: -DCQR_TRI_NOLL (no left-looking DMMAs), -DCQR_TRI_NODIAG (no
// diagonal recurrence) time the kernel's phases (results wrong; timing only).

#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"
#include "trisolve_common.cuh"

namespace cqr {

namespace {
using namespace tri;

// TMA SWIZZLE_64B layout of an 8-column tile (64-byte rows): 16-byte chunk u
// of row r sits at chunk u ^ ((r >> 1) & 3).
__device__ __forceinline__ int swz64(int r, int u) { return r * 8 + 2 * (u ^ ((r >> 1) & 3)); }

constexpr int kRW = 32;                  // rows per warp
constexpr int kTile = kRW * 8;           // doubles in an 8-column tile (2 KB)
constexpr int kSlab = kRW * 4;           // doubles in a 4-column slab (1 KB)
constexpr int kWarpDoubles = 6 * kTile;  // 2 staging tiles + an 8 KB input / left-looking buffer

template <int NP, bool BSMEM>
constexpr int head_doubles() {
  return ((NP / 8) * kDiagStride + (BSMEM ? (NP / 8) * (NP / 8 - 1) * 32 : 0) + 127) / 128 * 128;
}

// TMEM store of the left-looking operand: thread (gr, q) keeps, in its own TMEM lane, the DMMA A fragments
// af[g] of every solved k4 step its later passes need (8 32-bit columns per k4: column 8 k4 + 2 g); warp w
// uses lane quarter w % 4 at column slot w / 4.
__device__ __forceinline__ void tm_ld32(uint32_t taddr, double (&v)[16]) {
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
__device__ __forceinline__ void tm_st16(uint32_t taddr, const double (&v)[8]) {
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

template <int NP, int WPC, bool BSMEM, int TMW = 0>
__global__ void __launch_bounds__(WPC * 32, 1)
    trisolve_tma_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_ll,
                        const __grid_constant__ CUtensorMap tm_st, long long m, int n,
                        const double* __restrict__ bpack, const double* __restrict__ dpack,
                        const DevStatus* st) {
  constexpr int NT = NP / 8;
  constexpr int W = NT < 4 ? NT : 4;  // blocks per pass
  constexpr int NPASS = NT / W;
  constexpr int NB = BSMEM ? NT * (NT - 1) * 32 : 0;
  constexpr int ND = NT * kDiagStride;
  constexpr int HEAD = head_doubles<NP, BSMEM>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (failed(st)) return;
  // 512-byte alignment: the staging tiles' SWIZZLE_64B pattern repeats every 512 bytes (tiles sit at 2 KB steps)
  double* smem = reinterpret_cast<double*>(smem_raw + ((512u - (smem_u32(smem_raw) & 511u)) & 511u));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  double* sD = smem;
  const double* sB = bpack;
  double* sT = smem + HEAD + warp * kWarpDoubles;  // two staging tiles
  double* sL = sT + 2 * kTile;                     // input tiles / left-looking slabs
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + HEAD + WPC * kWarpDoubles) + 2 * warp;
  for (int e = threadIdx.x; e < ND; e += WPC * 32) sD[e] = dpack[e];
  if constexpr (BSMEM) {
    for (int e = threadIdx.x; e < NB; e += WPC * 32) smem[ND + e] = bpack[e];
    sB = smem + ND;
  }
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  __shared__ uint32_t tmem_base;
  if constexpr (TMW > 0) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  constexpr int kTmCols = (NT - W) * 16;  // TMEM columns per warp: the blocks later passes read
  static_assert(TMW == 0 || ((TMW + 3) / 4) * kTmCols <= 512, "TMEM: too many warps for this width");
  const bool tmw = warp < TMW;
  uint32_t tm_warp = 0;
  if constexpr (TMW > 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    tm_warp = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kTmCols);
  }

  // left-looking chunk ch (columns 16ch .. 16ch+15) -> buffer b, four slabs
  auto issue_ll = [&](int ch, int b, int row0) {
    mbar_expect_tx(bar + b, 4 * kSlab * 8);
#pragma unroll
    for (int s = 0; s < 4; ++s) tma_load_2d(sL + b * 2 * kTile + s * kSlab, &tm_ll, 16 * ch + 4 * s, row0, bar + b);
  };

  // the input tiles of (pass P, group grp) -> sL on bar[0]. L2 policy: the input is read once
  // (evict first), the solved rows are read back by the later passes' left-looking part (evict
  // last), so at wide n the recently solved rows, not the streamed input, stay in L2.
#ifndef CQR_TRI_NO_HINT
  const uint64_t pol_in = l2_policy_evict_first(), pol_out = l2_policy_evict_last();
#endif
  auto issue_in = [&](int P, long long grp) {
    mbar_expect_tx(bar, W * kTile * 8);
#pragma unroll
    for (int t = 0; t < W; ++t) {
#ifndef CQR_TRI_NO_HINT
      tma_load_2d_hint(sL + t * kTile, &tm_in, 8 * W * P + 8 * t, (int)(grp * kRW), bar, pol_in);
#else
      tma_load_2d(sL + t * kTile, &tm_in, 8 * W * P + 8 * t, (int)(grp * kRW), bar);
#endif
    }
  };

  uint32_t ph0 = 0, ph1 = 0;
  const long long groups = (m + kRW - 1) / kRW;
  const long long gstride = (long long)gridDim.x * WPC;
  // Whole rounds give group k * gstride + blockIdx.x * WPC + warp; the groups of the last, partial round
  // are dealt CTA-major (warp w of CTA b takes rounds * gstride + w * gridDim.x + b), so every SM keeps a
  // share of them instead of the first CTAs taking all (c1: 31250 groups, 1776 warps).
  const long long rounds = groups / gstride;
  auto next_grp = [&](long long g) -> long long {
    const long long k = g < rounds * gstride ? g / gstride : rounds;
    if (k + 1 < rounds) return g + gstride;
    if (k + 1 == rounds) return rounds * gstride + (long long)warp * gridDim.x + blockIdx.x;
    return groups;
  };
  long long grp = rounds > 0 ? (long long)blockIdx.x * WPC + warp : (long long)warp * gridDim.x + blockIdx.x;
  if (lane == 0 && grp < groups) issue_in(0, grp);
  for (; grp < groups; grp = next_grp(grp)) {
    const int row0 = (int)(grp * kRW);
#pragma unroll 1
    for (int P = 0; P < NPASS; ++P) {
      const int c0 = 8 * W * P;
      // 1. the pass's input columns (zero-filled beyond m and n), prefetched
      mbar_wait(bar, ph0);
      ph0 ^= 1;
      double acc[4][W][2];
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int t = 0; t < W; ++t) {
          const double2 v = *reinterpret_cast<const double2*>(sL + t * kTile + (8 * g + gr) * 8 + 2 * q);
          acc[g][t][0] = v.x;
          acc[g][t][1] = v.y;
        }
      // 2. left-looking: k in [0, c0) ascending, from this warp's stored rows
      if (P > 0 && TMW > 0 && tmw) {
        const int nch = c0 / 16;
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          double af16[16];
          tm_ld32(tm_warp + 32u * ch, af16);
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const int k4 = 4 * ch + s;
#pragma unroll
            for (int t = 0; t < W; ++t) {
              const int JJ = W * P + t;
              const int bi = (JJ * (JJ - 1) + k4) * 32 + lane;
              const double bv = BSMEM ? sB[bi] : __ldg(sB + bi);
#pragma unroll
              for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af16[4 * s + g], bv);
            }
          }
        }
      } else if (P > 0) {
        const int nch = c0 / 16;
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          bulk_wait<0>();  // this warp's earlier blocks have landed in global memory
          fence_async_global();
          issue_ll(0, 0, row0);
          if (nch > 1) issue_ll(1, 1, row0);
        }
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          const int b = ch & 1;
          if (b == 0) {
            mbar_wait(bar, ph0);
            ph0 ^= 1;
          } else {
            mbar_wait(bar + 1, ph1);
            ph1 ^= 1;
          }
          const double* buf = sL + b * 2 * kTile;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const int k4 = 4 * ch + s;
            double af[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) af[g] = buf[s * kSlab + (8 * g + gr) * 4 + q];
#pragma unroll
            for (int t = 0; t < W; ++t) {
              const int JJ = W * P + t;
              const int bi = (JJ * (JJ - 1) + k4) * 32 + lane;
              const double bv = BSMEM ? sB[bi] : __ldg(sB + bi);
#ifndef CQR_TRI_NOLL  // probe: without the left-looking DMMAs
#pragma unroll
              for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g], bv);
#else
              if (bv == 12345.0) acc[0][t][0] += af[0] + af[1] + af[2] + af[3];
#endif
            }
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0 && ch + 2 < nch) issue_ll(ch + 2, b, row0);
        }
      }
      // prefetch the next pass's input (sL is free again)
      {
        const bool last = P + 1 == NPASS;
        if (!last || next_grp(grp) < groups) {
          fence_async_shared();
          __syncwarp();
          if (lane == 0) issue_in(last ? 0 : P + 1, last ? next_grp(grp) : grp);
        }
      }
      // 3. right-looking inside the pass
#pragma unroll 1
      for (int Jl = 0; Jl < W; ++Jl) {
        const int J = W * P + Jl;
        double* tile = sT + (J & 1) * kTile;
        if (lane == 0) {
          if constexpr (NT == 1)
            bulk_wait_read<0>();
          else
            bulk_wait_read<1>();  // the store that last used this tile has read it
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 4; ++g)
          *reinterpret_cast<double2*>(tile + swz64(8 * g + gr, q)) = make_double2(acc[g][0][0], acc[g][0][1]);
        __syncwarp();
        {
          const double* D = sD + J * kDiagStride;
          double y[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 v = *reinterpret_cast<const double2*>(tile + swz64(lane, u));
            y[2 * u] = v.x;
            y[2 * u + 1] = v.y;
          }
          bool good = D[80] != 0.0;  // uniform: no zero in the strict upper block, safe divisors
#ifdef CQR_TRI_NODIAG  // probe: without the diagonal recurrence
          if (good) {
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] *= D[64 + j];
          } else
#endif
          if (good) {
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
          }
          if (!good) {  // rare: zeros in the block, extreme exponents or exact zeros
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = tile[swz64(lane, j >> 1) + (j & 1)];
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
            *reinterpret_cast<double2*>(tile + swz64(lane, u)) = make_double2(y[2 * u], y[2 * u + 1]);
        }
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
#ifndef CQR_TRI_NO_HINT
          tma_store_2d_hint(&tm_st, 8 * J, row0, tile, pol_out);
#else
          tma_store_2d(&tm_st, 8 * J, row0, tile);
#endif
          bulk_commit();
        }
        double af[4][2];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int kk4 = 0; kk4 < 2; ++kk4) {
            af[g][kk4] = tile[swz64(8 * g + gr, 2 * kk4 + (q >> 1)) + (q & 1)];
          }
        if (TMW > 0 && tmw && J < NT - W) {
          const double v8[8] = {af[0][0], af[1][0], af[2][0], af[3][0], af[0][1], af[1][1], af[2][1], af[3][1]};
          tm_st16(tm_warp + 16u * J, v8);
        }
        const double* bcol = sB + (2 * J) * 32 + lane;
#pragma unroll
        for (int t = 1; t < W; ++t) {
          if (Jl + t < W) {
            const int JJ = J + t;
            const double* bp = bcol + (JJ * (JJ - 1)) * 32;
#pragma unroll
            for (int kk4 = 0; kk4 < 2; ++kk4) {
              const double bv = BSMEM ? bp[kk4 * 32] : __ldg(bp + kk4 * 32);
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
    }
  }
  if (lane == 0) bulk_wait<0>();
  __syncwarp();
  if constexpr (TMW > 0) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

template <int NP, int WPC, bool BSMEM, int TMW = 0>
cudaError_t launch_t(const TrisolveArgs& a, cudaStream_t s) {
  CUtensorMap tin, tll, tst;
  if (!make_tmap_2d(&tin, a.in, a.n, a.m, a.ldi, 8, kRW, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_tmap_2d(&tll, a.out, a.n, a.m, a.ldo, 4, kRW, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_tmap_2d(&tst, a.out, a.n, a.m, a.ldo, 8, kRW, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorNotSupported;
  const size_t smem = (size_t)(head_doubles<NP, BSMEM>() + WPC * kWarpDoubles) * 8 + WPC * 16 + 512;
  auto k = trisolve_tma_kernel<NP, WPC, BSMEM, TMW>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  const long long groups = (a.m + kRW - 1) / kRW;
  long long grid = (groups + WPC - 1) / WPC;
  if (grid > (long long)a.num_sms) grid = a.num_sms;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, WPC * 32, smem, s>>>(tin, tll, tst, a.m, a.n, a.bpack, a.dpack, a.status);
  return cudaGetLastError();
}

}  // namespace

bool make_tmap_2d(CUtensorMap* map, const double* base, long long cols, long long rows, long long ld, int box_cols,
                  int box_rows, CUtensorMapSwizzle swizzle) {
  auto fn = encode_fn();
  if (!fn || ((uintptr_t)base & 15) || ((ld * 8) & 15) || cols < 1 || rows < 1 || ld < cols) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_colblocks(CUtensorMap* map, const double* base, long long cols, long long rows, long long ld,
                         int box_rows, int box_blocks, CUtensorMapSwizzle swizzle, int bw) {
  auto fn = encode_fn();
  if (!fn || ((uintptr_t)base & 15) || ((ld * 8) & 15) || cols < bw || (cols % bw) || rows < 1 || ld < cols)
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)bw, (cuuint64_t)rows, (cuuint64_t)(cols / bw)};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)bw * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)box_rows, (cuuint32_t)box_blocks};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool trisolve_tma_eligible(const TrisolveArgs& a, int np) {
  return np >= 32 && a.m <= (1LL << 31) - 64 && ((uintptr_t)a.in & 15) == 0 && ((uintptr_t)a.out & 15) == 0 &&
         (a.ldi & 1) == 0 && (a.ldo & 1) == 0 && encode_fn() != nullptr;
}

#ifndef CQR_TRI128_WPC
#define CQR_TRI128_WPC 12
#endif
#ifndef CQR_TRI128_BSMEM
#define CQR_TRI128_BSMEM true
#endif
#ifndef CQR_TRI256_WPC
#define CQR_TRI256_WPC 16  // 16 warps fit at 512-byte alignment (2.857 -> 2.820 ms); n = 512: 13 warps 15.4 vs 12 warps 10.0
#endif
#ifndef CQR_TRI512_WPC
#define CQR_TRI512_WPC 12
#endif
// warps whose left-looking operand stays in TMEM (the rest read it back from L2): n = 128, 12 warps:
// 0/8 TMEM warps 0.777/0.757 ms (all 8 warps TMEM, WPC 8: 0.815); n = 256: 0/4 of 16 warps 2.74/2.60 ms
#ifndef CQR_TRI128_TMW
#define CQR_TRI128_TMW 8
#endif
#ifndef CQR_TRI256_TMW
#define CQR_TRI256_TMW 4
#endif
#ifndef CQR_TRI64_TMW
#define CQR_TRI64_TMW 0
#endif
#ifndef CQR_TRI64_WPC
#define CQR_TRI64_WPC 12
#endif
cudaError_t launch_trisolve_tma(const TrisolveArgs& a, int np, cudaStream_t s) {
  switch (np) {
    case 32: return launch_t<32, 16, true>(a, s);
    case 64: return launch_t<64, CQR_TRI64_WPC, true, CQR_TRI64_TMW>(a, s);
    case 128: return launch_t<128, CQR_TRI128_WPC, CQR_TRI128_BSMEM, CQR_TRI128_TMW>(a, s);
    case 256: return launch_t<256, CQR_TRI256_WPC, false, CQR_TRI256_TMW>(a, s);
    case 512: return launch_t<512, CQR_TRI512_WPC, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cqr
