// trisolve_rr.cu — register-resident, right-looking right trisolve X R = A for
// n <= 128 (the c1 and c3 widths).
//
// A warp owns RW rows (32 at n <= 64, 16 at n = 128) and keeps the whole RW x NP
// row tile in its DMMA accumulators. Block by block (8 columns): the block's
// tile goes through a 64-byte-swizzled staging tile so that each lane owns one
// row for the diagonal recurrence (the in-block fma terms, then the correctly
// rounded division), leaves by TMA tensor store, and is read back as DMMA A
// fragments to update every later block of the tile at once (k = the 8 solved
// columns). Every element therefore receives k = 0, 1, ..., j-1 in ascending
// order -- the off-block terms through DMMA chains (the DMMA accumulates as the
// sequential fma chain in k order), the in-block terms as scalar fma -- then
// the division: the reference recurrence (kernels.hpp:116-123) bit for bit, as
// the left-looking kernels (trisolve.cu, trisolve_tma.cu).
//
// What changes against the left-looking TMA kernel: no pass re-reads this
// warp's solved rows from global memory (no store -> L2 -> TMA round trip per
// pass, no left-looking slabs): A is read once, X written once (16mn bytes), and
// the input of the next group is prefetched by one TMA batch into the buffer
// the current group has just consumed.

#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"
#include "trisolve_common.cuh"

namespace cqr {

namespace {
using namespace tri;

__device__ __forceinline__ int swz64r(int r, int u) { return r * 8 + 2 * (u ^ ((r >> 1) & 3)); }

template <int NP, int RW, int WPC, bool BSMEM>
struct RrCfg {
  static constexpr int NT = NP / 8;
  static constexpr int G = RW / 8;                 // 8-row DMMA tiles per warp
  static constexpr int IN = RW * NP;               // input buffer (doubles): NT tiles of RW x 8
  static constexpr int TILE = RW * 8;              // staging tile (doubles)
  static constexpr int WARP = IN + 2 * TILE;       // per-warp shared memory (doubles)
  static constexpr int ND = NT * kDiagStride;
  static constexpr int NB = BSMEM ? NT * (NT - 1) * 32 : 0;
  static constexpr int HEAD = (ND + NB + 127) / 128 * 128;
  static constexpr size_t SMEM = (size_t)(HEAD + WPC * WARP) * 8 + WPC * 16 + 512;
};

// DMMA without `volatile`, so that the compiler may interleave the pending updates with the
// diagonal recurrence (the recurrence's dependent DFMA chain and the independent DMMAs share the
// FP64 pipe; issued from one warp in alternation the chain's latency hides behind DMMA work).
__device__ __forceinline__ void dmma_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// lane 0 issues a TMA tensor store of `src` and commits it as a bulk group (predicated, no branch)
__device__ __forceinline__ void store_tile_lane0(int lane, const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0;\n\t"
      "@p cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%1, {%3, %4}], [%2];\n\t"
      "@p cp.async.bulk.commit_group;\n\t}" ::"r"(lane),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
// lane 0 waits until all but the newest bulk group have read their sources
__device__ __forceinline__ void wait_read1_lane0(int lane) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0;\n\t@p cp.async.bulk.wait_group.read 1;\n\t}" ::"r"(lane)
               : "memory");
}

template <int NP, int RW, int WPC, bool BSMEM>
__global__ void __launch_bounds__(WPC * 32, 1)
    trisolve_rr_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_st,
                       long long m, const double* __restrict__ bpack, const double* __restrict__ dpack,
                       const DevStatus* st) {
  using C = RrCfg<NP, RW, WPC, BSMEM>;
  constexpr int NT = C::NT, G = C::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (failed(st)) return;
  double* smem = reinterpret_cast<double*>(smem_raw + ((512u - (smem_u32(smem_raw) & 511u)) & 511u));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  const int row = RW == 32 ? lane : (lane & (RW - 1));  // the row a lane takes in the recurrence
  double* sD = smem;
  const double* sB = bpack;
  double* sIn = smem + C::HEAD + warp * C::WARP;  // NT input tiles (RW x 8 each)
  double* sT = sIn + C::IN;                        // two staging tiles
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::HEAD + WPC * C::WARP) + 2 * warp;
  for (int e = threadIdx.x; e < C::ND; e += WPC * 32) sD[e] = dpack[e];
  if constexpr (BSMEM) {
    for (int e = threadIdx.x; e < C::NB; e += WPC * 32) smem[C::ND + e] = bpack[e];
    sB = smem + C::ND;
  }
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  __syncthreads();
  // blocks whose fast path is valid (no zero in the strict upper part, safe divisors): one register
  unsigned goodmask = 0;
#pragma unroll
  for (int J = 0; J < NT; ++J) goodmask |= (sD[J * kDiagStride + 80] != 0.0 ? 1u : 0u) << J;

  const uint64_t pol_in = l2_policy_evict_first();
  auto issue_in = [&](long long grp) {
    mbar_expect_tx(bar, C::IN * 8);
#pragma unroll
    for (int t = 0; t < NT; ++t) tma_load_2d_hint(sIn + t * C::TILE, &tm_in, 8 * t, (int)(grp * RW), bar, pol_in);
  };

  uint32_t ph = 0;
  const long long groups = (m + RW - 1) / RW;
  const long long gstride = (long long)gridDim.x * WPC;
  const long long rounds = groups / gstride;
  auto next_grp = [&](long long g) -> long long {  // as trisolve_tma.cu: the last partial round dealt CTA-major
    const long long k = g < rounds * gstride ? g / gstride : rounds;
    if (k + 1 < rounds) return g + gstride;
    if (k + 1 == rounds) return rounds * gstride + (long long)warp * gridDim.x + blockIdx.x;
    return groups;
  };
  long long grp = rounds > 0 ? (long long)blockIdx.x * WPC + warp : (long long)warp * gridDim.x + blockIdx.x;
  if (lane == 0 && grp < groups) issue_in(grp);
  for (; grp < groups; grp = next_grp(grp)) {
    const int row0 = (int)(grp * RW);
    mbar_wait(bar, ph);
    ph ^= 1;
    double acc[G][NT][2];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double2 v = *reinterpret_cast<const double2*>(sIn + t * C::TILE + (8 * g + gr) * 8 + 2 * q);
        acc[g][t][0] = v.x;
        acc[g][t][1] = v.y;
      }
    {  // the buffer is consumed: prefetch the next group's rows into it
      const long long nx = next_grp(grp);
      fence_async_shared();
      __syncwarp();
      if (lane == 0 && nx < groups) issue_in(nx);
    }
    double afp[G][2];  // A fragments of the previous block: its updates into blocks >= J+1 are pending
#pragma unroll
    for (int J = 0; J < NT; ++J) {
      double* tile = sT + (J & 1) * C::TILE;
      wait_read1_lane0(lane);  // the store that last used this tile has read it
      __syncwarp();
#pragma unroll
      for (int g = 0; g < G; ++g)
        *reinterpret_cast<double2*>(tile + swz64r(8 * g + gr, q)) = make_double2(acc[g][J][0], acc[g][J][1]);
      __syncwarp();
      // diagonal recurrence (fast path, branch-free), one row per lane, interleaved with the pending
      // updates of block J-1 into the blocks after J
      const double* D = sD + J * kDiagStride;
      const double* Dc = D + kColBase;
      double y[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 v = *reinterpret_cast<const double2*>(tile + swz64r(row, u));
        y[2 * u] = v.x;
        y[2 * u + 1] = v.y;
      }
      bool ok = true;
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
      if (J >= 1) {
#pragma unroll
        for (int t = J + 1; t < NT; ++t) {
          const double* bp = sB + (t * (t - 1) + 2 * (J - 1)) * 32 + lane;
#pragma unroll
          for (int kk4 = 0; kk4 < 2; ++kk4) {
            const double bv = BSMEM ? bp[kk4 * 32] : __ldg(bp + kk4 * 32);
#pragma unroll
            for (int g = 0; g < G; ++g) dmma_nv(acc[g][t][0], acc[g][t][1], afp[g][kk4], bv);
          }
        }
      }
      if (!(((goodmask >> J) & 1u) && __all_sync(0xffffffffu, ok || lane >= RW))) {
        // rare: zeros in the block, extreme exponents or exact zeros -- the guarded recurrence
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = tile[swz64r(row, j >> 1) + (j & 1)];
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
      if (RW == 32 || lane < RW) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<double2*>(tile + swz64r(row, u)) = make_double2(y[2 * u], y[2 * u + 1]);
      }
      fence_async_shared();
      __syncwarp();
      store_tile_lane0(lane, &tm_st, 8 * J, row0, tile);
      if (J + 1 < NT) {
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int kk4 = 0; kk4 < 2; ++kk4) afp[g][kk4] = tile[swz64r(8 * g + gr, 2 * kk4 + (q >> 1)) + (q & 1)];
        // the next block's update now (the critical path); the later blocks' wait for the next recurrence
        const double* bp = sB + ((J + 1) * J + 2 * J) * 32 + lane;
#pragma unroll
        for (int kk4 = 0; kk4 < 2; ++kk4) {
          const double bv = BSMEM ? bp[kk4 * 32] : __ldg(bp + kk4 * 32);
#pragma unroll
          for (int g = 0; g < G; ++g) dmma_nv(acc[g][J + 1][0], acc[g][J + 1][1], afp[g][kk4], bv);
        }
      }
    }
  }
  if (lane == 0) bulk_wait<0>();
  __syncwarp();
}

template <int NP, int RW, int WPC, bool BSMEM>
cudaError_t launch_rr(const TrisolveArgs& a, cudaStream_t s) {
  using C = RrCfg<NP, RW, WPC, BSMEM>;
  CUtensorMap tin, tst;
  if (!make_tmap_2d(&tin, a.in, a.n, a.m, a.ldi, 8, RW, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_tmap_2d(&tst, a.out, a.n, a.m, a.ldo, 8, RW, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorNotSupported;
  auto k = trisolve_rr_kernel<NP, RW, WPC, BSMEM>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  const long long groups = (a.m + RW - 1) / RW;
  long long grid = (groups + WPC - 1) / WPC;
  if (grid > (long long)a.num_sms) grid = a.num_sms;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, WPC * 32, C::SMEM, s>>>(tin, tst, a.m, a.bpack, a.dpack, a.status);
  return cudaGetLastError();
}

}  // namespace

#ifndef CQR_RR128_WPC
#define CQR_RR128_WPC 8
#endif
#ifndef CQR_RR128_BSMEM
#define CQR_RR128_BSMEM true
#endif
#ifndef CQR_RR64_RW
#define CQR_RR64_RW 32
#endif
#ifndef CQR_RR64_WPC
#define CQR_RR64_WPC 8  // 226 registers, no spills (10 warps: 168 registers with spills, 1.32 vs 1.03 ms at c3)
#endif
cudaError_t launch_trisolve_rr(const TrisolveArgs& a, int np, cudaStream_t s) {
  switch (np) {
    case 32: return launch_rr<32, 32, 12, true>(a, s);
    case 64: return launch_rr<64, CQR_RR64_RW, CQR_RR64_WPC, true>(a, s);
    case 128: return launch_rr<128, 16, CQR_RR128_WPC, CQR_RR128_BSMEM>(a, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace cqr
