// panel.cu — the wide right trisolve X R = A (n = 256, 512: c2, c4) in 128-column panels.
//
// The left-looking TMA kernel re-reads, for every 32-column pass, all of a warp's earlier solved columns;
// at n = 512 those re-reads no longer fit in L2 (3.4x the algorithmic DRAM bytes). Here the solve runs in
// panels of 128 columns. For panel p > 0 a tall GEMM first applies every earlier panel at once,
//
//     X[:, P] <- A[:, P] - X[:, 0:128p] R[0:128p, P]          (P = columns 128p .. 128p + 127),
//
// on DMMA with each element's chain in k order starting from a_ij -- the reference recurrence's first
// 128p terms (kernels.hpp:116-119), bit for bit (DMMA accumulates as the sequential fma chain in k order) --
// and then the n = 128 TMA kernel solves the panel in place with R[P, P], continuing every chain at
// k = 128p. X[:, 0:128p] is read once per panel, by whole row tiles.
//
// GEMM tile: 128 rows x 128 columns per CTA, 8 DMMA warps (32 rows x 64 columns each) fed through a
// 4-stage ring by one producer warp: per stage a TMA box of 16 solved columns x 128 rows (SWIZZLE_128B:
// conflict-free A fragments) and the matching 16 x 128 block of -R from the full pack (pack_r's B
// fragment order, 16 bulk copies of 1 KB).

#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"
#include "trisolve_common.cuh"

namespace cqr {

namespace {

constexpr int kPM = 128;                     // rows per tile
constexpr int kPK = 16;                      // k per stage
constexpr int kPStages = 4;
constexpr int kPX = kPM * kPK;               // doubles of X per stage (16 KB)
constexpr int kPB = kPK / 4 * 16 * 32;       // doubles of B per stage: 4 k4 x 16 column blocks x 32 lanes (16 KB)
constexpr int kPWarps = 8;                   // DMMA warps; + 1 producer
constexpr size_t kPSmem = (size_t)kPStages * (kPX + kPB) * 8 + 1024;

__global__ void __launch_bounds__((kPWarps + 1) * 32, 1)
    panel_update_kernel(const __grid_constant__ CUtensorMap tm_x, const double* __restrict__ in, long long ldi,
                        double* __restrict__ out, long long ldo, long long m, int c0, int K,
                        const double* __restrict__ bpack, const DevStatus* st) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kPStages], empty[kPStages];
  if (failed(st)) return;
  double* sm = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long row0 = (long long)blockIdx.x * kPM;
  const int nst = K / kPK;
  if (tid == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  __syncthreads();
  if (warp == kPWarps) {  // ---- producer
    if (lane == 0) {
      const int J0 = c0 / 8;
      for (int kc = 0; kc < nst; ++kc) {
        const int s = kc % kPStages;
        mbar_wait(&empty[s], ((kc / kPStages) & 1) ^ 1);
        double* sx = sm + s * (kPX + kPB);
        double* sb = sx + kPX;
        mbar_expect_tx(&full[s], (kPX + kPB) * 8);
        tma_load_2d(sx, &tm_x, kc * kPK, (int)row0, &full[s]);
        // column block t = global block J0 + t: its k4 steps 4 kc .. 4 kc + 3 are contiguous in the pack
        for (int t = 0; t < 16; ++t) {
          const long long J = J0 + t;
          const double* src = bpack + (J * (J - 1) + 4LL * kc) * 32;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sb + t * 128)),
              "l"(src), "r"(1024), "r"(smem_u32(&full[s]))
              : "memory");
        }
      }
    }
    return;
  }
  // ---- DMMA warps: rows rw .. rw + 31, column blocks tb .. tb + 7 of the panel
  const int q = lane & 3, gr = lane >> 2;
  const int rw = 32 * (warp & 3), tb = 8 * (warp >> 2);
  double acc[4][8][2];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const long long r = row0 + rw + 8 * g + gr;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      double2 v = make_double2(0.0, 0.0);
      if (r < m) v = *reinterpret_cast<const double2*>(in + r * ldi + c0 + 8 * (tb + t) + 2 * q);
      acc[g][t][0] = v.x;
      acc[g][t][1] = v.y;
    }
  }
  for (int kc = 0; kc < nst; ++kc) {
    const int s = kc % kPStages;
    mbar_wait(&full[s], (kc / kPStages) & 1);
    const double* sx = sm + s * (kPX + kPB);
    const double* sb = sx + kPX;
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      double af[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        // SWIZZLE_128B: the 16-byte chunk c of row r sits at chunk c ^ (r & 7); here r & 7 == gr
        const int r = rw + 8 * g + gr, k = 4 * k4 + q;
        af[g] = sx[r * 16 + (((k >> 1) ^ gr) << 1) + (k & 1)];
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double bv = sb[((tb + t) * 4 + k4) * 32 + lane];
#pragma unroll
        for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g], bv);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const long long r = row0 + rw + 8 * g + gr;
    if (r < m) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        *reinterpret_cast<double2*>(out + r * ldo + c0 + 8 * (tb + t) + 2 * q) = make_double2(acc[g][t][0], acc[g][t][1]);
    }
  }
}

}  // namespace

// X[:, c0 : c0 + 128] <- A[:, c0 : c0 + 128] - X[:, 0 : c0] R[0 : c0, c0 : c0 + 128] (chains in k order)
cudaError_t launch_panel_update(const TrisolveArgs& a, int c0, cudaStream_t s) {
  CUtensorMap tm;
  if (!make_tmap_2d(&tm, a.out, c0, a.m, a.ldo, kPK, kPM, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
  cudaError_t e = allow_max_smem(panel_update_kernel);
  if (e != cudaSuccess) return e;
  const long long tiles = (a.m + kPM - 1) / kPM;
  panel_update_kernel<<<(unsigned)tiles, (kPWarps + 1) * 32, kPSmem, s>>>(tm, a.in, a.ldi, a.out, a.ldo, a.m, c0, c0,
                                                                         a.bpack, a.status);
  return cudaGetLastError();
}

}  // namespace cqr
