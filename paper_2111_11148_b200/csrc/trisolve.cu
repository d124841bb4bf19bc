// trisolve.cu — tall right triangular solve X R = A (kernels.hpp:94-127): the
// packed R, the dispatcher, and the register kernel used when A or X is not
// TMA-addressable (the default kernel is trisolve_tma.cu).
//
// Reference recurrence, per row and column j: y_j = a_j; for k < j:
// y_j = fma(-r_kj, x_k, y_j) (skipped when r_kj == 0); x_j = y_j / r_jj. A row's
// result depends only on that row, so any row partition gives the same bits
// (kernels.hpp:98-101).
//
// B200 mapping (both kernels). A warp owns 32 rows; columns go in blocks J of 8:
//  1. off-diagonal part, k < 8J: DMMA m8n8k4 with A = solved X columns and
//     B = -R fragments (pack_r). DMMA accumulates as the sequential fma chain
//     in k order (profiles/r01_fp64_probe.txt, r01_dmma_shapes.txt), so this is
//     the reference's chain bit for bit (zero terms are not skipped: only the
//     sign of an exact zero can differ);
//  2. diagonal 8x8 block, one lane per row: the remaining k in [8J, j) as
//     scalar fma, then the division: RN(1/r_jj) (computed once per column by
//     pack_r) and one Markstein correction, the correctly rounded quotient for
//     the operand window of trisolve_common.cuh (IEEE division outside it).
// Rows are independent, so warps never synchronise with each other.
//
// Per row: HBM 8n bytes read + 8n written; n^2 flops (n(n-1)/2 fma + n div).

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "trisolve_common.cuh"

namespace cqr {

namespace {
using namespace tri;

__global__ void pack_r_kernel(const double* __restrict__ r, int ldr, int n, int np, double* __restrict__ bpack,
                              double* __restrict__ dpack, int* __restrict__ bad_min, int degenerate,
                              const double* __restrict__ sgn, DevStatus* st) {
  if (failed(st)) return;
  // With column signs s (normalize_sign, engine.cpp:109-116) the pack holds diag(s) R: solving with it gives
  // Q = X R^-1 diag(s) directly, bit for bit (every product and quotient only changes sign, and
  // s_k R_kj * s_k x_k == R_kj x_k exactly, zeros included).
  auto R = [&](int i, int j) -> double {
    if (i < n && j < n) return sgn ? r[(long long)i * ldr + j] * sgn[i] : r[(long long)i * ldr + j];
    return (i == j) ? 1.0 : 0.0;
  };
  const int nt = np / 8;
  const long long nb = (long long)nt * (nt - 1) * 32;
  const long long nd = (long long)nt * kDiagStride;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nb + nd;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nb) {
      const int lane = (int)(e & 31);
      const long long f = e >> 5;
      int J = (int)((1.0 + sqrt(1.0 + 4.0 * (double)f)) * 0.5);
      while ((long long)J * (J - 1) > f) --J;
      while ((long long)(J + 1) * J <= f) ++J;
      const int k4 = (int)(f - (long long)J * (J - 1));
      bpack[e] = -R(4 * k4 + (lane & 3), 8 * J + (lane >> 2));
    } else {
      const long long d = e - nb;
      const int J = (int)(d / kDiagStride), w = (int)(d % kDiagStride);
      double v;
      if (w >= kColBase) {
        const int o = w - kColBase;
        int j = 0;
        while (j < 7 && col_start(j + 1) <= o) ++j;
        const int p = o - col_start(j), jj = 8 * J + j;
        v = p < j ? R(8 * J + p, jj) : p == j ? R(jj, jj) : p == j + 1 ? 1.0 / R(jj, jj) : 0.0;
      } else if (w < 64) {
        v = R(8 * J + w / 8, 8 * J + w % 8);
      } else if (w >= 80) {
        v = 0.0;
        if (w == 80) {
          bool ok = true;
          for (int a = 0; a < 8; ++a) {
            const double da = fabs(R(8 * J + a, 8 * J + a));
            ok = ok && da >= 0x1p-500 && da <= 0x1p+500;
            for (int b = a + 1; b < 8; ++b) ok = ok && R(8 * J + a, 8 * J + b) != 0.0;
          }
          v = ok ? 1.0 : 0.0;
        }
      } else {
        const int j = 8 * J + (w - 64) % 8;
        const double dj = R(j, j);
        if (w < 72) {
          v = 1.0 / dj;
        } else {
          const double a = fabs(dj);
          v = (a >= 0x1p-500 && a <= 0x1p+500) ? 1.0 : 0.0;
        }
      }
      dpack[d] = v;
    }
  }
  // diagonal check, lowest failing index (kernels.hpp:106-107 / engine.cpp:118-127)
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; bad_min && j < n; j += gridDim.x * blockDim.x) {
    const double dj = r[(long long)j * ldr + j];
    if (dj == 0.0 || (degenerate && !isfinite(dj))) atomicMin(bad_min, j);
  }
}

__global__ void pack_status_kernel(const int* bad_min, int n, DevStatus* st) {
  if (*bad_min < n) set_status(st, 2 /*CQR_SINGULAR_TRIANGULAR*/, *bad_min);
}

// Register kernel (the fallback when A or X is not TMA-addressable). A warp owns 32 rows (4 DMMA row groups;
// one lane per row in the scalar part, so all 32 lanes work). Columns go in
// passes of 64 (8 blocks of 8), the pass held in DMMA accumulator registers:
//  1. left-looking: contributions of all columns solved in earlier passes,
//     k ascending, A fragments re-read from the output (this warp's own rows,
//     L2-resident; column signs, when fused, are undone exactly by a second
//     multiplication by +-1), 32 independent accumulator chains per step;
//  2. right-looking inside the pass: block J solved one lane per row (scalar fma
//     + correctly rounded division), then its 8 columns update the pass's later
//     blocks with DMMA; the 8-block window rotates so the loop is not unrolled.
// Every element therefore receives k = 0, 1, ..., j-1 in ascending order, the
// in-block terms last, then the division: the reference recurrence exactly.
// The 8-column staging tile of a warp: row-major, 64 bytes per row, its four
// 16-byte chunks XOR-swizzled by bits 1-2 of the row so that the C-fragment
// stores, the row-per-lane loads/stores and the A-fragment loads are all
// bank-conflict free.
__device__ __forceinline__ int swz(int row, int u) {
  return row * 8 + 2 * (u ^ ((((row >> 1) & 1) << 1) | ((row >> 2) & 1)));
}

template <int NP, int WPC, bool BSMEM, int WIN, int MG>
__global__ void __launch_bounds__(WPC * 32, 1)
    trisolve_sb_kernel(const double* in, long long ldi, double* out, long long ldo, long long m, int n,
                       const double* __restrict__ bpack, const double* __restrict__ dpack,
                       int vec16, const DevStatus* st) {
  constexpr int NT = NP / 8;
  constexpr int RW = 8 * MG;   // rows per warp
  constexpr int RPL = MG / 4;  // rows per lane in the diagonal recurrence (independent chains)
  constexpr int W = NT < WIN ? NT : WIN;  // window (blocks per pass)
  constexpr int NPASS = NT / W;
  constexpr int NB = BSMEM ? NT * (NT - 1) * 32 : 0;
  constexpr int ND = NT * kDiagStride;
  extern __shared__ __align__(16) double smem[];
  if (failed(st)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  double* sD = smem;
  const double* sB = bpack;
  double* sS = smem + ND + NB + warp * RW * 8;
  for (int e = threadIdx.x; e < ND; e += WPC * 32) sD[e] = dpack[e];
  if constexpr (BSMEM) {
    for (int e = threadIdx.x; e < NB; e += WPC * 32) smem[ND + e] = bpack[e];
    sB = smem + ND;
  }
  __syncthreads();
  const long long groups = (m + RW - 1) / RW;
  const long long gstride = (long long)gridDim.x * WPC;
  for (long long grp = (long long)blockIdx.x * WPC + warp; grp < groups; grp += gstride) {
    const long long row0 = grp * RW;
    const int rows = (int)min((long long)RW, m - row0);
    if constexpr (NP >= 256) {  // pull this warp's next row group into L2 while this one is solved
      const long long nrow0 = (grp + gstride) * RW;
      const int nrows = (int)max(0LL, min((long long)RW, m - nrow0));
      const int lines = (n * 8 + 127) / 128;
      for (int e = lane; e < nrows * lines; e += 32) {
        const int r = e / lines, li = e - r * lines;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(in + (nrow0 + r) * ldi + li * 16));
      }
    }
#pragma unroll 1
    for (int P = 0; P < NPASS; ++P) {
      const int c0 = 8 * W * P;
      double acc[MG][W][2];
#pragma unroll
      for (int g = 0; g < MG; ++g) {
        const int r = g * 8 + gr;
        const double* src = in + (row0 + r) * ldi + c0 + 2 * q;
#pragma unroll
        for (int t = 0; t < W; ++t) {
          const int c = c0 + 8 * t + 2 * q;
          if (r < rows && vec16 && c + 1 < n) {
            const double2 v = *reinterpret_cast<const double2*>(src + 8 * t);
            acc[g][t][0] = v.x;
            acc[g][t][1] = v.y;
          } else {
            acc[g][t][0] = (r < rows && c < n) ? src[8 * t] : 0.0;
            acc[g][t][1] = (r < rows && c + 1 < n) ? src[8 * t + 1] : 0.0;
          }
        }
      }
      // 1. left-looking: k in [0, c0), ascending
      if (P > 0) {
        const double* xrow[MG];
#pragma unroll
        for (int g = 0; g < MG; ++g) {
          const int r = min(g * 8 + gr, rows - 1);
          xrow[g] = out + (row0 + r) * ldo + q;
        }
#pragma unroll 2
        for (int k4 = 0; k4 < c0 / 4; ++k4) {
          double af[MG];
#pragma unroll
          for (int g = 0; g < MG; ++g) af[g] = xrow[g][4 * k4];
#pragma unroll
          for (int t = 0; t < W; ++t) {
            const int JJ = W * P + t;
            const int bi = (JJ * (JJ - 1) + k4) * 32 + lane;
            const double b = BSMEM ? sB[bi] : __ldg(sB + bi);
#pragma unroll
            for (int g = 0; g < MG; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g], b);
          }
        }
      }
      // 2. right-looking inside the pass
#pragma unroll 1
      for (int Jl = 0; Jl < W; ++Jl) {
        const int J = W * P + Jl;
#pragma unroll
        for (int g = 0; g < MG; ++g)
          *reinterpret_cast<double2*>(sS + swz(g * 8 + gr, q)) = make_double2(acc[g][0][0], acc[g][0][1]);
        __syncwarp();
        {
          const double* D = sD + J * kDiagStride;
          double y[RPL][8];
#pragma unroll
          for (int rr = 0; rr < RPL; ++rr) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double2 v = *reinterpret_cast<const double2*>(sS + swz(lane + 32 * rr, u));
              y[rr][2 * u] = v.x;
              y[rr][2 * u + 1] = v.y;
            }
          }
          bool good = D[80] != 0.0;  // uniform: no zero in the strict upper block, safe divisors
          if (good) {
            bool ok = true;
            const double* Dc = D + kColBase;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              double v[10];  // column j: R[0..j-1][j], R_jj, RN(1/R_jj), as 16-byte loads
#pragma unroll
              for (int h = 0; h < (j + 3) / 2; ++h) {
                const double2 t = *reinterpret_cast<const double2*>(Dc + col_start(j) + 2 * h);
                v[2 * h] = t.x;
                v[2 * h + 1] = t.y;
              }
#pragma unroll
              for (int rr = 0; rr < RPL; ++rr) {
#pragma unroll
                for (int kk = 0; kk < j; ++kk) y[rr][j] = fma(-v[kk], y[rr][kk], y[rr][j]);
                bool okj;
                y[rr][j] = div_fast(y[rr][j], v[j], v[j + 1], okj);
                ok &= okj;
              }
            }
            good = __all_sync(0xffffffffu, ok);
          }
          if (!good) {  // rare: zeros in the block, extreme exponents or exact zeros
#pragma unroll
            for (int rr = 0; rr < RPL; ++rr) {
#pragma unroll
              for (int j = 0; j < 8; ++j) y[rr][j] = sS[swz(lane + 32 * rr, j >> 1) + (j & 1)];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
#pragma unroll
                for (int kk = 0; kk < j; ++kk) {
                  const double rv = D[kk * 8 + j];
                  if (rv != 0.0) y[rr][j] = fma(-rv, y[rr][kk], y[rr][j]);
                }
                y[rr][j] = fast_div(y[rr][j], D[j * 8 + j], D[64 + j], D[72 + j] != 0.0);
              }
            }
          }
          __syncwarp();
#pragma unroll
          for (int rr = 0; rr < RPL; ++rr) {
            const int rl = lane + 32 * rr;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<double2*>(sS + swz(rl, u)) = make_double2(y[rr][2 * u], y[rr][2 * u + 1]);
          }
        }
        __syncwarp();
        // write the solved block back, 8 rows x 64 bytes per store (the tile in C-fragment order)
        {
          const int c = 8 * J + 2 * q;
#pragma unroll
          for (int g = 0; g < MG; ++g) {
            const int r = g * 8 + gr;
            if (r < rows) {
              const double2 v = *reinterpret_cast<const double2*>(sS + swz(r, q));
              double* o = out + (row0 + r) * ldo + c;
              if (vec16 && c + 1 < n) {
                *reinterpret_cast<double2*>(o) = v;
              } else {
                if (c < n) o[0] = v.x;
                if (c + 1 < n) o[1] = v.y;
              }
            }
          }
        }
        __syncwarp();
        double af[MG][2];
#pragma unroll
        for (int g = 0; g < MG; ++g)
#pragma unroll
          for (int kk4 = 0; kk4 < 2; ++kk4) af[g][kk4] = sS[swz(g * 8 + gr, 2 * kk4 + (q >> 1)) + (q & 1)];
        const double* bcol = sB + (2 * J) * 32 + lane;
#pragma unroll
        for (int t = 1; t < W; ++t) {
          if (Jl + t < W) {
            const int JJ = J + t;
            const double* bp = bcol + (JJ * (JJ - 1)) * 32;
#pragma unroll
            for (int kk4 = 0; kk4 < 2; ++kk4) {
              const double b = BSMEM ? bp[kk4 * 32] : __ldg(bp + kk4 * 32);
#pragma unroll
              for (int g = 0; g < MG; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g][kk4], b);
            }
          }
#pragma unroll
          for (int g = 0; g < MG; ++g) {
            acc[g][t - 1][0] = acc[g][t][0];
            acc[g][t - 1][1] = acc[g][t][1];
          }
        }
        __syncwarp();
      }
    }
  }
}

template <int NP, int WPC, bool BSMEM, int WIN = 8, int MG = 4>
cudaError_t launch_trisolve_sb_t(const TrisolveArgs& a, cudaStream_t s) {
  constexpr int NT = NP / 8;
  const size_t smem =
      (size_t)(NT * kDiagStride + (BSMEM ? NT * (NT - 1) * 32 : 0) + WPC * 8 * MG * 8) * sizeof(double);
  auto k = trisolve_sb_kernel<NP, WPC, BSMEM, WIN, MG>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  const long long groups = (a.m + 8 * MG - 1) / (8 * MG);
  long long grid = (groups + WPC - 1) / WPC;
  if (grid > (long long)a.num_sms) grid = a.num_sms;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, WPC * 32, smem, s>>>(a.in, a.ldi, a.out, a.ldo, a.m, a.n, a.bpack, a.dpack, a.vec16,
                                           a.status);
  return cudaGetLastError();
}

}  // namespace

int trisolve_np(int n) {
  if (n <= 8) return 8;
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (n <= 256) return 256;
  return 512;
}

// The wide solve in 128-column panels (panel.cu): n a multiple of 128, at least 384 (m = 1e6: n = 512
// 9.98 -> 9.09 ms; n = 256 2.61 -> 2.64 ms, so the one-pass kernel stays there).
static bool panel_path(int n) {
  static const bool off = std::getenv("CQR_TRISOLVE_NO_PANELS") != nullptr;  // A/B: the one-pass kernel
  return !off && n >= 384 && n % 128 == 0 && n <= 512;
}
constexpr size_t kSubPack = 16 * 15 * 32 + 16 * kDiagStride + 128;  // one 128-column diagonal block's pack

static size_t full_pack_doubles(int np) {
  const int nt = np / 8;
  return ((size_t)nt * (nt - 1) * 32 + (size_t)nt * kDiagStride + 8 + 127) / 128 * 128;
}

size_t trisolve_pack_doubles(int n) {
  const int np = trisolve_np(n);
  return full_pack_doubles(np) + (panel_path(n) ? (size_t)(n / 128) * kSubPack : 0);
}

cudaError_t launch_pack_r(const double* r, int ldr, int n, double* pack, int degenerate, DevStatus* st,
                          cudaStream_t s, const double* sgn) {
  const int np = trisolve_np(n);
  const int nt = np / 8;
  double* bpack = pack;
  double* dpack = pack + (size_t)nt * (nt - 1) * 32;
  int* bad = reinterpret_cast<int*>(dpack + (size_t)nt * kDiagStride);
  const long long total = (long long)nt * (nt - 1) * 32 + (long long)nt * kDiagStride;
  long long g0 = (total + 255) / 256;
  int grid = (int)(g0 < 512 ? g0 : 512);
  if (grid < 1) grid = 1;
  cudaError_t e = cudaMemsetAsync(bad, 0x7f, sizeof(int), s);  // 0x7f7f7f7f > any n
  if (e != cudaSuccess) return e;
  pack_r_kernel<<<grid, 256, 0, s>>>(r, ldr, n, np, bpack, dpack, bad, degenerate, sgn, st);
  pack_status_kernel<<<1, 1, 0, s>>>(bad, n, st);
  if (panel_path(n)) {  // the diagonal 128 x 128 blocks, each packed as an n = 128 problem
    for (int p = 0; p < n / 128; ++p) {
      double* sp = pack + full_pack_doubles(np) + (size_t)p * kSubPack;
      pack_r_kernel<<<64, 256, 0, s>>>(r + (size_t)128 * p * ldr + 128 * p, ldr, 128, 128, sp, sp + 16 * 15 * 32,
                                       nullptr, degenerate, sgn ? sgn + 128 * p : nullptr, st);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_trisolve(TrisolveArgs a, cudaStream_t s) {
  const int np = trisolve_np(a.n);
  const int nt = np / 8;
  a.bpack = a.pack;
  a.dpack = a.pack + (size_t)nt * (nt - 1) * 32;
  // variant 0: the register-resident right-looking kernel (np <= 128) or the left-looking TMA kernel
  // (wider); 2: the left-looking TMA kernel at every width; 1: the register kernel (A/B runs)
  if (a.variant == 0 && panel_path(a.n) && trisolve_tma_eligible(a, np)) {
    // 128-column panels: the GEMM update of panel p by panels 0 .. p-1, then the n = 128 solve in place
    bool ok = true;
    for (int p = 0; p < a.n / 128 && ok; ++p) {
      if (p > 0) {
        const cudaError_t e = launch_panel_update(a, 128 * p, s);
        if (e == cudaErrorNotSupported) {
          ok = false;
          break;
        }
        if (e != cudaSuccess) return e;
      }
      TrisolveArgs b = a;
      b.in = p == 0 ? a.in : a.out + 128 * p;
      b.ldi = p == 0 ? a.ldi : a.ldo;
      b.out = a.out + 128 * p;
      b.n = 128;
      b.pack = a.pack + full_pack_doubles(np) + (size_t)p * kSubPack;
      b.bpack = b.pack;
      b.dpack = b.pack + 16 * 15 * 32;
      if (!trisolve_tma_eligible(b, 128)) {
        ok = false;
        break;
      }
      const cudaError_t e = launch_trisolve_tma(b, 128, s);
      if (e != cudaSuccess) return e;
    }
    if (ok) return cudaSuccess;
    // (only reachable before the first launch: the eligibility of the views matches the whole matrix's)
  }
  if ((a.variant == 0 || a.variant == 2) && trisolve_tma_eligible(a, np)) {
    // the right-looking kernel at np <= 64 (c3: 1.032 vs 1.058 ms per call; at np = 128 its 16-row
    // warps leave the diagonal recurrence on half the lanes: 0.97 vs 0.77 ms, so the left-looking kernel;
    // a variant with warp pairs sharing 32-row groups, each warp owning every other 8-column block and the
    // blocks handed over by named barriers, was bitwise equal but slower still: 1.22 ms -- the hand-over
    // serialises the two warps' recurrences and leaves the FP64 pipe idle while a warp waits)
    if (a.variant == 0 && np <= 64) {
      const cudaError_t e = launch_trisolve_rr(a, np, s);
      if (e != cudaErrorNotSupported) return e;
    }
    const cudaError_t e = launch_trisolve_tma(a, np, s);
    if (e != cudaErrorNotSupported) return e;
  }
  // register kernel (best measured configuration per width)
  switch (np) {
    case 8: return launch_trisolve_sb_t<8, 12, true>(a, s);
    case 16: return launch_trisolve_sb_t<16, 12, true>(a, s);
    case 32: return launch_trisolve_sb_t<32, 16, true, 4>(a, s);
    case 64: return launch_trisolve_sb_t<64, 16, true, 4>(a, s);
    case 128: return launch_trisolve_sb_t<128, 12, true, 4>(a, s);
    case 256: return launch_trisolve_sb_t<256, 12, false, 4>(a, s);
    case 512: return launch_trisolve_sb_t<512, 8, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cqr
