// trisolve.cu — tall right triangular solve X R = A (kernels.hpp:94-127).
//
// Reference recurrence, per row and column j: y_j = a_j; for k < j:
// y_j = fma(-r_kj, x_k, y_j); x_j = y_j / r_jj. A row's result depends only on
// that row, so any row partition gives the same bits (kernels.hpp:98-101).
//
// B200 mapping: each warp owns a panel of 8*MG rows staged in shared memory.
// Columns are processed in blocks J of 8. The contributions of all earlier
// blocks (k < 8J) are accumulated with DMMA m8n8k4 (A operand = solved X
// columns from smem, B operand = -R tile). DMMA accumulates as the sequential
// fma chain in k order, so this is the reference's chain bit for bit. The
// 8x8 diagonal block then runs the remaining k in [8J, j) as scalar fma + an
// IEEE division, inside the DMMA accumulator registers (4 lanes per row,
// shuffles broadcast x_k). Rows are independent, so warps never synchronise.
//
// HBM bytes per row: 8n read + 8n written; flops: n^2 (n(n-1)/2 fma + n div).

#include "common.cuh"
#include "kernels.h"

namespace cqr {

namespace {

// Bpack[(J*(J-1) + k4)*32 + lane] = -R[4*k4 + (lane&3)][8*J + (lane>>2)], k4 < 2J
// Dpack[J*64 + kk*8 + q*2 + e]     = R[8J+kk][8J + 2q + e]          (8x8 diagonal block)
// R is padded to np with the identity. Checks the diagonal first (lowest
// index wins): degenerate=1 flags zero or non-finite (engine.cpp:118-127),
// degenerate=0 flags exact zeros only (kernels.hpp:106-107).
__global__ void pack_r_kernel(const double* __restrict__ r, int ldr, int n, int np, double* __restrict__ bpack,
                              double* __restrict__ dpack, int degenerate, DevStatus* st) {
  if (failed(st)) return;
  __shared__ int bad;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int b = -1;
    for (int j = 0; j < n; ++j) {
      const double d = r[(long long)j * ldr + j];
      if (d == 0.0 || (degenerate && !isfinite(d))) {
        b = j;
        break;
      }
    }
    if (b >= 0) set_status(st, 2 /*CQR_SINGULAR_TRIANGULAR*/, b);
  }
  (void)bad;
  auto R = [&](int i, int j) -> double {
    if (i < n && j < n) return r[(long long)i * ldr + j];
    return (i == j) ? 1.0 : 0.0;
  };
  const int nt = np / 8;
  const long long nb = (long long)nt * (nt - 1) * 32;
  const long long nd = (long long)nt * 64;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nb + nd;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nb) {
      const int lane = (int)(e & 31);
      const long long f = e >> 5;
      // invert f = J*(J-1) + k4, 0 <= k4 < 2J
      int J = (int)((1.0 + sqrt(1.0 + 4.0 * (double)f)) * 0.5);
      while ((long long)J * (J - 1) > f) --J;
      while ((long long)(J + 1) * J <= f) ++J;
      const int k4 = (int)(f - (long long)J * (J - 1));
      bpack[e] = -R(4 * k4 + (lane & 3), 8 * J + (lane >> 2));
    } else {
      const long long d = e - nb;
      const int J = (int)(d / 64), w = (int)(d % 64);
      const int kk = w / 8, q = (w % 8) / 2, ee = w % 2;
      dpack[d] = R(8 * J + kk, 8 * J + 2 * q + ee);
    }
  }
}

template <int NP, int MG, int WPC, bool BSMEM>
__global__ void __launch_bounds__(WPC * 32) trisolve_kernel(const double* in, long long ldi, double* out,
                                                            long long ldo, long long m, int n,
                                                            const double* __restrict__ bpack,
                                                            const double* __restrict__ dpack,
                                                            const double* __restrict__ sgn, int vec16,
                                                            const DevStatus* st) {
  constexpr int NT = NP / 8;
  constexpr int RW = 8 * MG;
  constexpr int LDX = NP + 4;
  constexpr int NB = NT * (NT - 1) * 32;
  extern __shared__ __align__(16) double smem[];
  if (failed(st)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  const double* sB = bpack;
  double* sX = smem + (BSMEM ? NB : 0) + warp * RW * LDX;
  if constexpr (BSMEM) {
    double* s = smem;
    for (int e = threadIdx.x; e < NB; e += WPC * 32) s[e] = bpack[e];
    sB = s;
    __syncthreads();
  }
  const long long groups = (m + RW - 1) / RW;
  for (long long grp = (long long)blockIdx.x * WPC + warp; grp < groups; grp += (long long)gridDim.x * WPC) {
    const long long row0 = grp * RW;
    const int rows = (int)min((long long)RW, m - row0);
    stage_rows(sX, LDX, in + row0 * ldi, ldi, rows, RW, n, NP, lane, 32, vec16 != 0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll 1
    for (int J = 0; J < NT; ++J) {
      double c[MG][2];
#pragma unroll
      for (int g = 0; g < MG; ++g) {
        const double2 v = *reinterpret_cast<const double2*>(sX + (g * 8 + gr) * LDX + 8 * J + 2 * q);
        c[g][0] = v.x;
        c[g][1] = v.y;
      }
      const double* bj = sB + (long long)J * (J - 1) * 32 + lane;
      const double* xa = sX + gr * LDX + q;
#pragma unroll 4
      for (int k4 = 0; k4 < 2 * J; ++k4) {
        const double b = BSMEM ? bj[k4 * 32] : __ldg(bj + k4 * 32);
#pragma unroll
        for (int g = 0; g < MG; ++g) dmma(c[g][0], c[g][1], xa[g * 8 * LDX + 4 * k4], b);
      }
      // diagonal block: remaining k in [8J, j) then the division, per row
      double dv[8][2];
      const double* dp = dpack + J * 64 + q * 2;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(dp + kk * 8));
        dv[kk][0] = v.x;
        dv[kk][1] = v.y;
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int qo = kk >> 1, eo = kk & 1;
#pragma unroll
        for (int g = 0; g < MG; ++g) {
          double x = 0.0;
          if (q == qo) {
            x = (eo ? c[g][1] : c[g][0]) / (eo ? dv[kk][1] : dv[kk][0]);
            if (eo)
              c[g][1] = x;
            else
              c[g][0] = x;
          }
          x = __shfl_sync(0xffffffffu, x, (lane & ~3) | qo);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 2 * q + e;
            if (col > kk) {
              const double rr = dv[kk][e];
              if (rr != 0.0) c[g][e] = fma(-rr, x, c[g][e]);
            }
          }
        }
      }
      // publish the solved block: smem (operand for later blocks) and global
#pragma unroll
      for (int g = 0; g < MG; ++g) {
        *reinterpret_cast<double2*>(sX + (g * 8 + gr) * LDX + 8 * J + 2 * q) = make_double2(c[g][0], c[g][1]);
        const int r = g * 8 + gr;
        const int col = 8 * J + 2 * q;
        if (r < rows) {
          double* o = out + (row0 + r) * ldo + col;
          double v0 = c[g][0], v1 = c[g][1];
          if (sgn != nullptr) {
            if (col < n) v0 *= sgn[col];
            if (col + 1 < n) v1 *= sgn[col + 1];
          }
          if (vec16 && col + 1 < n) {
            *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
          } else {
            if (col < n) o[0] = v0;
            if (col + 1 < n) o[1] = v1;
          }
        }
      }
      __syncwarp();
    }
  }
}

template <int NP, int MG, int WPC, bool BSMEM>
cudaError_t launch_trisolve_t(const TrisolveArgs& a, cudaStream_t s) {
  constexpr int NT = NP / 8;
  const size_t smem = (size_t)((BSMEM ? NT * (NT - 1) * 32 : 0) + WPC * 8 * MG * (NP + 4)) * sizeof(double);
  auto k = trisolve_kernel<NP, MG, WPC, BSMEM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long groups = (a.m + 8 * MG - 1) / (8 * MG);
  long long grid = (groups + WPC - 1) / WPC;
  const long long cap = (long long)a.num_sms * 1;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, WPC * 32, smem, s>>>(a.in, a.ldi, a.out, a.ldo, a.m, a.n, a.bpack, a.dpack, a.sgn, a.vec16,
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

size_t trisolve_pack_doubles(int n) {
  const int np = trisolve_np(n);
  const int nt = np / 8;
  return (size_t)nt * (nt - 1) * 32 + (size_t)nt * 64 + 64;
}

cudaError_t launch_pack_r(const double* r, int ldr, int n, double* pack, int degenerate, DevStatus* st,
                          cudaStream_t s) {
  const int np = trisolve_np(n);
  const int nt = np / 8;
  double* bpack = pack;
  double* dpack = pack + (size_t)nt * (nt - 1) * 32;
  const long long total = (long long)nt * (nt - 1) * 32 + (long long)nt * 64;
  long long g0 = (total + 255) / 256;
  int grid = (int)(g0 < 1024 ? g0 : 1024);
  if (grid < 1) grid = 1;
  pack_r_kernel<<<grid, 256, 0, s>>>(r, ldr, n, np, bpack, dpack, degenerate, st);
  return cudaGetLastError();
}

cudaError_t launch_trisolve(TrisolveArgs a, cudaStream_t s) {
  const int np = trisolve_np(a.n);
  const int nt = np / 8;
  a.bpack = a.pack;
  a.dpack = a.pack + (size_t)nt * (nt - 1) * 32;
  switch (np) {
    case 8: return launch_trisolve_t<8, 2, 16, true>(a, s);
    case 16: return launch_trisolve_t<16, 2, 16, true>(a, s);
    case 32: return launch_trisolve_t<32, 2, 16, true>(a, s);
    case 64: return launch_trisolve_t<64, 2, 16, true>(a, s);
    case 128: return launch_trisolve_t<128, 2, 8, true>(a, s);
    case 256: return launch_trisolve_t<256, 2, 6, false>(a, s);
    case 512: return launch_trisolve_t<512, 1, 6, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cqr
