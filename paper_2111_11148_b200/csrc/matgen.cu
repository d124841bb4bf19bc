// matgen.cu — tall x small GEMM C = X * B (X m x n row-major with ldx, B n x n
// row-major, C m x n with ldc; C must not alias X), used by the device-side
// input synthesis (matgen.cpp:21-46: A = U * (diag(sigma) V^T), SURVEY 8f
// row 1). One warp per 32 rows, DMMA m8n8k4 over 64-column passes, k ascending.

#include "common.cuh"
#include "kernels.h"

namespace cqr {

namespace {

__global__ void __launch_bounds__(256) gemm_tall_kernel(const double* __restrict__ x, long long ldx,
                                                        const double* __restrict__ b, double* __restrict__ c,
                                                        long long ldc, long long m, int n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  const long long groups = (m + 31) / 32;
  for (long long grp = (long long)blockIdx.x * 8 + warp; grp < groups; grp += (long long)gridDim.x * 8) {
    const long long row0 = grp * 32;
    for (int c0 = 0; c0 < n; c0 += 64) {
      double acc[4][8][2];
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[g][t][0] = acc[g][t][1] = 0.0;
      for (int k4 = 0; k4 < (n + 3) / 4; ++k4) {
        const int k = 4 * k4 + q;
        double af[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const long long r = row0 + g * 8 + gr;
          af[g] = (r < m && k < n) ? x[r * ldx + k] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int col = c0 + 8 * t + gr;
          const double bv = (k < n && col < n) ? __ldg(b + (long long)k * n + col) : 0.0;
#pragma unroll
          for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g], bv);
        }
      }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const long long r = row0 + g * 8 + gr;
        if (r >= m) continue;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int col = c0 + 8 * t + 2 * q;
          if (col < n) c[r * ldc + col] = acc[g][t][0];
          if (col + 1 < n) c[r * ldc + col + 1] = acc[g][t][1];
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_gemm_tall(const double* x, long long ldx, const double* b, double* c, long long ldc, long long m,
                             int n, int num_sms, cudaStream_t s) {
  const long long groups = (m + 31) / 32;
  long long grid = (groups + 7) / 8;
  if (grid > (long long)num_sms * 4) grid = (long long)num_sms * 4;
  if (grid < 1) grid = 1;
  gemm_tall_kernel<<<(unsigned)grid, 256, 0, s>>>(x, ldx, b, c, ldc, m, n);
  return cudaGetLastError();
}

}  // namespace cqr
