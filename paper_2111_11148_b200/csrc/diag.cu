// diag.cu — device diagnostics (diagnostics.cpp:10-28): the residual
// ||A - QR||_F / ||A||_F and ||Q^T Q - I||_F (the latter from a Gram computed by
// gram.cu). Lets large configurations be validated without host passes over
// the tall matrices. Fixed reduction orders (deterministic).

#include "common.cuh"
#include "kernels.h"

namespace cqr {

namespace {

// One warp per row: lanes own columns j = lane + 32 t; q_i broadcast via shfl.
// Block partials -> partial[2*block + {0,1}] = (sum ||a - qR||^2, sum ||a||^2).
__global__ void residual_kernel(const double* __restrict__ a, long long lda, const double* __restrict__ q,
                                long long ldq, const double* __restrict__ r, long long m, int n,
                                double* __restrict__ partial) {
  __shared__ double sres[32], snorm[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double res = 0.0, nrm = 0.0;
  for (long long i = (long long)blockIdx.x * nw + warp; i < m; i += (long long)gridDim.x * nw) {
    const double* qi = q + i * ldq;
    const double* ai = a + i * lda;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      double acc = 0.0;
      for (int k = 0; k < n; ++k) {
        const double qk = qi[k];
        if (j < n) acc = fma(qk, r[(long long)k * n + j], acc);
      }
      if (j < n) {
        const double av = ai[j];
        const double d = av - acc;
        res = fma(d, d, res);
        nrm = fma(av, av, nrm);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    res += __shfl_xor_sync(0xffffffffu, res, o);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  }
  if (lane == 0) {
    sres[warp] = res;
    snorm[warp] = nrm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < nw; ++w) {
      s0 += sres[w];
      s1 += snorm[w];
    }
    partial[2 * blockIdx.x] = s0;
    partial[2 * blockIdx.x + 1] = s1;
  }
}

__global__ void residual_final_kernel(const double* __restrict__ partial, int nblocks, double* out) {
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      s0 += partial[2 * b];
      s1 += partial[2 * b + 1];
    }
    out[0] = s0;
    out[1] = s1;
  }
}

__global__ void orth_kernel(const double* __restrict__ g, int n, double* out) {
  __shared__ double sw[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double s = 0.0;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    const double v = g[e] - (i == j ? 1.0 : 0.0);
    s = fma(v, v, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sw[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sw[w];
    out[0] = sqrt(t);
  }
}

}  // namespace

cudaError_t launch_residual(const double* a, long long lda, const double* q, long long ldq, const double* r,
                            long long m, int n, double* partial, int nblocks, double* out, cudaStream_t s) {
  residual_kernel<<<nblocks, 256, 0, s>>>(a, lda, q, ldq, r, m, n, partial);
  residual_final_kernel<<<1, 32, 0, s>>>(partial, nblocks, out);
  return cudaGetLastError();
}

cudaError_t launch_orth_from_gram(const double* g, int n, double* out, cudaStream_t s) {
  orth_kernel<<<1, 1024, 0, s>>>(g, n, out);
  return cudaGetLastError();
}

}  // namespace cqr
