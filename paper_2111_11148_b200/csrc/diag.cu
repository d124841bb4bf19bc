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

// ---- cond(X) = cond(R^) for the diagnostics of engine.cpp:94-100 ----------------------------------------
// One-sided Jacobi on the columns of the n x n R^ (kernels.hpp:272-310 computes the same singular values with
// a cyclic sweep on the host; here the pairs of a sweep are scheduled as a round robin, n/2 disjoint pairs per
// round, one warp per pair), the rotation and convergence rule of the reference (|gamma| <= tol sqrt(alpha beta),
// tol = 10 u sqrt(rows)). One CTA; W column-major in global scratch (L2-resident, n <= 512). out[0] = sigma_max /
// sigma_min (inf when sigma_min == 0, NaN when 100 sweeps do not converge).
namespace cqr {
namespace {
__global__ void __launch_bounds__(1024) jacobi_cond_kernel(const double* __restrict__ r, int n, double* W,
                                                           double* out) {
  __shared__ int changed;
  __shared__ double smax[32], smin[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < n * n; e += blockDim.x) {  // W(:, k) = R^(:, k)
    const int i = e / n, k = e % n;
    W[(long long)k * n + i] = r[e];
  }
  __syncthreads();
  const double tol = 10.0 * 2.220446049250313e-16 * sqrt((double)n);
  const int np = n + (n & 1);  // round-robin players (a dummy when n is odd)
  bool conv = n <= 1;
  for (int sweep = 0; sweep < 100 && !conv; ++sweep) {
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int round = 0; round < np - 1; ++round) {
      for (int pr = warp; pr < np / 2; pr += nw) {
        // players 0 fixed, 1 .. np-1 rotated by `round`
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (np - 1); };
        int p = player(pr), q = player(np - 1 - pr);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= n) continue;  // the dummy
        double* wp = W + (long long)p * n;
        double* wq = W + (long long)q * n;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double a = wp[i], b = wq[i];
          al = fma(a, a, al);
          be = fma(b, b, be);
          ga = fma(a, b, ga);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (fabs(ga) <= tol * sqrt(al * be)) continue;
        if (lane == 0) changed = 1;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = lane; i < n; i += 32) {
          const double a = wp[i], b = wq[i];
          wp[i] = cs * a - sn * b;
          wq[i] = sn * a + cs * b;
        }
      }
      __syncthreads();
    }
    conv = changed == 0;
    __syncthreads();
  }
  // sigma_j = ||W(:, j)||
  double mx = 0.0, mn = 1.0 / 0.0;
  for (int j = warp; j < n; j += nw) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s = fma(W[(long long)j * n + i], W[(long long)j * n + i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    s = sqrt(s);
    mx = fmax(mx, s);
    mn = fmin(mn, s);
  }
  if (lane == 0) {
    smax[warp] = mx;
    smin[warp] = mn;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < nw; ++w) {
      mx = fmax(mx, smax[w]);
      mn = fmin(mn, smin[w]);
    }
    mx = fmax(mx, smax[0]);
    mn = fmin(mn, smin[0]);
    out[0] = !conv ? __longlong_as_double(0x7ff8000000000000ll) : (mn > 0.0 ? mx / mn : 1.0 / 0.0);
  }
}
}  // namespace

cudaError_t launch_jacobi_cond(const double* r, int n, double* work, double* out, cudaStream_t s) {
  jacobi_cond_kernel<<<1, 1024, 0, s>>>(r, n, work, out);
  return cudaGetLastError();
}
}  // namespace cqr
