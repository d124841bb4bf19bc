// householder.cu — tall Householder QR on the device: the dense baseline
// method (Method::HouseholderQr, engine.cpp:227-239, kernels.hpp:192-209) and
// the reference's matrix generator random_orthogonal (matgen.cpp:12-19: the
// thin Householder Q of a Gaussian matrix, signs as Householder leaves them).
//
// Column-by-column (unblocked) Householder on the row-major m x n working
// matrix W, the reflector of column c (the published algorithm behind Eigen's
// makeHouseholder, restated by the oracle): with x = W(c.., c),
//   beta = -sign(x_c) sqrt(x_c^2 + ||x_tail||^2),  tau = (beta - x_c) / beta,
//   v = x_tail / (x_c - beta)  (v_c = 1),          tau = 0 when ||x_tail||^2 <= tiny^2.
// Per column, one pass reduces the dot products x^T W(.., j) for every j >= c
// (block partials in a fixed order, summed over ranks by the engine's
// collectives when the rows are sharded), a one-block kernel forms beta, tau
// and w_j = v^T W(.., j), and one pass applies W(.., j) -= tau v w_j and stores
// v below the diagonal. The thin Q = H_0 ... H_{n-1} [I; 0] is accumulated
// backwards with the same two passes. Memory-bound (each column re-reads the
// trailing matrix): a baseline and an input generator, not the hot path.
// Deterministic run to run; parity with the oracle is a tolerance.

#include "common.cuh"
#include "kernels.h"

namespace cqr {

namespace {

constexpr int kHhThreads = 256;

// partial[b * w + t] = sum over this block's rows i (global index > c) of x_i * Y(i, c + t), t < w = n - c,
// x_i = X(i, c). Rows are this rank's [0, m_local) with global index row0 + i.
__global__ void hh_reduce_kernel(const double* __restrict__ X, long long ldx, const double* __restrict__ Y,
                                 long long ldy, long long m_local, long long row0, int c, int n, long long rpb,
                                 double* __restrict__ partial) {
  const int w = n - c;
  const long long lo0 = (long long)blockIdx.x * rpb;
  const long long first = max(lo0, (long long)c + 1 - row0);  // local index of the first row with global > c
  const long long hi = min(m_local, lo0 + rpb);
  for (int t = threadIdx.x; t < w; t += blockDim.x) {
    double s = 0.0;
    for (long long i = first; i < hi; ++i) s = fma(X[i * ldx + c], Y[i * ldy + c + t], s);
    partial[(long long)blockIdx.x * w + t] = s;
  }
}

// red[t] = sum_b partial[b * w + t] (block order), red[w + t] = Y(row c, c + t) when this rank holds row c
__global__ void hh_sum_kernel(const double* __restrict__ partial, int blocks, const double* __restrict__ Y,
                              long long ldy, long long m_local, long long row0, int c, int n, double* __restrict__ red) {
  const int w = n - c;
  const long long lc = (long long)c - row0;
  const bool own = lc >= 0 && lc < m_local;
  for (int t = threadIdx.x; t < w; t += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += partial[(long long)b * w + t];
    red[t] = s;
    red[w + t] = own ? Y[lc * ldy + c + t] : 0.0;
  }
}

// Factorization step: the reflector from red (tail squared norm at t = 0, x_c at red[w]), then
// coef[t] = tau * w_t (w_t = v^T W(.., c + t), t >= 1), coef[0] = x_c - beta (0 when tau = 0: the tail
// is zeroed), R(c, c..) and tau_c.
__global__ void hh_reflector_kernel(double* __restrict__ red, int c, int n, double* __restrict__ coef,
                                    double* __restrict__ R, double* __restrict__ tau_out) {
  const int w = n - c;
  const double tail = red[0], c0 = red[w];
  const double tol = 2.2250738585072014e-308 * 2.2250738585072014e-308;
  double tau, beta, denom;
  if (!(tail > tol)) {
    tau = 0.0;
    beta = c0;
    denom = 0.0;
  } else {
    beta = sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    denom = c0 - beta;
    tau = (beta - c0) / beta;
  }
  for (int t = threadIdx.x; t < w; t += blockDim.x) {
    if (t == 0) {
      coef[0] = denom;
      R[(long long)c * n + c] = beta;
    } else {
      // w_t = W(c, c+t) + sum_{i>c} v_i W(i, c+t) with v_i = x_i / (x_c - beta)
      const double wt = tau == 0.0 ? 0.0 : red[w + t] + red[t] / denom;
      const double ts = tau * wt;
      coef[t] = ts;
      R[(long long)c * n + c + t] = red[w + t] - ts;
    }
  }
  if (threadIdx.x == 0) tau_out[c] = tau;
}

// v below the diagonal: W(i, c) = x_i / (x_c - beta) (0 when tau = 0) for rows with global index > c
__global__ void hh_scale_kernel(double* __restrict__ W, long long ldw, long long m_local, long long row0, int c,
                                const double* __restrict__ coef) {
  const double denom = coef[0];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m_local;
       i += (long long)gridDim.x * blockDim.x)
    if (i + row0 > c) W[i * ldw + c] = denom == 0.0 ? 0.0 : W[i * ldw + c] / denom;
}

// W(i, c+t) -= coef[t] * v_i (t >= 1) for rows with global index > c; row c (its owner) takes R(c, c..)
__global__ void hh_update_kernel(double* __restrict__ W, long long ldw, long long m_local, long long row0, int c,
                                 int n, const double* __restrict__ coef, const double* __restrict__ R) {
  const int w = n - c;
  const long long lc = (long long)c - row0;
  const long long total = m_local * (long long)w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / w;
    const int t = (int)(e - i * w);
    if (i + row0 < c) continue;
    double* row = W + i * ldw + c;
    if (i == lc)
      row[t] = R[(long long)c * n + c + t];
    else if (t > 0)
      row[t] = fma(-coef[t], row[0], row[t]);
  }
}

// Q formation step for column c (backward): coef[t] = tau_c * z_t, z_t = Q(c, c+t) + sum_{i>c} v_i Q(i, c+t)
__global__ void hh_qcoef_kernel(const double* __restrict__ red, int c, int n, const double* __restrict__ tau,
                                double* __restrict__ coef) {
  const int w = n - c;
  const double tc = tau[c];
  for (int t = threadIdx.x; t < w; t += blockDim.x) coef[t] = tc * (red[w + t] + red[t]);
}

// Q(i, c+t) -= v_i coef[t] (v_c = 1, v_i = W(i, c) below)
__global__ void hh_qupdate_kernel(const double* __restrict__ W, long long ldw, double* __restrict__ Q, long long ldq,
                                  long long m_local, long long row0, int c, int n, const double* __restrict__ coef) {
  const int w = n - c;
  const long long total = m_local * (long long)w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / w;
    const int t = (int)(e - i * w);
    const long long gi = i + row0;
    if (gi < c) continue;
    const double v = gi == c ? 1.0 : W[i * ldw + c];
    Q[i * ldq + c + t] = fma(-coef[t], v, Q[i * ldq + c + t]);
  }
}

// Q = [I; 0] on this rank's rows
__global__ void hh_qinit_kernel(double* __restrict__ Q, long long ldq, long long m_local, long long row0, int n) {
  const long long total = m_local * (long long)n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n;
    const int j = (int)(e - i * n);
    Q[i * ldq + j] = (i + row0 == j) ? 1.0 : 0.0;
  }
}

// Q(:, j) *= sgn[j] (the sign normalisation of householder_qr_thin, kernels.hpp:203-208)
__global__ void col_sign_kernel(double* __restrict__ Q, long long ldq, long long m, int n,
                                const double* __restrict__ sgn) {
  const long long total = m * (long long)n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n;
    const int j = (int)(e - i * n);
    if (sgn[j] < 0.0) Q[i * ldq + j] = -Q[i * ldq + j];
  }
}

}  // namespace

int hh_blocks(long long m_local, int num_sms) {
  long long b = (m_local + 2047) / 2048;
  if (b > 4LL * num_sms) b = 4LL * num_sms;
  return b < 1 ? 1 : (int)b;
}

cudaError_t launch_hh_reduce(const double* X, long long ldx, const double* Y, long long ldy, long long m_local,
                             long long row0, int c, int n, int blocks, double* partial, double* red,
                             cudaStream_t s) {
  const long long rpb = (m_local + blocks - 1) / blocks;
  hh_reduce_kernel<<<blocks, kHhThreads, 0, s>>>(X, ldx, Y, ldy, m_local, row0, c, n, rpb > 0 ? rpb : 1, partial);
  hh_sum_kernel<<<1, 512, 0, s>>>(partial, blocks, Y, ldy, m_local, row0, c, n, red);
  return cudaGetLastError();
}

cudaError_t launch_hh_reflect_update(double* W, long long ldw, long long m_local, long long row0, int c, int n,
                                     double* red, double* coef, double* R, double* tau, int num_sms, cudaStream_t s) {
  hh_reflector_kernel<<<1, 512, 0, s>>>(red, c, n, coef, R, tau);
  hh_scale_kernel<<<num_sms, kHhThreads, 0, s>>>(W, ldw, m_local, row0, c, coef);
  hh_update_kernel<<<4 * num_sms, kHhThreads, 0, s>>>(W, ldw, m_local, row0, c, n, coef, R);
  return cudaGetLastError();
}

cudaError_t launch_hh_qinit(double* Q, long long ldq, long long m_local, long long row0, int n, int num_sms,
                            cudaStream_t s) {
  hh_qinit_kernel<<<4 * num_sms, kHhThreads, 0, s>>>(Q, ldq, m_local, row0, n);
  return cudaGetLastError();
}

cudaError_t launch_hh_qstep(const double* W, long long ldw, double* Q, long long ldq, long long m_local,
                            long long row0, int c, int n, const double* red, const double* tau, double* coef,
                            int num_sms, cudaStream_t s) {
  hh_qcoef_kernel<<<1, 512, 0, s>>>(red, c, n, tau, coef);
  hh_qupdate_kernel<<<4 * num_sms, kHhThreads, 0, s>>>(W, ldw, Q, ldq, m_local, row0, c, n, coef);
  return cudaGetLastError();
}

cudaError_t launch_col_sign(double* Q, long long ldq, long long m, int n, const double* sgn, int num_sms,
                            cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  col_sign_kernel<<<4 * num_sms, kHhThreads, 0, s>>>(Q, ldq, m, n, sgn);
  return cudaGetLastError();
}

}  // namespace cqr
