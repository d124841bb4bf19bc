// trisolve_common.cuh — packed-R layout and the division shared by the
// trisolve kernels (trisolve.cu, trisolve_tma.cu).
#pragma once

#include "common.cuh"

namespace cqr {
namespace tri {

// Packed R for a padded width np (R padded with the identity):
//   bpack[(J*(J-1) + k4)*32 + lane] = -R[4*k4 + (lane&3)][8J + (lane>>2)]   (k4 < 2J)
//   dpack[J*S + kk*8 + j]          =  R[8J+kk][8J+j]                       (8x8 diag block)
//   dpack[J*S + 64 + j]            =  RN(1 / R[8J+j][8J+j])
//   dpack[J*S + 72 + j]            =  1 if the fast division is safe for column j
//   dpack[J*S + 80]                =  1 if the block's strict upper part has no zero and
//                                      all its divisions are safe (uniform fast path)
//   dpack[J*S + 88 + kColStart[j] + p] = column j for the fast path, 16-byte aligned:
//                                      R[8J+p][8J+j] (p < j), R_jj (p = j), RN(1/R_jj) (p = j+1)
// (S = kDiagStride = 136 doubles per block)
constexpr int kDiagStride = 136;
constexpr int kColBase = 88;
// column j occupies [col_start(j), col_start(j) + 2*ceil((j+2)/2))
__host__ __device__ constexpr int col_start(int j) {
  return (j & 1) ? 2 * (j / 2) * (j / 2) + 4 * (j / 2) + 2 * (j / 2) + 2 : 2 * (j / 2) * (j / 2) + 4 * (j / 2);
}

// Correctly rounded y / d from inv = RN(1/d) and one Markstein correction
// (q0 = RN(y inv), r = y - q0 d exact by fma, q = RN(q0 + r inv)); exact
// whenever inv is correctly rounded and the quotient and residual stay normal,
// which |d| in [2^-500, 2^500] and |y| in [2^-400, 2^400] guarantee
// (tools/probe/markstein_check.c: 2e8 random and near-midpoint cases, 0
// mismatches). Other operands take the IEEE division.
__device__ __forceinline__ double fast_div(double y, double d, double inv, bool safe) {
  const double ay = fabs(y);
  if (!safe || !(ay >= 0x1p-400 && ay <= 0x1p+400)) {
    return (y == 0.0 && safe) ? y * inv : y / d;
  }
  const double q0 = y * inv;
  const double r = fma(-q0, d, y);
  return fma(r, inv, q0);
}

// Super-block kernels: every element receives k = 0, 1, ..., j-1 in ascending
// order, the in-block terms last, then the division: the reference recurrence.
__device__ __forceinline__ bool div_exponent_ok(double y) {
  const unsigned e = ((unsigned)__double2hiint(y) >> 20) & 0x7ffu;  // |y| in [2^-400, 2^401)
  return e - 623u < 801u;
}

// Straight-line correctly rounded division for the fast path (inv = RN(1/d),
// d in [2^-500, 2^500]); `ok` is false when y needs the IEEE fallback.
__device__ __forceinline__ double div_fast(double y, double d, double inv, bool& ok) {
  const double q0 = y * inv;
  const double r = fma(-q0, d, y);
  const double q = fma(r, inv, q0);
  ok = div_exponent_ok(y);
  return q;
}

}  // namespace tri
}  // namespace cqr
