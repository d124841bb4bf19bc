// boxmuller.cuh — branch-free FP64 Box-Muller for the in-kernel sketch
// (rng.hpp:47-55: r = sqrt(-2 ln u1), a = RN(2*pi)*u2, cos a / sin a).
//
// CUDA's log/sqrt/sincos carry special-case branches, which split basic
// blocks and keep the scheduler from interleaving the draws with the DMMA
// stream. These versions are straight-line for the arguments that occur
// (u1 in (0,1], a in [0, 2*pi)) and accurate to a few ulp in absolute terms
// (1e7 draws against glibc: max 12.5 ulp of max(|g|, 1) -- the absolute error of
// cos/sin near their zeros times r <= 8.6 -- and 70.7% bit-identical):
//  * log: u1 = 2^e f, f renormalised to [sqrt(2)/2, sqrt(2)), 128-entry table
//    of inv_i = RN(1/c_i) and -log(inv_i) (hi+lo, built in long double), r =
//    f*inv_i - 1 (one fma), log1p(r) by a degree-7 polynomial (|r| < 2^-7.9);
//  * sqrt: rsqrt.approx + one Newton step + one residual correction;
//  * sincos: 64-entry table of sin/cos(2*pi*i/64), 3-part Cody-Waite
//    reduction, degree-9/8 polynomials on |d| <= pi/64.
// Tables live in shared memory (BmTables, ~4 KB), filled from __constant__.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace cqr {

struct BmTables {
  double inv[128];
  double lhi[128];
  double llo[128];
  double s[66];
  double c[66];
};

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// Both outputs of Box-Muller pair p (counters 2p -> cos, 2p+1 -> sin).
__device__ __forceinline__ void gaussian_pair_fast(const BmTables& T, uint64_t seed, uint64_t p, double& g_even,
                                                   double& g_odd) {
  const uint64_t b1 = mix64(seed + (2 * p + 1) * 0x9E3779B97F4A7C15ull);
  const uint64_t b2 = mix64(seed + (2 * p + 2) * 0x9E3779B97F4A7C15ull);
  // u1 = N1 * 2^-53 with N1 = (b1 >> 11) + 1 in [1, 2^53]: the scaling is folded into the
  // exponent below (N1's double has u1's mantissa bits, its exponent is 53 higher)
  const double n1 = (double)((b1 >> 11) + 1);
  const double u2 = (double)(b2 >> 11) * 0x1.0p-53;
  // ---- log(u1)
  const int hi = __double2hiint(n1), lo = __double2loint(n1);
  int e = (hi >> 20) - 1023 - 53;
  const int mh = hi & 0xFFFFF;
  const int i = mh >> 13;
  double f = __hiloint2double(mh | 0x3FF00000, lo);
  const bool up = i >= 53;
  f = up ? f * 0.5 : f;
  e += up ? 1 : 0;
  const double r = fma(f, T.inv[i], -1.0);
  const double r2 = r * r;
  double pl = 1.0 / 7.0;
  pl = fma(pl, r, -1.0 / 6.0);
  pl = fma(pl, r, 1.0 / 5.0);
  pl = fma(pl, r, -1.0 / 4.0);
  pl = fma(pl, r, 1.0 / 3.0);
  pl = fma(pl, r, -0.5);
  const double l1p = fma(r2, pl, r);
  const double ed = (double)e;
  const double ln2_hi = 0x1.62e42fefa3800p-1, ln2_lo = 0x1.ef35793c76730p-45;
  const double L = fma(ed, ln2_hi, T.lhi[i]) + (fma(ed, ln2_lo, T.llo[i]) + l1p);
  // ---- sqrt(-2 L)
  const double x = -2.0 * L;
  double y = rsqrt_approx(x);
  y = y * fma(-0.5 * x, y * y, 1.5);  // one Newton step: a second one changed no draw in 1e7 (tools/gpu/bm_acc.py)
  double s = x * y;
  s = fma(0.5 * y, fma(-s, s, x), s);
  const double rad = (x > 0.0) ? s : 0.0;
  // ---- sincos(a), a = RN(2 pi) * u2
  const double a = 6.283185307179586 * u2;
  const double t = fma(a, 10.185916357881302, 0x1.8p52);  // a * 64/(2 pi) + rounding constant
  const int k = __double2loint(t) & 127;
  const double fk = t - 0x1.8p52;
  double d = fma(-fk, 0x1.921fb54400000p-4, a);  // 2 pi / 64, three parts
  d = fma(-fk, 0x1.0b4611a600000p-38, d);
  d = fma(-fk, 0x1.3198a2e037073p-73, d);
  const double d2 = d * d;
  double sp = 1.0 / 362880.0;
  sp = fma(sp, d2, -1.0 / 5040.0);
  sp = fma(sp, d2, 1.0 / 120.0);
  sp = fma(sp, d2, -1.0 / 6.0);
  const double sn = fma(sp * d2, d, d);
  double cp = 1.0 / 40320.0;
  cp = fma(cp, d2, -1.0 / 720.0);
  cp = fma(cp, d2, 1.0 / 24.0);
  cp = fma(cp, d2, -0.5);
  const double cs = fma(cp, d2, 1.0);
  const double S = T.s[k], C = T.c[k];
  const double ca = fma(C, cs, -(S * sn));
  const double sa = fma(S, cs, C * sn);
  g_even = rad * ca;
  g_odd = rad * sa;
}

// Host: fill the tables (long double arithmetic) and upload to the device copy.
void bm_tables_host(BmTables* t);

}  // namespace cqr
