// boxmuller.cuh — branch-free FP64 Box-Muller for the in-kernel sketch
// (rng.hpp:47-55: r = sqrt(-2 ln u1), a = RN(2*pi)*u2, cos a / sin a).
//
// CUDA's log/sqrt/sincos carry special-case branches, which split basic
// blocks and keep the scheduler from interleaving the draws with the DMMA
// stream. These versions are straight-line for the arguments that occur
// (u1 in (0,1], a in [0, 2*pi)) and stay within 3 ulp of max(|g|, 1) of the
// oracle (tools/gpu/bm_acc.py, 1e7 draws; tests/test_gpu_parity.py also drives
// the edge bits: u1 -> 1, u1 -> 0, quadrant and table boundaries of u2):
//  * log: u1 = 2^e f, f renormalised to [sqrt(2)/2, sqrt(2)), table points
//    c_i = 1 + i/256 (i = -75..106, rounded from the mantissa bits) with
//    inv_i = RN(1/c_i) and -log(inv_i) (hi+lo, long double), r = f*inv_i - 1
//    (one fma, |r| < 2^-8.5), log1p(r) by a degree-6 polynomial. c_0 = 1
//    exactly, so for u1 -> 1 the result is log1p(f - 1) with f - 1 exact: full
//    relative accuracy of ln u1 (and of r = sqrt(-2 ln u1)) down to u1 = 1 - 2^-53;
//  * sqrt: rsqrt.approx + one Newton step + one residual correction;
//  * sincos: sin/cos(2*pi*k/256) from a one-quadrant table (65 entries, quadrant
//    rotation by sign/swap on the integer pipe), k = round(256 u2) from the integer
//    counter bits, 3-part Cody-Waite reduction, degree-5/6 polynomials on |d| <= pi/256.
// The FP64 pipe is shared with the sketch's DMMA stream, which holds it whenever it
// has work (tools/probe/pipe_prio.cu): the draws' FP64 instructions mostly run in
// its gaps, so exact power-of-two scalings and the table indices go through the
// integer pipe, and P pairs are drawn side by side for instruction-level parallelism.
// Tables live in shared memory (BmTables, 4.9 KB), filled from __constant__.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace cqr {

constexpr int kBmLogLo = -75, kBmLogHi = 106;  // log table points c_i = 1 + i/256
constexpr int kBmLog = kBmLogHi - kBmLogLo + 1;
constexpr int kBmTrig = 256;  // table points 2 pi k / 256 over [0, 2 pi)
struct BmTables {
  double inv[kBmLog];
  double lhi[kBmLog];
  double llo[kBmLog];
  double q[kBmTrig / 4 + 1];  // sin(2 pi m / 256), m = 0..64 (one quadrant; the others by symmetry)
};

// sin and cos of 2 pi k / 256: k = 64 q + m, rotate the first-quadrant pair by q quarter turns
__device__ __forceinline__ void bm_table_sincos(const BmTables& T, int k, double& S, double& C) {
  const int q = k >> 6, m = k & 63;
  const bool swap = q & 1;  // odd quarter turns exchange sin and cos: swap the table index
  const long long sb = __double_as_longlong(T.q[swap ? 64 - m : m]), cb = __double_as_longlong(T.q[swap ? m : 64 - m]);
  const long long sneg = (long long)(q >> 1) << 63, cneg = (long long)((q ^ (q >> 1)) & 1) << 63;
  S = __longlong_as_double(sb ^ sneg);
  C = __longlong_as_double(cb ^ cneg);
}

// The same tables with the sines over the whole circle plus a quarter (320 entries, filled from the quadrant
// table by its own symmetry rule, so every draw is bit-identical): sin = s[k], cos = s[k + 64], no quadrant
// arithmetic (~10 integer instructions fewer per pair; the int8 sketch is issue-bound on its generator warps).
struct BmTablesX {
  double inv[kBmLog];
  double lhi[kBmLog];
  double llo[kBmLog];
  double s[kBmTrig + kBmTrig / 4];
};
__device__ __forceinline__ void bm_table_sincos(const BmTablesX& T, int k, double& S, double& C) {
  S = T.s[k];
  C = T.s[k + kBmTrig / 4];
}
// host: the full-circle copy of t (the quadrant rule of bm_table_sincos, bit for bit)
inline void bm_tables_expand(const BmTables& t, BmTablesX* x) {
  for (int i = 0; i < kBmLog; ++i) x->inv[i] = t.inv[i], x->lhi[i] = t.lhi[i], x->llo[i] = t.llo[i];
  for (int kk = 0; kk < kBmTrig + kBmTrig / 4; ++kk) {
    const int k = kk & (kBmTrig - 1), q = k >> 6, m = k & 63;
    const double v = t.q[(q & 1) ? 64 - m : m];
    x->s[kk] = (q >> 1) ? -v : v;  // the sign-bit flip of the device rule (-0.0 for a zero entry)
  }
}

// Polynomial and reduction constants in the constant bank: DFMA takes a c[][] operand
// directly, where an immediate double costs two register moves per use.
__constant__ double kBmK[] = {
    -1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -0.5,                           // 0-4: log1p
    0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45,                                   // 5-6: ln 2 hi, lo
    0x1.921fb54400000p-6, 0x1.0b4611a600000p-40, 0x1.3198a2e037073p-75,          // 7-9: 2 pi / 256, 3 parts
    1.5, 1.0 / 120.0, -1.0 / 720.0, 1.0 / 24.0, 1.0, 0x1.921fb54442d18p-51, -1.0  // 10-16
};

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

#define CQR_BM_EACH _Pragma("unroll") for (int j = 0; j < P; ++j)

// Box-Muller on raw counter bits: b1 -> u1 = ((b1 >> 11) + 1) 2^-53, b2 -> u2 =
// (b2 >> 11) 2^-53; g_even = r cos(a), g_odd = r sin(a). The pairs are independent;
// every step is issued for all P of them before the next one (P-way ILP).
// SCALED: the outputs times `scale`, a power of two (or zero) folded into the radius -- exact, so
// g * scale is bit for bit the scaled draw (one multiply per pair instead of one per draw).
// The core works on the 53-bit words m1 = b1 >> 11, m2 = b2 >> 11 (the only bits of the draws it uses).
template <int P, class TT, bool SCALED = false>
__device__ __forceinline__ void box_muller_top53(const TT& T, const uint64_t (&m1)[P], const uint64_t (&m2)[P],
                                                 double (&g_even)[P], double (&g_odd)[P], double scale = 1.0) {
  double n1[P], a[P], fk[P];
  int k[P];
  CQR_BM_EACH {
    // u1 = N1 * 2^-53 with N1 = (b1 >> 11) + 1 in [1, 2^53]: the scaling is folded into the
    // exponent below (N1's double has u1's mantissa bits, its exponent is 53 higher)
    n1[j] = (double)(m1[j] + 1);
    // a = RN(2 pi) * u2 with u2 = N2 * 2^-53: the power-of-two scaling commutes with the
    // rounding (a is 0 or >= 2^-51), so one multiply by RN(2 pi) * 2^-53 gives the same a
    const uint64_t n2 = m2[j];
    a[j] = (double)n2 * kBmK[15];
    // table point k = round(256 u2) in [0, 256] (k = 256 reduces with 2 pi and reads entry 0)
    const int kk = (int)((n2 + (1ull << 44)) >> 45);
    k[j] = kk & (kBmTrig - 1);
    fk[j] = (double)kk;
  }
  // ---- log(u1) = e ln 2 - log(inv_i) + log1p(f inv_i - 1)
  int e[P], ti[P];
  double r[P], r2[P], pl[P];
  CQR_BM_EACH {
    const int hi = __double2hiint(n1[j]), lo = __double2loint(n1[j]);
    const int mh = hi & 0xFFFFF;  // top 20 of the 52 mantissa bits m of f0 = 1 + m 2^-52
    const bool up = mh >= (213 << 11);  // f0 >= 1 + 106.5/256: use f = f0/2, e + 1
    // i = round((f - 1) * 256): round(m / 2^44) below, round(m / 2^45) - 128 above
    const int i = up ? ((mh + (1 << 12)) >> 13) - 128 : (mh + (1 << 11)) >> 12;
    ti[j] = i - kBmLogLo;
    e[j] = (hi >> 20) - 1023 - 53 + (up ? 1 : 0);
    const double f = __hiloint2double(mh | (up ? 0x3FE00000 : 0x3FF00000), lo);  // [0.708, 1.416)
    r[j] = fma(f, T.inv[ti[j]], kBmK[16]);
  }
  CQR_BM_EACH r2[j] = r[j] * r[j];
  CQR_BM_EACH pl[j] = fma(r[j], kBmK[0], kBmK[1]);
  CQR_BM_EACH pl[j] = fma(pl[j], r[j], kBmK[2]);
  CQR_BM_EACH pl[j] = fma(pl[j], r[j], kBmK[3]);
  CQR_BM_EACH pl[j] = fma(pl[j], r[j], kBmK[4]);
  double L[P];
  CQR_BM_EACH {
    const double l1p = fma(r2[j], pl[j], r[j]);
    const double ed = (double)e[j];
    L[j] = fma(ed, kBmK[5], T.lhi[ti[j]]) + (fma(ed, kBmK[6], T.llo[ti[j]]) + l1p);
  }
  // ---- sincos(a): d = a - k * 2 pi / 256 (three parts; k * part 1 and k * part 2 are exact)
  double d[P];
  CQR_BM_EACH {
    d[j] = fma(-fk[j], kBmK[7], a[j]);
    d[j] = fma(-fk[j], kBmK[8], d[j]);
    d[j] = fma(-fk[j], kBmK[9], d[j]);
  }
  // ---- sqrt(-2 L): L is +0 (never -0: its high part is +0 whenever the sum can vanish) or a
  // normal number (|L| >= 2^-54), so x = -2 L is a sign flip plus one on the exponent, and -x/2
  // is L itself; L = +0 maps to x = -2^-1022, which the x > 0 test below sends to r = 0
  double x[P], y[P];
  CQR_BM_EACH {
    x[j] = __longlong_as_double((__double_as_longlong(L[j]) ^ (1ll << 63)) + (1ll << 52));
    y[j] = rsqrt_approx(x[j]);
  }
  double d2[P], sp[P], cp[P];
  CQR_BM_EACH d2[j] = d[j] * d[j];
  CQR_BM_EACH y[j] = y[j] * fma(L[j], y[j] * y[j], kBmK[10]);  // one Newton step (a second one changed no draw in 1e7)
  // sin d = d + d^3 (-1/6 + d^2/120) (next term <= 8.6e-18); cos d to d^6 (next term <= 1.3e-20)
  CQR_BM_EACH sp[j] = fma(d2[j], kBmK[11], kBmK[0]);
  CQR_BM_EACH cp[j] = fma(d2[j], kBmK[12], kBmK[13]);
  CQR_BM_EACH cp[j] = fma(cp[j], d2[j], kBmK[4]);
  CQR_BM_EACH {
    double s = x[j] * y[j];
    const double hy = __longlong_as_double(__double_as_longlong(y[j]) - (1ll << 52));  // y / 2, y normal
    s = fma(hy, fma(-s, s, x[j]), s);
    const double rad = __double_as_longlong(x[j]) > 0 ? (SCALED ? s * scale : s) : 0.0;
    const double sn = fma(d[j] * d2[j], sp[j], d[j]);
    const double cs = fma(cp[j], d2[j], kBmK[14]);
    double S, C;
    bm_table_sincos(T, k[j], S, C);
    g_even[j] = rad * fma(C, cs, -(S * sn));
    g_odd[j] = rad * fma(S, cs, C * sn);
  }
}

template <int P, class TT, bool SCALED = false>
__device__ __forceinline__ void box_muller_bits(const TT& T, const uint64_t (&b1)[P], const uint64_t (&b2)[P],
                                                double (&g_even)[P], double (&g_odd)[P], double scale = 1.0) {
  uint64_t m1[P], m2[P];
  CQR_BM_EACH m1[j] = b1[j] >> 11, m2[j] = b2[j] >> 11;
  box_muller_top53<P, TT, SCALED>(T, m1, m2, g_even, g_odd, scale);
}
// mix64(z) >> 11 without forming mix64's last xor-shift: (z ^ (z >> 31)) >> 11 = (z >> 11) ^ (z >> 42), and
// z >> 42 has no high word (two instructions fewer per hash)
__device__ __forceinline__ uint64_t mix64_top53(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (z >> 11) ^ (z >> 42);
}

// Both outputs of Box-Muller pairs p[0..P) (counters 2p -> cos, 2p+1 -> sin; rng.hpp:47-55).
template <int P>
__device__ __forceinline__ void gaussian_pairs_fast(const BmTables& T, uint64_t seed, const uint64_t (&p)[P],
                                                    double (&g_even)[P], double (&g_odd)[P]) {
  uint64_t b1[P], b2[P];
  CQR_BM_EACH {
    b1[j] = mix64(seed + (2 * p[j] + 1) * 0x9E3779B97F4A7C15ull);
    b2[j] = mix64(seed + (2 * p[j] + 2) * 0x9E3779B97F4A7C15ull);
  }
  box_muller_bits<P, BmTables>(T, b1, b2, g_even, g_odd);
}
// Same, from each pair's first counter word z = seed + (2p + 1) G (the second is z + G).
template <int P, class TT>
__device__ __forceinline__ void gaussian_pairs_z(const TT& T, const uint64_t (&z)[P], double (&g_even)[P],
                                                 double (&g_odd)[P]) {
  uint64_t b1[P], b2[P];
  CQR_BM_EACH {
    b1[j] = mix64(z[j]);
    b2[j] = mix64(z[j] + 0x9E3779B97F4A7C15ull);
  }
  box_muller_bits<P, TT>(T, b1, b2, g_even, g_odd);
}
// the same draws times `scale` (a power of two or zero)
template <int P, class TT>
__device__ __forceinline__ void gaussian_pairs_z_scaled(const TT& T, const uint64_t (&z)[P], double scale,
                                                        double (&g_even)[P], double (&g_odd)[P]) {
  uint64_t m1[P], m2[P];
  CQR_BM_EACH {
    m1[j] = mix64_top53(z[j]);
    m2[j] = mix64_top53(z[j] + 0x9E3779B97F4A7C15ull);
  }
  box_muller_top53<P, TT, true>(T, m1, m2, g_even, g_odd, scale);
}
#undef CQR_BM_EACH

__device__ __forceinline__ void gaussian_pair_fast(const BmTables& T, uint64_t seed, uint64_t p, double& g_even,
                                                   double& g_odd) {
  const uint64_t pp[1] = {p};
  double ge[1], go[1];
  gaussian_pairs_fast<1>(T, seed, pp, ge, go);
  g_even = ge[0];
  g_odd = go[0];
}

// Host: fill the tables (long double arithmetic) and upload to the device copy.
void bm_tables_host(BmTables* t);

}  // namespace cqr
