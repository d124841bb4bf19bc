/* Exhaustive-random check that the trisolve division (inv = RN(1/d), then
 * Markstein corrections with fma) equals IEEE y/d bit for bit, for the operand
 * ranges the kernels take the fast path on (|d| in [2^-500, 2^500], |y| in
 * [2^-899, 2^900]). Tests the two-correction form used by the kernels and the
 * one-correction form (q0 = RN(y*inv); q = RN(q0 + RN(y - q0*d)*inv)).
 * Build: gcc -O2 -march=x86-64-v3 -ffp-contract=off -fopenmp -o markstein_check markstein_check.c -lm
 * Run:   ./markstein_check [cases_per_thread_millions]
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline double bits2d(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}
static inline uint64_t d2bits(double d) {
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
}
/* random double with exponent in [lo, hi] and a mantissa biased to hard cases */
static double pick(uint64_t r, int lo, int hi) {
  const int e = lo + (int)((r >> 52) % (uint64_t)(hi - lo + 1));
  uint64_t m = r & 0xFFFFFFFFFFFFFull;
  switch ((r >> 8) & 7) {
    case 0: m |= 0xFFFFFFFFF0000ull; break;        /* mantissa near 2 */
    case 1: m &= 0x000000000FFFFull; break;        /* mantissa near 1 */
    case 2: m = 0; break;                          /* power of two */
    case 3: m = 0xFFFFFFFFFFFFFull; break;         /* largest mantissa */
    default: break;
  }
  return bits2d(((uint64_t)(e + 1023) << 52) | m) * (((r >> 4) & 1) ? -1.0 : 1.0);
}

int main(int argc, char** argv) {
  const long per = (argc > 1 ? atol(argv[1]) : 25) * 1000000L;
  long bad2 = 0, bad1 = 0, total = 0;
#pragma omp parallel reduction(+ : bad2, bad1, total)
  {
    const uint64_t tid = (uint64_t)omp_get_thread_num();
    for (long i = 0; i < per; ++i) {
      const uint64_t r1 = mix(tid * 0x9E3779B97F4A7C15ull + 2 * (uint64_t)i + 1);
      const uint64_t r2 = mix(r1 ^ 0xD1B54A32D192ED03ull);
      const double d = pick(r1, -500, 500);
      double y;
      if (((r2 >> 60) & 3) == 0) {
        /* y close to a multiple of d: quotient near an integer or a midpoint */
        const double k = (double)(int64_t)(r2 & 0xFFFFF) + (((r2 >> 20) & 1) ? 0.5 : 0.0);
        y = k * d;
        y = bits2d(d2bits(y) + (int64_t)((r2 >> 24) & 7) - 3);
      } else {
        y = pick(r2, -YR, YR);
      }
      if (!(fabs(y) >= 0x1p-899 && fabs(y) <= 0x1p+900)) continue;
      if (!(fabs(y / d) >= 0x1p-1000 && fabs(y / d) <= 0x1p+1000)) continue; /* quotient in the normal range */
      const double inv = 1.0 / d;
      const double ref = y / d;
      const double q0 = y * inv;
      double rr = fma(-q0, d, y);
      const double q1 = fma(rr, inv, q0);
      rr = fma(-q1, d, y);
      const double q2 = fma(rr, inv, q1);
      bad2 += d2bits(q2) != d2bits(ref);
      bad1 += d2bits(q1) != d2bits(ref);
      ++total;
    }
  }
  printf("cases %ld: two corrections %ld mismatches, one correction %ld mismatches\n", total, bad2, bad1);
  return bad2 != 0;
}
