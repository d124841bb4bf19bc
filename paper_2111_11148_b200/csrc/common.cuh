// common.cuh — shared device helpers for the B200 (sm_100a) CholeskyQR path.
//
// FP64 on B200: tcgen05 has no f64 kind, so every tall contraction here runs
// on the FP64 tensor path, mma.sync m8n8k4 (SASS DMMA.8x8x4). Measured on the
// pool's B200s (profiles/r01_fp64_probe.txt): DMMA 37.1 TFLOP/s, DFMA 33.9,
// one shared pipe; and DMMA accumulates exactly like the sequential FMA chain
// c = fma(a0,b0,c); c = fma(a1,b1,c); ... in k order (262144/262144 bitwise
// matches). That last fact is what lets the DMMA kernels reproduce the fixed
// fma-chain orders of the oracle bit for bit.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cqr {

// ---- device status word ------------------------------------------------------
// code (cqr_status) + index; the first failure wins; every pipeline kernel
// exits early once it is set, so a failed attempt costs no host round trip
// until the engine reads the word at the end of the attempt.
struct DevStatus {
  int code;
  int pad;
  long long index;
};

__device__ __forceinline__ void set_status(DevStatus* st, int code, long long index) {
  if (atomicCAS(&st->code, 0, code) == 0) st->index = index;
}
// Non-finite input (engine.cpp:222) outranks any numerical failure: the check
// is fused into the first kernel that reads all of A.
__device__ __forceinline__ void set_status_invalid(DevStatus* st) {
  atomicExch(&st->code, 3 /*CQR_INVALID_ARGUMENT*/);
  st->index = -1;
}
__device__ __forceinline__ bool nonfinite(double v) {
  return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}
__device__ __forceinline__ bool failed(const DevStatus* st) {
  return st != nullptr && *(volatile const int*)&st->code != 0;
}

// ---- DMMA m8n8k4 (fp64) ----------------------------------------------------------
// A 8x4 row-major: lane holds A[lane>>2][lane&3]; B 4x8: lane holds
// B[lane&3][lane>>2]; C 8x8: lane holds C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- counter RNG (rng.hpp:18-55), bit-exact on the integer part ------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // counter stride (rng.hpp:29)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t bits_at(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
}
// Both Box-Muller outputs of pair p: counter 2p -> cos, 2p+1 -> sin (rng.hpp:47-55).
__device__ __forceinline__ void gaussian_pair(uint64_t seed, uint64_t p, double& g_even, double& g_odd) {
  const double u1 = (double)((bits_at(seed, 2 * p) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(bits_at(seed, 2 * p + 1) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586 * u2;  // RN(2*pi) * u2, as 2.0 * std::numbers::pi * u2
  double s, c;
  sincos(a, &s, &c);
  g_even = r * c;
  g_odd = r * s;
}

// ---- async copies ----------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Stage `rows` x `n` doubles (row stride ld in global, lds in smem) into smem,
// zero-filling columns [n, np) and rows [rows, rrows). Issued by `nthr` threads
// starting at thread `tid`. 16-byte copies when the layout allows.
__device__ __forceinline__ void stage_rows(double* s, int lds, const double* g, long long ld, int rows,
                                           int rrows, int n, int np, int tid, int nthr, bool vec16) {
  if (vec16) {
    const int hp = np / 2;  // pairs per row (np even)
    const int hn = n / 2;   // n even when vec16
    for (int e = tid; e < rrows * hp; e += nthr) {
      const int r = e / hp, c2 = e - r * hp;
      double* d = s + r * lds + 2 * c2;
      if (r < rows && c2 < hn) {
        cp_async16(d, g + (long long)r * ld + 2 * c2);
      } else {
        d[0] = 0.0;
        d[1] = 0.0;
      }
    }
  } else {
    for (int e = tid; e < rrows * np; e += nthr) {
      const int r = e / np, c = e - r * np;
      double* d = s + r * lds + c;
      if (r < rows && c < n)
        cp_async8(d, g + (long long)r * ld + c);
      else
        *d = 0.0;
    }
  }
}

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// The dynamic shared memory cap of a kernel, set once per (device, kernel) to the device's opt-in maximum
// minus the kernel's static shared memory. The attribute is process-wide per function: setting it to each
// launch's own size would let a concurrent host thread lower it under another thread's larger launch
// (cudaErrorInvalidValue). The launch still passes its actual size, which is what occupancy depends on.
cudaError_t allow_max_smem_impl(const void* kernel);
template <typename K>
inline cudaError_t allow_max_smem(K kernel) {
  return allow_max_smem_impl(reinterpret_cast<const void*>(kernel));
}

}  // namespace cqr
