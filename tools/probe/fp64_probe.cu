// FP64 pipe probe for B200 (sm_100a): DFMA vs DMMA throughput, whether the two
// pipes overlap, DMMA accumulation order, and the cost of the Box-Muller RNG.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double x, double y) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double x, double y) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = i; }
  double a = x + threadIdx.x * 1e-9, b = y;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// Every warp interleaves DMMA and DFMA.
template <int CH>
__global__ void k_mix(double* out, int iters, double x, double y) {
  double acc[CH][2];
  double f[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = i; f[i] = i; }
  double a = x + threadIdx.x * 1e-9, b = y;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      dmma(acc[i], a, b);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
      f[i] = fma(f[i], x, y);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1] + f[i];
  if (s == 12345.678) out[0] = s;
}

// One warp: C(8x8) += A(8x4) * B(4x8) for many random trials.
__global__ void k_dmma_order(const double* A, const double* B, const double* C, double* D, int trials) {
  int lane = threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const double* a = A + t * 32;
    const double* b = B + t * 32;
    const double* c = C + t * 64;
    double av = a[(lane >> 2) * 4 + (lane & 3)];          // A[row=lane/4][k=lane%4]
    double bv = b[(lane & 3) * 8 + (lane >> 2)];          // B[k=lane%4][col=lane/4]
    double acc[2];
    acc[0] = c[(lane >> 2) * 8 + 2 * (lane & 3)];
    acc[1] = c[(lane >> 2) * 8 + 2 * (lane & 3) + 1];
    dmma(acc, av, bv);
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = acc[0];
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc[1];
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_rng(double* out, uint64_t seed, uint64_t npairs_per_thread) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  double s = 0;
  for (uint64_t i = 0; i < npairs_per_thread; ++i) {
    uint64_t p = tid * npairs_per_thread + i;
    uint64_t b1 = mix64(seed + (2 * p + 1) * 0x9E3779B97F4A7C15ull);
    uint64_t b2 = mix64(seed + (2 * p + 2) * 0x9E3779B97F4A7C15ull);
    double u1 = (double)((b1 >> 11) + 1) * 0x1.0p-53;
    double u2 = (double)(b2 >> 11) * 0x1.0p-53;
    double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(2.0 * 3.141592653589793 * u2, &sn, &cs);
    s += r * cs + r * sn;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_rng_int(double* out, uint64_t seed, uint64_t npairs_per_thread) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t s = 0;
  for (uint64_t i = 0; i < npairs_per_thread; ++i) {
    uint64_t p = tid * npairs_per_thread + i;
    uint64_t b1 = mix64(seed + (2 * p + 1) * 0x9E3779B97F4A7C15ull);
    uint64_t b2 = mix64(seed + (2 * p + 2) * 0x9E3779B97F4A7C15ull);
    s ^= b1 + b2;
  }
  if (s == 12345) out[0] = (double)s;
}

__global__ void k_div(double* out, int iters, double d) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x + i + 1.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = acc[i] / d;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n4; i += stride) b[i] = a[i];
}

__global__ void k_read(const double4* __restrict__ a, double* out, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n4; i += stride) { double4 v = a[i]; s += v.x + v.y + v.z + v.w; }
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

static double host_seq(const double* a, const double* b, double c, int order[4]) {
  double acc = c;
  for (int q = 0; q < 4; ++q) acc = std::fma(a[order[q]], b[order[q]], acc);
  return acc;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms=%d clock(kHz)=%d\n", prop.name, sms, prop.clockRate);
  double* d_out; CK(cudaMalloc(&d_out, 64));

  const int iters = 4096;
  for (int bpsm : {4, 8}) {
    int grid = sms * bpsm, block = 256;
    float ms = time_ms([&] { k_dfma<8><<<grid, block>>>(d_out, iters, 1.0000001, 1e-9); });
    double flops = 2.0 * grid * block * 8.0 * iters;
    printf("DFMA  bpsm=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, flops / ms / 1e9);
    ms = time_ms([&] { k_dmma<8><<<grid, block>>>(d_out, iters, 1.0000001, 1e-9); });
    flops = 2.0 * (grid * block / 32) * 8.0 * iters * 256.0;
    printf("DMMA  bpsm=%d: %.3f ms  %.2f TFLOP/s\n", bpsm, ms, flops / ms / 1e9);
    ms = time_ms([&] { k_mix<4><<<grid, block>>>(d_out, iters, 1.0000001, 1e-9); });
    double f_dmma = 2.0 * (grid * block / 32) * 4.0 * iters * 256.0;
    double f_dfma = 2.0 * grid * block * 4.0 * 8.0 * iters;
    printf("MIX   bpsm=%d: %.3f ms  dmma %.2f + dfma %.2f = %.2f TFLOP/s (dmma-alone time %.3f, dfma-alone %.3f)\n",
           bpsm, ms, f_dmma / ms / 1e9, f_dfma / ms / 1e9, (f_dmma + f_dfma) / ms / 1e9,
           0.0, 0.0);
  }
  {
    int grid = sms * 8, block = 256;
    float ms = time_ms([&] { k_div<<<grid, block>>>(d_out, 512, 1.2345); });
    double ops = (double)grid * block * 8 * 512;
    printf("DDIV: %.3f ms  %.2f Gdiv/s\n", ms, ops / ms / 1e6);
  }
  {
    int grid = sms * 8, block = 256;
    uint64_t per = 256;
    float ms = time_ms([&] { k_rng<<<grid, block>>>(d_out, 12345, per); });
    double pairs = (double)grid * block * per;
    printf("RNG gaussian pairs: %.3f ms  %.2f Gpairs/s  (%.3f ns per entry chip-wide)\n", ms,
           pairs / ms / 1e6, ms * 1e6 / (2 * pairs));
    ms = time_ms([&] { k_rng_int<<<grid, block>>>(d_out, 12345, per); });
    printf("RNG int-only pairs: %.3f ms  %.2f Gpairs/s\n", ms, pairs / ms / 1e6);
  }
  {
    size_t bytes = (size_t)4 << 30;
    double4 *a, *b;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    size_t n4 = bytes / 32;
    float ms = time_ms([&] { k_copy<<<sms * 8, 256>>>(a, b, n4); });
    printf("copy 4GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
    ms = time_ms([&] { k_read<<<sms * 8, 256>>>(a, d_out, n4); });
    printf("read 4GiB: %.3f ms  %.1f GB/s\n", ms, 1.0 * bytes / ms / 1e6);
    cudaFree(a); cudaFree(b);
  }
  {
    const int T = 4096;
    std::vector<double> A(T * 32), B(T * 32), C(T * 64), D(T * 64);
    srand(7);
    auto rnd = [] { return (rand() / (double)RAND_MAX - 0.5) * std::ldexp(1.0, rand() % 20 - 10); };
    for (auto& v : A) v = rnd();
    for (auto& v : B) v = rnd();
    for (auto& v : C) v = rnd();
    double *dA, *dB, *dC, *dD;
    CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8));
    CK(cudaMalloc(&dC, C.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
    cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
    k_dmma_order<<<1, 32>>>(dA, dB, dC, dD, T);
    CK(cudaDeviceSynchronize());
    cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost);
    int orders[4][4] = {{0, 1, 2, 3}, {3, 2, 1, 0}, {1, 0, 3, 2}, {2, 3, 0, 1}};
    long match[5] = {0, 0, 0, 0, 0};
    long total = 0;
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          double a[4], b[4];
          for (int k = 0; k < 4; ++k) { a[k] = A[t * 32 + i * 4 + k]; b[k] = B[t * 32 + k * 8 + j]; }
          double c = C[t * 64 + i * 8 + j];
          double d = D[t * 64 + i * 8 + j];
          for (int o = 0; o < 4; ++o) if (host_seq(a, b, c, orders[o]) == d) match[o]++;
          // exactly rounded 5-term sum via long double products (approximate check)
          __float128 s = (__float128)c;
          for (int k = 0; k < 4; ++k) s += (__float128)a[k] * (__float128)b[k];
          if ((double)s == d) match[4]++;
          total++;
        }
    printf("DMMA order: seq0123 %ld/%ld, seq3210 %ld, seq1032 %ld, seq2301 %ld, single-round %ld\n",
           match[0], total, match[1], match[2], match[3], match[4]);
  }
  printf("done\n");
  return 0;
}
