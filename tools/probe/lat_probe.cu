// Latency probe: dependent-chain latency of DMMA, DFMA, DDIV, shfl, and the
// Markstein division sequence (one warp, clock64 around long chains).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k(double* out, long long* cyc, int iters, double x, double d) {
  double c0 = threadIdx.x, c1 = 1.0, a = x, b = x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(c0, c1, a, b);
  long long t1 = clock64();
  double f = threadIdx.x;
  for (int i = 0; i < iters; ++i) f = fma(f, x, d);
  long long t2 = clock64();
  double q = threadIdx.x + 1.0;
  for (int i = 0; i < iters; ++i) q = q / d;
  long long t3 = clock64();
  double s = threadIdx.x;
  for (int i = 0; i < iters; ++i) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31) * x;
  long long t4 = clock64();
  const double inv = 1.0 / d;
  double y = threadIdx.x + 1.0;
  for (int i = 0; i < iters; ++i) {
    double q0 = y * inv;
    double r = fma(-q0, d, y);
    double q1 = fma(r, inv, q0);
    r = fma(-q1, d, y);
    y = fma(r, inv, q1);
  }
  long long t5 = clock64();
  out[threadIdx.x] = c0 + c1 + f + q + s + y;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 64);
  const int it = 4096;
  k<<<1, 32>>>(o, c, it, 1.0000001, 1.0000003);
  k<<<1, 32>>>(o, c, it, 1.0000001, 1.0000003);
  long long h[5]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[5] = {"DMMA chain", "DFMA chain", "DDIV chain", "SHFL+DMUL chain", "Markstein div (5 ops) chain"};
  for (int i = 0; i < 5; ++i) printf("%-28s %.1f cycles/op\n", nm[i], (double)h[i] / it);
  return 0;
}
