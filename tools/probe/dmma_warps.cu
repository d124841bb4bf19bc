#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, int iters, double x, double y) {
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
int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int wpsm : {4, 8, 12, 16}) {
    for (int ch : {8, 16, 32}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto launch = [&] {
        if (ch == 8) k<8><<<sms, wpsm * 32>>>(out, iters, 1.0, 1e-3);
        if (ch == 16) k<16><<<sms, wpsm * 32>>>(out, iters, 1.0, 1e-3);
        if (ch == 32) k<32><<<sms, wpsm * 32>>>(out, iters, 1.0, 1e-3);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fl = (double)sms * wpsm * iters * ch * 512;
      printf("warps/SM %2d chains %2d: %.2f TFLOP/s\n", wpsm, ch, fl / (ms * 1e9));
    }
  }
}
