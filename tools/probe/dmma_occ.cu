// DMMA throughput vs warps per SM and independent accumulator chains per warp,
// and the same with the A operand streamed from shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, int iters, double x) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double a = x + threadIdx.x * 1e-9, b = x;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
__global__ void ks(double* out, int iters, double x) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = x + i;
  __syncthreads();
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      double a = sm[((it * CH + i) * 36 + lane) & 4095];
      double b = sm[((it * CH + i) * 36 + lane + 2048) & 4095];
      dmma(c[i][0], c[i][1], a, b);
    }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH, bool S>
void run(int warps, double* o) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  auto f = [&] { if (S) ks<CH><<<148, warps * 32>>>(o, iters, 1.0000001); else k<CH><<<148, warps * 32>>>(o, iters, 1.0000001); };
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 148 * warps * (double)CH * iters * 256.0;
  printf("%s warps/SM=%2d chains/warp=%d : %6.2f TFLOP/s\n", S ? "smemA" : "regs ", warps, CH, fl / ms / 1e9);
}
int main() {
  double* o; cudaMalloc(&o, 64);
  for (int w : {4, 8, 12, 16}) { run<1, false>(w, o); run<2, false>(w, o); run<4, false>(w, o); run<8, false>(w, o); }
  for (int w : {4, 8, 16}) { run<2, true>(w, o); run<4, true>(w, o); }
  return 0;
}
