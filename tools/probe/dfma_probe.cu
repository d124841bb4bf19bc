// Probe: FP64 DFMA issue throughput (independent chains) and dependent latency on one SM, and the
// same for DMUL / MUFU.RCP64H-based __drcp_rn / sqrt. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
template <int CH>
__global__ void thr(double* out, int iters, long long* cyc) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3 + c;
  const double b = 0.999999, d = 1e-7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fma(a[c], b, d);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void lat_sqrt(double* out, int iters, long long* cyc) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_rcp(double* out, int iters, long long* cyc) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __drcp_rn(x) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1024);
  long long h;
  const int iters = 4096;
  for (int threads : {32, 128, 256, 512, 1024}) {
    thr<8><<<1, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)threads * iters * 8;
    printf("DFMA throughput, %4d threads x 8 chains: %.1f DFMA/clk/SM\n", threads, ops / h);
  }
  thr<1><<<1, 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", (double)h / iters);
  lat_sqrt<<<1, 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("sqrt + add dependent latency: %.1f cycles\n", (double)h / iters);
  lat_rcp<<<1, 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("drcp_rn + add dependent latency: %.1f cycles\n", (double)h / iters);
  return 0;
}
