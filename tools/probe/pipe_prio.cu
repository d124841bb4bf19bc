// Does a DMMA stream starve DFMA chains of other warps on the same SM sub-partition?
// One CTA per SM: MMA warps (16 independent DMMA chains each) run a fixed number of steps;
// side warps run `chain` independent DFMA chains of fixed length. Each warp records its own
// elapsed clocks; we print how long the side warps took alone vs next to the MMA stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_prio pipe_prio.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CH, int MCH = 16, int SIDE_DMMA = 0, bool SWAP = false>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int mma_warps, int steps, int len) {
  const int warp = SWAP ? ((threadIdx.x >> 5) ^ 8) : (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const long long t0 = clock64();
  if (warp < mma_warps) {
    double acc[MCH][2];
#pragma unroll
    for (int i = 0; i < MCH; ++i) acc[i][0] = acc[i][1] = threadIdx.x + i;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
    for (int s = 0; s < steps * 16 / MCH; ++s) {
#pragma unroll
      for (int i = 0; i < MCH; ++i) dmma(acc[i][0], acc[i][1], a, b);
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < MCH; ++i) t += acc[i][0] + acc[i][1];
    if (t == 1234.5) out[0] = t;
  } else if (warp >= 8) {
    double x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = 1.0 + threadIdx.x * 1e-7 + i * 1e-3;
    double sacc[SIDE_DMMA > 0 ? SIDE_DMMA : 1][2];
#pragma unroll
    for (int i = 0; i < (SIDE_DMMA > 0 ? SIDE_DMMA : 1); ++i) sacc[i][0] = sacc[i][1] = i;
    for (int it = 0; it < len; ++it) {
#pragma unroll
      for (int i = 0; i < CH; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
#pragma unroll
      for (int i = 0; i < SIDE_DMMA; ++i) dmma(sacc[i][0], sacc[i][1], x[0], 1e-3);
    }
#pragma unroll
    for (int i = 0; i < (SIDE_DMMA > 0 ? SIDE_DMMA : 1); ++i) x[0] += sacc[i][0] + sacc[i][1];
    double t = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) t += x[i];
    if (t == 1234.5) out[0] = t;
  }
  const long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) cyc[warp] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 16 * 8);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  for (int ch : {1, 4, 8}) {
    for (int mw : {0, 4, 8}) {
      long long h[16] = {};
      const int len = 20000, steps = mw ? 4000 : 0;
      cudaMemset(cyc, 0, 128);
      if (ch == 1) k<1><<<sms, 512>>>(out, cyc, mw, steps, len);
      if (ch == 4) k<4><<<sms, 512>>>(out, cyc, mw, steps, len);
      if (ch == 8) k<8><<<sms, 512>>>(out, cyc, mw, steps, len);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
      long long mma = 0, side = 0;
      for (int w = 0; w < 8; ++w) mma = h[w] > mma ? h[w] : mma;
      for (int w = 8; w < 16; ++w) side = h[w] > side ? h[w] : side;
      printf("chains %d, %d MMA warps: MMA warps %lld clk, side warps %lld clk (%.2f clk per dependent DFMA step)\n",
             ch, mw, mma, side, (double)side / len);
    }
  }
  // side warps that also issue DMMAs (on independent accumulators) between their dependent DFMAs
  for (int sd : {0, 1, 2, 4}) {
    long long h[16] = {};
    const int len = 20000, steps = 4000;
    cudaMemset(cyc, 0, 128);
    if (sd == 0) k<1, 16, 0><<<sms, 512>>>(out, cyc, 8, steps, len);
    if (sd == 1) k<1, 16, 1><<<sms, 512>>>(out, cyc, 8, steps, len);
    if (sd == 2) k<1, 16, 2><<<sms, 512>>>(out, cyc, 8, steps, len);
    if (sd == 4) k<1, 16, 4><<<sms, 512>>>(out, cyc, 8, steps, len);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
    long long mma = 0, side = 0;
    for (int w = 0; w < 8; ++w) mma = h[w] > mma ? h[w] : mma;
    for (int w = 8; w < 16; ++w) side = h[w] > side ? h[w] : side;
    printf("side warps with %d DMMA per DFMA step: MMA warps %lld clk, side %.2f clk per step\n", sd, mma,
           (double)side / len);
  }
  {  // MMA warps on the high hardware warp ids
    long long h[16] = {};
    cudaMemset(cyc, 0, 128);
    k<1, 16, 0, true><<<sms, 512>>>(out, cyc, 8, 4000, 20000);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
    long long mma = 0, side = 0;
    for (int w = 0; w < 8; ++w) mma = h[w] > mma ? h[w] : mma;
    for (int w = 8; w < 16; ++w) side = h[w] > side ? h[w] : side;
    printf("MMA warps on hardware warps 8-15: MMA %lld clk, side %.2f clk per DFMA step\n", mma, (double)side / 20000);
  }
  // MMA warps with fewer independent DMMA chains: does the side chain get the pipe sooner?
  for (int mch : {2, 4, 8, 16}) {
    long long h[16] = {};
    const int len = 20000, steps = 4000;
    cudaMemset(cyc, 0, 128);
    if (mch == 2) k<1, 2><<<sms, 512>>>(out, cyc, 8, steps, len);
    if (mch == 4) k<1, 4><<<sms, 512>>>(out, cyc, 8, steps, len);
    if (mch == 8) k<1, 8><<<sms, 512>>>(out, cyc, 8, steps, len);
    if (mch == 16) k<1, 16><<<sms, 512>>>(out, cyc, 8, steps, len);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
    long long mma = 0, side = 0;
    for (int w = 0; w < 8; ++w) mma = h[w] > mma ? h[w] : mma;
    for (int w = 8; w < 16; ++w) side = h[w] > side ? h[w] : side;
    printf("8 MMA warps x %2d DMMA chains: MMA warps %lld clk (%.1f%% of 2.05M), side chain %.2f clk per DFMA step\n", mch,
           mma, 2.05e6 / mma * 100, (double)side / len);
  }
  return 0;
}
