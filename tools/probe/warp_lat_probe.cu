// Dependent-issue latency (SM cycles) of the warp primitives the small factorizations use:
// redux.sync max (u32), shfl.sync, vote.ballot, an LDS round trip, DFMA, DMUL, __drcp_rn, IEEE division.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o warp_lat_probe warp_lat_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k(long long* cyc, unsigned* outu, double* outd, int iters) {
  __shared__ unsigned sm[64];
  const int lane = threadIdx.x & 31;
  sm[lane] = lane;
  __syncwarp();
  unsigned v = lane * 7 + 1;
  double d = 1.0 + lane * 1e-3;
  long long t0, t1;
  // redux
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v + lane) & 0xffff;
  t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  // shfl
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  t1 = clock64();
  if (lane == 0) cyc[1] = t1 - t0;
  // ballot
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __ballot_sync(0xffffffffu, (v >> lane) & 1) + lane;
  t1 = clock64();
  if (lane == 0) cyc[2] = t1 - t0;
  // lds
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = sm[v & 31];
  t1 = clock64();
  if (lane == 0) cyc[3] = t1 - t0;
  // dfma
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = fma(d, 0.999999, 1e-7);
  t1 = clock64();
  if (lane == 0) cyc[4] = t1 - t0;
  // drcp
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = __drcp_rn(d) + 0.5;
  t1 = clock64();
  if (lane == 0) cyc[5] = t1 - t0;
  // div
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = 1.5 / d + 0.25;
  t1 = clock64();
  if (lane == 0) cyc[6] = t1 - t0;
  // fabs + compare + select chain (DADD for fabs?)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = fabs(d - 2.0) + 0.5;
  t1 = clock64();
  if (lane == 0) cyc[7] = t1 - t0;
  outu[threadIdx.x] = v;
  outd[threadIdx.x] = d;
}

int main() {
  long long* cyc;
  unsigned* ou;
  double* od;
  cudaMalloc(&cyc, 8 * 16);
  cudaMalloc(&ou, 4 * 32);
  cudaMalloc(&od, 8 * 32);
  const int iters = 4096;
  k<<<1, 32>>>(cyc, ou, od, iters);
  k<<<1, 32>>>(cyc, ou, od, iters);
  long long h[8];
  cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  const char* names[] = {"redux.max+iadd", "shfl+iadd", "ballot+iadd", "lds (dependent)", "dfma", "drcp_rn+dadd",
                         "ieee div+dadd", "dadd+fabs(dadd)"};
  for (int i = 0; i < 8; ++i) printf("%-18s %6.1f cycles per iteration\n", names[i], (double)h[i] / iters);
  return 0;
}
