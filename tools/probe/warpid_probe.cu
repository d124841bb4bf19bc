// Which SM sub-partition does warp w of a 384-thread CTA run on? (%warpid % 4 is the sub-partition)
#include <cstdio>
__global__ void k(int* out) {
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 12 + (threadIdx.x >> 5)] = (int)wid;
}
int main() {
  int* d;
  cudaMalloc(&d, 4 * 12 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<4, 384, 200 * 1024>>>(d);
  int h[48];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int b = 0; b < 4; ++b) {
    printf("cta %d:", b);
    for (int w = 0; w < 12; ++w) printf(" w%d->%d", w, h[b * 12 + w]);
    printf("\n");
  }
}
