// Probe: tcgen05.mma kind::i8 (s8 x s8 -> s32 in TMEM) on sm_100a, single CTA, M = 128.
// Validates the K-major SWIZZLE_NONE shared-memory descriptor layout and the instruction descriptor
// against a host GEMM, then times back-to-back MMAs (cycles per instruction) for N = 64, 128, 256.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8 umma_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 B contiguous); LBO = byte distance between the
// two 16-byte K halves of a 32-wide K step, SBO = byte distance between 8-row groups.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_s8(int M, int N, int asg = 1, int bsg = 1) {
  return (2u << 4)                      // D format s32
         | ((uint32_t)asg << 7) | ((uint32_t)bsg << 10)  // A, B signed (1) / unsigned (0) 8-bit
         | ((uint32_t)(N >> 3) << 17)   // N / 8
         | ((uint32_t)(M >> 4) << 24);  // M / 16
}

// element (r, k) of an R x Ktot K-major operand: k-step ks = k / 32 holds R/8 groups of 256 B
__host__ __device__ inline int koff(int r, int k, int R) {
  const int ks = k >> 5, kk = k & 31;
  return ks * (R * 32) + (r >> 3) * 256 + (kk >> 4) * 128 + (r & 7) * 16 + (kk & 15);
}

template <int N>
__global__ void umma_probe(const int8_t* __restrict__ ga, const int8_t* __restrict__ gb, int ktot, int reps,
                           int* __restrict__ out, long long* cycles, int asg, int bsg) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  int8_t* sa = reinterpret_cast<int8_t*>(sm);
  int8_t* sb = sa + 128 * ktot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * ktot; e += blockDim.x) sa[e] = ga[e];
  for (int e = tid; e < N * ktot; e += blockDim.x) sb[e] = gb[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int ks = 0; ks < ktot / 32; ++ks) {
        const uint64_t da = sdesc(smem_u32(sa + ks * 128 * 32), 128, 256);
        const uint64_t db = sdesc(smem_u32(sb + ks * N * 32), 128, 256);
        const uint32_t acc = (r > 0 || ks > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
            "l"(da), "l"(db), "r"(idesc_s8(128, N, asg, bsg)), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // everyone waits for the MMAs
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
  }
  if (tid == 0) {
    t1 = clock64();
    cycles[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // D row = TMEM lane: warp w reads lanes 32w.., 8 columns at a time
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) out[(32 * warp + lane) * N + c0 + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(N < 32 ? 32 : N));
}

template <int N>
int run(int ktot, int reps, int asg = 1, int bsg = 1) {
  std::vector<int8_t> A(128 * ktot), B(N * ktot), ha(128 * ktot), hb(N * ktot);
  srand(7 + N);
  for (auto& x : A) x = (int8_t)(rand() % 256 - 128);
  for (auto& x : B) x = (int8_t)(rand() % 256 - 128);
  // A logical 128 x ktot, B logical N x ktot (row = output column), both K-major in the core-matrix layout
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < ktot; ++k) ha[koff(r, k, 128)] = A[r * ktot + k];
  for (int r = 0; r < N; ++r)
    for (int k = 0; k < ktot; ++k) hb[koff(r, k, N)] = B[r * ktot + k];
  int8_t *da, *db;
  int* dout;
  long long* dcyc;
  CK(cudaMalloc(&da, ha.size()));
  CK(cudaMalloc(&db, hb.size()));
  CK(cudaMalloc(&dout, 128 * N * 4));
  CK(cudaMalloc(&dcyc, 8));
  CK(cudaMemcpy(da, ha.data(), ha.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb.data(), hb.size(), cudaMemcpyHostToDevice));
  const size_t smem = (size_t)(128 + N) * ktot + 1024;
  CK(cudaFuncSetAttribute(umma_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  umma_probe<N><<<1, 128, smem>>>(da, db, ktot, reps, dout, dcyc, asg, bsg);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> out(128 * N);
  long long cyc;
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  long long bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      long long s = 0;
      for (int k = 0; k < ktot; ++k)
        s += (long long)(asg ? (int)A[i * ktot + k] : (int)(uint8_t)A[i * ktot + k]) *
             (bsg ? (int)B[j * ktot + k] : (int)(uint8_t)B[j * ktot + k]);
      s *= reps;
      if ((int)s != out[i * N + j]) ++bad;
    }
  const long long nmma = (long long)reps * (ktot / 32);
  std::printf("a%c b%c N=%3d ktot=%d reps=%d: mismatches %lld of %d; %lld MMAs in %lld cycles = %.1f cycles/MMA (%.0f MAC/clk)\n",
              asg ? 's' : 'u', bsg ? 's' : 'u', N, ktot, reps, bad, 128 * N, nmma, cyc, (double)cyc / nmma, 128.0 * N * 32 * nmma / cyc);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dout);
  cudaFree(dcyc);
  return bad != 0;
}

int main() {
  int fails = 0;
  fails += run<64>(256, 1);
  fails += run<64>(256, 1, 0, 1);
  fails += run<64>(256, 1, 1, 0);
  fails += run<64>(256, 1, 0, 0);
  fails += run<128>(256, 1);
  fails += run<64>(256, 200);
  fails += run<128>(256, 200);
  fails += run<256>(256, 200);
  std::printf(fails ? "FAIL\n" : "ok\n");
  return fails;
}
