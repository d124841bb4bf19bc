// FP64 MMA shapes on B200 (sm_100a): throughput of m8n8k4 / m16n8k4 / m16n8k8 /
// m16n8k16 and whether each accumulates like the sequential fma chain in k order
// (the property the bitwise kernels rely on).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes dmma_shapes.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e = (x);                                                                       \
    if (e != cudaSuccess) {                                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);           \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

template <int K>
struct Mma;
// m16n8kK: A 16xK (K/2 regs... see frag maps below), B Kx8, C 16x8 (4 regs)
template <>
struct Mma<4> {
  static __device__ __forceinline__ void run(double (&c)[4], const double (&a)[2], const double (&b)[1]) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  }
};
template <>
struct Mma<8> {
  static __device__ __forceinline__ void run(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
};
template <>
struct Mma<16> {
  static __device__ __forceinline__ void run(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
};

__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int K, int CH>
__global__ void k_tp(double* out, int iters, double x, double y) {
  double acc[CH][4];
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = x + threadIdx.x * 1e-9 + i;
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = y + i;
#pragma unroll
  for (int i = 0; i < CH; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = threadIdx.x + i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) Mma<K>::run(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_tp884(double* out, int iters, double x, double y) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    acc[i][0] = threadIdx.x;
    acc[i][1] = i;
  }
  double a = x + threadIdx.x * 1e-9, b = y;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) mma884(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// One warp per trial: D(16x8) = C + A(16xK) B(Kx8), fragments per the PTX ISA
// (g = lane>>2, t = lane&3): A a[i] = A[g + 8*(i&1)][t + 4*(i>>1)], B b[i] = B[t + 4i][g],
// C c[i] = C[g + 8*(i>>1)][2t + (i&1)].
template <int K>
__global__ void k_order(const double* A, const double* B, const double* C, double* D, int trials) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  for (int tr = 0; tr < trials; ++tr) {
    const double* a = A + (size_t)tr * 16 * K;
    const double* b = B + (size_t)tr * K * 8;
    const double* c = C + (size_t)tr * 128;
    double af[K / 2], bf[K / 4], acc[4];
#pragma unroll
    for (int i = 0; i < K / 2; ++i) af[i] = a[(g + 8 * (i & 1)) * K + t + 4 * (i >> 1)];
#pragma unroll
    for (int i = 0; i < K / 4; ++i) bf[i] = b[(t + 4 * i) * 8 + g];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = c[(g + 8 * (i >> 1)) * 8 + 2 * t + (i & 1)];
    Mma<K>::run(acc, af, bf);
#pragma unroll
    for (int i = 0; i < 4; ++i) D[(size_t)tr * 128 + (g + 8 * (i >> 1)) * 8 + 2 * t + (i & 1)] = acc[i];
  }
}

template <int K>
void order_test(int trials) {
  std::vector<double> A((size_t)trials * 16 * K), B((size_t)trials * K * 8), C((size_t)trials * 128),
      D((size_t)trials * 128);
  srand(7 + K);
  auto rnd = [] {
    // wide dynamic range so that summation order matters
    double v = (double)rand() / RAND_MAX - 0.5;
    return ldexp(v, rand() % 40 - 20);
  };
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  for (auto& v : C) v = rnd();
  double *dA, *dB, *dC, *dD;
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMalloc(&dB, B.size() * 8));
  CK(cudaMalloc(&dC, C.size() * 8));
  CK(cudaMalloc(&dD, D.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
  k_order<K><<<1, 32>>>(dA, dB, dC, dD, trials);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
  long seq = 0, seq4 = 0, tot = 0;
  for (int tr = 0; tr < trials; ++tr)
    for (int r = 0; r < 16; ++r)
      for (int col = 0; col < 8; ++col) {
        const double* a = &A[(size_t)tr * 16 * K + r * K];
        const double* b = &B[(size_t)tr * K * 8];
        double s = C[(size_t)tr * 128 + r * 8 + col];
        for (int k = 0; k < K; ++k) s = fma(a[k], b[k * 8 + col], s);
        // alternative: chunks of 4 summed exactly-ish then added? (record plain chain only)
        double s4 = C[(size_t)tr * 128 + r * 8 + col];
        for (int k0 = 0; k0 < K; k0 += 4) {
          double p = 0;
          for (int k = k0; k < k0 + 4; ++k) p = fma(a[k], b[k * 8 + col], p);
          s4 += p;
        }
        const double d = D[(size_t)tr * 128 + r * 8 + col];
        seq += (d == s);
        seq4 += (d == s4);
        ++tot;
      }
  printf("m16n8k%-2d order: sequential fma chain %ld/%ld, 4-chunk partials %ld/%ld\n", K, seq, tot, seq4, tot);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  cudaFree(dD);
}

template <typename F>
float time_it(F f) {
  cudaEvent_t s, ev;
  cudaEventCreate(&s);
  cudaEventCreate(&ev);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(s);
  f();
  cudaEventRecord(ev);
  CK(cudaEventSynchronize(ev));
  float ms;
  cudaEventElapsedTime(&ms, s, ev);
  return ms;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms=%d\n", p.name, p.multiProcessorCount);
  double* out;
  CK(cudaMalloc(&out, 8));
  const int sms = p.multiProcessorCount, iters = 4096;
  for (int bpsm : {4, 8}) {
    const int blocks = sms * bpsm, thr = 128;
    const double warps = (double)blocks * thr / 32;
    float ms = time_it([&] { k_tp884<8><<<blocks, thr>>>(out, iters, 1.0, 1e-3); });
    printf("m8n8k4   bpsm=%d %.3f ms %.2f TFLOP/s\n", bpsm, ms, warps * iters * 8 * 512 / (ms * 1e9));
    ms = time_it([&] { k_tp<4, 8><<<blocks, thr>>>(out, iters, 1.0, 1e-3); });
    printf("m16n8k4  bpsm=%d %.3f ms %.2f TFLOP/s\n", bpsm, ms, warps * iters * 8 * 1024 / (ms * 1e9));
    ms = time_it([&] { k_tp<8, 8><<<blocks, thr>>>(out, iters, 1.0, 1e-3); });
    printf("m16n8k8  bpsm=%d %.3f ms %.2f TFLOP/s\n", bpsm, ms, warps * iters * 8 * 2048 / (ms * 1e9));
    ms = time_it([&] { k_tp<16, 8><<<blocks, thr>>>(out, iters, 1.0, 1e-3); });
    printf("m16n8k16 bpsm=%d %.3f ms %.2f TFLOP/s\n", bpsm, ms, warps * iters * 8 * 4096 / (ms * 1e9));
  }
  order_test<4>(4096);
  order_test<8>(4096);
  order_test<16>(4096);
  printf("done\n");
  return 0;
}
