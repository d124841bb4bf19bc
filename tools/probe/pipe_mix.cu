// How DFMA work from other warps slows a DMMA stream on B200 (they share the FP64 pipe).
// One CTA per SM: 8 "MMA" warps issue independent DMMA.8x8x4 chains; 8 "side" warps issue
// a fixed number of DFMA per step in one of several patterns:
//   mode 0: no side work
//   mode 1: DFMA interleaved 1:3 with integer ops, 4 independent chains
//   mode 2: dense DFMA, 8 independent chains, then the same integer ops
//   mode 3: integer ops only
//   mode 4: FP32 FFMA instead of DFMA, interleaved like mode 1
//   mode 5: dense DFMA, 16 chains
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix pipe_mix.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double* out, int steps, int side_ops) {
  const int warp = threadIdx.x >> 5;
  if (warp < 8) {
    double acc[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = threadIdx.x + i;
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
    for (int s = 0; s < steps; ++s) {
#pragma unroll
      for (int i = 0; i < 16; ++i) dmma(acc[i][0], acc[i][1], a, b);
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += acc[i][0] + acc[i][1];
    if (t == 1234.5) out[0] = t;
    return;
  }
  if (MODE == 0) return;
  // side warps: total work = steps * side_ops "units" (scaled so that they finish about when the MMA warps do)
  double x[16];
  float fx[16];
  unsigned u[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    x[i] = 1.0 + threadIdx.x * 1e-7 + i * 1e-3;
    fx[i] = 1.0f + i * 1e-3f;
    u[i] = threadIdx.x * 7 + i;
  }
  const int iters = steps * side_ops / 16;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1 || MODE == 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (MODE == 1) x[i] = fma(x[i], 0.999999, 1e-7);
          else fx[i] = fmaf(fx[i], 0.999999f, 1e-7f);
          u[i] = (u[i] ^ (u[i] >> 7)) + 0x9E3779B9u;
          u[i + 4] = u[i + 4] * 3u + u[i];
          u[i + 8] = __funnelshift_r(u[i + 8], u[i], 3);
        }
      }
    } else if (MODE == 2 || MODE == 5) {
      constexpr int CH = MODE == 2 ? 8 : 16;
#pragma unroll
      for (int j = 0; j < 16 / CH; ++j)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        u[i & 3] = (u[i & 3] ^ (u[i & 3] >> 7)) + 0x9E3779B9u;
        u[4 + (i & 3)] = u[4 + (i & 3)] * 3u + u[i & 3];
        u[8 + (i & 3)] = __funnelshift_r(u[8 + (i & 3)], u[i & 3], 3);
      }
    } else if (MODE >= 10) {  // one op kind, 8 independent chains, 16 ops per iteration
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (MODE == 10) x[i] = x[i] * 0.999999;
          if (MODE == 11) x[i] = x[i] + 1e-9;
          if (MODE == 12) u[i] = u[i] + u[i + 8];
          if (MODE == 13) u[i] = u[i] ^ (u[i + 8] & 0x5555u) ^ 0x77u;
          if (MODE == 14) u[i] = u[i] * 0x9E3779B9u + u[i + 8];
          if (MODE == 15) u[i] = __funnelshift_r(u[i], u[i + 8], 5);
          if (MODE == 16) fx[i] = fmaf(fx[i], 0.999f, 1e-7f);
          if (MODE == 17) { asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(*(unsigned long long*)&x[i]) : "r"(u[i]), "r"(u[i + 8])); u[i] += 1; }
          if (MODE == 18) x[i] = (double)(u[i] + j);
          if (MODE == 19) x[i] = fma(x[i], 0.999999, 1e-7);
        }
    } else if (MODE == 3) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        u[i & 3] = (u[i & 3] ^ (u[i & 3] >> 7)) + 0x9E3779B9u;
        u[4 + (i & 3)] = u[4 + (i & 3)] * 3u + u[i & 3];
        u[8 + (i & 3)] = __funnelshift_r(u[8 + (i & 3)], u[i & 3], 3);
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += x[i] + fx[i] + u[i];
  if (t == 1234.5) out[0] = t;
}

template <int MODE>
float run(double* out, int sms, int steps, int side_ops) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<sms, 512>>>(out, steps, side_ops);
  cudaEventRecord(a);
  k<MODE><<<sms, 512>>>(out, steps, side_ops);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int sms = p.multiProcessorCount, steps = 8192;
  const double mma_flops = (double)sms * 8 * steps * 16 * 512;
  float t0 = run<0>(out, sms, steps, 0);
  printf("MMA only: %.3f ms (%.1f TFLOP/s)\n", t0, mma_flops / t0 / 1e9);
  // side DFMA lane-ops per step per warp: side_ops * 32 lanes
  {
    const int side = 8;
    const double ops = (double)sms * 8 * steps * side;
    auto cyc = [&](float t) { return (t - t0) * 1e-3 * 1.9e9 / (ops / (sms * 4)); };
    const char* names[] = {"DMUL", "DADD", "IADD3", "LOP3", "IMAD", "SHF", "FFMA", "IMAD.WIDE", "I2F.F64", "DFMA"};
    float ts[] = {run<10>(out, sms, steps, side), run<11>(out, sms, steps, side), run<12>(out, sms, steps, side),
                  run<13>(out, sms, steps, side), run<14>(out, sms, steps, side), run<15>(out, sms, steps, side),
                  run<16>(out, sms, steps, side), run<17>(out, sms, steps, side), run<18>(out, sms, steps, side),
                  run<19>(out, sms, steps, side)};
    for (int i = 0; i < 10; ++i) printf("  %-9s x%d/step/warp: %.3f ms, %.2f SMSP clk per warp instruction\n", names[i], side, ts[i], cyc(ts[i]));
  }
  for (int side : {2, 4, 8, 16}) {
    const double dfma = (double)sms * 8 * steps * side;  // warp-level DFMA instructions in the side warps
    float t1 = run<1>(out, sms, steps, side), t2 = run<2>(out, sms, steps, side), t5 = run<5>(out, sms, steps, side);
    float t3 = run<3>(out, sms, steps, side), t4 = run<4>(out, sms, steps, side);
    // extra time per side warp-DFMA, in SM-sub-partition clocks (1.9 GHz nominal)
    auto cyc = [&](float t) { return (t - t0) * 1e-3 * 1.9e9 / (dfma / (sms * 4)); };
    printf("side %2d DFMA/step/warp: interleaved %.3f ms (%.2f clk/DFMA) dense8 %.3f (%.2f) dense16 %.3f (%.2f) | "
           "int-only %.3f  ffma-interleaved %.3f\n",
           side, t1, cyc(t1), t2, cyc(t2), t5, cyc(t5), t3, t4);
  }
  return 0;
}
