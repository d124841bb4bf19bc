// sketch.cu — Gaussian sketch A1 = Omega A with Omega generated in-kernel
// (sketch.cpp:94-116), uniform row extraction (sketch.cpp:27-55) and the
// device RNG fills used by the parity tests (rng.hpp:22-92).
//
// Omega(i, j) = gaussian_at(seed, i*m + j) with the GLOBAL row index j, so a
// row-sharded A (one GPU per block, parexec.cpp:9-18) sketches to partials that
// sum to the single-GPU sketch. Omega never touches HBM: each CTA owns an
// (ST rows of Omega) x (a contiguous range of A's rows) block, generates the
// Omega tile for each 32-row step into shared memory exactly once (both
// Box-Muller outputs of a pair are used, rng.hpp:47-55), and multiplies it
// with the staged A rows on DMMA m8n8k4. Per-CTA partials are summed in a
// fixed k-chunk order by a second kernel (deterministic run to run).
//
// Algorithmic work: 2*l*m*n flops + l*m Gaussian draws; HBM: 8*m*n bytes of A
// (each A row is read by l/ST CTAs that run together, the repeats hit L2).

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "boxmuller.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace cqr {

namespace {

constexpr int kST = 64;  // Omega rows per CTA
constexpr int kKS = 32;  // A rows per step
constexpr int kThreads = 256;

int sketch_np(int n) {
  if (n <= 8) return 8;
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (n <= 256) return 256;
  return 512;
}

__constant__ BmTables c_bm;

// Generate the Box-Muller pairs of Omega[s0 .. s0+ST) x [kb .. kb+KS) (kb =
// global row index of A) into sOm (row stride KS+4). Straight-line code:
// invalid slots compute a clamped pair and skip the (predicated) stores; Omega
// rows at or beyond l are zero. ALIGNED: every row's counter range starts
// even (m_global and kb even), so a row is exactly KS/2 pairs.
template <bool ALIGNED>
__device__ __forceinline__ void gen_pair_slot(const BmTables& T, double* sOm, int s0, int l, long long m_global,
                                              long long kb, uint64_t seed, int e) {
  constexpr int LDO = kKS + 4;
  if (ALIGNED) {
    const int i = e >> 4, pp = e & 15;
    const unsigned long long c_lo = (unsigned long long)(s0 + i) * (unsigned long long)m_global + kb;
    double ge, go;
    gaussian_pair_fast(T, seed, (c_lo >> 1) + pp, ge, go);
    const bool live = s0 + i < l;
    *reinterpret_cast<double2*>(sOm + i * LDO + 2 * pp) = make_double2(live ? ge : 0.0, live ? go : 0.0);
  } else {
    constexpr int PPR = kKS / 2 + 1;
    const bool valid = e < kST * PPR;
    const int ee = valid ? e : 0;
    const int i = ee / PPR, pp = ee - i * PPR;
    const unsigned long long c_lo = (unsigned long long)(s0 + i) * (unsigned long long)m_global + kb;
    const unsigned long long p = (c_lo >> 1) + pp;
    double ge, go;
    gaussian_pair_fast(T, seed, p, ge, go);
    const bool live = s0 + i < l;
    const long long ce = (long long)(2 * p - c_lo);
    double* row = sOm + i * LDO;
    if (valid && ce >= 0 && ce < kKS) row[ce] = live ? ge : 0.0;
    if (valid && ce + 1 >= 0 && ce + 1 < kKS) row[ce + 1] = live ? go : 0.0;
  }
}

// NP = columns handled by one CTA (<= 128); wider A is split over gridDim.z
// column parts of NP, each regenerating the same Omega tile. Per 32-row step:
// one barrier; the DMMAs of step i are interleaved (same basic block) with the
// Box-Muller draws of step i+1 into the other Omega buffer, and the A rows of
// step i+1 stream in by cp.async meanwhile.
template <int NP, bool ALIGNED>
__global__ void __launch_bounds__(kThreads, 2) sketch_kernel(const double* __restrict__ a, long long lda,
                                                             long long m_local, long long m_global, long long row0,
                                                             int n, int l, uint64_t seed, long long rows_per_chunk,
                                                             double* __restrict__ partial, int lp, int np_total,
                                                             int vec16, int check, int y0, DevStatus* st) {
  constexpr int NT = NP / 8;
  constexpr int WN = NT < 8 ? NT : 8;  // warps along n
  constexpr int WM = 8 / WN;           // warps along Omega rows
  constexpr int MG = kST / 8 / WM;     // 8-row groups per warp
  constexpr int NG = NT / WN;          // 8-col groups per warp
  constexpr int LDA = NP + 4;
  constexpr int LDO = kKS + 4;
  constexpr int SLOTS = ALIGNED ? kST * kKS / 2 : kST * (kKS / 2 + 1);
  constexpr int PER = (SLOTS + kThreads - 1) / kThreads;  // pair slots per thread per step
  constexpr int K4 = kKS / 4;
  extern __shared__ __align__(16) double smem[];
  __shared__ BmTables T;
  if (failed(st)) return;
  // buffers as offsets into smem[] (keeps every access in the shared window: LDS/STS)
  constexpr int OFF_OM = 0, OFF_A = 2 * kST * LDO;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, gr = lane >> 2;
  const int wm = warp / WN, wn = warp - (warp / WN) * WN;
  const int s0 = blockIdx.x * kST;
  const int col0 = blockIdx.z * NP;
  a += col0;
  n = min(NP, n - col0);
  const int ky = blockIdx.y + y0;  // k-chunk index (launches may cover a sub-range of chunks)
  const long long k_begin = (long long)ky * rows_per_chunk;
  const long long k_end = min(m_local, k_begin + rows_per_chunk);
  {
    const double* src = reinterpret_cast<const double*>(&c_bm);
    double* dst = reinterpret_cast<double*>(&T);
    for (int e = tid; e < (int)(sizeof(BmTables) / sizeof(double)); e += kThreads) dst[e] = src[e];
  }
  double acc[MG][NG][2];
#pragma unroll
  for (int g = 0; g < MG; ++g)
#pragma unroll
    for (int h = 0; h < NG; ++h) acc[g][h][0] = acc[g][h][1] = 0.0;
  const int nsteps = k_end > k_begin ? (int)((k_end - k_begin + kKS - 1) / kKS) : 0;
  bool bad = false;  // non-finite A values seen in this warp's B fragments (they cover all of A)
  if (nsteps > 0) {
    stage_rows(smem + OFF_A, LDA, a + k_begin * lda, lda, (int)min((long long)kKS, k_end - k_begin), kKS, n, NP, tid,
               kThreads, vec16 != 0);
    cp_async_commit();
    __syncthreads();  // tables
#pragma unroll
    for (int u = 0; u < PER; ++u)
      gen_pair_slot<ALIGNED>(T, smem + OFF_OM, s0, l, m_global, row0 + k_begin, seed, tid + kThreads * u);
  }
  for (int st_i = 0; st_i < nsteps; ++st_i) {
    const long long kb = k_begin + (long long)st_i * kKS;
    cp_async_wait<0>();
    __syncthreads();
    if (st_i + 1 < nsteps) {
      const long long kn = kb + kKS;
      stage_rows(smem + OFF_A + ((st_i + 1) & 1) * kKS * LDA, LDA, a + kn * lda, lda, (int)min((long long)kKS, k_end - kn), kKS, n, NP, tid,
                 kThreads, vec16 != 0);
      cp_async_commit();
    }
    const int offA = OFF_A + (st_i & 1) * kKS * LDA;
    const int offO = OFF_OM + (st_i & 1) * kST * LDO + (wm * MG * 8 + gr) * LDO + q;
    double* On = smem + OFF_OM + ((st_i + 1) & 1) * kST * LDO;
    const long long kbn = row0 + kb + kKS;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      gen_pair_slot<ALIGNED>(T, On, s0, l, m_global, kbn, seed, tid + kThreads * u);
#pragma unroll
      for (int k4 = u * K4 / PER; k4 < (u + 1) * K4 / PER; ++k4) {
        double af[MG], bf[NG];
#pragma unroll
        for (int g = 0; g < MG; ++g) af[g] = smem[offO + g * 8 * LDO + 4 * k4];
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          bf[h] = smem[offA + (4 * k4 + q) * LDA + (wn * NG + h) * 8 + gr];
          bad |= nonfinite(bf[h]);
        }
#pragma unroll
        for (int g = 0; g < MG; ++g)
#pragma unroll
          for (int h = 0; h < NG; ++h) dmma(acc[g][h][0], acc[g][h][1], af[g], bf[h]);
      }
    }
  }
  if (check && __any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  // partial[chunk][s0 + i][col0 + col], lp rows per chunk, np_total columns
  double* out = partial + (long long)ky * lp * np_total + col0;
#pragma unroll
  for (int g = 0; g < MG; ++g) {
    const int i = s0 + (wm * MG + g) * 8 + gr;
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      const int j = (wn * NG + h) * 8 + 2 * q;
      *reinterpret_cast<double2*>(out + (long long)i * np_total + j) = make_double2(acc[g][h][0], acc[g][h][1]);
    }
  }
}

// Warp-specialised variant (the default for n in (64, 128], even counters,
// TMA-addressable A). The Box-Muller draws and the DMMA stream share the FP64
// pipe; in the kernel above every warp alternates between them, and the
// draw latency leaves the pipe ~25% idle (a constant-Omega build of the same
// kernel runs the sketch in 2.14 ms vs 2.94). Here 8 generator warps fill a
// 3-stage ring of Omega tiles (64 x 32, the same counters and pair layout) while
// a TMA load brings the matching 32 x 128 A tile (SWIZZLE_128B boxes of 16
// columns, one box per MMA warp), and 8 MMA warps consume the stages behind
// full/empty mbarriers. Per-element arithmetic and k order are those of
// sketch_kernel<128, true>: the partials are bit-identical.
// The DMMA stream holds the FP64 pipe whenever it has work (tools/probe/pipe_prio.cu:
// a DFMA chain next to 8 DMMA warps advances only when they stall), so the draws'
// FP64 instructions run in its gaps and in the windows where the ring runs dry
// (per-warp timeline: -DCQR_WS_TRACE + tools/gpu/ws_trace.py). Each generator
// thread draws its ILP pairs side by side (box_muller_bits<P>): 2.66 -> 2.55 ms at
// c1; constant draws (-DCQR_WS_FAKEGEN) bound the kernel at 1.89 ms.
#ifndef CQR_WS_STAGES
#define CQR_WS_STAGES 3
#endif
#ifndef CQR_WS_GEN
#define CQR_WS_GEN 8
#endif
constexpr int kWsStages = CQR_WS_STAGES;
constexpr int kWsGen = CQR_WS_GEN;
#ifndef CQR_WS_ILP
#define CQR_WS_ILP 4
#endif
constexpr int kWsIlp = CQR_WS_ILP;
#ifndef CQR_WS_MMA
#define CQR_WS_MMA 8
#endif
constexpr int kWsMma = CQR_WS_MMA;
// n <= 64 (NPC = 64: each drawn entry feeds only 64 columns) draws with 16 generator warps,
// 2 pairs side by side (c3 shape: 0.923 -> 0.850 ms at m = 1e6); wider A keeps 8 x 4.
#ifndef CQR_WS_GEN256
#define CQR_WS_GEN256 kWsGen
#endif
#ifndef CQR_WS_MMA256
#define CQR_WS_MMA256 kWsMma
#endif
#ifndef CQR_WS_GEN64
#define CQR_WS_GEN64 16
#endif
#ifndef CQR_WS_ILP64
#define CQR_WS_ILP64 2
#endif
template <int NPC>
constexpr int ws_gen() {
  return NPC == 64 ? CQR_WS_GEN64 : NPC == 256 ? CQR_WS_GEN256 : kWsGen;
}
template <int NPC>
constexpr int ws_ilp() {
  return NPC == 64 ? CQR_WS_ILP64 : kWsIlp;
}
template <int NPC>
constexpr int ws_mma() {
  return NPC == 256 ? CQR_WS_MMA256 : kWsMma;
}
template <int NPC>
constexpr int ws_threads() {
  return (ws_gen<NPC>() + ws_mma<NPC>()) * 32;
}

// NPC columns of A per CTA (128, or 256 for wider A with 32 Omega rows per CTA so
// that each drawn Omega entry feeds twice the DMMA work), ST Omega rows per CTA.
#ifdef CQR_WS_TRACE  // probe: per-warp step timeline of CTA 0 (read with cqr_debug_trace)
constexpr int kTraceSteps = 64;
__device__ long long g_trace[16 * kTraceSteps * 2];
#endif

template <int NPC, int ST>
struct WsShape {
  // A tile boxes: 8 columns (64-byte rows: a fragment's four rows fall in alternating bank halves,
  // two wavefronts) for NPC = 64 (0.851 -> 0.832 ms at m = 1e6); wider tiles keep 16-column
  // SWIZZLE_128B boxes (narrow boxes: 2.515 -> 2.52 ms at n = 128, 8.97 -> 9.14 at n = 256)
  static constexpr int BW = NPC <= 64 ? 8 : 16;
  static constexpr int ATILE = kKS * NPC;       // doubles per A stage (NPC/BW boxes of 32 x BW)
  static constexpr int OTILE = ST * (kKS + 4);  // doubles per Omega stage (stride 36)
  static constexpr int MMA = ws_mma<NPC>();
  static constexpr int NGW = NPC / (8 * MMA);  // 8-column groups per MMA warp
  static constexpr int MGW = ST / 8;            // 8-row groups per MMA warp
  static constexpr int GEN = ws_gen<NPC>();
  static constexpr int PAIRS = ST * kKS / 2 / (GEN * 32);  // Box-Muller pairs per generator thread per step
  static constexpr int ILP = PAIRS < ws_ilp<NPC>() ? PAIRS : ws_ilp<NPC>();  // pairs drawn side by side
  static constexpr size_t SMEM = (size_t)kWsStages * (ATILE + OTILE) * sizeof(double) + 1024;
};

template <int NPC, int ST>
__global__ void __launch_bounds__(ws_threads<NPC>(), 1)
    sketch_ws_kernel(const __grid_constant__ CUtensorMap tma_a, long long m_local, long long m_global, long long row0,
                     int l, uint64_t seed, long long rows_per_chunk, double* __restrict__ partial, int lp,
                     int np_total, int check, int y0, int tma3, DevStatus* st) {
  using S = WsShape<NPC, ST>;
  constexpr int LDO = kKS + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BmTables T;
  __shared__ __align__(8) uint64_t full[kWsStages], empty[kWsStages];
  if (failed(st)) return;
  double* sm = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* sA = sm;                            // [stage][box][32 rows][BW cols]
  double* sO = sm + kWsStages * S::ATILE;     // [stage][ST][36]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s0 = blockIdx.x * ST;
  const int ky = blockIdx.y + y0;
  const int col0 = blockIdx.z * NPC;
  const long long k_begin = (long long)ky * rows_per_chunk;
  const long long k_end = min(m_local, k_begin + rows_per_chunk);
  const int nsteps = k_end > k_begin ? (int)((k_end - k_begin + kKS - 1) / kKS) : 0;
  {
    const double* src = reinterpret_cast<const double*>(&c_bm);
    double* dst = reinterpret_cast<double*>(&T);
    for (int e = tid; e < (int)(sizeof(BmTables) / sizeof(double)); e += ws_threads<NPC>()) dst[e] = src[e];
  }
  if (tid == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], S::GEN * 32 + 1);  // every generator thread + the TMA issuer's expect_tx
      mbar_init(&empty[s], S::MMA);          // one elected lane per MMA warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  __syncthreads();
  if (warp >= S::MMA) {
    // ---- generator warps: Omega tiles + the A tile's TMA
    const int gt = tid - S::MMA * 32;
    // Counter state of each of this thread's pairs: pair p = (c >> 1) + pp with c = (s0 + i) m_global
    // + row0 + k (even: m_global, row0 and the chunk starts are even), so from one step to the next
    // p grows by kKS/2 and the pair's first counter word seed + (2p + 1) G by kKS G.
    const bool all_live = s0 + ST <= l;
    uint64_t z[S::PAIRS];
#pragma unroll
    for (int u = 0; u < S::PAIRS; ++u) {
      const int e = gt + S::GEN * 32 * u;
      const unsigned long long c0 = (unsigned long long)(s0 + (e >> 4)) * (unsigned long long)m_global + row0 + k_begin;
      z[u] = seed + (2 * ((c0 >> 1) + (e & 15)) + 1) * kGolden;
    }
    for (int stp = 0; stp < nsteps; ++stp) {
      const int s = stp % kWsStages;
      mbar_wait(&empty[s], ((stp / kWsStages) & 1) ^ 1);
#ifdef CQR_WS_TRACE
      if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && stp < kTraceSteps) g_trace[(warp * kTraceSteps + stp) * 2] = clock64();
#endif
      const long long kb = k_begin + (long long)stp * kKS;
      if (gt == 0) {
        mbar_expect_tx(&full[s], S::ATILE * 8);
        if (tma3) {  // all NPC/BW column boxes in one 3-D load
          tma_load_3d(sA + s * S::ATILE, &tma_a, 0, (int)kb, col0 / S::BW, &full[s]);
        } else {
#pragma unroll
          for (int b = 0; b < NPC / S::BW; ++b)
            tma_load_2d(sA + s * S::ATILE + b * (kKS * S::BW), &tma_a, col0 + S::BW * b, (int)kb, &full[s]);
        }
      }
      double* Om = sO + s * S::OTILE;
#pragma unroll
      for (int u0 = 0; u0 < S::PAIRS; u0 += S::ILP) {
        uint64_t zz[S::ILP];
        double ge[S::ILP], go[S::ILP];
#pragma unroll
        for (int j = 0; j < S::ILP; ++j) {
          zz[j] = z[u0 + j];
          z[u0 + j] += (uint64_t)kKS * kGolden;
        }
#ifdef CQR_WS_FAKEGEN  // probe: constant draws (the MMA-side bound of this kernel)
#pragma unroll
        for (int j = 0; j < S::ILP; ++j) ge[j] = (double)(zz[j] & 255) * 0x1.0p-8, go[j] = 0.5;
#else
        gaussian_pairs_z<S::ILP>(T, zz, ge, go);
#endif
#pragma unroll
        for (int j = 0; j < S::ILP; ++j) {
          const int e = gt + S::GEN * 32 * (u0 + j);
          const int i = e >> 4, pp = e & 15;
          if (!all_live && s0 + i >= l) ge[j] = go[j] = 0.0;  // Omega rows past l (last s-tile only)
          *reinterpret_cast<double2*>(Om + i * LDO + 2 * pp) = make_double2(ge[j], go[j]);
        }
      }
#ifdef CQR_WS_TRACE
      if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && stp < kTraceSteps) g_trace[(warp * kTraceSteps + stp) * 2 + 1] = clock64();
#endif
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
    return;
  }
  // ---- MMA warps: all ST Omega rows x NPC/8 columns each
  const int q = lane & 3, gr = lane >> 2;
  double acc[S::MGW][S::NGW][2];
#pragma unroll
  for (int g = 0; g < S::MGW; ++g)
#pragma unroll
    for (int h = 0; h < S::NGW; ++h) acc[g][h][0] = acc[g][h][1] = 0.0;
  bool bad = false;
  for (int stp = 0; stp < nsteps; ++stp) {
    const int s = stp % kWsStages;
    mbar_wait(&full[s], (stp / kWsStages) & 1);
#ifdef CQR_WS_TRACE
    if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && stp < kTraceSteps) g_trace[(warp * kTraceSteps + stp) * 2] = clock64();
#endif
    const double* Om = sO + s * S::OTILE + gr * LDO + q;
    const double* As = sA + s * S::ATILE;
#ifdef CQR_WS_NOMMA  // probe: generator-only throughput (the MMA warps just cycle the ring)
    if (nsteps > 0) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      continue;
    }
#endif
#pragma unroll
    for (int k4 = 0; k4 < kKS / 4; ++k4) {
      const int r = 4 * k4 + q;
      double af[S::MGW], bf[S::NGW];
#pragma unroll
      for (int g = 0; g < S::MGW; ++g) af[g] = Om[g * 8 * LDO + 4 * k4];
#pragma unroll
      for (int h = 0; h < S::NGW; ++h) {
        const int cg = warp * S::NGW + h;  // 8-column group: box cg (BW = 8) or box cg/2, half cg&1
        if constexpr (S::BW == 8)
          bf[h] = As[cg * (kKS * 8) + r * 8 + gr];
        else
          bf[h] = As[(cg >> 1) * (kKS * 16) + r * 16 + 2 * ((4 * (cg & 1) + (gr >> 1)) ^ (r & 7)) + (gr & 1)];
        bad |= nonfinite(bf[h]);
      }
#pragma unroll
      for (int g = 0; g < S::MGW; ++g)
#pragma unroll
        for (int h = 0; h < S::NGW; ++h) dmma(acc[g][h][0], acc[g][h][1], af[g], bf[h]);
    }
    __syncwarp();
#ifdef CQR_WS_TRACE
    if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && stp < kTraceSteps) g_trace[(warp * kTraceSteps + stp) * 2 + 1] = clock64();
#endif
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
  if (check && __any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  double* out = partial + (long long)ky * lp * np_total + col0;
#pragma unroll
  for (int g = 0; g < S::MGW; ++g) {
    const int i = s0 + g * 8 + gr;
#pragma unroll
    for (int h = 0; h < S::NGW; ++h) {
      const int j = (warp * S::NGW + h) * 8 + 2 * q;
      *reinterpret_cast<double2*>(out + (long long)i * np_total + j) = make_double2(acc[g][h][0], acc[g][h][1]);
    }
  }
}

template <int NPC, int ST>
cudaError_t launch_ws(const SketchPlan& p, const double* a, long long lda, long long m_global, long long row0,
                      uint64_t seed, double* partial, int check, const DevStatus* st, cudaStream_t s, int y0,
                      int y1) {
  CUtensorMap tm;
  static const bool no3d = std::getenv("CQR_SKETCH_TMA2D") != nullptr;  // tuning: per-box 2-D loads
  constexpr int BW = WsShape<NPC, ST>::BW;
  constexpr CUtensorMapSwizzle SW = BW == 8 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B;
  const int tma3 = !no3d && p.n % BW == 0 && p.np % NPC == 0 &&
                   make_tmap_colblocks(&tm, a, p.n, p.m_local, lda, kKS, NPC / BW, SW, BW);
  if (!tma3 && !make_tmap_2d(&tm, a, p.n, p.m_local, lda, BW, kKS, SW)) return cudaErrorInvalidValue;
  auto k = sketch_ws_kernel<NPC, ST>;
  cudaError_t e =
      allow_max_smem(k);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)p.s_tiles, (unsigned)(y1 - y0), (unsigned)(p.np / NPC));
  k<<<grid, ws_threads<NPC>(), WsShape<NPC, ST>::SMEM, s>>>(tm, p.m_local, m_global, row0, p.l, seed, p.rows_per_chunk,
                                                      partial, p.lp, p.np, check, y0, tma3,
                                                      const_cast<DevStatus*>(st));
  return cudaGetLastError();
}

__global__ void sketch_reduce_kernel(const double* __restrict__ partial, int kchunks, int lp, int np, int l,
                                     int n, double* __restrict__ a1, const DevStatus* st) {
  if (failed(st)) return;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)l * n) return;
  const int i = (int)(e / n), c = (int)(e - (long long)i * n);
  const double* p = partial + (long long)i * np + c;
  const long long stride = (long long)lp * np;
  // the sum stays in k order (a fixed order: run-to-run identical); only the loads run ahead, 16 in flight
  double s = 0.0;
  int k = 0;
  for (; k + 16 <= kchunks; k += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(p + (k + u) * stride);
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u];
  }
  for (; k < kchunks; ++k) s += __ldg(p + k * stride);
  a1[e] = s;
}

__global__ void gather_rows_kernel(const double* __restrict__ a, long long lda, long long m_local,
                                   long long m_global, long long row0, int n, int l, uint64_t seed,
                                   const long long* __restrict__ idx_in, double* __restrict__ a1,
                                   long long* __restrict__ idx_out, const DevStatus* st) {
  if (failed(st)) return;
  const int k = blockIdx.x;
  long long idx;
  if (idx_in) {
    idx = idx_in[k];
  } else {
    const double u = (double)(bits_at(seed, (uint64_t)k) >> 11) * 0x1.0p-53;  // Stream(seed).next_index, rng.hpp:69-71
    idx = (long long)(u * (double)m_global);
  }
  if (idx_out && threadIdx.x == 0) idx_out[k] = idx;
  const long long loc = idx - row0;
  const bool mine = loc >= 0 && loc < m_local;
  for (int c = threadIdx.x; c < n; c += blockDim.x) a1[(long long)k * n + c] = mine ? a[loc * lda + c] : 0.0;
}

__global__ void rng_bits_kernel(uint64_t seed, uint64_t k0, long long count, uint64_t* out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = bits_at(seed, k0 + (uint64_t)e);
}

// The same Box-Muller code as the sketch kernel (the parity tests compare it to glibc).
__global__ void rng_gauss_kernel(uint64_t seed, uint64_t k0, long long count, double* out) {
  __shared__ BmTables T;
  {
    const double* src = reinterpret_cast<const double*>(&c_bm);
    double* dst = reinterpret_cast<double*>(&T);
    for (int e = threadIdx.x; e < (int)(sizeof(BmTables) / sizeof(double)); e += blockDim.x) dst[e] = src[e];
  }
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    const uint64_t k = k0 + (uint64_t)e;
    double ge, go;
    gaussian_pair_fast(T, seed, k >> 1, ge, go);
    out[e] = (k & 1) ? go : ge;
  }
}

// The Box-Muller tables are uploaded once per device, ordered on the launching
// stream (a non-blocking stream is not ordered after the legacy stream) and
// completed before any kernel is allowed to read them.
cudaError_t ensure_tables(cudaStream_t s) {
  static std::mutex mu;
  static unsigned long long done = 0;  // bit per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (dev < 64 && (done >> dev) & 1ull) return cudaSuccess;
  BmTables t;
  bm_tables_host(&t);
  e = cudaMemcpyToSymbolAsync(c_bm, &t, sizeof(t), 0, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && dev < 64) done |= 1ull << dev;
  return e;
}

template <int NP>
cudaError_t launch_sketch_t(const SketchPlan& p, const double* a, long long lda, long long m_global, long long row0,
                            uint64_t seed, double* partial, int vec16, int check, const DevStatus* st,
                            cudaStream_t s, int y0, int y1) {
  if (y1 < 0) y1 = p.kchunks;
  if (y1 <= y0) return cudaSuccess;
  cudaError_t e0 = ensure_tables(s);
  if (e0 != cudaSuccess) return e0;
  const size_t smem = (size_t)(2 * kST * (kKS + 4) + 2 * kKS * (NP + 4)) * sizeof(double);
  const bool aligned = (m_global % 2 == 0) && (row0 % 2 == 0) && (p.rows_per_chunk % 2 == 0);
  if (!aligned) {
    auto k = sketch_kernel<NP, false>;
    cudaError_t e = allow_max_smem(k);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)p.s_tiles, (unsigned)(y1 - y0), (unsigned)(p.np / NP));
    k<<<grid, kThreads, smem, s>>>(a, lda, p.m_local, m_global, row0, p.n, p.l, seed, p.rows_per_chunk, partial,
                                   p.lp, p.np, vec16, check, y0, const_cast<DevStatus*>(st));
    return cudaGetLastError();
  }
  auto k = sketch_kernel<NP, true>;
  cudaError_t e = allow_max_smem(k);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)p.s_tiles, (unsigned)(y1 - y0), (unsigned)(p.np / NP));
  k<<<grid, kThreads, smem, s>>>(a, lda, p.m_local, m_global, row0, p.n, p.l, seed, p.rows_per_chunk, partial, p.lp,
                                 p.np, vec16, check, y0, const_cast<DevStatus*>(st));
  return cudaGetLastError();
}

}  // namespace

#ifdef CQR_WS_TRACE
extern "C" int cqr_debug_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
}
#endif

void bm_tables_host(BmTables* t) {
  for (int i = 0; i < kBmLog; ++i) {
    const long double c = 1.0L + (long double)(i + kBmLogLo) / 256.0L;  // exact; c = 1 at i = -kBmLogLo
    const double inv = (double)(1.0L / c);
    const long double v = 0.0L - logl((long double)inv);  // +0 for inv = 1
    t->inv[i] = inv;
    t->lhi[i] = (double)v;
    t->llo[i] = (double)(v - (long double)t->lhi[i]);
  }
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int m = 0; m <= kBmTrig / 4; ++m) t->q[m] = (double)sinl(two_pi * (long double)m / kBmTrig);
}

bool sketch_ws_ok(const double* a, long long lda, long long m_global, long long row0, int n) {
  static const bool off = std::getenv("CQR_SKETCH_LEGACY") != nullptr;  // tuning: force the interleaved kernel
  if (off || n <= 32 || n > 512 || (m_global & 1) || (row0 & 1) || m_global > (1LL << 31) - 64) return false;
  CUtensorMap probe;
  return make_tmap_2d(&probe, a, n, std::max<long long>(1, m_global), lda, 8, kKS, CU_TENSOR_MAP_SWIZZLE_NONE);
}

SketchPlan sketch_plan(long long m_local, int n, int l, int num_sms, bool ws_ok, int splits) {
  SketchPlan p;
  p.n = n;
  p.l = l;
  p.np = sketch_np(n);
  p.m_local = m_local;
  // interleaved kernel: about 2 resident CTAs per SM over 2 waves; warp-specialised:
  // one CTA per SM, one wave (n = 128: 64 Omega rows x 128 columns per CTA; wider:
  // 32 Omega rows x 256 columns). Chunks are multiples of KS rows.
  p.ws = ws_ok && p.np >= 64 ? 1 : 0;
  p.st = !p.ws ? kST : p.np == 64 ? 128 : p.np == 128 ? 64 : 32;  // Omega rows per CTA: DMMA work per draw
  p.npc = p.ws ? std::min(p.np, 256) : std::min(p.np, 128);
  p.s_tiles = (l + p.st - 1) / p.st;
  p.lp = p.s_tiles * p.st;
  const long long target = (long long)num_sms * (p.ws ? std::max(1, splits) : 4);
  const int zparts = p.np / p.npc;
  // warp-specialised: whole waves (round down), the interleaved kernel: round up
  const long long per = (long long)p.s_tiles * zparts;
  long long kc = p.ws ? target / per : (target + per - 1) / per;
  const long long max_kc = (m_local + kKS - 1) / kKS;
  if (kc > max_kc) kc = max_kc;
  if (kc < 1) kc = 1;
  long long rpc = (m_local + kc - 1) / kc;
  rpc = (rpc + kKS - 1) / kKS * kKS;
  if (rpc < kKS) rpc = kKS;
  p.rows_per_chunk = rpc;
  p.kchunks = (int)((m_local + rpc - 1) / rpc);
  if (p.kchunks < 1) p.kchunks = 1;
  p.partial_doubles = (size_t)p.kchunks * p.lp * p.np;
  return p;
}

cudaError_t launch_sketch_gaussian(const SketchPlan& p, const double* a, long long lda, long long m_global,
                                   long long row0, uint64_t seed, double* partial, int vec16, int check,
                                   const DevStatus* st, cudaStream_t s, int y0, int y1) {
  if (p.ws) {
    if (y1 < 0) y1 = p.kchunks;
    if (y1 <= y0) return cudaSuccess;
    cudaError_t e0 = ensure_tables(s);
    if (e0 != cudaSuccess) return e0;
    if (p.npc == 64) return launch_ws<64, 128>(p, a, lda, m_global, row0, seed, partial, check, st, s, y0, y1);
    if (p.npc == 128) return launch_ws<128, kST>(p, a, lda, m_global, row0, seed, partial, check, st, s, y0, y1);
    return launch_ws<256, 32>(p, a, lda, m_global, row0, seed, partial, check, st, s, y0, y1);
  }
  switch (p.np) {
    case 8: return launch_sketch_t<8>(p, a, lda, m_global, row0, seed, partial, vec16, check, st, s, y0, y1);
    case 16: return launch_sketch_t<16>(p, a, lda, m_global, row0, seed, partial, vec16, check, st, s, y0, y1);
    case 32: return launch_sketch_t<32>(p, a, lda, m_global, row0, seed, partial, vec16, check, st, s, y0, y1);
    case 64: return launch_sketch_t<64>(p, a, lda, m_global, row0, seed, partial, vec16, check, st, s, y0, y1);
    case 128: return launch_sketch_t<128>(p, a, lda, m_global, row0, seed, partial, vec16, check, st, s, y0, y1);
    case 256:
    case 512: return launch_sketch_t<128>(p, a, lda, m_global, row0, seed, partial, vec16, check, st, s, y0, y1);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_sketch_reduce(const SketchPlan& p, const double* partial, double* a1, const DevStatus* st,
                                 cudaStream_t s) {
  const long long total = (long long)p.l * p.n;
  sketch_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(partial, p.kchunks, p.lp, p.np, p.l, p.n,
                                                                       a1, st);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* a, long long lda, long long m_local, long long m_global, long long row0,
                               int n, int l, uint64_t seed, const long long* idx_dev, double* a1, long long* idx_out,
                               const DevStatus* st, cudaStream_t s) {
  gather_rows_kernel<<<(unsigned)l, 128, 0, s>>>(a, lda, m_local, m_global, row0, n, l, seed, idx_dev, a1, idx_out,
                                                 st);
  return cudaGetLastError();
}

cudaError_t launch_rng_bits(uint64_t seed, uint64_t k0, long long count, uint64_t* out, cudaStream_t s) {
  rng_bits_kernel<<<256, 256, 0, s>>>(seed, k0, count, out);
  return cudaGetLastError();
}

// Box-Muller on given counter bits (bits[2i] -> u1, bits[2i+1] -> u2): out[2i] = r cos a,
// out[2i+1] = r sin a. Drives the edge cases (u1 -> 1, table and quadrant boundaries) in tests.
__global__ void box_muller_bits_kernel(const uint64_t* __restrict__ bits, long long pairs, double* __restrict__ out) {
  __shared__ BmTables T;
  {
    const double* src = reinterpret_cast<const double*>(&c_bm);
    double* dst = reinterpret_cast<double*>(&T);
    for (int e = threadIdx.x; e < (int)(sizeof(BmTables) / sizeof(double)); e += blockDim.x) dst[e] = src[e];
  }
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < pairs;
       e += (long long)gridDim.x * blockDim.x) {
    const uint64_t b1[1] = {bits[2 * e]}, b2[1] = {bits[2 * e + 1]};
    double ge[1], go[1];
    box_muller_bits<1>(T, b1, b2, ge, go);
    out[2 * e] = ge[0];
    out[2 * e + 1] = go[0];
  }
}

cudaError_t launch_box_muller_bits(const uint64_t* bits, long long pairs, double* out, cudaStream_t s) {
  cudaError_t e = ensure_tables(s);
  if (e != cudaSuccess) return e;
  box_muller_bits_kernel<<<148, 256, 0, s>>>(bits, pairs, out);
  return cudaGetLastError();
}

cudaError_t launch_rng_gaussian(uint64_t seed, uint64_t k0, long long count, double* out, cudaStream_t s) {
  cudaError_t e = ensure_tables(s);
  if (e != cudaSuccess) return e;
  rng_gauss_kernel<<<256, 256, 0, s>>>(seed, k0, count, out);
  return cudaGetLastError();
}

}  // namespace cqr
