// sketch_i8.cu — the Gaussian sketch A1 = Omega A (sketch.cpp:94-116) as an exact integer product on
// the 5th-generation tensor cores (tcgen05.mma kind::i8, s32 accumulators in TMEM).
//
// FP64 has no tcgen05 kind; DMMA (sketch.cu) tops out at 37 TFLOP/s and shares its pipe with the
// Box-Muller draws. Here both operands become 56-bit fixed-point integers cut into 7 signed byte digits
// ("Ozaki" splitting):
//   Omega(i,k) = N_ik 2^-51,        N_ik = round(w 2^51),          |N| < 2^55 (|w| < 9 for every draw);
//   A(k,j)     = M_kj 2^(E_j - 54), M_kj = round(a 2^(54 - E_j)),  |M| < 2^54,
// E_j the exponent bound of column j over the current sub-chunk of the CTA's rows (max |a| < 2^E_j), found by
// scanner warps of this kernel one sub-chunk ahead (they also check finiteness). The digits are balanced: N = sum_s D_s 2^(8(6-s)) with every D_s in [-128, 127],
// read off the bytes of N + 0x808080808080 (the lower six bytes with their top bit flipped), so the
// dropped low-order products are zero-mean and do not drift with K. The 28 digit products with
// s + t <= 6 accumulate per level u = s + t in TMEM -- exactly: |level| <= 7 * 128^2 * K < 2^31 for
// k-chunks of <= 16384 rows -- and the epilogue recombines sum_u ACC_u 2^(8(6-u)) in 64-bit integers,
// converts (two roundings) and scales by 2^(E_j - 57). The dropped levels weigh <= 2^-56 of the leading
// one: as accurate as an FP64 GEMM (tests: <= 1e-13 against the oracle's sequential fma chains). Omega
// is still the reference's gaussian_at(seed, i*m + k), draw for draw (boxmuller.cuh); it never touches
// HBM.
//
// Warp roles (one CTA per SM, 128 Omega rows x 64 columns of A x one k-chunk):
//   warp 0      TMEM allocation; lane 0 issues the 10 MMAs of each 32-row step (M=128, N<=256, K=32)
//               and commits them to the stages' `empty` barriers (Omega planes and A planes are two rings);
//   warp 1      lane 0 streams A's FP64 rows (32 x 64 tiles) by TMA into its own ring;
//   warps 2-5   cut A's tile into the 7 digit planes (K-major core-matrix layout, SWIZZLE_NONE: one exact
//               scaling, conversion, four 4x4 byte transposes per 8 entries) and run the epilogue of every
//               sub-chunk (each warp one TMEM lane quadrant);
//   next 16     (12 for clusters of 8) draw Omega (Box-Muller pairs, 4 side by side, in teams that take
//               alternate steps) and cut each draw into its digit planes; with a cluster each CTA draws its
//               share of the rows and ships it to the partners by bulk copies;
//   last 4      scan the next sub-chunk's column exponent bounds (and finiteness) from A's high words.
// The kernel is bound by the SM's issue rate for this mix (profiles/r04_sketch_probes.txt): its time follows the
// generators' and slicers' instruction counts, hence the care for every prmt and xor below.

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "boxmuller.cuh"
#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace cqr {

namespace {

constexpr int kI8Rows = 128;      // Omega rows per CTA (MMA M)
constexpr int kI8Cols = 64;       // A columns per CTA (MMA N)
constexpr int kI8K = 32;          // rows of A per step (MMA K for kind::i8)
// ring depths per cluster size C (digit-plane stages S, FP64 A stages AS; S >= generator teams, smem
// S 42 KB + AS 16 KB <= 218 KB): C = 1 (c3) S 3 AS 4: 2.65 vs 2.70 ms (S 4 AS 2); C = 2 (c1) S 4 AS 3: 1.77 vs 1.80;
// C = 4, 8 (c2, c4) S 4 AS 3: 23.79 / 16.32 vs 23.98 / 16.40 ms (AS 2)
// r04: the Omega planes (28 KB per stage) and A's digit planes (14 KB) are separate rings of S and P stages: a
// generator team owns every teams-th step, and with S = teams its next step had to wait for the MMAs of its
// previous one (ncu: 35% of the generators' samples at c1 sat in that wait); S > teams gives a step of slack.
#ifndef CQR_I8_S1
#define CQR_I8_S1 4
#endif
#ifndef CQR_I8_P1
#define CQR_I8_P1 3
#endif
#ifndef CQR_I8_AS1
#define CQR_I8_AS1 3
#endif
#ifndef CQR_I8_S2
#define CQR_I8_S2 4
#endif
#ifndef CQR_I8_P2
#define CQR_I8_P2 4
#endif
#ifndef CQR_I8_AS2
#define CQR_I8_AS2 3
#endif
#ifndef CQR_I8_S4
#define CQR_I8_S4 4
#endif
#ifndef CQR_I8_P4
#define CQR_I8_P4 4
#endif
#ifndef CQR_I8_AS4
#define CQR_I8_AS4 3
#endif
#ifndef CQR_I8_S8
#define CQR_I8_S8 4
#endif
#ifndef CQR_I8_P8
#define CQR_I8_P8 4
#endif
#ifndef CQR_I8_AS8
#define CQR_I8_AS8 3
#endif
#ifndef CQR_I8_GEN
#define CQR_I8_GEN 16
#endif
#ifndef CQR_I8_GEN8
#define CQR_I8_GEN8 12  // generator warps for clusters of 8 (c4: 12 vs 16 warps 17.0 vs 18.6 ms)
#endif
#ifndef CQR_I8_SLEEP_NS
#define CQR_I8_SLEEP_NS 100
#endif
#ifndef CQR_I8_SLICE
#define CQR_I8_SLICE 4
#endif
constexpr int kI8Slice = CQR_I8_SLICE;  // slicer warps (the first four also run the epilogue)
constexpr long long kI8MaxChunk = 16384;  // rows per k-chunk: 7 * 128^2 * 16384 < 2^31
constexpr int kDig = 7;                 // byte digits per operand
constexpr int kOmPlane = kI8Rows * kI8K;  // bytes per Omega digit plane (4 KB)
constexpr int kAPlane = kI8Cols * kI8K;   // bytes per A digit plane (2 KB)
constexpr int kOmStage = kDig * kOmPlane;  // 28 KB
constexpr int kApStage = kDig * kAPlane;   // 14 KB
constexpr int kATile = kI8K * kI8Cols;    // doubles per FP64 A stage
__host__ __device__ constexpr size_t i8_smem(int stages, int pstages, int astages) {
  return (size_t)stages * kOmStage + (size_t)pstages * kApStage + (size_t)astages * kATile * 8 + 1024;
}

__constant__ BmTablesX c_bm_i8;  // full-circle sine table: no quadrant arithmetic in the draws

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t sbo = 256) {
  // K-major, SWIZZLE_NONE: 8-row x 16-byte core matrices, LBO = 128 B (the two K halves), SBO = the stride
  // between 8-row groups (256 B when a plane's row groups are consecutive)
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46);
}
// Omega planes, row-group-major: an 8-row group holds its 256-byte core-matrix pair of every digit plane
// (1792 B), so the rows one CTA of a cluster draws are ONE contiguous chunk across all planes
constexpr int kOmGroup = 7 * 256;
// s32 accumulator, M = 128, N columns, K-major s8 operands
__host__ __device__ constexpr uint32_t idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kI8Rows >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// every CTA of the cluster (ctaMask) gets one arrival on its barrier at this smem offset
__device__ __forceinline__ void umma_commit_cluster(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// shared::cta -> another CTA's shared memory (shared::cluster address), completing on that CTA's barrier
__device__ __forceinline__ void bulk_copy_cluster(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                                  uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// a wait that backs off: producers and the epilogue park here for long stretches, and a tight try_wait loop
// would burn the issue slots the generator warps need
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#ifndef CQR_I8_NOSLEEP
  while (!mbar_try_wait(bar, parity)) __nanosleep(CQR_I8_SLEEP_NS);
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// byte offset of element (r, k) (k < 32) of an R-row K-major digit plane
__device__ __forceinline__ int plane_off(int r, int k) {
  return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}
// the same element in the row-group-major Omega planes (plane p at + p * 256)
__device__ __forceinline__ int om_off(int r, int k) {
  return (r >> 3) * kOmGroup + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

// 8 consecutive entries (k = 8o .. 8o+7 of one row) as 64-bit two's complement integers (lo, hi words)
// -> digit plane s (byte 6 - s) receives the 8 bytes [entry 0 .. entry 7] at plane s + off: an 8x7
// byte transpose as four 4x4 byte transposes (two prmt stages each: 30 prmt, 3 per stored word pair;
// a per-plane gather took 42)
__device__ __forceinline__ void transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&t)[4],
                                           bool need3) {
  const uint32_t a0 = __byte_perm(w0, w1, 0x5140u), a2 = __byte_perm(w2, w3, 0x5140u);  // bytes 0, 1 of each pair
  const uint32_t a1 = __byte_perm(w0, w1, 0x7362u), a3 = __byte_perm(w2, w3, 0x7362u);  // bytes 2, 3
  t[0] = __byte_perm(a0, a2, 0x5410u);  // byte 0 of w0..w3
  t[1] = __byte_perm(a0, a2, 0x7632u);  // byte 1
  t[2] = __byte_perm(a1, a3, 0x5410u);  // byte 2
  t[3] = need3 ? __byte_perm(a1, a3, 0x7632u) : 0u;  // byte 3 (byte 7 of an entry is not a digit)
}
__device__ __forceinline__ void transpose_store(const uint32_t (&lo)[8], const uint32_t (&hi)[8],
                                                unsigned char* planes, int plane_bytes, int off) {
  uint32_t la[4], lb[4], ha[4], hb[4];  // bytes 0-3 (lo) and 4-7 (hi) of entries 0-3 (a) and 4-7 (b)
  transpose4(lo[0], lo[1], lo[2], lo[3], la, true);
  transpose4(lo[4], lo[5], lo[6], lo[7], lb, true);
  transpose4(hi[0], hi[1], hi[2], hi[3], ha, false);
  transpose4(hi[4], hi[5], hi[6], hi[7], hb, false);
#pragma unroll
  for (int s = 0; s < kDig; ++s) {
    const int b = 6 - s;
    // the lower six digits are balanced by flipping each byte's top bit (split64 leaves that to the planes:
    // 12 xors per 8 entries here instead of 16 there)
    *reinterpret_cast<uint2*>(planes + s * plane_bytes + off) =
        b < 4   ? make_uint2(la[b] ^ 0x80808080u, lb[b] ^ 0x80808080u)
        : b < 6 ? make_uint2(ha[b - 4] ^ 0x80808080u, hb[b - 4] ^ 0x80808080u)
                : make_uint2(ha[2], hb[2]);
  }
}

// balanced byte digits of v (|v| < 2^55 - 2^48): the bytes of v + 0x808080808080, the lower six with
// their top bit flipped (byte - 128), the top one as is
__device__ __forceinline__ void split64(long long v, uint32_t& lo, uint32_t& hi) {
  const unsigned long long w = (unsigned long long)v + 0x0000808080808080ull;
  lo = (uint32_t)w;  // the top-bit flips of the lower six bytes are applied to the transposed planes
  hi = (uint32_t)(w >> 32);
}

// Generator teams: with C CTAs sharing an Omega tile each CTA draws 1/C of it per step, too little work to
// hide one thread's Box-Muller latency; T teams then take every T-th step, so T steps are drawn at once.
#ifndef CQR_I8_TEAMS2
#define CQR_I8_TEAMS2 4  // clusters of 2 (c1): 2/4 teams 1.89/1.80 ms
#endif
#ifndef CQR_I8_TEAMS4
#define CQR_I8_TEAMS4 4  // clusters of 4/8 (c2/c4): 2 teams 24.6/16.8 ms vs 4 teams 24.0/16.4 (<= 7: bar ids 1..7)
#endif
#ifndef CQR_I8_TEAMS1
#define CQR_I8_TEAMS1 4  // no cluster (c3): 1/2/4 teams 2.652/2.622/2.614 ms (4 teams: S 4, P 3, AS 3)
#endif
__host__ __device__ constexpr int gen_teams(int ncta) {
  return ncta >= 4 ? CQR_I8_TEAMS4 : ncta == 2 ? CQR_I8_TEAMS2 : CQR_I8_TEAMS1;
}

// Sub-chunks: a CTA's rows [k_begin, k_end) are accumulated in TMEM in sub-chunks of kSubFirst, 4x, 16x ...
// steps (capped at 512 steps = kI8MaxChunk rows, the s32 exactness bound), each with its own column
// exponent bounds. The scanner warps find sub-chunk t+1's bounds while sub-chunk t is on the tensor cores
// (4x its rows in the same time: they read A at ~4x the MMA side's rate, L2-prefetched by TMA), so only the
// first, short sub-chunk's scan is exposed -- the separate exponent pre-pass over all of A is gone. Between
// sub-chunks the epilogue warps drain TMEM into the FP64 partial (+=), while the producers run ahead.
#ifndef CQR_I8_SUBGROW
#define CQR_I8_SUBGROW 2  // sub-chunk growth 2^CQR_I8_SUBGROW (x2: c1 1.90 ms, x4: 1.84)
#endif
#ifndef CQR_I8_SUBFIRST
#define CQR_I8_SUBFIRST 16
#endif
constexpr int kSubFirst = CQR_I8_SUBFIRST;  // steps (32 rows each) of a CTA's first sub-chunk
constexpr int kI8MaxSteps = (int)(kI8MaxChunk / kI8K);
__host__ __device__ constexpr int sub_steps(int t) {
  return t * CQR_I8_SUBGROW >= 5 ? kI8MaxSteps
                                 : (kSubFirst << (CQR_I8_SUBGROW * t)) < kI8MaxSteps ? (kSubFirst << (CQR_I8_SUBGROW * t))
                                                                                     : kI8MaxSteps;
}
#ifndef CQR_I8_SCAN
#define CQR_I8_SCAN 4
#endif
constexpr int kI8Scan = CQR_I8_SCAN;  // scanner warps (2 or 4; 4: c1 1.84 vs 1.99 ms at x4 growth)
constexpr int kExpSlots = 4;    // exponent-bound ring (sub-chunks in flight)
#ifndef CQR_I8_AHEAD
#define CQR_I8_AHEAD 6
#endif
constexpr int kScanAhead = CQR_I8_AHEAD;  // 32-row blocks prefetched into L2 ahead of the scan (0: none)

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

// GEN generator warps (16; 12 for clusters of 8 CTAs, where each CTA draws 1/8 of the tile: measured
// c4 17.0 vs 18.6 ms, every other config within noise or slower)
template <int GEN, int kI8Stages, int kI8PStages, int kI8AStages>
__global__ void __launch_bounds__((2 + kI8Slice + GEN + kI8Scan) * 32, 1)
    sketch_i8_kernel(const __grid_constant__ CUtensorMap tma_a, const double* __restrict__ a, long long lda,
                     long long m_local, long long m_global, long long row0, int l, int n, uint64_t seed,
                     long long rows_per_chunk, double* __restrict__ partial, int lp, int np_total, int y0,
                     DevStatus* st) {
  static_assert(kI8Slice == 4 || kI8Slice == 8, "warps 2-5 (the first four slicers) are the epilogue");
  constexpr int NTHR = (2 + kI8Slice + GEN + kI8Scan) * 32;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ BmTablesX T;
  __shared__ __align__(8) uint64_t full[kI8Stages], empty[kI8Stages], afull[kI8AStages], aempty[kI8AStages];
  __shared__ __align__(8) uint64_t pfull[kI8PStages], pempty[kI8PStages];
  __shared__ __align__(8) uint64_t subdone, tfree, expfull[kExpSlots];
  __shared__ uint32_t tmem_base;
  __shared__ int sexp[kExpSlots][kI8Cols];
  __shared__ unsigned sexpw[kI8Scan][kI8Cols];
  __shared__ int drained;
  if (failed(st)) return;
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sOm = sm;                                    // [stage][plane][4 KB]
  unsigned char* sAp = sm + kI8Stages * kOmStage;             // [pstage][plane][2 KB]
  double* sAf = reinterpret_cast<double*>(sm + kI8Stages * kOmStage + kI8PStages * kApStage);  // [astage][32 x 64]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s0 = blockIdx.x * kI8Rows;
  const int ky = blockIdx.y + y0;
  const int col0 = blockIdx.z * kI8Cols;
  // the column tiles of one (Omega tile, k-chunk) form a cluster (gridDim.z CTAs): CTA r draws Omega rows
  // [r 128 / C, (r + 1) 128 / C) once and stores their digits into every CTA's planes
  const int ncta = (int)gridDim.z, crank = (int)blockIdx.z;
  const long long k_begin = (long long)ky * rows_per_chunk;
  const long long k_end = min(m_local, k_begin + rows_per_chunk);
  const int nsteps = k_end > k_begin ? (int)((k_end - k_begin + kI8K - 1) / kI8K) : 0;
  {
    const double* src = reinterpret_cast<const double*>(&c_bm_i8);
    double* dst = reinterpret_cast<double*>(&T);
    for (int e = tid; e < (int)(sizeof(BmTablesX) / sizeof(double)); e += NTHR) dst[e] = src[e];
  }
  if (tid == 0) {
    for (int s = 0; s < kI8Stages; ++s) {
      // one generator team; the partners' Omega rows arrive as bulk-copy bytes (expect_tx)
      mbar_init(&full[s], GEN * 32 / gen_teams(ncta));
      mbar_init(&empty[s], ncta);                              // every CTA's MMAs have read the stage
    }
    for (int s = 0; s < kI8PStages; ++s) {
      mbar_init(&pfull[s], kI8Slice * 32);  // the slicers
      mbar_init(&pempty[s], 1);             // this CTA's MMAs have read A's digit planes
    }
    for (int s = 0; s < kI8AStages; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], kI8Slice * 32);
    }
    mbar_init(&subdone, 1);
    mbar_init(&tfree, 4 * 32);  // the four epilogue warps
    for (int s = 0; s < kExpSlots; ++s) mbar_init(&expfull[s], 32);
    drained = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();  // the partners' barriers are initialised before anyone arrives on them
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---- MMA issuer: per step, D[level s+t] += Omega digit s x A digit t (s + t <= 7)
    if (lane == 0) {
      int t = 0, t_end = sub_steps(0);  // current sub-chunk and its end step
      for (int stp = 0; stp < nsteps; ++stp) {
        const int s = stp % kI8Stages, sp = stp % kI8PStages;
        const bool first = stp == t_end - sub_steps(t);
        if (first && t > 0) mbar_wait(&tfree, (t - 1) & 1);  // the epilogue has drained sub-chunk t-1
        mbar_wait(&pfull[sp], (stp / kI8PStages) & 1);
        mbar_wait(&full[s], (stp / kI8Stages) & 1);  // partners' bulk copies included
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t om = smem_u32(sOm + s * kOmStage), ap = smem_u32(sAp + sp * kApStage);
#ifndef CQR_I8_NOMMA  // probe: the producers' bound (no MMAs)
        // Omega digit sd against the stacked A digit planes 0 .. 6-sd (consecutive 2 KB planes = one taller
        // K-major B operand): its N = 64 (7 - sd) output columns land on TMEM levels sd .. 6, i.e. on
        // columns [64 sd, 448) -- one or two MMAs (N <= 256) per Omega digit, 10 per step
#pragma unroll
        for (int sd = 0; sd < kDig; ++sd) {
          const uint32_t acc = (!first || sd > 0) ? 1u : 0u;  // sd = 0 of a sub-chunk's first step writes every level
          const uint64_t da = umma_sdesc(om + sd * 256, kOmGroup);
          const int nt = kDig - sd;                      // A digit planes 0 .. nt-1
          const int n1 = nt > 4 ? 4 : nt;                // first MMA: up to 4 planes (N <= 256)
          umma_i8(tmem + 64u * (uint32_t)sd, da, umma_sdesc(ap), idesc_i8(64 * n1), acc);
          if (nt > n1)
            umma_i8(tmem + 64u * (uint32_t)(sd + n1), da, umma_sdesc(ap + n1 * kAPlane), idesc_i8(64 * (nt - n1)), acc);
        }
#endif
        // the stage's smem (in every CTA of the cluster) may be rewritten once every CTA's MMAs have read it
        umma_commit_cluster(&empty[s], (uint16_t)((1u << ncta) - 1u));
        umma_commit(&pempty[sp]);
        if (stp + 1 == t_end || stp + 1 == nsteps) {  // sub-chunk t complete in TMEM -> the epilogue
          umma_commit(&subdone);
          ++t;
          t_end += sub_steps(t);
        }
      }
    }
  } else if (warp == 1) {
    // ---- A's FP64 rows by TMA
    if (lane == 0) {
      for (int stp = 0; stp < nsteps; ++stp) {
        const int s = stp % kI8AStages;
        mbar_wait_sleep(&aempty[s], ((stp / kI8AStages) & 1) ^ 1);
#ifdef CQR_I8_NOTMA  // probe: no A loads
        mbar_arrive(&afull[s]);
#else
        mbar_expect_tx(&afull[s], kATile * 8);
        tma_load_2d(sAf + s * kATile, &tma_a, col0, (int)(k_begin + (long long)stp * kI8K), &afull[s]);
#endif
      }
    }
  } else if (warp < 2 + kI8Slice) {
    // ---- A slicers: unit u = (column j, k-octet o), 256 units per step; then (warps 2-5, TMEM lane quadrants
    // 2, 3, 0, 1) the epilogue of every sub-chunk: row i = 32 (warp % 4) + lane
    const int st_id = tid - 64;
    constexpr int SUPT = 256 / (kI8Slice * 32);  // units per thread
    const int j = st_id & 63;                    // this thread's column (units st_id + 128 uu)
    const int quad = warp & 3;
    const int i = 32 * quad + lane;
    const bool epi = warp < 6;  // warps 2-5: TMEM lane quadrants 2, 3, 0, 1
    double* out = partial + ((long long)ky * lp + s0 + i) * np_total + col0;
    if (nsteps == 0 && epi) {  // an empty chunk: no MMA initialised the accumulators
      for (int c = 0; c < kI8Cols; ++c) out[c] = 0.0;
    }
    double f1 = 0.0, f2 = 0.0;
    bool two = true;  // the second scaling factor is needed (warp-uniform)
    int t = 0, t_end = sub_steps(0);
    for (int stp = 0; stp < nsteps; ++stp) {
      const int s = stp % kI8PStages, sa = stp % kI8AStages;
      if (stp == t_end - sub_steps(t)) {  // a sub-chunk's first step: its exponent bound for column j
        mbar_wait_sleep(&expfull[t % kExpSlots], (t / kExpSlots) & 1);
        // a 2^(54 - E_j) as two exact power-of-two scalings (54 - E_j may exceed the double range)
        const int sh = 54 - sexp[t % kExpSlots][j], sh1 = sh / 2;
        // one exact scaling 2^sh when it is a finite double (always, short of columns below 2^-969 and
        // all-zero columns); else two (the warp takes one path: c1 sketch 1.66 -> 1.56 ms with the row select gone)
        const int s1 = sh <= 1000 ? sh : sh1;
        f1 = ldexp(1.0, s1);
        f2 = ldexp(1.0, sh - s1);
        two = __any_sync(0xffffffffu, sh > 1000);
      }
      mbar_wait_sleep(&afull[sa], (stp / kI8AStages) & 1);
      mbar_wait_sleep(&pempty[s], ((stp / kI8PStages) & 1) ^ 1);
      const double* At = sAf + sa * kATile;
      unsigned char* planes = sAp + s * kApStage;
#ifndef CQR_I8_NOSLICE  // probe: without the A slicing
      // rows past the chunk end are rows past m_local (chunks are whole 32-row steps): TMA zero-fills them
      auto slice_units = [&](auto two_muls) {
#pragma unroll
        for (int uu = 0; uu < SUPT; ++uu) {
          const int u = st_id + kI8Slice * 32 * uu;
          const int o = u >> 6;
          uint32_t lo[8], hi[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            double sv = At[(8 * o + e) * kI8Cols + j] * f1;
            if (decltype(two_muls)::value) sv *= f2;
            split64(__double2ll_rn(sv), lo[e], hi[e]);
          }
          transpose_store(lo, hi, planes, kAPlane, plane_off(j, 8 * o));
        }
      };
      if (two)
        slice_units(std::true_type{});
      else
        slice_units(std::false_type{});
#endif
      fence_async_shared();  // generic-proxy stores -> visible to the tensor core (async proxy)
      mbar_arrive(&pfull[s]);
      mbar_arrive(&aempty[sa]);
      if ((stp + 1 == t_end || stp + 1 == nsteps) && !epi) {
        ++t;
        t_end += sub_steps(t);
      } else if (stp + 1 == t_end || stp + 1 == nsteps) {
        // ---- epilogue of sub-chunk t: sum_u ACC_u 2^(8(6-u)) in 64-bit integers, scaled, into the partial
        mbar_wait_sleep(&subdone, t & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int* E = sexp[t % kExpSlots];
#pragma unroll 1
        for (int c0 = 0; c0 < kI8Cols; c0 += 8) {
          long long hi[8], lo[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) hi[jj] = lo[jj] = 0;
#pragma unroll
          for (int u = 0; u < kDig; ++u) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                           "=r"(v[7])
                         : "r"(tmem + ((uint32_t)(32 * quad) << 16) + 64u * u + c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const long long a8 = (long long)(int)v[jj];
              if (u < 3)
                hi[jj] += a8 << (8 * (2 - u));
              else
                lo[jj] += a8 << (8 * (6 - u));
            }
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            // N M ~ sum_u ACC_u 2^(8(12-u)) = 2^48 (hi 2^32 + lo); value = N M 2^-51 2^(E_j - 54)
            const double v = ldexp(fma((double)hi[jj], 0x1p32, (double)lo[jj]), E[c0 + jj] - 57);
            out[c0 + jj] = t == 0 ? v : out[c0 + jj] + v;
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __threadfence_block();
        atomicAdd(&drained, 1);  // the exponent slot of sub-chunk t is free again
        mbar_arrive(&tfree);
        ++t;
        t_end += sub_steps(t);
      }
    }
  } else if (warp < 2 + kI8Slice + GEN) {
    // ---- Omega generators: unit u = (Omega row i, k-octet o) = 4 Box-Muller pairs; this CTA draws the
    // units [crank UNITS / C, (crank + 1) UNITS / C) of each step for the whole cluster
    const int gt0 = tid - 32 * (2 + kI8Slice);
    const int teams = gen_teams(ncta), tsize = GEN * 32 / teams;
    const int team = gt0 / tsize, gt = gt0 - team * tsize;  // this thread's team and rank in it
    constexpr int UNITS = kI8Rows * (kI8K / 8);
    const int u_lo = crank * UNITS / ncta, u_hi = (crank + 1) * UNITS / ncta;
    constexpr int UPT = (UNITS + GEN * 32 - 1) / (GEN * 32) * 4;  // units per thread per step (at most)
    const int upt = (u_hi - u_lo + tsize - 1) / tsize;
    uint64_t z[UPT];
    bool live[UPT];
#pragma unroll
    for (int uu = 0; uu < UPT; ++uu) {
      const int u = min(u_lo + gt + tsize * uu, UNITS - 1);
      const int i = u >> 2, o = u & 3;
      // first counter word of the unit's first pair at the team's first step: c = (s0 + i) m_global + row0 + k
      const unsigned long long c0 = (unsigned long long)(s0 + i) * (unsigned long long)m_global + row0 + k_begin +
                                    8 * o + (unsigned long long)kI8K * team;
      z[uu] = seed + (2 * (c0 >> 1) + 1) * kGolden;
      live[uu] = s0 + i < l;
    }
    const uint32_t slice = (uint32_t)(kDig * kOmPlane / ncta);  // this CTA's rows of all planes: one chunk
    for (int stp = team; stp < nsteps; stp += teams) {
      const int s = stp % kI8Stages;
      mbar_wait_sleep(&empty[s], ((stp / kI8Stages) & 1) ^ 1);  // every CTA's MMAs are done with stage s
      unsigned char* planes = sOm + s * kOmStage;
#pragma unroll 1
      for (int uu = 0; uu < upt; ++uu) {
        const int u = u_lo + gt + tsize * uu;
        if (u >= u_hi) break;
        const int i = u >> 2, o = u & 3;
        uint64_t zz[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) zz[q] = z[uu] + (uint64_t)(2 * q) * kGolden;
        z[uu] += (uint64_t)(kI8K * teams) * kGolden;
        // round(w 2^51): the scaling is exact (folded into the Box-Muller radius: one multiply per pair), the
        // conversion rounds; rows past l draw zeros (a zero factor instead of 16 selects per unit: c3 2.65 ->
        // 2.60 ms, c1 1.767 -> 1.747)
        const double lv = live[uu] ? 0x1p51 : 0.0;
        double ge[4], go[4];
#ifdef CQR_I8_NOGEN  // probe: the MMA side's bound (constant draws)
#pragma unroll
        for (int q = 0; q < 4; ++q) ge[q] = (double)(zz[q] & 255) * 0x1p45 * (lv != 0.0), go[q] = 0x1p50;
#else
        gaussian_pairs_z_scaled<4>(T, zz, lv, ge, go);
#endif
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          split64(__double2ll_rn(ge[q]), lo[2 * q], hi[2 * q]);
          split64(__double2ll_rn(go[q]), lo[2 * q + 1], hi[2 * q + 1]);
        }
#ifndef CQR_I8_NOGENSTORE  // probe: no Omega digit stores
        transpose_store(lo, hi, planes, 256, om_off(i, 8 * o));
#endif
      }
#ifndef CQR_I8_NOGENFENCE  // probe: no proxy fence after the digit stores
      fence_async_shared();  // the digit stores -> the tensor core's and the bulk copies' (async) view
#endif
      if (ncta > 1) {
        // the team's stores are done; its lanes 0 .. C-2 ship this CTA's rows (one contiguous chunk of whole
        // row groups, all planes) to one partner each
        asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(tsize) : "memory");
        if (gt < ncta - 1) {
          const int r = gt < crank ? gt : gt + 1;
          const uint32_t dst = mapa_rank(smem_u32(planes), (uint32_t)r);
          const uint32_t bar = mapa_rank(smem_u32(&full[s]), (uint32_t)r);
          bulk_copy_cluster(dst + crank * slice, planes + crank * slice, slice, bar);
        }
        if (gt == 0)
          mbar_arrive_expect(&full[s], (uint32_t)(ncta - 1) * slice);  // the partners' chunks to come
        else
          mbar_arrive(&full[s]);
      } else {
        mbar_arrive(&full[s]);
      }
    }
  } else {
    // ---- exponent scanners: the bound of each column of this CTA over each sub-chunk (max |a| < 2^E, an
    // all-zero column keeps -1074), ahead of the slicers; non-finite entries set the status (engine.cpp:222).
    // Scanner w takes the rows k = w (mod kI8Scan) of each group of 16 kI8Scan rows; lane l the columns
    // col0 + l and col0 + 32 + l. Only the exponent matters (frexp(x) = biased exponent - 1022 for normal
    // x; 2^-1022 bounds the subnormals), so each load is the 4-byte high word: 32 loads in flight per lane
    // in 32 registers. Non-finite entries (exponent field 0x7ff) set the status (engine.cpp:222).
    const int w = warp - (2 + kI8Slice + GEN);
    const bool ok0 = col0 + lane < n, ok1 = col0 + 32 + lane < n;
    const unsigned* h0 = reinterpret_cast<const unsigned*>(a + (ok0 ? col0 + lane : 0)) + 1;
    const unsigned* h1 = reinterpret_cast<const unsigned*>(a + (ok1 ? col0 + 32 + lane : 0)) + 1;
    const long long ldw = 2 * lda;  // row stride in 32-bit words
    if (kScanAhead > 0 && w == 0 && lane == 0)
      for (int b = 0; b < min(kScanAhead, nsteps); ++b) tma_prefetch_2d(&tma_a, col0, (int)(k_begin + 32LL * b));
    unsigned badbits = 0;
    int t = 0;
    for (int b0 = 0; b0 < nsteps; b0 += sub_steps(t), ++t) {
      const int b1 = min(nsteps, b0 + sub_steps(t));
      const long long kend = min(k_end, k_begin + 32LL * b1);
      if (t >= kExpSlots) {  // slot t % 4 is free once the epilogue has drained sub-chunk t - 4
        while (*(volatile int*)&drained < 4 * 32 * (t - kExpSlots + 1)) __nanosleep(200);
      }
      unsigned m0 = 0, m1 = 0;
#ifdef CQR_I8_NOSCAN  // probe: no scan (bound 2^1: right for |a| < 2 only)
      m0 = m1 = 0x3ff80000u;
#else
#pragma unroll 1
      for (long long k0 = k_begin + 32LL * b0 + w; k0 < kend; k0 += 16 * kI8Scan) {
        if (kScanAhead > 0 && w == 0 && lane == 0) {
          const long long bb = (k0 - k_begin) / 32 + kScanAhead;
          if (bb < nsteps && ((k0 - k_begin) & 31) < kI8Scan) tma_prefetch_2d(&tma_a, col0, (int)(k_begin + 32 * bb));
        }
        unsigned x0[16], x1[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const long long k = k0 + kI8Scan * r;
          const unsigned pr = k < kend;
          x0[r] = x1[r] = 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@p ld.global.nc.L1::no_allocate.u32 %0, [%2];\n\t@p ld.global.nc.L1::no_allocate.u32 %1, [%3];\n\t}"
              : "+r"(x0[r]), "+r"(x1[r])
              : "l"(h0 + k * ldw), "l"(h1 + k * ldw), "r"(pr));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          m0 = max(m0, x0[r] & 0x7fffffffu);
          m1 = max(m1, x1[r] & 0x7fffffffu);
        }
      }
#endif
      // non-finite entries: the running maximum reaches the exponent field 0x7ff iff some entry does (bit 31 of
      // the sum), so one check per sub-chunk replaces one per entry
      badbits |= (m0 + 0x00100000u) | (m1 + 0x00100000u);
      sexpw[w][lane] = ok0 ? m0 : 0u;
      sexpw[w][32 + lane] = ok1 ? m1 : 0u;
      asm volatile("bar.sync %0, %1;" ::"r"(8), "r"(kI8Scan * 32) : "memory");
      if (w == 0) {
        int* E = sexp[t % kExpSlots];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          unsigned mm = 0;
#pragma unroll
          for (int ww = 0; ww < kI8Scan; ++ww) mm = max(mm, sexpw[ww][32 * h + lane]);
          const int be = (int)(mm >> 20);  // biased exponent of the column's largest |a|
          E[32 * h + lane] = mm == 0 ? -1074 : be == 0 ? -1022 : be - 1022;
        }
        mbar_arrive(&expfull[t % kExpSlots]);
      }
      asm volatile("bar.sync %0, %1;" ::"r"(8), "r"(kI8Scan * 32) : "memory");  // sexpw reusable
    }
    const bool bad = (badbits >> 31) != 0;
    if (__any_sync(0xffffffffu, bad) && lane == 0) set_status_invalid(st);
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();  // no partner still stores into this CTA's smem or arrives on its barriers
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

cudaError_t ensure_tables_i8(cudaStream_t s) {
  static std::mutex mu;
  static unsigned long long done = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (dev < 64 && (done >> dev) & 1ull) return cudaSuccess;
  BmTables t;
  bm_tables_host(&t);
  static BmTablesX x;  // static: the async copy reads it until the synchronize below (under the mutex)
  bm_tables_expand(t, &x);
  e = cudaMemcpyToSymbolAsync(c_bm_i8, &x, sizeof(x), 0, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && dev < 64) done |= 1ull << dev;
  return e;
}

}  // namespace

bool sketch_i8_ok(const double* a, long long lda, long long m_global, long long row0, int n) {
  static const bool off = std::getenv("CQR_SKETCH_DMMA") != nullptr;  // A/B: the DMMA kernels
  if (off || n < 1 || n > 512 || (m_global & 1) || (row0 & 1) || m_global > (1LL << 31) - 64) return false;
  CUtensorMap probe;
  return make_tmap_2d(&probe, a, n, std::max<long long>(1, m_global), lda, kI8Cols, kI8K,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
}

namespace {
// the kernel instance, block size and dynamic smem for clusters of C CTAs
struct I8Launch {
  void (*kern)(CUtensorMap, const double*, long long, long long, long long, long long, int, int, uint64_t, long long,
               double*, int, int, int, DevStatus*);
  int warps;
  size_t smem;
};
I8Launch i8_launch(int C) {
  if (C >= 8)
    return {sketch_i8_kernel<CQR_I8_GEN8, CQR_I8_S8, CQR_I8_P8, CQR_I8_AS8>, 2 + kI8Slice + CQR_I8_GEN8 + kI8Scan,
            i8_smem(CQR_I8_S8, CQR_I8_P8, CQR_I8_AS8)};
  if (C >= 4)
    return {sketch_i8_kernel<CQR_I8_GEN, CQR_I8_S4, CQR_I8_P4, CQR_I8_AS4>, 2 + kI8Slice + CQR_I8_GEN + kI8Scan,
            i8_smem(CQR_I8_S4, CQR_I8_P4, CQR_I8_AS4)};
  if (C >= 2)
    return {sketch_i8_kernel<CQR_I8_GEN, CQR_I8_S2, CQR_I8_P2, CQR_I8_AS2>, 2 + kI8Slice + CQR_I8_GEN + kI8Scan,
            i8_smem(CQR_I8_S2, CQR_I8_P2, CQR_I8_AS2)};
  return {sketch_i8_kernel<CQR_I8_GEN, CQR_I8_S1, CQR_I8_P1, CQR_I8_AS1>, 2 + kI8Slice + CQR_I8_GEN + kI8Scan,
          i8_smem(CQR_I8_S1, CQR_I8_P1, CQR_I8_AS1)};
}
}  // namespace

namespace {
// concurrent clusters of C sketch CTAs on this device (cached per (device, C))
long long max_active_clusters(int C, int num_sms) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, long long> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return std::max(1, num_sms / C);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find({dev, C});
  if (it != cache.end()) return it->second;
  const I8Launch L = i8_launch(C);
  auto kern = L.kern;
  const int warps = L.warps;
  long long v = std::max(1, num_sms / C);
  int nc = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, 1, (unsigned)C);
  cfg.blockDim = dim3(warps * 32, 1, 1);
  cfg.dynamicSmemBytes = L.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)C;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (allow_max_smem(kern) == cudaSuccess && cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc > 0)
    v = nc;
  cudaGetLastError();
  cache[{dev, C}] = v;
  return v;
}
}  // namespace

void sketch_i8_plan(SketchPlan& p, long long m_local, int n, int l, int num_sms, int splits) {
  p.i8 = 1;
  p.ws = 0;
  p.n = n;
  p.l = l;
  p.np = (n + kI8Cols - 1) / kI8Cols * kI8Cols;
  p.npc = kI8Cols;
  p.st = kI8Rows;
  p.m_local = m_local;
  p.s_tiles = (l + kI8Rows - 1) / kI8Rows;
  p.lp = p.s_tiles * kI8Rows;
  // the fewest k-chunks whose clusters (s_tiles per k-chunk, C = np / 64 CTAs each) fill whole rounds of
  // the device's concurrent clusters (cudaOccupancyMaxActiveClusters: clusters of 4 or 8 do not tile all
  // 148 SMs); every CTA runs its chunk as sub-chunks (sub_steps), so a chunk has no size bound. The host
  // pipeline launches the chunks in `splits` row ranges: splits x as many.
  const long long slots = max_active_clusters(p.np / kI8Cols, num_sms);
  long long g = slots, b = p.s_tiles;
  while (b) {
    const long long r = g % b;
    g = b;
    b = r;
  }
  long long kc = std::max<long long>(1, slots / g) * std::max(1, splits);
  const long long max_kc = (m_local + kI8K - 1) / kI8K;
  if (kc > max_kc) kc = max_kc;
  if (kc < 1) kc = 1;
  long long rpc = (m_local + kc - 1) / kc;
  rpc = (rpc + kI8K - 1) / kI8K * kI8K;
  if (rpc < kI8K) rpc = kI8K;
  p.rows_per_chunk = rpc;
  p.kchunks = (int)((m_local + rpc - 1) / rpc);
  if (p.kchunks < 1) p.kchunks = 1;
  p.partial_doubles = (size_t)p.kchunks * p.lp * p.np;
  static const bool dbg = std::getenv("CQR_DEBUG_PLAN") != nullptr;
  if (dbg)
    std::fprintf(stderr, "sketch_i8_plan: m=%lld n=%d l=%d s_tiles=%d C=%d slots=%lld kchunks=%d rows/chunk=%lld\n",
                 m_local, n, l, p.s_tiles, p.np / kI8Cols, slots, p.kchunks, p.rows_per_chunk);
}

cudaError_t launch_sketch_i8(const SketchPlan& p, const double* a, long long lda, long long m_global, long long row0,
                             uint64_t seed, double* partial, const DevStatus* st, cudaStream_t s, int y0, int y1) {
  if (y1 < 0) y1 = p.kchunks;
  if (y1 <= y0) return cudaSuccess;
  cudaError_t e = ensure_tables_i8(s);
  if (e != cudaSuccess) return e;
  CUtensorMap tm;
  if (!make_tmap_2d(&tm, a, p.n, p.m_local, lda, kI8Cols, kI8K, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  const int ncta = p.np / kI8Cols;
  const I8Launch L = i8_launch(ncta);
  auto kern = L.kern;
  const int warps = L.warps;
  e = allow_max_smem(kern);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.s_tiles, (unsigned)(y1 - y0), (unsigned)(p.np / kI8Cols));
  cfg.blockDim = dim3(warps * 32, 1, 1);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // the column tiles share their Omega draws
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)(p.np / kI8Cols);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tm, a, lda, p.m_local, m_global, row0, p.l, p.n, seed, p.rows_per_chunk,
                            partial, p.lp, p.np, y0, const_cast<DevStatus*>(st));
}

}  // namespace cqr
