// Experiment (round 3), removed from the product: see profiles/r01_pipe_share.txt.
// ---- n = 128 with the diagonal recurrences on their own SM sub-partition -----------------------------------
// The recurrence is a ~31-deep dependent FP64 chain per block; on a sub-partition that also issues DMMAs it
// waits behind them (the DMMA takes the shared FP64 pipe first), so a warp spends most of its time in it. Here
// the warps w with w % 4 == 3 (sub-partition 3) run ONLY recurrences: DMMA warp d (the other nine) stages its
// block in its staging tile, posts a request, and the chain warp of its row of four (warp 4 (d / 4) + 3)
// solves the block on an otherwise idle FP64 pipe and posts it back; the DMMA warp then stores it and applies
// it to the pass's later blocks, as trisolve_tma_kernel does. Three DMMA sub-partitions at full DMMA rate
// instead of four throttled by the recurrences. Same arithmetic, bit for bit.
template <int NP>
__global__ void __launch_bounds__(384, 1)
    trisolve_split_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_ll,
                          const __grid_constant__ CUtensorMap tm_st, long long m, const double* __restrict__ bpack,
                          const double* __restrict__ dpack, const DevStatus* st) {
  constexpr int WPC = 12, NDW = 9;
  constexpr int NT = NP / 8;
  constexpr int W = 4;
  constexpr int NPASS = NT / W;
  constexpr int NB = NT * (NT - 1) * 32;
  constexpr int ND = NT * kDiagStride;
  constexpr int HEAD = head_doubles<NP, true>();
  constexpr int kTmCols = (NT - W) * 16;
  static_assert(2 * kTmCols <= 512, "two DMMA warps' operands per TMEM lane quarter");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t tmem_base;
  __shared__ int job[NDW], finished[NDW];
  if (failed(st)) return;
  double* smem = reinterpret_cast<double*>(smem_raw + ((512u - (smem_u32(smem_raw) & 511u)) & 511u));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, gr = lane >> 2;
  const bool chain = (warp & 3) == 3;
  const int dwi = (warp >> 2) * 3 + (warp & 3);  // DMMA warp index 0..8 (chain warps: unused)
  double* sD = smem;
  double* sB = smem + ND;
  auto warp_T = [&](int d) { return smem + HEAD + d * kWarpDoubles; };  // DMMA warp d's two staging tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + HEAD + NDW * kWarpDoubles);  // [d][4]: in, ll, req, done
  for (int e = threadIdx.x; e < ND; e += WPC * 32) sD[e] = dpack[e];
  for (int e = threadIdx.x; e < NB; e += WPC * 32) sB[e] = bpack[e];
  if (threadIdx.x < NDW) {
    mbar_init(bars + 4 * threadIdx.x, 1);
    mbar_init(bars + 4 * threadIdx.x + 1, 1);
    mbar_init(bars + 4 * threadIdx.x + 2, 32);
    mbar_init(bars + 4 * threadIdx.x + 3, 32);
    finished[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (chain) {
    // ---- chain warp c serves DMMA warps 3c, 3c+1, 3c+2
    const int c = warp >> 2;
    uint32_t rp[3] = {0, 0, 0};
    int live = 3;
    bool done_[3] = {false, false, false};
    while (live > 0) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int d = 3 * c + i;
        if (done_[i]) continue;
        if (mbar_try_wait(bars + 4 * d + 2, rp[i])) {
          rp[i] ^= 1;
          const int J = job[d];
          double* tile = warp_T(d) + (J & 1) * kTile;
          const double* D = sD + J * kDiagStride;
          double y[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 v = *reinterpret_cast<const double2*>(tile + swz64(lane, u));
            y[2 * u] = v.x;
            y[2 * u + 1] = v.y;
          }
          bool good = D[80] != 0.0;
          if (good) {
            bool ok = true;
            const double* Dc = D + kColBase;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              double v[10];
#pragma unroll
              for (int h = 0; h < (j + 3) / 2; ++h) {
                const double2 t2 = *reinterpret_cast<const double2*>(Dc + col_start(j) + 2 * h);
                v[2 * h] = t2.x;
                v[2 * h + 1] = t2.y;
              }
#pragma unroll
              for (int kk = 0; kk < j; ++kk) y[j] = fma(-v[kk], y[kk], y[j]);
              bool okj;
              y[j] = div_fast(y[j], v[j], v[j + 1], okj);
              ok &= okj;
            }
            good = __all_sync(0xffffffffu, ok);
          }
          if (!good) {
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = tile[swz64(lane, j >> 1) + (j & 1)];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
#pragma unroll
              for (int kk = 0; kk < j; ++kk) {
                const double rv = D[kk * 8 + j];
                if (rv != 0.0) y[j] = fma(-rv, y[kk], y[j]);
              }
              y[j] = fast_div(y[j], D[j * 8 + j], D[64 + j], D[72 + j] != 0.0);
            }
          }
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<double2*>(tile + swz64(lane, u)) = make_double2(y[2 * u], y[2 * u + 1]);
          mbar_arrive_cta(bars + 4 * d + 3);  // every lane: its rows are in the tile
        } else if (*(volatile int*)&finished[d]) {
          done_[i] = true;
          --live;
        }
      }
    }
  } else {
    // ---- DMMA warp dwi: the groups, passes and left-looking phase of trisolve_tma_kernel
    const int d = dwi;
    double* sT = warp_T(d);
    double* sL = sT + 2 * kTile;
    uint64_t* bar = bars + 4 * d;  // [0] input + left-looking buffer 0, [1] left-looking buffer 1
    const bool tmw = (warp >> 2) < 2;
    const uint32_t tm_warp = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kTmCols);
    auto issue_ll = [&](int ch, int b, int row0) {
      mbar_expect_tx(bar + b, 4 * kSlab * 8);
#pragma unroll
      for (int s = 0; s < 4; ++s) tma_load_2d(sL + b * 2 * kTile + s * kSlab, &tm_ll, 16 * ch + 4 * s, row0, bar + b);
    };
    const uint64_t pol_in = l2_policy_evict_first(), pol_out = l2_policy_evict_last();
    auto issue_in = [&](int P, long long grp) {
      mbar_expect_tx(bar, W * kTile * 8);
#pragma unroll
      for (int t = 0; t < W; ++t)
        tma_load_2d_hint(sL + t * kTile, &tm_in, 8 * W * P + 8 * t, (int)(grp * kRW), bar, pol_in);
    };
    uint32_t ph0 = 0, ph1 = 0, pdone = 0;
    const long long groups = (m + kRW - 1) / kRW;
    const long long gstride = (long long)gridDim.x * NDW;
    const long long rounds = groups / gstride;
    auto next_grp = [&](long long g) -> long long {
      const long long k = g < rounds * gstride ? g / gstride : rounds;
      if (k + 1 < rounds) return g + gstride;
      if (k + 1 == rounds) return rounds * gstride + (long long)d * gridDim.x + blockIdx.x;
      return groups;
    };
    long long grp = rounds > 0 ? (long long)blockIdx.x * NDW + d : (long long)d * gridDim.x + blockIdx.x;
    if (lane == 0 && grp < groups) issue_in(0, grp);
    for (; grp < groups; grp = next_grp(grp)) {
      const int row0 = (int)(grp * kRW);
#pragma unroll 1
      for (int P = 0; P < NPASS; ++P) {
        const int c0 = 8 * W * P;
        mbar_wait(bar, ph0);
        ph0 ^= 1;
        double acc[4][W][2];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int t = 0; t < W; ++t) {
            const double2 v = *reinterpret_cast<const double2*>(sL + t * kTile + (8 * g + gr) * 8 + 2 * q);
            acc[g][t][0] = v.x;
            acc[g][t][1] = v.y;
          }
        if (P > 0 && tmw) {
          const int nch = c0 / 16;
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll 1
          for (int ch = 0; ch < nch; ++ch) {
            double af16[16];
            tm_ld32(tm_warp + 32u * ch, af16);
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int k4 = 4 * ch + s;
#pragma unroll
              for (int t = 0; t < W; ++t) {
                const int JJ = W * P + t;
                const double bv = sB[(JJ * (JJ - 1) + k4) * 32 + lane];
#pragma unroll
                for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af16[4 * s + g], bv);
              }
            }
          }
        } else if (P > 0) {
          const int nch = c0 / 16;
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            bulk_wait<0>();
            fence_async_global();
            issue_ll(0, 0, row0);
            if (nch > 1) issue_ll(1, 1, row0);
          }
#pragma unroll 1
          for (int ch = 0; ch < nch; ++ch) {
            const int b = ch & 1;
            if (b == 0) {
              mbar_wait(bar, ph0);
              ph0 ^= 1;
            } else {
              mbar_wait(bar + 1, ph1);
              ph1 ^= 1;
            }
            const double* buf = sL + b * 2 * kTile;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const int k4 = 4 * ch + s;
              double af[4];
#pragma unroll
              for (int g = 0; g < 4; ++g) af[g] = buf[s * kSlab + (8 * g + gr) * 4 + q];
#pragma unroll
              for (int t = 0; t < W; ++t) {
                const int JJ = W * P + t;
                const double bv = sB[(JJ * (JJ - 1) + k4) * 32 + lane];
#pragma unroll
                for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g], bv);
              }
            }
            fence_async_shared();
            __syncwarp();
            if (lane == 0 && ch + 2 < nch) issue_ll(ch + 2, b, row0);
          }
        }
        {
          const bool last = P + 1 == NPASS;
          if (!last || next_grp(grp) < groups) {
            fence_async_shared();
            __syncwarp();
            if (lane == 0) issue_in(last ? 0 : P + 1, last ? next_grp(grp) : grp);
          }
        }
#pragma unroll 1
        for (int Jl = 0; Jl < W; ++Jl) {
          const int J = W * P + Jl;
          double* tile = sT + (J & 1) * kTile;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 4; ++g)
            *reinterpret_cast<double2*>(tile + swz64(8 * g + gr, q)) = make_double2(acc[g][0][0], acc[g][0][1]);
          if (lane == 0) job[d] = J;
          __syncwarp();
          mbar_arrive_cta(bar + 2);  // request: the chain warp solves the block in place
          mbar_wait(bar + 3, pdone);
          pdone ^= 1;
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d_hint(&tm_st, 8 * J, row0, tile, pol_out);
            bulk_commit();
          }
          double af[4][2];
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int kk4 = 0; kk4 < 2; ++kk4) af[g][kk4] = tile[swz64(8 * g + gr, 2 * kk4 + (q >> 1)) + (q & 1)];
          if (tmw && J < NT - W) {
            const double v8[8] = {af[0][0], af[1][0], af[2][0], af[3][0], af[0][1], af[1][1], af[2][1], af[3][1]};
            tm_st16(tm_warp + 16u * J, v8);
          }
          const double* bcol = sB + (2 * J) * 32 + lane;
#pragma unroll
          for (int t = 1; t < W; ++t) {
            if (Jl + t < W) {
              const int JJ = J + t;
              const double* bp = bcol + (JJ * (JJ - 1)) * 32;
#pragma unroll
              for (int kk4 = 0; kk4 < 2; ++kk4) {
                const double bv = bp[kk4 * 32];
#pragma unroll
                for (int g = 0; g < 4; ++g) dmma(acc[g][t][0], acc[g][t][1], af[g][kk4], bv);
              }
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              acc[g][t - 1][0] = acc[g][t][0];
              acc[g][t - 1][1] = acc[g][t][1];
            }
          }
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
    if (lane == 0) *(volatile int*)&finished[d] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

