// Warp-specialised FP64 GEMM: one producer warp streams A/B tiles with
// cp.async into a STAGES-deep shared-memory ring and signals per-stage
// mbarriers (cp.async.mbarrier.arrive.noinc); the consumer warps wait only on
// the "full" barrier of the stage they need, issue their DMMA.8x8x4 tiles and
// release the stage on its "empty" barrier.  Compared with the lockstep
// kernel (one __syncthreads per k tile) the consumer warps drift freely, so a
// warp waiting on shared-memory loads no longer stalls the whole CTA.
// Shared-memory layout (padded rows, conflict-free fragment loads) and the
// epilogue are those of dgemm_kernel in gemm.cu.
#pragma once

namespace td {

// mbar_init / mbar_wait: gemm_tma.cuh
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)));
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct WsCfg {
  using Base = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  static constexpr int CONSUMERS = Base::WARPS_M * Base::WARPS_N;
  static constexpr int THREADS = (CONSUMERS + 1) * 32;
  static constexpr int BAR_OFFSET = Base::SMEM_BYTES;                // bytes
  static constexpr int SMEM_BYTES = Base::SMEM_BYTES + 2 * STAGES * 8;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int VEC>
__global__ void __launch_bounds__(WsCfg<BM, BN, BK, WM, WN, STAGES>::THREADS, 1)
dgemm_ws_kernel(GemmArgs p) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  using W = WsCfg<BM, BN, BK, WM, WN, STAGES>;
  extern __shared__ __align__(128) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + W::BAR_OFFSET);
  uint64_t* empty = full + STAGES;

  const int tile = blockIdx.x;
  const int group = p.group;
  const int per_group = group * p.tiles_n;
  const int g = tile / per_group;
  const int first_m = g * group;
  const int gsize = min(p.tiles_m - first_m, group);
  const int in_g = tile % per_group;
  const int64_t m0 = int64_t(first_m + in_g % gsize) * BM;
  const int64_t n0 = int64_t(in_g / gsize) * BN;
  const int64_t bz = blockIdx.y;
  const double* __restrict__ A = p.A + bz * p.sA;
  const double* __restrict__ B = p.B + bz * p.sB;
  double* __restrict__ C = p.C + bz * p.sC;
  const int64_t M = p.M, N = p.N, K = p.K;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int ktiles = (int)ceil_div(K, BK);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], W::CONSUMERS);
    }
  }
  __syncthreads();

  if (warp == W::CONSUMERS) {
    // ---------------- producer warp
    for (int t = 0; t < ktiles; ++t) {
      const int s = t % STAGES;
      if (t >= STAGES) mbar_wait(&empty[s], ((t / STAGES) - 1) & 1);
      const int64_t k0 = int64_t(t) * BK;
      double* as = As + s * Cfg::A_STAGE;
      double* bs = Bs + s * Cfg::B_STAGE;
      constexpr int A_PER_ROW = BK / VEC;
#pragma unroll 4
      for (int c = lane; c < BM * A_PER_ROW; c += 32) {
        const int r = c / A_PER_ROW;
        const int col = (c % A_PER_ROW) * VEC;
        const int64_t gm = m0 + r, gk = k0 + col;
        int valid = 0;
        const double* src = A;
        if (gm < M && gk < K) {
          valid = (int)(K - gk < VEC ? K - gk : VEC);
          src = A + gm * p.lda + gk;
        }
        cp_async_f64<VEC>(as + r * Cfg::SA + col, src, valid);
      }
      constexpr int B_PER_ROW = BN / VEC;
#pragma unroll 4
      for (int c = lane; c < BK * B_PER_ROW; c += 32) {
        const int r = c / B_PER_ROW;
        const int col = (c % B_PER_ROW) * VEC;
        const int64_t gk = k0 + r, gn = n0 + col;
        int valid = 0;
        const double* src = B;
        if (gk < K && gn < N) {
          valid = (int)(N - gn < VEC ? N - gn : VEC);
          src = B + gk * p.ldb + gn;
        }
        cp_async_f64<VEC>(bs + r * Cfg::SB + col, src, valid);
      }
      cp_async_arrive_noinc(&full[s]);
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumer warps
  const int wm0 = (warp / Cfg::WARPS_N) * WM;
  const int wn0 = (warp % Cfg::WARPS_N) * WN;
  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int arow = wm0 + (lane >> 2);
  const int acol = lane & 3;
  const int brow = lane & 3;
  const int bcol = wn0 + (lane >> 2);

  for (int t = 0; t < ktiles; ++t) {
    const int s = t % STAGES;
    mbar_wait(&full[s], (t / STAGES) & 1);
    const double* as = As + s * Cfg::A_STAGE;
    const double* bs = Bs + s * Cfg::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(arow + i * 8) * Cfg::SA + kk + acol];
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) bf[j] = bs[(kk + brow) * Cfg::SB + bcol + j * 8];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    const int64_t r = m0 + wm0 + i * 8 + (lane >> 2);
    if (r >= M) continue;
    double* crow = C + r * p.ldc;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
      const int64_t c = n0 + wn0 + j * 8 + (lane & 3) * 2;
      if (c + 1 < N && ((reinterpret_cast<uintptr_t>(crow + c) & 15) == 0)) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (p.accumulate) {
          const double2 o = *reinterpret_cast<const double2*>(crow + c);
          v.x += o.x;
          v.y += o.y;
        }
        *reinterpret_cast<double2*>(crow + c) = v;
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (c + h < N) {
            double v = acc[i][j][h];
            if (p.accumulate) v += crow[c + h];
            crow[c + h] = v;
          }
        }
      }
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int VEC>
static int launch_gemm_ws(cudaStream_t st, int64_t batch, GemmArgs a) {
  using W = WsCfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = dgemm_ws_kernel<BM, BN, BK, WM, WN, STAGES, VEC>;
  TD_CUDA(ensure_smem(kern, W::SMEM_BYTES));
  a.tiles_m = (int)ceil_div(a.M, BM);
  a.tiles_n = (int)ceil_div(a.N, BN);
  a.group = raster_group(1, BM, BN);
  const int64_t tiles = int64_t(a.tiles_m) * a.tiles_n;
  TD_REQUIRE(tiles < (1ll << 31) && batch <= 65535, "dgemm: grid too large (%lld tiles, batch %lld)",
             (long long)tiles, (long long)batch);
  dim3 grid((unsigned)tiles, (unsigned)batch);
  kern<<<grid, W::THREADS, W::SMEM_BYTES, st>>>(a);
  return check_launch("dgemm_ws_kernel");
}

}  // namespace td
