// FP64 GEMM / TTM leaf kernels (DMMA m8n8k4 tiles, cp.async multistage smem).
//
// Replaces the reference's per-point evaluation of the GEMM leaf
// C(i,j) += A(i,k) * B(k,j) (reference pkg/src/tendist/algorithms.py:80-83,
// evaluated point by point at cin.py:399-417) and the TTM leaf
// Y(i,j,l) += B(i,j,k) * C(k,l) (algorithms.py:300-301).
//
// Kernel shape (BM x BN x 16 CTA tile, warps of WM x WN):
//   * STAGES-deep cp.async ring: A tile [BM][16+4], B tile [16][BN+4]
//     (row pads of 4 doubles make every fragment LDS.64 conflict-free:
//     rows r=0..3 x cols c=0..3 land on 16 distinct 8-byte banks);
//   * each warp owns (WM/8) x (WN/8) accumulators of DMMA.8x8x4 in
//     registers and issues all of them per k4 slice;
//   * grouped tile rasterisation (8 M-tiles per group) for L2 reuse;
//   * epilogue writes (or accumulates into) row-major C with bounds checks.
// The default path is the TMA-fed variant of the same body (gemm_tma.cuh:
// k4-sliced tensor-map views, mbarrier-completed stages, 4 CTAs/SM); this
// LDGSTS kernel serves operands TMA cannot address (odd leading dimensions,
// K or N not a multiple of 4, unaligned bases).
// Summation order: k tiles ascending, within a tile the DMMA's own order --
// exact on integer-valued data, |err| <= gamma_K |A||B| on real data.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "dmma.cuh"
#include "gemm.cuh"

namespace td {

constexpr int PAD = 4;

// KP = 1: "k-pair" fragments -- one LDS.128 fetches A[row][2q], A[row][2q+1]
// for two consecutive k4 slices (lane q owns k = 2q + s within each k8 group;
// B is read with the same permutation).  Row strides change so both stay
// conflict-free: A rows of BK+8 (quarter-warp rows 192 B apart), B rows of
// BN+2 (k rows 2q land on distinct 8-byte bank groups).
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int KP = 0>
struct GemmCfg {
  static constexpr int GEMM_BK = BK;
  static constexpr int WARPS_M = BM / WM;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int SA = GEMM_BK + (KP ? 8 : PAD);  // A row stride (doubles)
  static constexpr int SB = BN + (KP ? 2 : PAD);       // B row stride (doubles)
  static constexpr int A_STAGE = BM * SA;
  static constexpr int B_STAGE = GEMM_BK * SB;
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
  static constexpr int FM = WM / 8;
  static constexpr int FN = WN / 8;
  // resident CTAs per SM the register budget is sized for: 4-warp CTAs share
  // an SM (2 with 64x32 / 32x64 warp tiles, 3 with 32x32 ones)
  static constexpr int MIN_BLOCKS = THREADS > 128 ? 1 : (FM * FN <= 16 ? 3 : 2);
};


template <int BM, int BN, int BK, int WM, int WN, int STAGES, int VEC, int KP = 0, int EPI = 0>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, STAGES, KP>::THREADS,
                                  GemmCfg<BM, BN, BK, WM, WN, STAGES, KP>::MIN_BLOCKS)
dgemm_kernel(GemmArgs p) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, KP>;
  constexpr int GEMM_BK = BK;
  extern __shared__ __align__(128) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;

  // grouped rasterisation
  const int tile = blockIdx.x;
  const int group = p.group;
  const int per_group = group * p.tiles_n;
  const int g = tile / per_group;
  const int first_m = g * group;
  const int gsize = min(p.tiles_m - first_m, group);
  const int in_g = tile % per_group;
  const int tm = first_m + in_g % gsize;
  const int tn = in_g / gsize;
  const int64_t m0 = int64_t(tm) * BM;
  const int64_t n0 = int64_t(tn) * BN;

  const int64_t bz = blockIdx.y;
  const double* __restrict__ A = p.A + bz * p.sA;
  const double* __restrict__ B = p.B + bz * p.sB;
  double* __restrict__ C = p.C + bz * p.sC;
  const int64_t M = p.M, N = p.N, K = p.K;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm0 = (warp / Cfg::WARPS_N) * WM;
  const int wn0 = (warp % Cfg::WARPS_N) * WN;

  // Fast path for interior tiles: each thread's chunks sit at fixed rows /
  // columns, only k advances, so the global addresses are one base pointer
  // plus compile-time row steps (no per-chunk index math or predicates).
  constexpr int FA_PER_ROW = GEMM_BK / VEC, FB_PER_ROW = BN / VEC;
  constexpr bool FAST_OK = (BM * FA_PER_ROW) % Cfg::THREADS == 0 && (GEMM_BK * FB_PER_ROW) % Cfg::THREADS == 0 &&
                           Cfg::THREADS % FA_PER_ROW == 0 && Cfg::THREADS % FB_PER_ROW == 0;
  constexpr int FA_ITERS = BM * FA_PER_ROW / Cfg::THREADS, FA_STEP = Cfg::THREADS / FA_PER_ROW;
  constexpr int FB_ITERS = GEMM_BK * FB_PER_ROW / Cfg::THREADS, FB_STEP = Cfg::THREADS / FB_PER_ROW;
  const int fa_r = tid / FA_PER_ROW, fa_c = (tid % FA_PER_ROW) * VEC;
  const int fb_r = tid / FB_PER_ROW, fb_c = (tid % FB_PER_ROW) * VEC;
  const bool interior = FAST_OK && m0 + BM <= M && n0 + BN <= N;
  const double* fa_base = A + (interior ? (m0 + fa_r) * p.lda + fa_c : 0);
  const double* fb_base = B + (interior ? fb_r * p.ldb + n0 + fb_c : 0);
  const int64_t fa_step = int64_t(FA_STEP) * p.lda, fb_step = int64_t(FB_STEP) * p.ldb;

  auto load_tile = [&](int stage, int64_t k0) {
    double* as = As + stage * Cfg::A_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    if constexpr (FAST_OK) {
      if (interior && k0 + GEMM_BK <= K) {
        const double* a = fa_base + k0;
#pragma unroll
        for (int it = 0; it < FA_ITERS; ++it)
          cp_async_f64<VEC>(as + (fa_r + it * FA_STEP) * Cfg::SA + fa_c, a + it * fa_step, VEC);
        const double* b = fb_base + k0 * p.ldb;
#pragma unroll
        for (int it = 0; it < FB_ITERS; ++it)
          cp_async_f64<VEC>(bs + (fb_r + it * FB_STEP) * Cfg::SB + fb_c, b + it * fb_step, VEC);
        return;
      }
    }
    constexpr int A_CHUNKS = BM * GEMM_BK / VEC;
    constexpr int A_PER_ROW = GEMM_BK / VEC;
#pragma unroll
    for (int c = tid; c < A_CHUNKS; c += Cfg::THREADS) {
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
    constexpr int B_CHUNKS = GEMM_BK * BN / VEC;
    constexpr int B_PER_ROW = BN / VEC;
#pragma unroll
    for (int c = tid; c < B_CHUNKS; c += Cfg::THREADS) {
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
  };

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = (int)ceil_div(K, GEMM_BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, int64_t(s) * GEMM_BK);
    cp_async_commit();
  }

  const int arow = wm0 + (lane >> 2);
  const int acol = lane & 3;
  const int brow = lane & 3;
  const int bcol = wn0 + (lane >> 2);

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = kt + STAGES - 1;
      if (nt < ktiles) load_tile(nt % STAGES, int64_t(nt) * GEMM_BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE;
    if constexpr (KP) {
#pragma unroll
      for (int kk = 0; kk < GEMM_BK; kk += 8) {
        double2 a2[Cfg::FM];
        double b0[Cfg::FN], b1[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
          a2[i] = *reinterpret_cast<const double2*>(as + (arow + i * 8) * Cfg::SA + kk + 2 * acol);
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          b0[j] = bs[(kk + 2 * brow) * Cfg::SB + bcol + j * 8];
          b1[j] = bs[(kk + 2 * brow + 1) * Cfg::SB + bcol + j * 8];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a2[i].x, b0[j]);
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a2[i].y, b1[j]);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < GEMM_BK; kk += 4) {
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
    }
  }
  cp_async_wait<0>();

  if constexpr (EPI == 1) {
    // Hadamard with H and sum over the tile's rows: lanes sharing (lane & 3)
    // hold the same columns (shuffle), then the WARPS_M warps of a column
    // strip add up in shared memory in warp order -- a fixed summation order.
    double part[Cfg::FN][2];
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) part[j][0] = part[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) {
      const int64_t r = m0 + wm0 + i * 8 + (lane >> 2);
      const double* hrow = p.H + r * p.ldh;
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int64_t c = n0 + wn0 + j * 8 + (lane & 3) * 2;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (r < M && c + h < N) part[j][h] += hrow[c + h] * acc[i][j][h];
      }
    }
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = part[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        part[j][h] = v;
      }
    __syncthreads();  // the ring is drained: reuse it as [WARPS_M][BN]
    double* red = smem;
    if (lane < 4) {
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) red[(warp / Cfg::WARPS_N) * BN + wn0 + j * 8 + lane * 2 + h] = part[j][h];
    }
    __syncthreads();
    for (int c = tid; c < BN; c += Cfg::THREADS) {
      double v = red[c];
#pragma unroll
      for (int w = 1; w < Cfg::WARPS_M; ++w) v += red[w * BN + c];
      if (n0 + c < N) C[int64_t(tm) * N + n0 + c] = v;
    }
    return;
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    const int64_t r = m0 + wm0 + i * 8 + (lane >> 2);
    if (r >= M) continue;
    double* crow = C + r * p.ldc;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
      const int64_t c = n0 + wn0 + j * 8 + (lane & 3) * 2;
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

// M-tiles per raster group (consecutive CTAs walk down M inside a group, then
// along N): controls how much A/B one wave keeps live in the 126 MB L2.
static int raster_group(int blocks_per_sm, int BM, int BN) {
  static const int forced = [] {
    const char* e = std::getenv("TD_GEMM_GROUP");
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  // Measured on B200 at 16384^3 with 64x64 tiles (tools/tuning/group_sweep.sh):
  // DRAM read per launch 558/290/164/115/128/263 GB for groups 1/2/4/8/16/32
  // with the same 35.5 TFLOP/s -- 8 M-tiles per group minimises re-reads.
  // Round 2, TMA kernel (4 CTAs/SM): 164/119/130/160/218/288 GB for groups
  // 4/8/12/16/24/32 at an unchanged 36.40 TFLOP/s (the squarer waves re-read
  // more: concurrently running CTAs drift apart in k) -- 8 again.
  (void)blocks_per_sm;
  (void)BM;
  (void)BN;
  return 8;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int VEC, int KP = 0, int EPI = 0>
static int launch_gemm(cudaStream_t st, int64_t batch, GemmArgs a) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, KP>;
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, VEC, KP, EPI>;
  static bool configured = false;  // attribute is per-device; cheap to re-set
  (void)configured;
  TD_CUDA(ensure_smem(kern, Cfg::SMEM_BYTES));
  a.tiles_m = (int)ceil_div(a.M, BM);
  a.tiles_n = (int)ceil_div(a.N, BN);
  a.group = raster_group(Cfg::MIN_BLOCKS, BM, BN);
  const int64_t tiles = int64_t(a.tiles_m) * a.tiles_n;
  TD_REQUIRE(tiles < (1ll << 31) && batch <= 65535, "dgemm: grid too large (%lld tiles, batch %lld)",
             (long long)tiles, (long long)batch);
  dim3 grid((unsigned)tiles, (unsigned)batch);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(a);
  return check_launch("dgemm_kernel");
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace td
#include "gemm_tma.cuh"
#include "mttkrp_tma.cuh"
#ifdef TD_TUNING
#include "gemm_ws.cuh"
#endif
namespace td {

static int zero_or_keep(cudaStream_t st, int64_t batch, int64_t M, int64_t N, double* C, int64_t ldc,
                        int64_t sC, int accumulate);

// Tile configurations (BM, BN, BK, WM, WN, STAGES).  `config` < 0 picks by N.
// The default build keeps the configurations the library uses or tests
// (LDGSTS fallbacks 20 / 34, the MTTKRP row-sum tiles 21 / 26 / 29 / 35, every
// TMA tile); `make TUNING=1` adds the tuning history below (td_dgemm_config).
#define TD_GEMM_CORE_CONFIGS(X)             \
  X(20, 64, 64, 16, 32, 32, 4)              \
  X(21, 128, 32, 16, 64, 16, 4)             \
  X(26, 128, 32, 16, 32, 32, 3)             \
  X(29, 128, 32, 8, 32, 32, 5)              \
  X(34, 128, 32, 8, 32, 32, 4)              \
  X(35, 128, 32, 16, 32, 32, 4)

#ifdef TD_TUNING
#define TD_GEMM_TUNING_CONFIGS(X)           \
  X(0, 128, 128, 16, 64, 32, 4)             \
  X(1, 128, 128, 32, 64, 32, 3)             \
  X(2, 128, 128, 16, 32, 32, 4)             \
  X(3, 128, 128, 32, 32, 32, 3)             \
  X(4, 256, 64, 16, 64, 32, 4)              \
  X(5, 256, 64, 32, 64, 32, 2)              \
  X(6, 256, 32, 16, 32, 32, 4)              \
  X(7, 128, 64, 32, 32, 32, 3)              \
  X(16, 64, 128, 16, 32, 64, 3)             \
  X(17, 64, 128, 32, 32, 64, 2)             \
  X(18, 128, 64, 16, 64, 32, 3)             \
  X(19, 64, 128, 16, 32, 64, 4)             \
  X(22, 128, 64, 32, 64, 32, 2)             \
  X(23, 128, 64, 16, 32, 64, 3)             \
  X(24, 64, 64, 16, 32, 32, 3)              \
  X(25, 64, 64, 32, 32, 32, 2)              \
  X(27, 64, 32, 16, 32, 32, 4)              \
  X(28, 64, 32, 16, 32, 32, 6)

// k-pair fragment variants (KP = 1)
#define TD_GEMM_KP_CONFIGS(X)               \
  X(30, 64, 64, 16, 32, 32, 4)              \
  X(31, 64, 128, 16, 32, 64, 3)             \
  X(32, 128, 64, 16, 64, 32, 3)             \
  X(33, 64, 64, 16, 32, 32, 3)

// warp-specialised (producer warp + mbarrier ring) variants: measured slower
// (29.6 TFLOP/s at 16384^3), kept for tuning only
#define TD_GEMM_WS_CONFIGS(X)               \
  X(10, 128, 128, 32, 64, 32, 3)            \
  X(11, 128, 128, 16, 64, 32, 5)            \
  X(12, 256, 64, 32, 64, 32, 2)             \
  X(13, 128, 64, 32, 32, 32, 4)             \
  X(14, 256, 64, 16, 64, 32, 4)             \
  X(15, 128, 128, 16, 32, 32, 6)
#else
#define TD_GEMM_TUNING_CONFIGS(X)
#define TD_GEMM_KP_CONFIGS(X)
#define TD_GEMM_WS_CONFIGS(X)
#endif

#define TD_GEMM_CONFIGS(X) TD_GEMM_CORE_CONFIGS(X) TD_GEMM_TUNING_CONFIGS(X)

// TMA-fed variants (gemm_tma.cuh); operands the copy engine cannot address
// (odd leading dimensions, K or N not a multiple of 4) take the LDGSTS kernel
#define TD_GEMM_TMA_CONFIGS(X)                 \
  X(40, 64, 64, 16, 32, 32, 4, 0)              \
  X(43, 128, 32, 16, 32, 32, 3, 0)             \
  X(44, 64, 128, 16, 32, 64, 3, 0)             \
  X(47, 64, 64, 16, 32, 32, 3, 4)              \
  X(48, 128, 32, 16, 32, 32, 3, 4)             \
  X(50, 128, 64, 16, 64, 32, 4, 0)             \
  X(51, 256, 32, 16, 32, 32, 3, 2)

// Tile history on B200 (tools/tuning/tune2.py, tune_n32.py, tune_n64.py; 16384^3
// unless noted):
//   LDGSTS 128x64x16, 4 warps of 64x32, 3 stages, 2 CTAs/SM          34.2 TFLOP/s
//   + fixed-address load path, 64x128x16 (cuBLAS's own d884 tile)       35.2
//   64x64x16, 4 warps of 32x32, 4 stages, 3 CTAs/SM (config 20)         35.6
//   TMA 64x64x16, 3 stages, 4 CTAs/SM (<= 128 registers; config 47)     36.5  (98.5 %, cuBLAS 36.1)
// TTM shape (M = 2^20, N = 64, K = 1024): config 20 35.0, config 47 36.0 (round 2,
// tools/ttm_configs.py: 47 36.09, 40 (4 stages) 35.79, 50 (128x64) 35.52).
// N <= 32 (MTTKRP / TTM with a rank-32 factor; the A panel streams from HBM
// at ~4.4 TB/s): LDGSTS 128x32x8 4 stages (config 34) 33.6, TMA 128x32x16
// 3 stages (config 48) 35.2.  Also measured at N = 32 (round 1, no gain):
// TMA 128x32 with BK 12 / 3 stages 34.8, BK 16 / 2 stages / 4 CTAs 35.3,
// BK 8 / 5 stages 34.7, 64x32 / 6 CTAs 34.9, 256x32 33.7, 8 warps of 32x16
// 34.3, 64x32 with 16x32 warps 35.1; and the MTTKRP tail wave split into
// half-k CTAs 34.8-35.1 (CTA waves are not synchronous); a persistent
// row-sum kernel keeping the TMA ring running across tiles 31.0-31.7.
// Round 2 (tools/kernel_probe.py): the tail of the last wave costs MTTKRP
// ~1.7 % at I = 1024 (35.0 TFLOP/s; 35.3 at I = 999 = 18 full waves, 35.6
// at I = 4096), and a persistent TMA kernel with dynamically claimed tiles
// (atomic counter, claim latency hidden one tile ahead, the ring running
// across tile boundaries, both EPI forms) measured 33.8 (MTTKRP) and 35.8
// (TTM) against 35.0 / 36.1 here: co-resident CTAs already hide a new
// tile's cold pipeline, so the per-tile CTAs stay.  With the per-stage empty
// barriers, deeper rings for MTTKRP (tools/mttkrp_configs.py): 128x32x8 with 6
// stages / 3 CTAs 34.45, 128x32x16 with 4 stages / 2 CTAs 32.07, vs 34.95.
// Also not kept (tools/ab_kernels.py, A/B builds on one box): refilling a
// slot from the LAST warp to release it (shared-memory arrival counter, no
// producer wait, all STAGES slots in flight) -- DGEMM 36.0 vs 36.38, TTM 35.7
// vs 36.05, MTTKRP 256-row 34.97 vs 35.29; and an L2 prefetch
// (cp.async.bulk.prefetch.tensor) of the A panel 2-16 k-tiles beyond the ring
// -- MTTKRP 27.5 vs 35.3 (even an idle prefetch cursor on the issuing thread
// cost the stream-K kernel 35.42 -> 34.62: the issue path is latency-critical).
static int default_config(int64_t N) {
  if (N <= 32) return 34;
  return 20;
}

static int default_tma_config(int64_t N) {
  if (N <= 32) return 48;
  return 47;
}

int dgemm_dispatch(cudaStream_t st, int64_t batch, GemmArgs a, int config = -1) {
  if (a.M <= 0 || a.N <= 0 || batch <= 0) return TD_OK;
  if (a.K <= 0) return zero_or_keep(st, batch, a.M, a.N, a.C, a.ldc, a.sC, a.accumulate);
  const bool vec2 = aligned16(a.A) && aligned16(a.B) && (a.lda % 2 == 0) && (a.ldb % 2 == 0) &&
                    (batch == 1 || (a.sA % 2 == 0 && a.sB % 2 == 0));
  if (config < 0) config = tma_ok(batch, a) ? default_tma_config(a.N) : default_config(a.N);
  switch (config) {
#define TD_GEMM_CASE(id, BM, BN, BK, WM, WN, ST) \
  case id:                                        \
    return vec2 ? launch_gemm<BM, BN, BK, WM, WN, ST, 2>(st, batch, a) : launch_gemm<BM, BN, BK, WM, WN, ST, 1>(st, batch, a);
    TD_GEMM_CONFIGS(TD_GEMM_CASE)
#undef TD_GEMM_CASE
#define TD_GEMM_KP_CASE(id, BM, BN, BK, WM, WN, ST) \
  case id:                                           \
    return vec2 ? launch_gemm<BM, BN, BK, WM, WN, ST, 2, 1>(st, batch, a) : launch_gemm<BM, BN, BK, WM, WN, ST, 1, 1>(st, batch, a);
    TD_GEMM_KP_CONFIGS(TD_GEMM_KP_CASE)
#undef TD_GEMM_KP_CASE
#define TD_GEMM_TMA_CASE(id, BM, BN, BK, WM, WN, ST, MINB)                                     \
  case id:                                                                                      \
    if (tma_ok(batch, a)) return launch_gemm_tma<BM, BN, BK, WM, WN, ST, 0, MINB>(st, batch, a); \
    return vec2 ? launch_gemm<BM, BN, BK, WM, WN, 3, 2>(st, batch, a)                           \
                : launch_gemm<BM, BN, BK, WM, WN, 3, 1>(st, batch, a);
    TD_GEMM_TMA_CONFIGS(TD_GEMM_TMA_CASE)
#undef TD_GEMM_TMA_CASE
#define TD_GEMM_WS_CASE(id, BM, BN, BK, WM, WN, ST) \
  case id:                                           \
    return vec2 ? launch_gemm_ws<BM, BN, BK, WM, WN, ST, 2>(st, batch, a) : launch_gemm_ws<BM, BN, BK, WM, WN, ST, 1>(st, batch, a);
    TD_GEMM_WS_CONFIGS(TD_GEMM_WS_CASE)
#undef TD_GEMM_WS_CASE
    default:
      set_error("dgemm: unknown tile config %d", config);
      return TD_ERR_ARG;
  }
}

// MTTKRP on the GEMM body (EPI = 1): for every batch b (an i of B(i,k,l)),
// work[b][tm][n] = sum over the rows r of M-tile tm of H(r,n) * (A_b . B)(r,n).
// The caller sums the tm partials in ascending order (mttkrp.cu).
#define TD_ROWSUM_CONFIGS(X)                \
  X(26, 128, 32, 16, 32, 32, 3)             \
  X(29, 128, 32, 8, 32, 32, 5)              \
  X(21, 128, 32, 16, 64, 16, 4)             \
  X(20, 64, 64, 16, 32, 32, 4)              \
  X(34, 128, 32, 8, 32, 32, 4)              \
  X(35, 128, 32, 16, 32, 32, 4)

int dgemm_rowsum_tile_rows(int config) {
  switch (config) {
#define TD_ROWSUM_BM(id, BM, BN, BK, WM, WN, ST) \
  case id:                                        \
    return BM;
    TD_ROWSUM_CONFIGS(TD_ROWSUM_BM)
#define TD_ROWSUM_TMA_BM(id, BM, BN, BK, WM, WN, ST, MINB) TD_ROWSUM_BM(id, BM, BN, BK, WM, WN, ST)
    TD_GEMM_TMA_CONFIGS(TD_ROWSUM_TMA_BM)
#undef TD_ROWSUM_TMA_BM
#undef TD_ROWSUM_BM
    default:
      return 0;
  }
}

bool dgemm_rowsum_fusable(int config, int64_t batch, const GemmArgs& a) {
  switch (config) {
#define TD_ROWSUM_TMA_ID(id, BM, BN, BK, WM, WN, ST, MINB) case id:
    TD_GEMM_TMA_CONFIGS(TD_ROWSUM_TMA_ID)
#undef TD_ROWSUM_TMA_ID
      return tma_ok(std::min<int64_t>(batch, 2), a);
    default:
      return false;
  }
}

int dgemm_rowsum(cudaStream_t st, int config, int64_t batch, GemmArgs a) {
  const bool vec2 = aligned16(a.A) && aligned16(a.B) && (a.lda % 2 == 0) && (a.ldb % 2 == 0) &&
                    (batch == 1 || a.sA % 2 == 0);
  for (int64_t done = 0; done < batch;) {  // grid.y is limited to 65535
    const int64_t chunk = std::min<int64_t>(batch - done, 65535);
    GemmArgs c = a;
    c.A += done * a.sA;
    c.C += done * a.sC;
    if (c.counters) {
      c.counters += done * a.N;
      c.out += done * a.ldo;
    }
    int rc = TD_ERR_ARG;
    switch (config) {
#define TD_ROWSUM_CASE(id, BM, BN, BK, WM, WN, ST)                                              \
  case id:                                                                                      \
    rc = vec2 ? launch_gemm<BM, BN, BK, WM, WN, ST, 2, 0, 1>(st, chunk, c)                      \
              : launch_gemm<BM, BN, BK, WM, WN, ST, 1, 0, 1>(st, chunk, c);                     \
    break;
      TD_ROWSUM_CONFIGS(TD_ROWSUM_CASE)
#undef TD_ROWSUM_CASE
#define TD_ROWSUM_TMA_CASE(id, BM, BN, BK, WM, WN, ST, MINB)                                    \
  case id:                                                                                      \
    rc = tma_ok(chunk, c) ? launch_gemm_tma<BM, BN, BK, WM, WN, ST, 1, MINB>(st, chunk, c)      \
                          : (vec2 ? launch_gemm<BM, BN, BK, WM, WN, 3, 2, 0, 1>(st, chunk, c)   \
                                  : launch_gemm<BM, BN, BK, WM, WN, 3, 1, 0, 1>(st, chunk, c)); \
    break;
      TD_GEMM_TMA_CONFIGS(TD_ROWSUM_TMA_CASE)
#undef TD_ROWSUM_TMA_CASE
      default:
        set_error("mttkrp: unknown GEMM row-sum config %d", config);
    }
    if (rc) return rc;
    done += chunk;
  }
  return TD_OK;
}

__global__ void zero_rows_kernel(double* C, int64_t M, int64_t N, int64_t ldc, int64_t sC) {
  const int64_t b = blockIdx.y;
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    C[b * sC + (e / N) * ldc + e % N] = 0.0;
  }
}

static int zero_or_keep(cudaStream_t st, int64_t batch, int64_t M, int64_t N, double* C, int64_t ldc,
                        int64_t sC, int accumulate) {
  if (accumulate) return TD_OK;
  const int64_t total = M * N;
  dim3 grid((unsigned)std::min<int64_t>(ceil_div(total, 256), 4096), (unsigned)batch);
  zero_rows_kernel<<<grid, 256, 0, st>>>(C, M, N, ldc, sC);
  return check_launch("zero_rows_kernel");
}

}  // namespace td

extern "C" {

int td_dgemm(void* stream, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
             const double* B, int64_t ldb, double* C, int64_t ldc, int accumulate) {
  td::StreamDevice sd(stream);
  td::GemmArgs a{M, N, K, A, lda, 0, B, ldb, 0, C, ldc, 0, accumulate, 0, 0, 0, nullptr, 0};
  return td::dgemm_dispatch(td::as_stream(stream), 1, a);
}

int td_dgemm_config(void* stream, int config, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                    const double* B, int64_t ldb, double* C, int64_t ldc, int accumulate) {
  td::StreamDevice sd(stream);
  td::GemmArgs a{M, N, K, A, lda, 0, B, ldb, 0, C, ldc, 0, accumulate, 0, 0, 0, nullptr, 0};
  return td::dgemm_dispatch(td::as_stream(stream), 1, a, config);
}

int td_dgemm_batched(void* stream, int64_t batch, int64_t M, int64_t N, int64_t K, const double* A,
                     int64_t lda, int64_t strideA, const double* B, int64_t ldb, int64_t strideB,
                     double* C, int64_t ldc, int64_t strideC, int accumulate) {
  td::StreamDevice sd(stream);
  td::GemmArgs a{M, N, K, A, lda, strideA, B, ldb, strideB, C, ldc, strideC, accumulate, 0, 0, 0, nullptr, 0};
  int64_t done = 0;
  while (done < batch) {  // grid.y is limited to 65535
    const int64_t chunk = std::min<int64_t>(batch - done, 65535);
    td::GemmArgs c = a;
    c.A += done * strideA;
    c.B += done * strideB;
    c.C += done * strideC;
    int rc = td::dgemm_dispatch(td::as_stream(stream), chunk, c);
    if (rc) return rc;
    done += chunk;
  }
  return TD_OK;
}

int td_dgemm_grouped(void* stream, int count, const td_gemm_problem* problems, int accumulate) {
  TD_REQUIRE(count >= 0 && count <= TD_GEMM_GROUP_MAX && (count == 0 || problems),
             "dgemm_grouped: 0..%d problems", TD_GEMM_GROUP_MAX);
  td::StreamDevice sd(stream);
  const cudaStream_t st = td::as_stream(stream);
  td::GemmArgs args[TD_GEMM_GROUP_MAX];
  int n = 0;
  bool tma = true, seg2 = false;
  int64_t maxN = 0;
  for (int q = 0; q < count; ++q) {
    const td_gemm_problem& pr = problems[q];
    td::GemmArgs a{pr.M, pr.N, pr.K, pr.A, pr.lda, 0, pr.B, pr.ldb, 0, pr.C, pr.ldc, 0, accumulate, 0, 0, 0,
                   nullptr, 0};
    if (a.M <= 0 || a.N <= 0) continue;
    if (pr.K2 > 0) {
      if (a.K <= 0) {  // only the second segment
        a.K = pr.K2; a.A = pr.A2; a.lda = pr.lda2; a.B = pr.B2; a.ldb = pr.ldb2;
      } else {
        a.K2 = pr.K2; a.A2 = pr.A2; a.lda2 = pr.lda2; a.B2 = pr.B2; a.ldb2 = pr.ldb2;
        td::GemmArgs s2 = a;
        s2.K = a.K2; s2.A = a.A2; s2.lda = a.lda2; s2.B = a.B2; s2.ldb = a.ldb2;
        tma = tma && td::tma_ok(1, s2);
        seg2 = true;
      }
    }
    if (a.K <= 0) {  // nothing to multiply: only the Assign form writes zeros
      if (int rc = td::dgemm_dispatch(st, 1, a)) return rc;
      continue;
    }
    tma = tma && td::tma_ok(1, a);
    maxN = std::max(maxN, a.N);
    args[n++] = a;
  }
  if (n == 0) return TD_OK;
  if (!tma || (n == 1 && !seg2)) {  // one plain problem, or one TMA cannot address: separate launches
    for (int q = 0; q < n; ++q) {
      td::GemmArgs a = args[q];
      const int64_t K2 = a.K2;
      a.K2 = 0;
      if (int rc = td::dgemm_dispatch(st, 1, a)) return rc;
      if (K2 > 0) {  // the second segment accumulates after the first (same stream)
        a.K = K2; a.A = args[q].A2; a.lda = args[q].lda2; a.B = args[q].B2; a.ldb = args[q].ldb2;
        a.accumulate = 1;
        if (int rc = td::dgemm_dispatch(st, 1, a)) return rc;
      }
    }
    return TD_OK;
  }
  // the default TMA tiles (config 47 / 48 by N, gemm.cu default_tma_config)
  if (seg2) {
    if (maxN <= 32) return td::launch_gemm_tma_grouped<128, 32, 16, 32, 32, 3, 4, true>(st, n, args);
    return td::launch_gemm_tma_grouped<64, 64, 16, 32, 32, 3, 4, true>(st, n, args);
  }
  if (maxN <= 32) return td::launch_gemm_tma_grouped<128, 32, 16, 32, 32, 3, 4>(st, n, args);
  return td::launch_gemm_tma_grouped<64, 64, 16, 32, 32, 3, 4>(st, n, args);
}

int td_ttm(void* stream, int64_t I, int64_t J, int64_t K, int64_t L, const double* B, int64_t sBi,
           int64_t sBj, const double* C, int64_t ldc, double* Y, int64_t sYi, int64_t sYj,
           int accumulate) {
  // Y(i,j,:) = B(i,j,:) . C : rows (i,j) of B times C[K x L].
  if (sBi == J * sBj && sYi == J * sYj) {  // (i,j) rows flatten into one M = I*J GEMM
    return td_dgemm(stream, I * J, L, K, B, sBj, C, ldc, Y, sYj, accumulate);
  }
  return td_dgemm_batched(stream, I, J, L, K, B, sBj, sBi, C, ldc, 0, Y, sYj, sYi, accumulate);
}

}  // extern "C"
