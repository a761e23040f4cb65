// Fused MTTKRP leaf:  A(i,j) (+)= sum_k C(k,j) * sum_l B(i,k,l) * D(l,j)
// (reference statement pkg/src/tendist/algorithms.py:339-340, evaluated per
// point at cin.py:399-417 in the reference).
//
// A CTA owns one i, one 32-wide block of j and KPC consecutive k-blocks of
// ROWS = 32*WARPS rows.  For each k-block:
//     T[ROWS x 32] = B(i, kblk, :) . D[:, jblk]  on DMMA.8x8x4 tiles (every
//     warp 32 x 32, 16 DMMA per k4 slice) fed by one cp.async ring over
//     (k-block, l-tile) pairs, so the pipeline never drains between k-blocks;
//     epilogue: partial(j) += sum_k C(k,j) * T(k,j) in registers (C read from
//     a shared-memory copy loaded with the first stage, or from L2).
// At the end a fixed-order shuffle + shared-memory tree reduces the partial
// over the warps and the CTA writes it to a stream-ordered workspace
// [I][groups][R]; `mttkrp_reduce` then sums the groups of every A(i, :) in
// ascending order and writes (or accumulates) A.  No atomics: the summation
// order is a fixed function of the shape, runs are bitwise reproducible, and
// integer-valued inputs give exact results.
// B is streamed once from HBM (8 B per 64 flop at R = 32); D and C stay in L2.
// Unlike the GEMM, every B byte comes from DRAM, so the ring must keep many
// bytes in flight per SM: the configurations trade l-tile depth (BK), stages
// and resident CTAs per SM (MINB) against shared memory.
//
// The defaults run the same algorithm on the tuned GEMM body instead: a
// batched GEMM over i, M = k rows, N = j, K = l, whose epilogue (gemm.cu /
// gemm_tma.cuh, EPI = 1) does the Hadamard with C and the fixed-order sum over
// the tile's k rows; large shapes take whole-item CTAs plus a stream-K last
// wave (mttkrp_tma.cuh, config 22), smaller ones the per-i kernel on 256- or
// 128-row tiles (19 / 18) -- see default_mttkrp_config.  Round 1 measured
// 34.8 (TMA-fed body) and 33.4 (LDGSTS body) vs 30.9 TFLOP/s for the best
// fused configuration.
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "dmma.cuh"
#include "gemm.cuh"

namespace td {

constexpr int MK_R = 32;               // j columns per CTA
constexpr int MK_SD = MK_R + 4;        // D / C tile row stride (doubles)

template <int WARPS, int STAGES, int BK, bool CSMEM>
struct MkCfg {
  static constexpr int ROWS = WARPS * 32;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int SA = BK + 4;    // B-tile row stride: conflict-free fragment loads for BK = 8, 16
  static constexpr int A_STAGE = ROWS * SA;
  static constexpr int D_STAGE = BK * MK_SD;
  static constexpr int SMEM = STAGES * (A_STAGE + D_STAGE) * 8 + WARPS * MK_R * 8 + (CSMEM ? ROWS * MK_SD * 8 : 0);
};

struct MttkrpArgs {
  int64_t I, K, L, R;
  const double* B;
  int64_t sBi, sBk;
  const double* C;
  int64_t ldc;
  const double* D;
  int64_t ldd;
  double* A;
  int64_t lda;
  int accumulate;
  double* work;   // [I][groups][R] partials
  int kblocks, groups;
};

template <int WARPS, int STAGES, int KPC, int BK, bool CSMEM, int MINB, int VEC>
__global__ void __launch_bounds__(WARPS * 32, MINB) mttkrp_kernel(MttkrpArgs p) {
  using Cfg = MkCfg<WARPS, STAGES, BK, CSMEM>;
  static_assert(!CSMEM || KPC == 1, "the shared C block holds one k-block");
  constexpr int ROWS = Cfg::ROWS;
  constexpr int SA = Cfg::SA;
  extern __shared__ __align__(128) double smem[];
  double* Bs = smem;
  double* Ds = smem + STAGES * Cfg::A_STAGE;
  double* red = Ds + STAGES * Cfg::D_STAGE;  // [WARPS][32]
  double* Cs = red + WARPS * MK_R;            // [ROWS][MK_SD] C block (CSMEM)

  const int64_t i = blockIdx.x / p.groups;
  const int grp = blockIdx.x % p.groups;
  const int kb0 = grp * KPC;
  const int nkb = min(KPC, p.kblocks - kb0);
  const int64_t j0 = int64_t(blockIdx.y) * MK_R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* __restrict__ Bi = p.B + i * p.sBi;
  const int64_t K = p.K, L = p.L, R = p.R;
  const int ltiles = (int)ceil_div(L, BK);
  const int total = nkb * ltiles;

  // fixed-address fast path (full k-block, full l tile, full 32-wide j block)
  constexpr int FB_PER_ROW = BK / VEC, FD_PER_ROW = MK_R / VEC;
  constexpr int FB_ITERS = ROWS * FB_PER_ROW / Cfg::THREADS, FB_STEP = Cfg::THREADS / FB_PER_ROW;
  constexpr int FD_ITERS = BK * FD_PER_ROW / Cfg::THREADS, FD_STEP = Cfg::THREADS / FD_PER_ROW;
  constexpr bool FD_FAST = FD_ITERS * Cfg::THREADS == BK * FD_PER_ROW && FD_ITERS > 0;
  static_assert(FB_ITERS * Cfg::THREADS == ROWS * FB_PER_ROW, "mttkrp tile / thread mismatch");
  const int fb_r = tid / FB_PER_ROW, fb_c = (tid % FB_PER_ROW) * VEC;
  const int fd_r = tid / FD_PER_ROW, fd_c = (tid % FD_PER_ROW) * VEC;
  const bool jfull = j0 + MK_R <= R;
  const double* fd_base = p.D + int64_t(fd_r) * p.ldd + j0 + fd_c;
  const int64_t fb_step = int64_t(FB_STEP) * p.sBk, fd_step = int64_t(FD_STEP) * p.ldd;

  auto load = [&](int stage, int t) {
    const int64_t k0 = int64_t(kb0 + t / ltiles) * ROWS;
    const int64_t l0 = int64_t(t % ltiles) * BK;
    double* bs = Bs + stage * Cfg::A_STAGE;
    double* ds = Ds + stage * Cfg::D_STAGE;
    if constexpr (CSMEM) {
      if (t == 0) {  // the CTA's C block rides in the first stage: the epilogue reads smem, not L2
        for (int c = tid; c < ROWS * MK_R; c += Cfg::THREADS) {
          const int r = c / MK_R, col = c % MK_R;
          const int64_t gk = k0 + r, gj = j0 + col;
          const bool ok = gk < K && gj < R;
          cp_async_f64<1>(Cs + r * MK_SD + col, ok ? p.C + gk * p.ldc + gj : p.C, ok ? 1 : 0);
        }
      }
    }
    if (jfull && k0 + ROWS <= K && l0 + BK <= L) {
      const double* b = Bi + (k0 + fb_r) * p.sBk + fb_c + l0;
#pragma unroll
      for (int it = 0; it < FB_ITERS; ++it)
        cp_async_f64<VEC>(bs + (fb_r + it * FB_STEP) * SA + fb_c, b + it * fb_step, VEC);
      if constexpr (FD_FAST) {
        const double* d = fd_base + l0 * p.ldd;
#pragma unroll
        for (int it = 0; it < FD_ITERS; ++it)
          cp_async_f64<VEC>(ds + (fd_r + it * FD_STEP) * MK_SD + fd_c, d + it * fd_step, VEC);
        return;
      }
    } else {
      constexpr int B_PER_ROW = BK / VEC;
#pragma unroll 4
      for (int c = tid; c < ROWS * B_PER_ROW; c += Cfg::THREADS) {
        const int r = c / B_PER_ROW, col = (c % B_PER_ROW) * VEC;
        const int64_t gk = k0 + r, gl = l0 + col;
        int valid = 0;
        const double* src = p.B;
        if (gk < K && gl < L) {
          valid = (int)(L - gl < VEC ? L - gl : VEC);
          src = Bi + gk * p.sBk + gl;
        }
        cp_async_f64<VEC>(bs + r * SA + col, src, valid);
      }
    }
    constexpr int D_PER_ROW = MK_R / VEC;
    for (int c = tid; c < BK * D_PER_ROW; c += Cfg::THREADS) {
      const int r = c / D_PER_ROW, col = (c % D_PER_ROW) * VEC;
      const int64_t gl = l0 + r, gj = j0 + col;
      int valid = 0;
      const double* src = p.D;
      if (gl < L && gj < R) {
        valid = (int)(R - gj < VEC ? R - gj : VEC);
        src = p.D + gl * p.ldd + gj;
      }
      cp_async_f64<VEC>(ds + r * MK_SD + col, src, valid);
    }
  };

  double acc[4][4][2];
  double part[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) part[a][0] = part[a][1] = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) load(s, s);
    cp_async_commit();
  }
  const int arow = warp * 32 + (lane >> 2);
  const int acol = lane & 3;
  const int brow = lane & 3;
  const int bcol = lane >> 2;

  for (int t = 0; t < total; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < total) load(nt % STAGES, nt);
      cp_async_commit();
    }
    const double* bs = Bs + (t % STAGES) * Cfg::A_STAGE;
    const double* ds = Ds + (t % STAGES) * Cfg::D_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = bs[(arow + m * 8) * SA + kk + acol];
#pragma unroll
      for (int n = 0; n < 4; ++n) bf[n] = ds[(kk + brow) * MK_SD + bcol + n * 8];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
    if (t % ltiles == ltiles - 1) {  // k-block finished: Hadamard with C, reduce over its k rows
      const int64_t k0 = int64_t(kb0 + t / ltiles) * ROWS;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int64_t k = k0 + warp * 32 + m * 8 + (lane >> 2);
        const bool kin = k < K;
        const double* crow = p.C + k * p.ldc;
        const double* srow = Cs + (warp * 32 + m * 8 + (lane >> 2)) * MK_SD;
#pragma unroll
        for (int n = 0; n < 4; ++n) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jl = n * 8 + (lane & 3) * 2 + h;
            const int64_t j = j0 + jl;
            if (kin && j < R) part[n][h] += (CSMEM ? srow[jl] : crow[j]) * acc[m][n][h];
            acc[m][n][h] = 0.0;
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  // reduce partials: lanes sharing (lane & 3) hold the same columns
#pragma unroll
  for (int n = 0; n < 4; ++n)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = part[n][h];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      part[n][h] = v;
    }
  if (lane < 4) {
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[warp * MK_R + n * 8 + lane * 2 + h] = part[n][h];
  }
  __syncthreads();
  if (tid < MK_R) {
    double v = red[tid];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) v += red[w * MK_R + tid];
    const int64_t j = j0 + tid;
    if (j < R) p.work[(i * p.groups + grp) * R + j] = v;
  }
}

// A(i, j) (+)= sum over the CTA groups of row i, ascending (fixed order)
__global__ void mttkrp_reduce(const double* __restrict__ work, int groups, int64_t I, int64_t R, double* A,
                              int64_t lda, int accumulate) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < I * R; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / R, j = e - (e / R) * R;
    const double* w = work + i * groups * R + j;
    double v = 0.0;
    for (int g = 0; g < groups; ++g) v += w[int64_t(g) * R];
    double* dst = A + i * lda + j;
    *dst = accumulate ? *dst + v : v;
  }
}

static bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

static int retain_pool() {  // keep the stream-ordered pool's memory across syncs
  int dev = 0;
  TD_CUDA(cudaGetDevice(&dev));
  static bool retained[64] = {false};
  if (dev < 64 && !retained[dev]) {
    cudaMemPool_t pool;
    TD_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    TD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    retained[dev] = true;
  }
  return TD_OK;
}

template <int WARPS, int STAGES, int KPC, int BK, bool CSMEM, int MINB>
static int launch_mttkrp(cudaStream_t st, MttkrpArgs a, bool vec2) {
  using Cfg = MkCfg<WARPS, STAGES, BK, CSMEM>;
  a.kblocks = (int)std::max<int64_t>(1, ceil_div(a.K, Cfg::ROWS));
  a.groups = (int)ceil_div(a.kblocks, KPC);
  TD_REQUIRE(a.I * a.groups < (1ll << 31), "mttkrp: grid too large");
  if (int rc = retain_pool()) return rc;
  TD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.work), sizeof(double) * a.I * a.groups * a.R, st));
  if (a.K > 0) {
    dim3 grid((unsigned)(a.I * a.groups), (unsigned)ceil_div(a.R, MK_R));
    if (vec2) {
      auto kern = mttkrp_kernel<WARPS, STAGES, KPC, BK, CSMEM, MINB, 2>;
      TD_CUDA(ensure_smem(kern, Cfg::SMEM));
      kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(a);
    } else {
      auto kern = mttkrp_kernel<WARPS, STAGES, KPC, BK, CSMEM, MINB, 1>;
      TD_CUDA(ensure_smem(kern, Cfg::SMEM));
      kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(a);
    }
    if (int rc = check_launch("mttkrp_kernel")) return rc;
  } else {
    TD_CUDA(cudaMemsetAsync(a.work, 0, sizeof(double) * a.I * a.groups * a.R, st));
  }
  const int64_t outs = a.I * a.R;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(outs, 256), 148 * 8));
  mttkrp_reduce<<<blocks, 256, 0, st>>>(a.work, a.groups, a.I, a.R, a.A, a.lda, a.accumulate);
  int rc = check_launch("mttkrp_reduce");
  TD_CUDA(cudaFreeAsync(a.work, st));
  return rc;
}

// MTTKRP as a batched GEMM over i whose epilogue does the Hadamard with C and
// the sum over the k rows of each tile (gemm.cu, EPI = 1): the tile loop is
// the tuned GEMM body, so B streams at the GEMM's rate.
// Workspace of the GEMM-body MTTKRP, cached per (device, stream): the
// [I][groups][R] partials and the per-(i, N-tile) arrival counters of the
// fused finish (zeroed once; the last CTA of each row resets its counter).
// One stream's launches are ordered, so they can share it; growth happens on
// the first (largest) launch, outside any CUDA-graph capture.
struct MkScratch {
  double* work = nullptr;
  size_t work_bytes = 0;
  int* counters = nullptr;
  size_t counter_bytes = 0;
};

static int mk_scratch(cudaStream_t st, size_t work_bytes, size_t counter_bytes, double** work, int** counters) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, MkScratch> cache;
  int dev = 0;
  TD_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  MkScratch& s = cache[{dev, st}];
  if (s.work_bytes < work_bytes || s.counter_bytes < counter_bytes) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    TD_CUDA(cudaStreamIsCapturing(st, &cap));
    TD_REQUIRE(cap == cudaStreamCaptureStatusNone,
               "mttkrp: workspace must grow during CUDA-graph capture (run the launch once before capturing)");
    TD_CUDA(cudaStreamSynchronize(st));
    if (s.work) TD_CUDA(cudaFree(s.work));
    if (s.counters) TD_CUDA(cudaFree(s.counters));
    s.work_bytes = std::max(work_bytes, s.work_bytes);
    s.counter_bytes = std::max(counter_bytes, s.counter_bytes);
    TD_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.work), s.work_bytes));
    TD_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.counters), s.counter_bytes));
    TD_CUDA(cudaMemsetAsync(s.counters, 0, s.counter_bytes, st));
  }
  *work = s.work;
  *counters = s.counters;
  return TD_OK;
}

static int launch_mttkrp_gemm(cudaStream_t st, MttkrpArgs a, int gemm_config) {
  const int bm = dgemm_rowsum_tile_rows(gemm_config);
  TD_REQUIRE(bm > 0, "mttkrp: unknown GEMM row-sum config %d", gemm_config);
  a.groups = (int)std::max<int64_t>(1, ceil_div(a.K, bm));
  int* counters = nullptr;
  if (int rc = mk_scratch(st, sizeof(double) * std::max<int64_t>(1, a.I * a.groups * a.R),
                          sizeof(int) * std::max<int64_t>(1, a.I * a.R), &a.work, &counters))
    return rc;
  int rc = TD_OK;
  bool fused = false;
  if (a.K > 0 && a.L > 0) {
    GemmArgs g{};
    g.M = a.K; g.N = a.R; g.K = a.L;
    g.A = a.B; g.lda = a.sBk; g.sA = a.sBi;
    g.B = a.D; g.ldb = a.ldd; g.sB = 0;
    g.C = a.work; g.ldc = a.R; g.sC = int64_t(a.groups) * a.R;
    g.H = a.C; g.ldh = a.ldc;
    fused = dgemm_rowsum_fusable(gemm_config, a.I, g);
    if (fused) {  // the last CTA of every (i, N-tile) finishes the sum and writes A
      g.counters = counters;
      g.out = a.A; g.ldo = a.lda; g.out_acc = a.accumulate;
    }
    rc = dgemm_rowsum(st, gemm_config, a.I, g);
  } else {
    TD_CUDA(cudaMemsetAsync(a.work, 0, sizeof(double) * a.I * a.groups * a.R, st));
  }
  if (rc == TD_OK && !fused) {
    const int64_t outs = a.I * a.R;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(outs, 256), 148 * 8));
    mttkrp_reduce<<<blocks, 256, 0, st>>>(a.work, a.groups, a.I, a.R, a.A, a.lda, a.accumulate);
    rc = check_launch("mttkrp_reduce");
  }
  return rc;
}

// Stream-K MTTKRP (gemm.cu / mttkrp_tma.cuh); `required` = false lets shapes
// the plan rejects fall back to the per-i GEMM body.
static int launch_mttkrp_streamk(cudaStream_t st, const MttkrpArgs& a, int variant, bool required) {
  const MkSplitArgs s{a.I, a.K, a.L, a.R, a.B, a.sBi, a.sBk, a.C, a.ldc, a.D, a.ldd, a.A, a.lda, a.accumulate};
  int ctas = 0;
  const int64_t words = mttkrp_streamk_plan(variant, s, &ctas);
  if (words == 0) {
    TD_REQUIRE(!required, "mttkrp: stream-K variant %d cannot take this shape", variant);
    return launch_mttkrp_gemm(st, a, 51);
  }
  double* work = nullptr;
  int* counters = nullptr;
  if (int rc = mk_scratch(st, sizeof(double) * words, sizeof(int), &work, &counters)) return rc;
  return mttkrp_streamk(st, variant, s, ctas, work);
}

// configurations 0-7: the fused kernel above, <WARPS, STAGES, k-blocks per CTA,
// l per stage, C in smem, CTAs per SM>; 8-13, 15, 18: the GEMM body with the
// row-sum epilogue on GEMM tile configs 26, 29, 21, 20, 34, 35, 43, 48 (the
// last two TMA-fed)
// Default by the number of 256-row items per wave of resident CTAs (2 per SM),
// measured at K = L = 1024, R = 32 (tools/mttkrp_clocks.py, TFLOP/s):
//   I      waves | 18 (128-row, 3/SM) | 19 (256-row, 2/SM) | 22 (DP + stream-K)
//   1024   13.8  | 34.95              | 35.29              | 35.42
//   256     3.5  | 33.59              | 34.41              | 33.84
//   128     1.7  | 32.23              | 29.56              | 32.05
//   4096   55    | 35.53              | 35.81              | --
// Deeper rings at 256 rows do not help (BK 8: 6 stages 34.93, 5 stages 35.02;
// the stream-K form with BK 8 / 6 stages 34.67), so the per-k-tile overhead,
// not the bytes in flight, is what the wider l-tiles save.  A dedicated producer
// warp (warp-specialised 128-row tiles, 4 compute warps + 1 TMA warp, 3 CTAs/SM,
// all slots in flight) is slower too: 34.53 (BK 16) / 33.75 (BK 8, 6 stages) vs
// 34.99 with the issuing thread inside warp 0; 35.07 vs 35.53 at I = 4096.
// Round-1 baseline (the per-i kernel, fused kernel configs 0-7 and the LDGSTS
// bodies): 34.8 / 30.9 / 33.4.
static int default_mttkrp_config(const MttkrpArgs& a) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = a.I * ceil_div(std::max<int64_t>(a.K, 1), 256) * ceil_div(a.R, 32);
  const int64_t waves = items / (2 * int64_t(sms));
  if (waves >= 8) return 22;
  if (waves >= 3) return 19;
  return 18;
}

int mttkrp_dispatch(cudaStream_t st, const MttkrpArgs& a, int config) {
  const bool vec2 = al16(a.B) && al16(a.D) && a.sBi % 2 == 0 && a.sBk % 2 == 0 && a.ldd % 2 == 0;
  // 18 / 19: the TMA-fed GEMM body (128- / 256-row tiles, 16-wide l-tiles, 3
  // stages); 22: whole-item CTAs plus a stream-K last wave (mttkrp_tma.cuh).
  // Operands the copy engine cannot address take the LDGSTS body.
  switch (config < 0 ? default_mttkrp_config(a) : config) {
    case 0: return launch_mttkrp<4, 4, 1, 16, false, 2>(st, a, vec2);
    case 1: return launch_mttkrp<4, 3, 1, 16, true, 2>(st, a, vec2);
    case 2: return launch_mttkrp<4, 3, 2, 16, false, 2>(st, a, vec2);
    case 3: return launch_mttkrp<4, 5, 1, 8, false, 3>(st, a, vec2);
    case 4: return launch_mttkrp<4, 6, 1, 8, false, 3>(st, a, vec2);
    case 5: return launch_mttkrp<4, 4, 1, 8, true, 3>(st, a, vec2);
    case 6: return launch_mttkrp<4, 3, 1, 16, false, 3>(st, a, vec2);
    case 7: return launch_mttkrp<4, 8, 1, 8, false, 2>(st, a, vec2);
    case 8: return launch_mttkrp_gemm(st, a, 26);
    case 9: return launch_mttkrp_gemm(st, a, 29);
    case 10: return launch_mttkrp_gemm(st, a, 21);
    case 11: return launch_mttkrp_gemm(st, a, 20);
    case 12: return launch_mttkrp_gemm(st, a, 34);
    case 13: return launch_mttkrp_gemm(st, a, 35);
    case 15: return launch_mttkrp_gemm(st, a, 43);
    case 18: return launch_mttkrp_gemm(st, a, 48);
    case 19: return launch_mttkrp_gemm(st, a, 51);
    case 22: return launch_mttkrp_streamk(st, a, 0, config >= 0);
    default:
      set_error("mttkrp: unknown config %d", config);
      return TD_ERR_ARG;
  }
}

}  // namespace td

extern "C" int td_mttkrp_config(void* stream, int config, int64_t I, int64_t K, int64_t L, int64_t R,
                                const double* B, int64_t sBi, int64_t sBk, const double* C, int64_t ldc,
                                const double* D, int64_t ldd, double* A, int64_t lda, int accumulate) {
  using namespace td;
  if (I <= 0 || R <= 0) return TD_OK;
  StreamDevice sd(stream);
  TD_REQUIRE(I <= 2147483647, "mttkrp: I too large");
  MttkrpArgs a{I, K, L, R, B, sBi, sBk, C, ldc, D, ldd, A, lda, accumulate, nullptr, 0, 0};
  return mttkrp_dispatch(as_stream(stream), a, config);
}

extern "C" int td_mttkrp(void* stream, int64_t I, int64_t K, int64_t L, int64_t R, const double* B,
                         int64_t sBi, int64_t sBk, const double* C, int64_t ldc, const double* D,
                         int64_t ldd, double* A, int64_t lda, int accumulate) {
  return td_mttkrp_config(stream, -1, I, K, L, R, B, sBi, sBk, C, ldc, D, ldd, A, lda, accumulate);
}
