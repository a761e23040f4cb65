// MTTKRP with a stream-K last wave, on the per-i GEMM formulation (included by
// gemm.cu after gemm_tma.cuh):
//
//     T(i, k, j) = sum_l B(i, k, l) D(l, j)        (DMMA.8x8x4, M = k rows, N = j, K = l)
//     A(i, j)   (+)= sum_k C(k, j) T(i, k, j)      (row-sum epilogue)
//
// An item is one (i, BM k-rows, 32 j) tile -- B(i, k0:k0+BM, :) is one
// contiguous run -- and a unit is one BK-wide l-tile of an item.  The first
// n_dp blocks (all full waves of resident CTAs but the last) take one whole
// item each; the last n_sk blocks (one per resident slot) walk equal
// contiguous runs [c U / n_sk, (c+1) U / n_sk) of the remaining U units with
// ONE TMA ring running across item boundaries, so the last wave has no tail
// (the per-i kernel's 4096-8192 short CTAs lost ~1.5 % to it).  At each item
// end (or the end of its range) every warp does its own row-sum epilogue --
// Hadamard with C, fixed shuffle tree over its 32 rows -- and stores a 32-wide
// partial, no CTA-wide barrier: the item's head (first unit) into the item's
// slot, a continuation (an sk block starting mid-item) into the block's own
// slot.  `mttkrp_st_reduce` sums, per output, the warp groups of every k-tile
// in ascending order (head + the following sk blocks' continuations in block
// order), in four contiguous quarters combined as (q0 + q1) + (q2 + q3).
// No atomics: the order is a fixed function of the shape and the resident-CTA
// count, runs are bitwise reproducible, integer-valued inputs exact.
//
// Not kept (tools/mttkrp_configs.py, round 2): the same split-K over the whole
// (k, l) plane with M = i (Khatri-Rao rows scaled in registers, one partial
// per CTA) -- bit-exact but 7.4 ms vs 1.97: a 128-row box of i rows 8 MB
// apart touches 128 pages per copy and B streams at 1.2 TB/s.
#pragma once

namespace td {

template <int BM, int BK, int STAGES>
struct StCfg {
  static constexpr int BN = 32;
  static constexpr int THREADS = BM;  // one warp per 32 rows, each warp 32 x 32
  static constexpr int FM = 4, FN = 4;
  static constexpr int A_STAGE = BM * BK;  // doubles
  static constexpr int B_STAGE = BK * BN;
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 128;
  static_assert(BM % 32 == 0 && BK % 4 == 0, "stream-K MTTKRP tile");
};

struct StParams {
  int64_t dp_units;        // units of the whole-item blocks (n_dp * ltiles)
  int64_t tail_units;      // units of the remaining items, spread over the sk CTAs
  int n_dp, n_sk;
  int ltiles, tiles_m, tiles_n;
  int64_t K, R, ldc;
  const double* C;
  double* work;            // [I][tiles_m * BM / 32][tiles_n * 32]: item heads
  double* cont;            // [n_sk][BM / 32][32]: the continuation of an sk CTA's first item
};

__device__ __forceinline__ int64_t st_begin(int64_t units, int ctas, int c) { return units * c / ctas; }

template <int BM, int BK, int STAGES, int MINB>
__global__ void __launch_bounds__(BM, MINB)
mttkrp_st_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmD, StParams p) {
  using Cfg = StCfg<BM, BK, STAGES>;
  extern __shared__ __align__(128) unsigned char st_smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(st_smem_raw) + 127) & ~uintptr_t(127));
  double* As = smem;
  double* Ds = As + STAGES * Cfg::A_STAGE;

  const int sk = int(blockIdx.x) - p.n_dp;  // >= 0: a stream-K block over the tail items
  const int64_t begin = sk < 0 ? int64_t(blockIdx.x) * p.ltiles
                               : p.dp_units + st_begin(p.tail_units, p.n_sk, sk);
  const int n = sk < 0 ? p.ltiles : int(st_begin(p.tail_units, p.n_sk, sk + 1) - st_begin(p.tail_units, p.n_sk, sk));
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int groups = p.tiles_m * (BM / 32);
  const int64_t rpad = int64_t(p.tiles_n) * Cfg::BN;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // item x = (i * tiles_m + tm) * tiles_n + tn; both the producer (thread 0)
  // and the consumers step their (i, tm, tn, l-tile) counters incrementally
  // (no 64-bit division on the issue path)
  struct Pos {
    int i, tm, tn, l;
    __device__ void next(const StParams& q) {
      if (++l < q.ltiles) return;
      l = 0;
      if (++tn < q.tiles_n) return;
      tn = 0;
      if (++tm < q.tiles_m) return;
      tm = 0;
      ++i;
    }
  };
  Pos start;
  {
    const int64_t x = begin / p.ltiles;
    const int64_t it = x / p.tiles_n;
    start.l = int(begin - x * p.ltiles);
    start.tn = int(x - it * p.tiles_n);
    start.tm = int(it % p.tiles_m);
    start.i = int(it / p.tiles_m);
  }
  Pos pp = start;
  auto issue = [&](int t) {
    const int s = t % STAGES;
    mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
    tma_load_4d(As + s * Cfg::A_STAGE, &tmB, 0, pp.tm * BM, pp.l * (BK / 4), pp.i, &full[s]);
    tma_load_4d(Ds + s * Cfg::B_STAGE, &tmD, 0, pp.l * BK, pp.tn * (Cfg::BN / 4), 0, &full[s]);
    pp.next(p);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s)
      if (s < n) issue(s);
  }

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int a_off = (warp * 32 + (lane >> 2)) * 4 + (lane & 3);
  const int b_off = ((lane >> 2) / 4) * BK * 4 + (lane & 3) * 4 + ((lane >> 2) & 3);

  Pos cp = start;
  bool head = cp.l == 0;  // this CTA owns the item's first unit (slot 0)
  for (int t = 0; t < n; ++t) {
    const int s = t % STAGES;
    mbar_wait(&full[s], (t / STAGES) & 1);
    if (tid == 0 && t + STAGES - 1 < n) {
      if (t >= 1) mbar_wait(&empty[(t - 1) % STAGES], ((t - 1) / STAGES) & 1);
      issue(t + STAGES - 1);
    }
    const double* as = As + s * Cfg::A_STAGE + a_off;
    const double* bs = Ds + s * Cfg::B_STAGE + b_off;
#pragma unroll
    for (int kq = 0; kq < BK / 4; ++kq) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) af[i] = as[kq * BM * 4 + i * 32];
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) bf[j] = bs[kq * 16 + j * 2 * BK * 4];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (cp.l == p.ltiles - 1 || t == n - 1) {  // item done in this CTA: the warp's row-sum partial
      const int tn = cp.tn, tm = cp.tm;
      const int64_t i = cp.i;
      double part[Cfg::FN][2];
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) part[j][0] = part[j][1] = 0.0;
#pragma unroll
      for (int f = 0; f < Cfg::FM; ++f) {
        const int64_t r = int64_t(tm) * BM + warp * 32 + f * 8 + (lane >> 2);
        const double* crow = p.C + r * p.ldc;
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int64_t c = int64_t(tn) * Cfg::BN + j * 8 + (lane & 3) * 2;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double cv = (r < p.K && c + h < p.R) ? __ldg(crow + c + h) : 0.0;
            part[j][h] += cv * acc[f][j][h];
            acc[f][j][h] = 0.0;
          }
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
      if (lane < 4) {
        double* w = head ? p.work + (i * groups + tm * (BM / 32) + warp) * rpad + tn * Cfg::BN
                         : p.cont + (int64_t(sk) * (BM / 32) + warp) * Cfg::BN;
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
          *reinterpret_cast<double2*>(w + j * 8 + lane * 2) = make_double2(part[j][0], part[j][1]);
      }
      head = true;
    }
    cp.next(p);
  }
}

// One CTA of 4 warps per (output row i, 32-column tile): warp q sums the q-th
// contiguous quarter of the row's 32-row groups in ascending order (each the
// item head plus, for a tail item cut by sk range boundaries, the
// continuations of the following sk CTAs in order), then (q0 + q1) + (q2 + q3).
__global__ void __launch_bounds__(128) mttkrp_st_reduce(const double* __restrict__ work, StParams p, int bm,
                                                       double* __restrict__ A, int64_t lda, int accumulate) {
  __shared__ double part[4][32];
  const int64_t i = blockIdx.x;
  const int tn = blockIdx.y;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int per_tile = bm / 32;
  const int groups = p.tiles_m * per_tile;
  const int64_t rpad = int64_t(p.tiles_n) * 32;
  const double* src = work + i * groups * rpad + tn * 32 + lane;
  const int g0 = groups * q / 4, g1 = groups * (q + 1) / 4;
  double v = 0.0;
  for (int g = g0; g < g1; ++g) {
    double x = __ldcg(src + int64_t(g) * rpad);
    const int64_t first = ((i * p.tiles_m + g / per_tile) * p.tiles_n + tn) * p.ltiles - p.dp_units;
    if (first >= 0) {  // a tail item: sk CTAs c0 < c <= c1 hold its continuations
      const int64_t c0 = ((first + 1) * p.n_sk - 1) / p.tail_units;
      const int64_t c1 = ((first + p.ltiles) * p.n_sk - 1) / p.tail_units;
      for (int64_t c = c0 + 1; c <= c1; ++c) x += __ldcg(p.cont + (c * per_tile + g % per_tile) * 32 + lane);
    }
    v += x;
  }
  part[q][lane] = v;
  __syncthreads();
  if (q == 0) {
    const double t = (part[0][lane] + part[1][lane]) + (part[2][lane] + part[3][lane]);
    const int64_t col = int64_t(tn) * 32 + lane;
    if (col < p.R) {
      double* dst = A + i * lda + col;
      *dst = accumulate ? *dst + t : t;
    }
  }
}

// Resident CTAs of a kernel on the current device (cached per kernel, device).
template <typename Kernel>
static int resident_ctas(Kernel kern, int threads, int smem) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  const uint64_t key = (reinterpret_cast<uintptr_t>(reinterpret_cast<const void*>(kern)) << 8) ^ uint64_t(dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0, sms = 0;
  if (ensure_smem(kern, smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = per_sm * sms;
  return per_sm * sms;
}

template <int BM, int BK, int STAGES, int MINB>
static int64_t st_plan(const MkSplitArgs& a, int* ctas) {
  using Cfg = StCfg<BM, BK, STAGES>;
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!al(a.B) || !al(a.D) || a.sBi % 2 || a.sBk % 2 || a.ldd % 2 || a.L % 4 || a.R % 4 || a.K < 1 ||
      a.L < 1 || a.I >= (1ll << 31) || a.K >= (1ll << 31) || a.L >= (1ll << 31) || tma_encoder() == nullptr)
    return 0;
  const int slots = resident_ctas(mttkrp_st_kernel<BM, BK, STAGES, MINB>, Cfg::THREADS, Cfg::SMEM_BYTES);
  const int64_t tiles_m = ceil_div(a.K, BM), tiles_n = ceil_div(a.R, Cfg::BN);
  const int64_t items = a.I * tiles_m * tiles_n;
  if (slots <= 0) return 0;
  // whole-item blocks for all but the last `dp_back` full waves; the rest stream-K over one wave
  static const int dp_back = [] {
    const char* e = std::getenv("TD_MK_DP_BACK");
    return e ? std::atoi(e) : 1;
  }();
  const int64_t waves = items / slots;
  const int64_t n_dp = std::max<int64_t>(0, waves - dp_back) * slots;
  const int64_t tail_units = (items - n_dp) * ceil_div(a.L, BK);
  const int64_t n_sk = std::min<int64_t>(slots, tail_units);
  *ctas = (int)n_dp;
  return a.I * tiles_m * (BM / 32) * tiles_n * Cfg::BN + n_sk * (BM / 32) * Cfg::BN;
}

template <int BM, int BK, int STAGES, int MINB>
static int st_launch(cudaStream_t st, const MkSplitArgs& a, int ctas, double* work) {
  using Cfg = StCfg<BM, BK, STAGES>;
  auto kern = mttkrp_st_kernel<BM, BK, STAGES, MINB>;
  TD_CUDA(ensure_smem(kern, Cfg::SMEM_BYTES));
  CUtensorMap mb, md;
  if (int rc = make_sliced_map(&mb, a.B, a.K, a.L, a.sBk, a.I, a.sBi, BM, BK)) return rc;
  if (int rc = make_sliced_map(&md, a.D, a.L, a.R, a.ldd, 1, 0, BK, Cfg::BN)) return rc;
  const int slots = resident_ctas(kern, Cfg::THREADS, Cfg::SMEM_BYTES);
  StParams p;
  p.ltiles = (int)ceil_div(a.L, BK);
  p.tiles_m = (int)ceil_div(a.K, BM);
  p.tiles_n = (int)ceil_div(a.R, Cfg::BN);
  const int64_t items = a.I * p.tiles_m * p.tiles_n;
  p.n_dp = ctas;  // from st_plan
  p.dp_units = int64_t(p.n_dp) * p.ltiles;
  p.tail_units = (items - p.n_dp) * p.ltiles;
  p.n_sk = (int)std::min<int64_t>(slots, p.tail_units);
  p.K = a.K;
  p.R = a.R;
  p.ldc = a.ldc;
  p.C = a.C;
  p.work = work;
  p.cont = work + a.I * p.tiles_m * (BM / 32) * p.tiles_n * Cfg::BN;
  TD_REQUIRE(int64_t(p.n_dp) + p.n_sk < (1ll << 31), "mttkrp: grid too large");
  kern<<<(unsigned)(p.n_dp + p.n_sk), Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(mb, md, p);
  if (int rc = check_launch("mttkrp_st_kernel")) return rc;
  mttkrp_st_reduce<<<dim3((unsigned)a.I, (unsigned)p.tiles_n), 128, 0, st>>>(work, p, BM, a.A, a.lda, a.accumulate);
  return check_launch("mttkrp_st_reduce");
}

// variants: <BM, BK, STAGES, CTAs per SM>
// (A separate straight-line loop for the whole-item blocks, epilogue after it,
// measured 35.20 vs 35.42 TFLOP/s: one loop body for both kinds of block stays.)
// (measured at 1024^3 r32 as pure stream-K, before the whole-item blocks:
// 128x16 / 3 stages / 3 per SM 32.5, the same at <= 128 registers 33.2,
// 128x8 / 5 / 4 31.5, 128x8 / 6 / 3 31.8, 256x16 / 3 / 2 34.8)
#define TD_MK_SPLITK_VARIANTS(X) \
  X(0, 256, 16, 3, 2)

int64_t mttkrp_streamk_plan(int variant, const MkSplitArgs& a, int* ctas) {
  switch (variant) {
#define TD_SK_PLAN(id, BM, BK, ST, MINB) \
  case id:                               \
    return st_plan<BM, BK, ST, MINB>(a, ctas);
    TD_MK_SPLITK_VARIANTS(TD_SK_PLAN)
#undef TD_SK_PLAN
    default:
      return 0;
  }
}

int mttkrp_streamk(cudaStream_t st, int variant, const MkSplitArgs& a, int ctas, double* work) {
  switch (variant) {
#define TD_SK_LAUNCH(id, BM, BK, ST, MINB) \
  case id:                                 \
    return st_launch<BM, BK, ST, MINB>(st, a, ctas, work);
    TD_MK_SPLITK_VARIANTS(TD_SK_LAUNCH)
#undef TD_SK_LAUNCH
    default:
      set_error("mttkrp: unknown stream-K variant %d", variant);
      return TD_ERR_ARG;
  }
}

}  // namespace td
