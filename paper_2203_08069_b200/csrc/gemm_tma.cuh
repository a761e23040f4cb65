// TMA-fed variant of the DMMA GEMM body (included by gemm.cu).
//
// Operand tiles arrive by `cp.async.bulk.tensor` (one elected thread issues
// two bulk copies per stage, completion counted on an mbarrier with
// expect_tx) instead of per-thread LDGSTS.  The tensor maps are k4-sliced
// views of the row-major operands, so the copies land in the layouts the
// DMMA fragments want:
//   A tile  [BK/4][BM][4]   (view dims {4 k, M, K/4, batch}, strides {lda, 4, sA})
//   B tile  [BN/4][BK][4]   (view dims {4 n, K, N/4, batch}, strides {ldb, 4, sB})
// A fragment (8 rows x 4 k) and B fragment (4 k x 8 cols) of a warp are then
// two contiguous 128-byte runs: conflict-free LDS.64 with no padding, and the
// out-of-bounds parts of edge tiles are zero-filled by the copy engine (no
// predicated loads).  Needs 16-byte aligned bases, even leading dimensions
// and K, N multiples of 4; gemm.cu falls back to the LDGSTS kernel otherwise.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

namespace td {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_4d(void* sdst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(sdst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB = 0>
struct TmaCfg {
  static constexpr int WARPS_M = BM / WM;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int FM = WM / 8;
  static constexpr int FN = WN / 8;
  static constexpr int A_STAGE = BM * BK;  // doubles
  static constexpr int B_STAGE = BK * BN;
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 128;  // + alignment slack
  static constexpr int MIN_BLOCKS = MINB ? MINB : (THREADS > 128 ? 1 : (FM * FN <= 16 ? 3 : 2));
  static_assert(BK % 4 == 0 && BN % 8 == 0 && BM <= 256 && BK * BN / 4 <= 256 * 64, "tma tile");
};

// Epilogue of one tile: EPI = 0 stores (or accumulates) the accumulators
// into C; EPI = 1 (MTTKRP) multiplies by H, sums the tile's rows in a fixed
// order through `red` (WARPS_M x BN doubles of shared memory) into the
// workspace row of the M-tile, and with p.counters the last CTA of the
// (batch, N-tile) finishes the ordered sum over the M-tiles.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int EPI, int MINB>
__device__ __forceinline__ void tma_epilogue(double (&acc)[TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>::FM]
                                                           [TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>::FN][2],
                                             const GemmArgs& p, double* __restrict__ C, const int tm, const int tn,
                                             const int m0, const int n0, const int bz, double* red) {
  using Cfg = TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>;
  const int64_t M = p.M, N = p.N;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm0 = (warp / Cfg::WARPS_N) * WM;
  const int wn0 = (warp % Cfg::WARPS_N) * WN;
  if constexpr (EPI == 1) {  // MTTKRP row-sum epilogue (see dgemm_kernel)
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
    if (p.counters != nullptr) {
      // fused finish (replaces mttkrp_reduce): the last CTA of this (batch, N-tile)
      // to arrive sums the M-tile partials in ascending order -- the same order,
      // so the same bits -- and writes the output row
      __shared__ int last_arrival;
      __threadfence();
      __syncthreads();
      int* counter = p.counters + int64_t(bz) * p.N + tn;
      if (tid == 0) last_arrival = atomicAdd(counter, 1) == p.tiles_m - 1;
      __syncthreads();
      if (last_arrival) {
        __threadfence();
        for (int c = tid; c < BN; c += Cfg::THREADS) {
          if (n0 + c >= N) continue;
          double v = 0.0;
          for (int g = 0; g < p.tiles_m; ++g) v += __ldcg(C + int64_t(g) * N + n0 + c);
          double* dst = p.out + int64_t(bz) * p.ldo + n0 + c;
          *dst = p.out_acc ? *dst + v : v;
        }
        if (tid == 0) *counter = 0;  // ready for the next launch on this workspace
      }
    }
    return;
  }

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

// One CTA tile of the TMA-fed GEMM: tile `tile` (raster order) of batch
// entry `bz`, operands through the tensor maps tmA / tmB (kernel-parameter
// addresses: __grid_constant__).  Shared by the plain kernel and the
// grouped one below.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int EPI, int MINB, bool SEG2 = false>
__device__ __forceinline__ void tma_gemm_tile(const CUtensorMap* tmA_, const CUtensorMap* tmB_, const GemmArgs& p,
                                              const int tile, const int bz, const CUtensorMap* tmA2 = nullptr,
                                              const CUtensorMap* tmB2 = nullptr) {
  using Cfg = TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>;
  extern __shared__ __align__(128) unsigned char tma_smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];   // per stage: every warp has read it
  double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(tma_smem_raw) + 127) & ~uintptr_t(127));
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  const CUtensorMap& tmA = *tmA_;
  const CUtensorMap& tmB = *tmB_;

  // grouped rasterisation (as dgemm_kernel)
  const int per_group = p.group * p.tiles_n;
  const int first_m = (tile / per_group) * p.group;
  const int gsize = min(p.tiles_m - first_m, p.group);
  const int in_g = tile % per_group;
  const int tm = first_m + in_g % gsize;
  const int tn = in_g / gsize;
  const int m0 = tm * BM;
  const int n0 = tn * BN;
  const int bzB = p.sB ? bz : 0;
  double* __restrict__ C = p.C + int64_t(bz) * p.sC;
  const int64_t M = p.M, N = p.N, K = p.K;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm0 = (warp / Cfg::WARPS_N) * WM;
  const int wn0 = (warp % Cfg::WARPS_N) * WN;
  const int kt1 = (int)ceil_div(K, BK);  // k-tiles of the first segment
  const int ktiles = kt1 + (SEG2 && p.K2 > 0 ? (int)ceil_div(p.K2, BK) : 0);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
    if (SEG2 && kt >= kt1) {  // second segment: its own operands, k from 0 again
      tma_load_4d(As + s * Cfg::A_STAGE, tmA2, 0, m0, (kt - kt1) * (BK / 4), bz, &full[s]);
      tma_load_4d(Bs + s * Cfg::B_STAGE, tmB2, 0, (kt - kt1) * BK, n0 / 4, bzB, &full[s]);
      return;
    }
    tma_load_4d(As + s * Cfg::A_STAGE, &tmA, 0, m0, kt * (BK / 4), bz, &full[s]);
    tma_load_4d(Bs + s * Cfg::B_STAGE, &tmB, 0, kt * BK, n0 / 4, bzB, &full[s]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s)
      if (s < ktiles) issue(s);
  }

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // fragment offsets inside a stage (doubles)
  const int a_off = (wm0 + (lane >> 2)) * 4 + (lane & 3);                 // + kq*BM*4 + i*32
  const int b_off = ((wn0 + (lane >> 2)) / 4) * BK * 4 + (lane & 3) * 4 + ((lane >> 2) & 3);  // + kq*16 + j*2*BK*4

  for (int kt = 0; kt < ktiles; ++kt) {
    mbar_wait(&full[kt % STAGES], (kt / STAGES) & 1);
    if (tid == 0 && kt + STAGES - 1 < ktiles) {
      // the slot the next copy overwrites was read in iteration kt - 1: wait until every
      // warp released it (per-stage "empty" barrier instead of a CTA-wide __syncthreads,
      // so the other warps never wait for each other)
      if (kt >= 1) mbar_wait(&empty[(kt - 1) % STAGES], ((kt - 1) / STAGES) & 1);
      issue(kt + STAGES - 1);
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE + a_off;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE + b_off;
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
    if (lane == 0) mbar_arrive(&empty[kt % STAGES]);
  }

  if constexpr (EPI == 1) __syncthreads();  // every stage has been consumed: the ring serves as scratch
  tma_epilogue<BM, BN, BK, WM, WN, STAGES, EPI, MINB>(acc, p, C, tm, tn, m0, n0, bz, smem);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int EPI, int MINB = 0>
__global__ void __launch_bounds__(TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>::THREADS,
                                  TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>::MIN_BLOCKS)
dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs p) {
  tma_gemm_tile<BM, BN, BK, WM, WN, STAGES, EPI, MINB>(&tmA, &tmB, p, blockIdx.x, blockIdx.y);
}

// Grouped launch: up to TD_GEMM_GROUP_MAX problems, their tiles laid end to
// end along grid.x (problem q owns tiles [start[q], start[q+1])).
template <bool SEG2>
struct alignas(64) GroupedTmaT {
  CUtensorMap map[2 * TD_GEMM_GROUP_MAX];
  CUtensorMap map2[SEG2 ? 2 * TD_GEMM_GROUP_MAX : 1];  // second k-segments (SEG2 only)
  GemmArgs args[TD_GEMM_GROUP_MAX];
  int start[TD_GEMM_GROUP_MAX + 1];
  int count;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB = 0, bool SEG2 = false>
__global__ void __launch_bounds__(TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>::THREADS,
                                  TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>::MIN_BLOCKS)
dgemm_tma_grouped_kernel(const __grid_constant__ GroupedTmaT<SEG2> g) {
  const int x = blockIdx.x;
  int q = 0;
  while (q + 1 < g.count && x >= g.start[q + 1]) ++q;
  const GemmArgs p = g.args[q];
  tma_gemm_tile<BM, BN, BK, WM, WN, STAGES, 0, MINB, SEG2>(&g.map[2 * q], &g.map[2 * q + 1], p, x - g.start[q], 0,
                                                           &g.map2[SEG2 ? 2 * q : 0], &g.map2[SEG2 ? 2 * q + 1 : 0]);
}

// ---- host side: tensor maps through the driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// k4-sliced 4-D view {4, rows, cols/4, batch} of a row-major [batch][rows][cols] operand.
// Encoded maps are cached by their parameters (repeated launches on the same
// tiles -- every step of a launch plan -- skip the driver call).
static int encode_sliced_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                             int64_t batch, int64_t batch_stride, int box_rows, int box_cols);

struct MapKey {
  const double* base;
  int64_t rows, cols, ld, batch, stride;
  int box_rows, box_cols;
  bool operator==(const MapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld && batch == o.batch &&
           stride == o.stride && box_rows == o.box_rows && box_cols == o.box_cols;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = reinterpret_cast<uintptr_t>(k.base);
    for (int64_t v : {k.rows, k.cols, k.ld, k.batch, k.stride, int64_t(k.box_rows) << 32 | k.box_cols})
      h = (h ^ uint64_t(v)) * 0x9E3779B97F4A7C15ull;
    return size_t(h ^ (h >> 29));
  }
};

static int make_sliced_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                           int64_t batch, int64_t batch_stride, int box_rows, int box_cols) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{base, rows, cols, ld, batch, batch > 1 ? batch_stride : 0, box_rows, box_cols};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *map = it->second;
      return TD_OK;
    }
  }
  if (int rc = encode_sliced_map(map, base, rows, cols, ld, batch, batch_stride, box_rows, box_cols)) return rc;
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() > 8192) cache.clear();
  cache.emplace(key, *map);
  return TD_OK;
}

static int encode_sliced_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                             int64_t batch, int64_t batch_stride, int box_rows, int box_cols) {
  auto enc = tma_encoder();
  TD_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[4] = {4, (cuuint64_t)rows, (cuuint64_t)(cols / 4), (cuuint64_t)batch};
  const cuuint64_t strides[3] = {(cuuint64_t)ld * 8, 32, (cuuint64_t)(batch > 1 ? batch_stride * 8 : 16)};
  const cuuint32_t box[4] = {4, (cuuint32_t)box_rows, (cuuint32_t)(box_cols / 4), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TD_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TD_OK;
}

static bool tma_ok(int64_t batch, const GemmArgs& a) {
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return al(a.A) && al(a.B) && a.lda % 2 == 0 && a.ldb % 2 == 0 && a.K % 4 == 0 && a.N % 4 == 0 &&
         a.M < (1ll << 31) && a.K < (1ll << 31) && a.N < (1ll << 31) &&
         (batch == 1 || (a.sA % 2 == 0 && a.sB % 2 == 0)) && tma_encoder() != nullptr;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int EPI, int MINB = 0>
static int launch_gemm_tma(cudaStream_t st, int64_t batch, GemmArgs a) {
  using Cfg = TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>;
  auto kern = dgemm_tma_kernel<BM, BN, BK, WM, WN, STAGES, EPI, MINB>;
  TD_CUDA(ensure_smem(kern, Cfg::SMEM_BYTES));
  CUtensorMap ma, mb;
  if (int rc = make_sliced_map(&ma, a.A, a.M, a.K, a.lda, batch, a.sA, BM, BK)) return rc;
  if (int rc = make_sliced_map(&mb, a.B, a.K, a.N, a.ldb, a.sB ? batch : 1, a.sB, BK, BN)) return rc;
  a.tiles_m = (int)ceil_div(a.M, BM);
  a.tiles_n = (int)ceil_div(a.N, BN);
  a.group = raster_group(Cfg::MIN_BLOCKS, BM, BN);
  const int64_t tiles = int64_t(a.tiles_m) * a.tiles_n;
  TD_REQUIRE(tiles < (1ll << 31) && batch <= 65535, "dgemm: grid too large (%lld tiles, batch %lld)",
             (long long)tiles, (long long)batch);
  dim3 grid((unsigned)tiles, (unsigned)batch);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(ma, mb, a);
  return check_launch("dgemm_tma_kernel");
}

}  // namespace td

namespace td {

// Grouped form of launch_gemm_tma (plain epilogue, batch 1 per problem).
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB = 0, bool SEG2 = false>
static int launch_gemm_tma_grouped(cudaStream_t st, int count, const GemmArgs* probs) {
  using Cfg = TmaCfg<BM, BN, BK, WM, WN, STAGES, MINB>;
  auto kern = dgemm_tma_grouped_kernel<BM, BN, BK, WM, WN, STAGES, MINB, SEG2>;
  TD_CUDA(ensure_smem(kern, Cfg::SMEM_BYTES));
  GroupedTmaT<SEG2> g;
  std::memset(&g, 0, sizeof g);
  g.count = count;
  int64_t tiles = 0;
  for (int q = 0; q < count; ++q) {
    GemmArgs a = probs[q];
    if (int rc = make_sliced_map(&g.map[2 * q], a.A, a.M, a.K, a.lda, 1, 0, BM, BK)) return rc;
    if (int rc = make_sliced_map(&g.map[2 * q + 1], a.B, a.K, a.N, a.ldb, 1, 0, BK, BN)) return rc;
    if constexpr (SEG2) {
      if (a.K2 > 0) {
        if (int rc = make_sliced_map(&g.map2[2 * q], a.A2, a.M, a.K2, a.lda2, 1, 0, BM, BK)) return rc;
        if (int rc = make_sliced_map(&g.map2[2 * q + 1], a.B2, a.K2, a.N, a.ldb2, 1, 0, BK, BN)) return rc;
      }
    } else {
      a.K2 = 0;
    }
    a.tiles_m = (int)ceil_div(a.M, BM);
    a.tiles_n = (int)ceil_div(a.N, BN);
    a.group = raster_group(Cfg::MIN_BLOCKS, BM, BN);
    g.args[q] = a;
    g.start[q] = (int)tiles;
    tiles += int64_t(a.tiles_m) * a.tiles_n;
  }
  g.start[count] = (int)tiles;
  TD_REQUIRE(tiles < (1ll << 31), "dgemm_grouped: grid too large (%lld tiles)", (long long)tiles);
  if (tiles == 0) return TD_OK;
  kern<<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(g);
  return check_launch("dgemm_tma_grouped_kernel");
}

}  // namespace td

