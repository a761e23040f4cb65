// Fused MTTKRP leaf:  A(i,j) (+)= sum_k C(k,j) * sum_l B(i,k,l) * D(l,j)
// (reference statement pkg/src/tendist/algorithms.py:339-340, evaluated per
// point at cin.py:399-417 in the reference).
//
// One CTA owns one i (and one 32-wide block of j):
//   for each k-block of 128 rows:  T[128 x 32] = B(i, kblk, :) . D[:, jblk]
//        on DMMA.8x8x4 tiles fed by a cp.async ring over l (16 per stage);
//   epilogue per k-block: partial(j) += sum_k C(k,j) * T(k,j) in registers;
//   end: fixed-order shuffle + shared-memory tree over the 8 warps, then one
//   write (or accumulate) of A(i, jblk).
// No atomics: the summation order is a fixed function of the shape, so runs
// are bitwise reproducible; exact on integer-valued data.
// B is streamed once from HBM (8 B per 64 flop at R = 32); D and C stay in L2.
#include "common.cuh"
#include "dmma.cuh"

namespace td {

constexpr int MK_BK = 16;              // l per pipeline stage
constexpr int MK_ROWS = 128;           // k rows per block
constexpr int MK_R = 32;               // j columns per CTA
constexpr int MK_THREADS = 256;        // 8 warps x 16 rows
constexpr int MK_STAGES = 4;
constexpr int MK_SA = MK_BK + 4;       // B-tile row stride (doubles)
constexpr int MK_SD = MK_R + 4;        // D-tile row stride
constexpr int MK_A_STAGE = MK_ROWS * MK_SA;
constexpr int MK_D_STAGE = MK_BK * MK_SD;
constexpr int MK_SMEM = MK_STAGES * (MK_A_STAGE + MK_D_STAGE) * 8 + 8 * MK_R * 8;

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
};

template <int VEC>
__global__ void __launch_bounds__(MK_THREADS, 2) mttkrp_kernel(MttkrpArgs p) {
  extern __shared__ __align__(128) double smem[];
  double* Bs = smem;
  double* Ds = smem + MK_STAGES * MK_A_STAGE;
  double* red = Ds + MK_STAGES * MK_D_STAGE;  // [8 warps][32]

  const int64_t i = blockIdx.x;
  const int64_t j0 = int64_t(blockIdx.y) * MK_R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* __restrict__ Bi = p.B + i * p.sBi;
  const int64_t K = p.K, L = p.L, R = p.R;

  const int kblocks = (int)ceil_div(K, MK_ROWS);
  const int ltiles = (int)ceil_div(L, MK_BK);
  const int total = kblocks * ltiles;

  auto load = [&](int stage, int t) {
    const int64_t k0 = int64_t(t / ltiles) * MK_ROWS;
    const int64_t l0 = int64_t(t % ltiles) * MK_BK;
    double* bs = Bs + stage * MK_A_STAGE;
    double* ds = Ds + stage * MK_D_STAGE;
    constexpr int B_PER_ROW = MK_BK / VEC;
    for (int c = tid; c < MK_ROWS * B_PER_ROW; c += MK_THREADS) {
      const int r = c / B_PER_ROW, col = (c % B_PER_ROW) * VEC;
      const int64_t gk = k0 + r, gl = l0 + col;
      int valid = 0;
      const double* src = p.B;
      if (gk < K && gl < L) {
        valid = (int)(L - gl < VEC ? L - gl : VEC);
        src = Bi + gk * p.sBk + gl;
      }
      cp_async_f64<VEC>(bs + r * MK_SA + col, src, valid);
    }
    constexpr int D_PER_ROW = MK_R / VEC;
    for (int c = tid; c < MK_BK * D_PER_ROW; c += MK_THREADS) {
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

  double acc[2][4][2];
  double part[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) part[a][0] = part[a][1] = 0.0;
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

#pragma unroll
  for (int s = 0; s < MK_STAGES - 1; ++s) {
    if (s < total) load(s, s);
    cp_async_commit();
  }
  const int arow = warp * 16 + (lane >> 2);
  const int acol = lane & 3;
  const int brow = lane & 3;
  const int bcol = lane >> 2;

  for (int t = 0; t < total; ++t) {
    cp_async_wait<MK_STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + MK_STAGES - 1;
      if (nt < total) load(nt % MK_STAGES, nt);
      cp_async_commit();
    }
    const double* bs = Bs + (t % MK_STAGES) * MK_A_STAGE;
    const double* ds = Ds + (t % MK_STAGES) * MK_D_STAGE;
#pragma unroll
    for (int kk = 0; kk < MK_BK; kk += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int m = 0; m < 2; ++m) af[m] = bs[(arow + m * 8) * MK_SA + kk + acol];
#pragma unroll
      for (int n = 0; n < 4; ++n) bf[n] = ds[(kk + brow) * MK_SD + bcol + n * 8];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
    if (t % ltiles == ltiles - 1) {  // k-block finished: Hadamard with C, reduce over k
      const int64_t k0 = int64_t(t / ltiles) * MK_ROWS;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int64_t k = k0 + warp * 16 + m * 8 + (lane >> 2);
        const bool kin = k < K;
#pragma unroll
        for (int n = 0; n < 4; ++n) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t j = j0 + n * 8 + (lane & 3) * 2 + h;
            if (kin && j < R) part[n][h] += p.C[k * p.ldc + j] * acc[m][n][h];
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
    for (int w = 1; w < 8; ++w) v += red[w * MK_R + tid];
    const int64_t j = j0 + tid;
    if (j < R) {
      double* dst = p.A + i * p.lda + j;
      *dst = p.accumulate ? *dst + v : v;
    }
  }
}

static bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

}  // namespace td

extern "C" int td_mttkrp(void* stream, int64_t I, int64_t K, int64_t L, int64_t R, const double* B,
                         int64_t sBi, int64_t sBk, const double* C, int64_t ldc, const double* D,
                         int64_t ldd, double* A, int64_t lda, int accumulate) {
  using namespace td;
  if (I <= 0 || R <= 0) return TD_OK;
  TD_REQUIRE(I <= 2147483647, "mttkrp: I too large");
  MttkrpArgs a{I, K, L, R, B, sBi, sBk, C, ldc, D, ldd, A, lda, accumulate};
  const bool vec2 = al16(B) && al16(D) && sBi % 2 == 0 && sBk % 2 == 0 && ldd % 2 == 0;
  dim3 grid((unsigned)I, (unsigned)ceil_div(R, MK_R));
  cudaStream_t st = as_stream(stream);
  if (vec2) {
    TD_CUDA(cudaFuncSetAttribute(mttkrp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, MK_SMEM));
    mttkrp_kernel<2><<<grid, MK_THREADS, MK_SMEM, st>>>(a);
  } else {
    TD_CUDA(cudaFuncSetAttribute(mttkrp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, MK_SMEM));
    mttkrp_kernel<1><<<grid, MK_THREADS, MK_SMEM, st>>>(a);
  }
  return check_launch("mttkrp_kernel");
}
