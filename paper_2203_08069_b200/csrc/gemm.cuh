// Arguments of the DMMA GEMM body shared by the GEMM / TTM leaves (gemm.cu)
// and the MTTKRP row-sum variant (mttkrp.cu).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace td {

struct GemmArgs {
  int64_t M, N, K;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  int accumulate;
  int tiles_m, tiles_n;
  int group;   // M-tiles per raster group (~sqrt of the resident CTAs: square L2 working set per wave)
  // EPI = 1 (MTTKRP row-sum epilogue): C[bz][tm][n] = sum over the tile's rows r
  // of H(r, n) * (A.B)(r, n) -- one partial per M-tile, C is the workspace
  const double* H;
  int64_t ldh;
  // EPI = 1, TMA body, fused finish: per-(batch, N-tile) arrival counters (zero
  // between launches) and the output rows out + batch * ldo (+= if out_acc)
  int* counters;
  double* out;
  int64_t ldo;
  int out_acc;
  // TMA body, grouped kernel: an optional second k-segment (K2 > 0) accumulated
  // after the first in the same registers (td_gemm_problem.K2)
  int64_t K2;
  const double* A2;
  int64_t lda2;
  const double* B2;
  int64_t ldb2;
};

// MTTKRP row-sum GEMMs (EPI = 1 in gemm.cu): rows per M-tile of a config, launch
int dgemm_rowsum_tile_rows(int config);
int dgemm_rowsum(cudaStream_t st, int config, int64_t batch, GemmArgs a);
// Does `config` take the TMA body (whose epilogue can finish the sum itself)?
bool dgemm_rowsum_fusable(int config, int64_t batch, const GemmArgs& a);

// Stream-K MTTKRP (mttkrp_tma.cuh): A(i, j) (+)= sum_(k,l) B(i, k, l) * C(k, j) * D(l, j)
struct MkSplitArgs {
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
// Workspace doubles the variant needs for this shape and its CTA count, or 0
// when the copy engine cannot address the operands (per-i kernel instead).
int64_t mttkrp_streamk_plan(int variant, const MkSplitArgs& a, int* ctas);
int mttkrp_streamk(cudaStream_t st, int variant, const MkSplitArgs& a, int ctas, double* work);

}  // namespace td
