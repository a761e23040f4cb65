// FP64 tensor-core building blocks for sm_100a.
//
// sm_100a has no FP64 form of tcgen05.mma (ptxas: "Unknown modifier
// '.kind::f64'") and wgmma is sm_90a-only, so the FP64 tensor path on B200 is
// the warp-level `mma.sync.aligned.m8n8k4.f64` (SASS: DMMA.8x8x4).  Measured on
// this pool's B200 (tools/tuning/dmma.cu): 37.06 TFLOP/s at 1965 MHz, i.e. the full
// 148 SM x 128 flop/clk FP64 peak, identical to DFMA.  Operands are staged
// through shared memory by TMA bulk tensor copies (gemm_tma.cuh, the default
// wherever the copy engine can address the operands) or by cp.async (LDGSTS)
// multistage pipelines.
#pragma once
#include <cstdint>

namespace td {

// D(8x8) += A(8x4, row) * B(4x8, col); per lane: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = {D[lane/4][2*(lane%4)], D[lane/4][2*(lane%4)+1]}.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async of VEC doubles (VEC = 2 -> 16 B .cg, VEC = 1 -> 8 B .ca); `valid`
// doubles are read from global, the rest of the destination is zero-filled.
template <int VEC>
__device__ __forceinline__ void cp_async_f64(double* sdst, const double* gsrc, int valid) {
  const uint32_t d = smem_u32(sdst);
  const int bytes = valid * 8;
  if constexpr (VEC == 2) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(bytes));
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace td
