// Shared plumbing of the C ABI: thread-local error text, status macros,
// launch accounting.  See include/distal_b200.h for the conventions.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <atomic>
#include "../../include/distal_b200.h"

namespace td {

void set_error(const char* fmt, ...);
void clear_error();
extern std::atomic<long long> g_launches;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Makes the stream's device current for the duration of a call (one host
// thread may drive several GPUs); restores the caller's device afterwards.
struct StreamDevice {
  int prev = -1;
  explicit StreamDevice(void* s) {
    if (!s) return;
    int dev = -1, cur = -1;
    cudaGetDevice(&cur);  // also initialises this (static) runtime before the stream query
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(as_stream(s), &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();  // under CUDA-graph capture: leave the device alone (no stream queries)
      return;
    }
    if (cudaStreamGetDevice(as_stream(s), &dev) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    if (cur != dev) {
      prev = cur;
      cudaSetDevice(dev);
    }
  }
  ~StreamDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device
// (it is a host round trip; launches of the same kernel repeat it otherwise).
bool smem_attr_done(const void* kern, int dev, int bytes);   // capi.cu
void smem_attr_mark(const void* kern, int dev, int bytes);

template <class Kernel>
inline cudaError_t ensure_smem(Kernel kern, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorUnknown;
  const void* key = reinterpret_cast<const void*>(kern);
  if (smem_attr_done(key, dev, bytes)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) smem_attr_mark(key, dev, bytes);
  return e;
}

inline int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return TD_ERR_CUDA;
  }
  return TD_OK;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace td

#define TD_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      td::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e),    \
                    __FILE__, __LINE__);                                       \
      return TD_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

#define TD_REQUIRE(cond, ...)                                                  \
  do {                                                                         \
    if (!(cond)) {                                                             \
      td::set_error(__VA_ARGS__);                                              \
      return TD_ERR_ARG;                                                       \
    }                                                                          \
  } while (0)
