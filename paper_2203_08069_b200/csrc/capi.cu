// Library-level entry points: version, errors, devices, launch counter.
#include "common.cuh"
#include <cstring>
#include <mutex>
#include <set>
#include <tuple>

namespace td {
static thread_local char t_err[1024] = {0};
std::atomic<long long> g_launches{0};

// kernels whose dynamic-shared-memory limit was already raised, per device
static std::mutex g_attr_mu;
static std::set<std::tuple<const void*, int, int>> g_attr_done;

bool smem_attr_done(const void* kern, int dev, int bytes) {
  std::lock_guard<std::mutex> lock(g_attr_mu);
  return g_attr_done.count({kern, dev, bytes}) != 0;
}

void smem_attr_mark(const void* kern, int dev, int bytes) {
  std::lock_guard<std::mutex> lock(g_attr_mu);
  g_attr_done.insert({kern, dev, bytes});
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}
void clear_error() { t_err[0] = 0; }
}  // namespace td

extern "C" {

int td_version(void) { return 10000; }  // 1.0.0

const char* td_last_error(void) { return td::t_err; }

int td_device_count(void) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    return 0;
  }
  if (e != cudaSuccess) {
    td::set_error("cudaGetDeviceCount: %s", cudaGetErrorString(e));
    return TD_ERR_CUDA;
  }
  return n;
}

int td_set_device(int device) {
  TD_CUDA(cudaSetDevice(device));
  return TD_OK;
}

long long td_launch_count(void) { return td::g_launches.load(); }

int td_init(int ndev, const int* devices) {
  TD_REQUIRE(ndev >= 0 && (ndev == 0 || devices), "init: bad device list");
  int prev = 0;
  TD_CUDA(cudaGetDevice(&prev));
  for (int k = 0; k < ndev; ++k) {  // create the primary contexts up front (not inside the first launch)
    TD_CUDA(cudaSetDevice(devices[k]));
    TD_CUDA(cudaFree(nullptr));
  }
  TD_CUDA(cudaSetDevice(prev));
  return TD_OK;
}

int td_finalize(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return TD_OK;
  }
  int prev = 0;
  TD_CUDA(cudaGetDevice(&prev));
  for (int d = 0; d < n; ++d) {  // drain every device this process touched
    TD_CUDA(cudaSetDevice(d));
    TD_CUDA(cudaDeviceSynchronize());
  }
  TD_CUDA(cudaSetDevice(prev));
  return TD_OK;
}

int td_stream_device(void* stream) {
  int dev = -1;
  TD_CUDA(cudaStreamGetDevice(td::as_stream(stream), &dev));
  return dev;
}

int td_memcpy_2d(void* stream, double* dst, int64_t dst_pitch, const double* src, int64_t src_pitch,
                 int64_t width, int64_t rows) {
  if (width <= 0 || rows <= 0) return TD_OK;
  td::StreamDevice sd(stream);
  TD_CUDA(cudaMemcpy2DAsync(dst, size_t(dst_pitch) * 8, src, size_t(src_pitch) * 8, size_t(width) * 8,
                            size_t(rows), cudaMemcpyDefault, td::as_stream(stream)));
  return TD_OK;
}

}  // extern "C"
