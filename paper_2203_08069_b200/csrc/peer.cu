// Peer memory over NVLink 5 / NVSwitch: buffers that a leaf kernel running on
// one GPU writes directly in another GPU's HBM.
//
// Used for the reduce write-back of the reference's commit phase
// (pkg/src/tendist/simulator.py:624-654, the `reduce` events of :635-645):
// when a task's whole partial output goes to a home piece on another GPU
// (Johnson-3D / COSMA depth partials), the task's DMMA GEMM epilogue stores
// its tiles straight into an "inbox" in the home GPU's HBM as they finish,
// so the transfer overlaps the math tile by tile instead of following it.
// Two process models:
//   * one process driving several GPUs: plain cudaMalloc + peer access
//     (td_peer_enable), the pointer is used as is;
//   * one process per GPU (torchrun): the home exports a CUDA IPC handle
//     (td_peer_alloc), the writer maps it into its own context
//     (td_peer_open, cudaIpcMemLazyEnablePeerAccess).
#include "common.cuh"
#include <cstring>

static_assert(sizeof(cudaIpcMemHandle_t) == TD_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");

namespace {
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != dev) {
      prev = cur;
      cudaSetDevice(dev);
    }
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

int td_peer_can_access(int device, int peer) {
  int ok = 0;
  TD_CUDA(cudaDeviceCanAccessPeer(&ok, device, peer));
  return ok;
}

int td_peer_enable(int device, int peer) {
  if (device == peer) return TD_OK;
  DeviceScope scope(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return TD_OK;
  }
  TD_CUDA(e);
  return TD_OK;
}

int td_peer_alloc(int device, int64_t bytes, void** ptr, char* ipc_handle) {
  TD_REQUIRE(ptr && bytes >= 0, "peer_alloc: bad arguments");
  DeviceScope scope(device);
  void* p = nullptr;
  TD_CUDA(cudaMalloc(&p, bytes > 0 ? (size_t)bytes : 8));
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      TD_CUDA(e);
    }
    std::memcpy(ipc_handle, &h, sizeof(h));
  }
  *ptr = p;
  return TD_OK;
}

int td_peer_free(int device, void* ptr) {
  if (!ptr) return TD_OK;
  DeviceScope scope(device);
  TD_CUDA(cudaFree(ptr));
  return TD_OK;
}

int td_peer_open(int device, const char* ipc_handle, void** ptr) {
  TD_REQUIRE(ipc_handle && ptr, "peer_open: bad arguments");
  DeviceScope scope(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  TD_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TD_OK;
}

int td_peer_close(int device, void* ptr) {
  if (!ptr) return TD_OK;
  DeviceScope scope(device);
  TD_CUDA(cudaIpcCloseMemHandle(ptr));
  return TD_OK;
}

}  // extern "C"
