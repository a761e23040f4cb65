// NCCL over NVLink 5 / NVSwitch: the lowering of the reference's simulated
// transfers.  Each compute-phase CommEvent (reference
// pkg/src/tendist/simulator.py:563-581, write-backs :635-645) becomes one
// ncclSend/ncclRecv pair inside the step's ncclGroupStart/End, issued on the
// per-GPU communication stream so it overlaps the previous step's leaf
// kernels; fan-outs and reductions also have ncclBroadcast / ncclReduce forms.
// Links against the NCCL that PyTorch ships (nvidia-nccl-cu12, 2.28.x) so the
// process holds a single libnccl.
#include "common.cuh"
#include <nccl.h>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <thread>

#define TD_NCCL(call)                                                          \
  do {                                                                         \
    ncclResult_t _r = (call);                                                  \
    if (_r != ncclSuccess) {                                                   \
      td::set_error("%s failed: %s", #call, ncclGetErrorString(_r));           \
      return TD_ERR_NCCL;                                                      \
    }                                                                          \
  } while (0)

static_assert(sizeof(ncclUniqueId) == TD_UNIQUE_ID_BYTES, "ncclUniqueId size");

extern "C" {

int td_nccl_version(void) {
  int v = 0;
  if (ncclGetVersion(&v) != ncclSuccess) return TD_ERR_NCCL;
  return v;
}

int td_comm_unique_id(char* out) {
  ncclUniqueId id;
  TD_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return TD_OK;
}

int td_comm_init_rank(void** comm, int nranks, int rank, const char* unique_id, int device) {
  TD_REQUIRE(comm && unique_id && nranks > 0 && rank >= 0 && rank < nranks, "comm_init_rank: bad arguments");
  TD_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c;
  TD_NCCL(ncclCommInitRank(&c, nranks, id, rank));
  *comm = c;
  return TD_OK;
}

int td_comm_init_all(void** comms, int ndev, const int* devices) {
  TD_REQUIRE(comms && devices && ndev > 0, "comm_init_all: bad arguments");
  ncclComm_t* cs = reinterpret_cast<ncclComm_t*>(comms);
  TD_NCCL(ncclCommInitAll(cs, ndev, devices));
  return TD_OK;
}

int td_comm_split(void* comm, int color, int key, void** newcomm) {
  TD_REQUIRE(comm && newcomm, "comm_split: bad arguments");
  // inside ncclGroupStart/End (one thread splitting several communicators) NCCL
  // fills the handle only at ncclGroupEnd: hand it the caller's slot, not a local
  *newcomm = nullptr;
  TD_NCCL(ncclCommSplit(static_cast<ncclComm_t>(comm), color < 0 ? NCCL_SPLIT_NOCOLOR : color, key,
                        reinterpret_cast<ncclComm_t*>(newcomm), nullptr));
  return TD_OK;
}

int td_comm_destroy(void* comm) {
  if (!comm) return TD_OK;
  TD_NCCL(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
  return TD_OK;
}

int td_group_start(void) {
  TD_NCCL(ncclGroupStart());
  return TD_OK;
}

int td_group_end(void) {
  TD_NCCL(ncclGroupEnd());
  return TD_OK;
}

int td_send(void* comm, void* stream, const double* buf, int64_t count, int peer) {
  TD_NCCL(ncclSend(buf, (size_t)count, ncclDouble, peer, static_cast<ncclComm_t>(comm), td::as_stream(stream)));
  return TD_OK;
}

int td_recv(void* comm, void* stream, double* buf, int64_t count, int peer) {
  TD_NCCL(ncclRecv(buf, (size_t)count, ncclDouble, peer, static_cast<ncclComm_t>(comm), td::as_stream(stream)));
  return TD_OK;
}

int td_bcast(void* comm, void* stream, double* buf, int64_t count, int root) {
  TD_NCCL(ncclBroadcast(buf, buf, (size_t)count, ncclDouble, root, static_cast<ncclComm_t>(comm),
                        td::as_stream(stream)));
  return TD_OK;
}

int td_reduce_sum(void* comm, void* stream, const double* send, double* recv, int64_t count, int root) {
  TD_NCCL(ncclReduce(send, recv, (size_t)count, ncclDouble, ncclSum, root, static_cast<ncclComm_t>(comm),
                     td::as_stream(stream)));
  return TD_OK;
}

int td_allgather(void* comm, void* stream, const double* send, double* recv, int64_t count) {
  TD_NCCL(ncclAllGather(send, recv, (size_t)count, ncclDouble, static_cast<ncclComm_t>(comm),
                        td::as_stream(stream)));
  return TD_OK;
}

int td_shift(void* comm, void* stream, const double* send, double* recv, int64_t count, int delta) {
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int n = 0, me = 0;
  TD_NCCL(ncclCommCount(c, &n));
  TD_NCCL(ncclCommUserRank(c, &me));
  const int to = ((me + delta) % n + n) % n;
  const int from = ((me - delta) % n + n) % n;
  if (to == me) {  // a shift by a multiple of the ring: a local copy
    if (send != recv)
      TD_CUDA(cudaMemcpyAsync(recv, send, size_t(count) * 8, cudaMemcpyDeviceToDevice, td::as_stream(stream)));
    return TD_OK;
  }
  TD_NCCL(ncclGroupStart());
  ncclResult_t r1 = ncclSend(send, (size_t)count, ncclDouble, to, c, td::as_stream(stream));
  ncclResult_t r2 = ncclRecv(recv, (size_t)count, ncclDouble, from, c, td::as_stream(stream));
  TD_NCCL(ncclGroupEnd());
  TD_NCCL(r1);
  TD_NCCL(r2);
  return TD_OK;
}

int td_comm_wait(void* const* comms, int ncomms, void* const* streams, int nstreams, double timeout_s) {
  TD_REQUIRE((ncomms == 0 || comms) && (nstreams == 0 || streams), "comm_wait: null arrays");
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    bool done = true;
    for (int k = 0; k < nstreams; ++k) {
      const cudaError_t e = cudaStreamQuery(td::as_stream(streams[k]));
      if (e == cudaErrorNotReady) {
        done = false;
      } else if (e != cudaSuccess) {
        td::set_error("comm_wait: stream %d failed: %s", k, cudaGetErrorString(e));
        return TD_ERR_CUDA;
      }
    }
    if (done) return TD_OK;
    const char* why = nullptr;
    char buf[256];
    for (int k = 0; k < ncomms && !why; ++k) {
      ncclResult_t ar = ncclSuccess;
      if (ncclCommGetAsyncError(static_cast<ncclComm_t>(comms[k]), &ar) != ncclSuccess ||
          (ar != ncclSuccess && ar != ncclInProgress)) {
        std::snprintf(buf, sizeof buf, "NCCL communicator %d reported %s", k, ncclGetErrorString(ar));
        why = buf;
      }
    }
    const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!why && timeout_s > 0 && waited > timeout_s) {
      std::snprintf(buf, sizeof buf, "no progress after %.1f s (a peer never posted its side of a transfer?)",
                    waited);
      why = buf;
    }
    if (why) {
      // abort every communicator: pending NCCL kernels return, the job can shut down
      if (std::getenv("TD_DEBUG")) std::fprintf(stderr, "td_comm_wait: %s; aborting %d comm(s)\n", why, ncomms);
      for (int k = 0; k < ncomms; ++k) ncclCommAbort(static_cast<ncclComm_t>(comms[k]));
      if (std::getenv("TD_DEBUG")) std::fprintf(stderr, "td_comm_wait: aborted\n");
      td::set_error("comm_wait: %s; communicators aborted", why);
      return TD_ERR_NCCL;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int td_allreduce_sum(void* comm, void* stream, const double* send, double* recv, int64_t count) {
  TD_NCCL(ncclAllReduce(send, recv, (size_t)count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm),
                        td::as_stream(stream)));
  return TD_OK;
}

}  // extern "C"
