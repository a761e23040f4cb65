// Launch plans: the per-step loop of one distributed launch in C++.
//
// The reference runs a launch (reference pkg/src/tendist/simulator.py:557-663:
// per step the fetches of phase one, then every task's leaf, then the
// commits) as a Python loop.  Here the host planner lowers that loop once
// into a flat array of td_op records -- every leaf kernel, box copy, fill,
// NCCL group / send / receive / broadcast and cross-stream event edge, in
// issue order, with the device pointers of the HBM tiles baked in -- and
// td_execute_plan issues the whole array in one ABI call.  A host in any
// language can build the array itself: each op names one td_* entry point of
// this header and carries that entry point's arguments as 64-bit words, in
// order (pointers and integers as-is, doubles bit-cast).
#include "common.cuh"
#include <cstring>

extern "C" {

int td_event_create(int device, void** event) {
  TD_REQUIRE(event != nullptr, "event_create: null out pointer");
  int prev = -1;
  TD_CUDA(cudaGetDevice(&prev));
  TD_CUDA(cudaSetDevice(device));
  cudaEvent_t e = nullptr;
  cudaError_t rc = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaSetDevice(prev);
  TD_CUDA(rc);
  *event = e;
  return TD_OK;
}

int td_event_destroy(void* event) {
  if (event) TD_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)));
  return TD_OK;
}

// `device` owns the event and the stream (it also names the device whose
// legacy default stream a NULL `stream` means).
namespace {
struct OnDevice {
  int prev = -1;
  explicit OnDevice(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~OnDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

int td_event_record(void* event, void* stream, int device) {
  OnDevice on(device);
  TD_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), td::as_stream(stream)));
  return TD_OK;
}

int td_stream_wait_event(void* stream, void* event, int device) {
  OnDevice on(device);
  TD_CUDA(cudaStreamWaitEvent(td::as_stream(stream), reinterpret_cast<cudaEvent_t>(event), 0));
  return TD_OK;
}

}  // extern "C"

namespace {

template <class T>
inline T P(int64_t w) {
  return reinterpret_cast<T>(static_cast<intptr_t>(w));
}
inline double D(int64_t w) {
  double d;
  std::memcpy(&d, &w, sizeof d);
  return d;
}
inline int I(int64_t w) { return static_cast<int>(w); }

int run_op(const td_op& o) {
  const int64_t* a = o.arg;
  switch (o.kind) {
    case TD_OP_DGEMM:
      return td_dgemm(P<void*>(a[0]), a[1], a[2], a[3], P<const double*>(a[4]), a[5], P<const double*>(a[6]),
                      a[7], P<double*>(a[8]), a[9], I(a[10]));
    case TD_OP_DGEMM_BATCHED:
      return td_dgemm_batched(P<void*>(a[0]), a[1], a[2], a[3], a[4], P<const double*>(a[5]), a[6], a[7],
                              P<const double*>(a[8]), a[9], a[10], P<double*>(a[11]), a[12], a[13], I(a[14]));
    case TD_OP_DGEMM_GROUPED:
      return td_dgemm_grouped(P<void*>(a[0]), I(a[1]), P<const td_gemm_problem*>(a[2]), I(a[3]));
    case TD_OP_TTV:
      return td_ttv(P<void*>(a[0]), a[1], a[2], a[3], P<const double*>(a[4]), a[5], a[6], P<const double*>(a[7]),
                    P<double*>(a[8]), a[9], a[10], I(a[11]));
    case TD_OP_TTM:
      return td_ttm(P<void*>(a[0]), a[1], a[2], a[3], a[4], P<const double*>(a[5]), a[6], a[7],
                    P<const double*>(a[8]), a[9], P<double*>(a[10]), a[11], a[12], I(a[13]));
    case TD_OP_MTTKRP:
      return td_mttkrp(P<void*>(a[0]), a[1], a[2], a[3], a[4], P<const double*>(a[5]), a[6], a[7],
                       P<const double*>(a[8]), a[9], P<const double*>(a[10]), a[11], P<double*>(a[12]), a[13],
                       I(a[14]));
    case TD_OP_INNERPROD:
      return td_innerprod(P<void*>(a[0]), a[1], a[2], P<const double*>(a[3]), a[4], P<const double*>(a[5]), a[6],
                          P<double*>(a[7]), P<double*>(a[8]), I(a[9]));
    case TD_OP_NEST_EVAL:
      return td_nest_eval(P<void*>(a[0]), P<const void*>(a[1]), a[2]);
    case TD_OP_COPY_BOX:
      return td_copy_box(P<void*>(a[0]), I(a[1]), P<const int64_t*>(a[2]), P<double*>(a[3]),
                         P<const int64_t*>(a[4]), P<const double*>(a[5]), P<const int64_t*>(a[6]), I(a[7]));
    case TD_OP_MEMCPY_2D:
      return td_memcpy_2d(P<void*>(a[0]), P<double*>(a[1]), a[2], P<const double*>(a[3]), a[4], a[5], a[6]);
    case TD_OP_FILL:
      return td_fill(P<void*>(a[0]), P<double*>(a[1]), a[2], D(a[3]));
    case TD_OP_GROUP_START:
      return td_group_start();
    case TD_OP_GROUP_END:
      return td_group_end();
    case TD_OP_SEND:
      return td_send(P<void*>(a[0]), P<void*>(a[1]), P<const double*>(a[2]), a[3], I(a[4]));
    case TD_OP_RECV:
      return td_recv(P<void*>(a[0]), P<void*>(a[1]), P<double*>(a[2]), a[3], I(a[4]));
    case TD_OP_BCAST:
      return td_bcast(P<void*>(a[0]), P<void*>(a[1]), P<double*>(a[2]), a[3], I(a[4]));
    case TD_OP_REDUCE_SUM:
      return td_reduce_sum(P<void*>(a[0]), P<void*>(a[1]), P<const double*>(a[2]), P<double*>(a[3]), a[4],
                           I(a[5]));
    case TD_OP_EVENT_RECORD:
      return td_event_record(P<void*>(a[0]), P<void*>(a[1]), I(a[2]));
    case TD_OP_STREAM_WAIT:
      return td_stream_wait_event(P<void*>(a[0]), P<void*>(a[1]), I(a[2]));
    default:
      td::set_error("unknown op kind %d", o.kind);
      return TD_ERR_ARG;
  }
}

}  // namespace

extern "C" int td_execute_plan(const td_op* ops, int64_t count) {
  TD_REQUIRE(count == 0 || ops != nullptr, "execute_plan: null op array");
  int in_group = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int rc = run_op(ops[i]);
    if (ops[i].kind == TD_OP_GROUP_START) ++in_group;
    if (ops[i].kind == TD_OP_GROUP_END) --in_group;
    if (rc != TD_OK) {
      char msg[768];
      std::snprintf(msg, sizeof msg, "%s", td_last_error());
      // never leave an NCCL group open behind a failed op
      while (in_group-- > 0) td_group_end();
      td::set_error("plan op %lld (kind %d) failed: %s", (long long)i, ops[i].kind, msg);
      return rc;
    }
  }
  return TD_OK;
}
