/*
 * distal_b200.h -- C ABI of the B200-native distributed dense tensor-algebra path.
 *
 * The reference (`tendist`, pure Python) has no FFI; its drop-in boundary for
 * this path is two-level:
 *   (1) the leaf-kernel plugin API -- register_leaf_kernel / substitute_leaf /
 *       LeafRuntime (reference pkg/src/tendist/cin.py:344-379,
 *       scheduling.py:263-299), whose per-point body is cin.py:399-417
 *       (_run_leaf) and whose accumulation contract is cin.py:363-365;
 *   (2) the simulated transfers of execute() phase one
 *       (reference pkg/src/tendist/simulator.py:563-581 `fetch`, :635-645
 *       write-back) which on B200 become real NCCL traffic.
 * Every entry point below replaces one of those; the Python host
 * (paper_2203_08069_b200/_native.py) binds them with ctypes.
 *
 * Conventions
 *   - All tensors are row-major float64 in device memory owned by the caller
 *     (PyTorch allocations); leading dimensions / strides are in ELEMENTS.
 *   - Every call is asynchronous on the given stream (cudaStream_t passed as
 *     void*; NULL = legacy default stream) and returns int: 0 on success,
 *     < 0 on failure, with a thread-local message from td_last_error().
 *   - No C++ exception crosses this ABI; no torch type appears in it.
 *   - `accumulate` != 0 means OUT += result (the reference's Reduce leaf,
 *     cin.py:416-417); 0 means OUT = result (Assign, cin.py:414-415).
 */
#ifndef DISTAL_B200_H
#define DISTAL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TD_OK 0
#define TD_ERR_CUDA (-1)
#define TD_ERR_NCCL (-2)
#define TD_ERR_ARG (-3)
#define TD_ERR_UNSUPPORTED (-4)

/* ---- library / device ------------------------------------------------- */
/* ABI version (major*10000 + minor*100 + patch). */
int td_version(void);
/* Message for the last failing call on this thread ("" if none). */
const char* td_last_error(void);
/* Number of visible CUDA devices (0 when no GPU); negative on driver error. */
int td_device_count(void);
/* Selects the current device of the calling thread. */
int td_set_device(int device);
/* Number of kernel launches this library issued since load (all threads). */
long long td_launch_count(void);
/* Lifecycle: create the CUDA contexts of `devices` up front; drain every
 * device (host-visible completion) at the end.  Communicators are created
 * with td_comm_init_rank / td_comm_init_all (+ td_comm_split for the axis
 * sub-communicators of a processor grid) and freed with td_comm_destroy. */
int td_init(int ndev, const int* devices);
int td_finalize(void);
/* Device ordinal a stream belongs to (every compute entry point makes that
 * device current for the call, so one thread can drive several GPUs). */
int td_stream_device(void* stream);

/* ---- leaf kernels (replace the per-point interpreter, cin.py:399-417) ---- */

/* GEMM leaf  C(i,j) (+)= A(i,k) * B(k,j)   -- statement of algorithms.py:80-83.
 * Row-major, k contiguous in A, j contiguous in B and C.  FP64 mma.sync DMMA
 * tiles staged through a cp.async multistage shared-memory pipeline.
 * Batched form: `batch` independent problems at the given element strides
 * (strideB may be 0 to share B) -- used for TTM, algorithms.py:300-301. */
int td_dgemm(void* stream, int64_t M, int64_t N, int64_t K,
             const double* A, int64_t lda, const double* B, int64_t ldb,
             double* C, int64_t ldc, int accumulate);
/* Same GEMM with a forced tile configuration (tuning / tests; csrc/gemm.cu
 * TD_GEMM_CONFIGS lists them); config < 0 = the default choice. */
int td_dgemm_config(void* stream, int config, int64_t M, int64_t N, int64_t K,
                    const double* A, int64_t lda, const double* B, int64_t ldb,
                    double* C, int64_t ldc, int accumulate);
int td_dgemm_batched(void* stream, int64_t batch, int64_t M, int64_t N, int64_t K,
                     const double* A, int64_t lda, int64_t strideA,
                     const double* B, int64_t ldb, int64_t strideB,
                     double* C, int64_t ldc, int64_t strideC, int accumulate);

/* Grouped GEMM: `count` (<= TD_GEMM_GROUP_MAX) independent GEMMs of any
 * shapes in ONE launch (the tiles of all problems share the grid).  Used for
 * the same-step GEMM leaves of the tasks co-located on one GPU (reference
 * simulator.py:615-622 runs them one after another): every output element
 * gets exactly the arithmetic of a separate td_dgemm call.  `problems` is
 * read during the call only.  Falls back to per-problem launches when a
 * problem cannot be addressed by TMA. */
#define TD_GEMM_GROUP_MAX 8
typedef struct td_gemm_problem {
  int64_t M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  /* optional second k-segment (K2 = 0: none), accumulated in the same registers
   * after the first: C (+)= A.B + A2.B2, A2 M x K2, B2 K2 x N (two k-slabs of a
   * task's steps that live in different pieces -> one launch instead of two) */
  int64_t K2;
  const double* A2;
  int64_t lda2;
  const double* B2;
  int64_t ldb2;
} td_gemm_problem;
int td_dgemm_grouped(void* stream, int count, const td_gemm_problem* problems, int accumulate);

/* TTV leaf  A(i,j) (+)= sum_k B(i,j,k) * c(k)   -- algorithms.py:280-281.
 * Rows (i,j) with element strides (sBi, sBj) in B and (sAi, sAj) in A; k
 * stride of B and c is 1.  Bandwidth-bound: 128-bit loads, one warp per row,
 * warp-shuffle row reduction. */
int td_ttv(void* stream, int64_t I, int64_t J, int64_t K,
           const double* B, int64_t sBi, int64_t sBj,
           const double* c, double* A, int64_t sAi, int64_t sAj, int accumulate);

/* TTM leaf  Y(i,j,l) (+)= sum_k B(i,j,k) * C(k,l)   -- algorithms.py:300-301.
 * Lowered onto the DMMA GEMM (rows (i,j) flattened when contiguous, else
 * batched over i). */
int td_ttm(void* stream, int64_t I, int64_t J, int64_t K, int64_t L,
           const double* B, int64_t sBi, int64_t sBj,
           const double* C, int64_t ldc,
           double* Y, int64_t sYi, int64_t sYj, int accumulate);

/* MTTKRP leaf  A(i,j) (+)= sum_{k,l} B(i,k,l) * C(k,j) * D(l,j)
 * -- algorithms.py:339-340.  Fused: T = B(i,k,:) . D on DMMA tiles, epilogue
 * multiplies by C(k,:) and reduces over k inside the CTA (deterministic, no
 * atomics).  l stride of B is 1; j stride of A, C, D is 1. */
int td_mttkrp(void* stream, int64_t I, int64_t K, int64_t L, int64_t R,
              const double* B, int64_t sBi, int64_t sBk,
              const double* C, int64_t ldc, const double* D, int64_t ldd,
              double* A, int64_t lda, int accumulate);
/* Same with a forced CTA configuration (csrc/mttkrp.cu; < 0 = default). */
int td_mttkrp_config(void* stream, int config, int64_t I, int64_t K, int64_t L, int64_t R,
                     const double* B, int64_t sBi, int64_t sBk,
                     const double* C, int64_t ldc, const double* D, int64_t ldd,
                     double* A, int64_t lda, int accumulate);

/* innerprod leaf  a (+)= sum B(x) * C(x) over a rows x n box
 * -- algorithms.py:320 and the 3-order form.
 * Rows at element strides sB / sC (contiguous within a row).  Deterministic
 * two-pass reduction: per-CTA partials into `work` (>= td_innerprod_work_size()
 * doubles), then one CTA sums them in fixed order into *out. */
int td_innerprod(void* stream, int64_t rows, int64_t n,
                 const double* B, int64_t sB, const double* C, int64_t sC,
                 double* out, double* work, int accumulate);
int64_t td_innerprod_work_size(void);

/* Generic exact-order nest evaluator: runs an arbitrary leaf statement over
 * an arbitrary loop nest (split / divide / rotate relations, guards) with the
 * reference interpreter's per-point accumulation order (cin.py:420-477).
 * `prog` points to a host struct td_nest_prog (csrc/interp.cuh), `bytes` its
 * size; it is copied into the launch. */
int td_nest_eval(void* stream, const void* prog, int64_t bytes);

/* ---- data movement helpers (tiles, commits, packing) ----------------- */
/* dst[box] (+)= src[box] for an n-d box (ndim <= 8), element strides. */
int td_copy_box(void* stream, int ndim, const int64_t* shape,
                double* dst, const int64_t* dst_strides,
                const double* src, const int64_t* src_strides, int accumulate);
/* Pitched 2-D copy between host (pinned) and device or device and device:
 * `rows` rows of `width` float64, row pitches in elements (cudaMemcpy2DAsync,
 * direction inferred from the pointers).  Used to upload / download
 * k-slabs of resident pieces while the leaves of earlier steps run. */
int td_memcpy_2d(void* stream, double* dst, int64_t dst_pitch, const double* src, int64_t src_pitch,
                 int64_t width, int64_t rows);
/* fill a contiguous range with a constant */
int td_fill(void* stream, double* dst, int64_t n, double value);
/* Synthetic input generator: writes the box [origin, origin+shape) of a
 * global tensor with dims `gdims` into dst (row-major, strides dst_strides).
 * Value at global linear index g: mode 0 -> integer in [-4,4],
 * mode 1 -> uniform(-1,1); both from splitmix64(seed, tensor_id, g)
 * (numpy twin: oracle/generator.py). */
int td_generate(void* stream, int ndim, const int64_t* gdims, const int64_t* origin,
                const int64_t* shape, double* dst, const int64_t* dst_strides,
                uint64_t seed, uint64_t tensor_id, int mode);

/* ---- NCCL over NVLink: the lowering of communicate / rotate --------------
 * (reference simulator.py:563-581 fetch events, :635-645 write-back events) */
#define TD_UNIQUE_ID_BYTES 128
int td_nccl_version(void);
int td_comm_unique_id(char* out /* TD_UNIQUE_ID_BYTES */);
/* one rank per process: comm over nranks GPUs, this process is `rank` on `device` */
int td_comm_init_rank(void** comm, int nranks, int rank, const char* unique_id, int device);
/* single process driving ndev devices */
int td_comm_init_all(void** comms, int ndev, const int* devices);
int td_comm_destroy(void* comm);
/* Sub-communicator over the ranks that pass the same color >= 0 (ranked by
 * key); color < 0 = not a member (*newcomm = NULL).  Collective over `comm`.
 * Used for the broadcast groups of fan-out transfers (SUMMA/COSMA panels). */
/* Inside td_group_start/end (one thread splitting several communicators) NCCL
 * writes *newcomm at td_group_end: keep the slot alive until then. */
int td_comm_split(void* comm, int color, int key, void** newcomm);
int td_group_start(void);
int td_group_end(void);
/* point-to-point transfer of `count` float64 (one CommEvent) */
int td_send(void* comm, void* stream, const double* buf, int64_t count, int peer);
int td_recv(void* comm, void* stream, double* buf, int64_t count, int peer);
/* broadcast / sum-reduce / sum-allreduce of float64 over the communicator */
int td_bcast(void* comm, void* stream, double* buf, int64_t count, int root);
int td_reduce_sum(void* comm, void* stream, const double* send, double* recv, int64_t count, int root);
int td_allreduce_sum(void* comm, void* stream, const double* send, double* recv, int64_t count);
/* recv[r*count ..] = send of rank r (SUMMA's row-panel gather along a grid axis). */
int td_allgather(void* comm, void* stream, const double* send, double* recv, int64_t count);
/* Cyclic shift along the communicator's ring: send to rank+delta, receive
 * from rank-delta (mod size) -- Cannon's systolic step, rotate() of
 * scheduling.py:222-260. */
int td_shift(void* comm, void* stream, const double* send, double* recv, int64_t count, int delta);
/* Host-side wait with a watchdog: returns when every stream is idle; while
 * waiting polls ncclCommGetAsyncError on every communicator, and on an async
 * error or after timeout_s seconds (<= 0: never) aborts ALL of them
 * (ncclCommAbort, so stuck NCCL kernels return) and fails with TD_ERR_NCCL
 * instead of hanging. */
int td_comm_wait(void* const* comms, int ncomms, void* const* streams, int nstreams, double timeout_s);

/* ---- peer memory over NVLink (csrc/peer.cu) ------------------------------
 * Reduce write-backs of the commit phase (reference simulator.py:624-654,
 * reduce events :635-645) whose whole partial goes to another GPU's home
 * piece: the task's leaf epilogue stores its tiles straight into an inbox in
 * the home GPU's HBM while the rest of the GEMM still computes; an 8-byte
 * NCCL token then orders the home's task-order accumulation after it.
 * One process, several GPUs: td_peer_enable + td_peer_alloc(handle = NULL).
 * One process per GPU: the home calls td_peer_alloc with a handle buffer and
 * the writer maps it with td_peer_open. */
#define TD_IPC_HANDLE_BYTES 64
/* 1 if `device` can map `peer`'s memory, 0 if not, < 0 on error. */
int td_peer_can_access(int device, int peer);
/* Let kernels on `device` access `peer`'s allocations (idempotent). */
int td_peer_enable(int device, int peer);
/* cudaMalloc `bytes` on `device`; if ipc_handle != NULL also export a CUDA
 * IPC handle (TD_IPC_HANDLE_BYTES bytes) for td_peer_open in another process. */
int td_peer_alloc(int device, int64_t bytes, void** ptr, char* ipc_handle);
int td_peer_free(int device, void* ptr);
/* Map another process's td_peer_alloc buffer into `device`'s context. */
int td_peer_open(int device, const char* ipc_handle, void** ptr);
int td_peer_close(int device, void* ptr);

/* ---- launch plans: the per-step loop in one call (csrc/plan.cu) ----------
 * One launch of a scheduled statement (reference simulator.py:557-663: per
 * step the fetches, every task's leaf, then the commits) lowered to a flat
 * array of ops in issue order.  Each op names one entry point of this header
 * and carries its arguments, in order, as 64-bit words (pointers and
 * integers as-is, doubles bit-cast); arrays an op points to (copy_box
 * shapes/strides, nest programs, grouped-GEMM problems) must outlive the
 * plan.  td_execute_plan issues every op, stops at the first failure (its
 * index in td_last_error(); an open NCCL group is closed), and is
 * asynchronous like the calls it replays. */
enum {
  TD_OP_DGEMM = 1, TD_OP_DGEMM_BATCHED = 2, TD_OP_DGEMM_GROUPED = 3, TD_OP_TTV = 4, TD_OP_TTM = 5,
  TD_OP_MTTKRP = 6, TD_OP_INNERPROD = 7, TD_OP_NEST_EVAL = 8, TD_OP_COPY_BOX = 9, TD_OP_MEMCPY_2D = 10,
  TD_OP_FILL = 11, TD_OP_GROUP_START = 12, TD_OP_GROUP_END = 13, TD_OP_SEND = 14, TD_OP_RECV = 15,
  TD_OP_BCAST = 16, TD_OP_REDUCE_SUM = 17, TD_OP_EVENT_RECORD = 18, TD_OP_STREAM_WAIT = 19
};
#define TD_OP_MAX_ARGS 16
typedef struct td_op {
  int32_t kind;
  int32_t nargs;
  int64_t arg[TD_OP_MAX_ARGS];
} td_op;
int td_execute_plan(const td_op* ops, int64_t count);

/* Cross-stream edges of a plan (no timing): record on the producer stream,
 * wait on the consumer stream.  `device` is the stream's device (a NULL
 * stream is that device's legacy default stream). */
int td_event_create(int device, void** event);
int td_event_destroy(void* event);
int td_event_record(void* event, void* stream, int device);
int td_stream_wait_event(void* stream, void* event, int device);

#ifdef __cplusplus
}
#endif
#endif /* DISTAL_B200_H */
