/* A non-Python host driving the B200 path through the C ABI alone
 * (include/distal_b200.h): one launch plan -- C = 0, then C += A_k0 B_k0 and
 * C += A_k1 B_k1 over two k-halves -- issued by td_execute_plan in one call,
 * checked against a host product.  Build: `make examples` (links
 * libdistal_b200.so); run: examples/plan_demo  (prints "plan_demo OK"). */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "distal_b200.h"

static int64_t bits_of(double d) {
  int64_t w;
  memcpy(&w, &d, sizeof w);
  return w;
}

int main(void) {
  const int64_t M = 192, N = 160, K = 256;
  double *hA = (double*)malloc(sizeof(double) * M * K), *hB = (double*)malloc(sizeof(double) * K * N);
  double *hC = (double*)malloc(sizeof(double) * M * N);
  for (int64_t i = 0; i < M * K; ++i) hA[i] = (double)((i * 7) % 9) - 4.0;   /* integers: exact */
  for (int64_t i = 0; i < K * N; ++i) hB[i] = (double)((i * 5) % 9) - 4.0;
  double *dA, *dB, *dC;
  cudaStream_t st;
  if (cudaMalloc((void**)&dA, sizeof(double) * M * K) || cudaMalloc((void**)&dB, sizeof(double) * K * N) ||
      cudaMalloc((void**)&dC, sizeof(double) * M * N) || cudaStreamCreate(&st)) {
    fprintf(stderr, "plan_demo: no usable GPU\n");
    return 2;
  }
  cudaMemcpy(dA, hA, sizeof(double) * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(double) * K * N, cudaMemcpyHostToDevice);

  td_op ops[3];
  memset(ops, 0, sizeof ops);
  const int64_t half = K / 2;
  int64_t fill[] = {(int64_t)st, (int64_t)dC, M * N, bits_of(0.0)};
  int64_t g0[] = {(int64_t)st, M, N, half, (int64_t)dA, K, (int64_t)dB, N, (int64_t)dC, N, 1};
  int64_t g1[] = {(int64_t)st, M, N, K - half, (int64_t)(dA + half), K, (int64_t)(dB + half * N), N,
                  (int64_t)dC, N, 1};
  ops[0].kind = TD_OP_FILL, ops[0].nargs = 4, memcpy(ops[0].arg, fill, sizeof fill);
  ops[1].kind = TD_OP_DGEMM, ops[1].nargs = 11, memcpy(ops[1].arg, g0, sizeof g0);
  ops[2].kind = TD_OP_DGEMM, ops[2].nargs = 11, memcpy(ops[2].arg, g1, sizeof g1);
  if (td_execute_plan(ops, 3) != TD_OK) {
    fprintf(stderr, "plan_demo: %s\n", td_last_error());
    return 1;
  }
  cudaStreamSynchronize(st);
  cudaMemcpy(hC, dC, sizeof(double) * M * N, cudaMemcpyDeviceToHost);
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) {
      double want = 0.0;
      for (int64_t k = 0; k < K; ++k) want += hA[i * K + k] * hB[k * N + j];
      if (hC[i * N + j] != want) {
        fprintf(stderr, "plan_demo: C[%lld,%lld] = %g, want %g\n", (long long)i, (long long)j, hC[i * N + j], want);
        return 1;
      }
    }
  printf("plan_demo OK (%lld x %lld x %lld, 3 ops in one td_execute_plan)\n", (long long)M, (long long)N,
         (long long)K);
  return 0;
}
