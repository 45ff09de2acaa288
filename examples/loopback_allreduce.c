/* Plain-C use of libddl on a GPU (no Python): 8 virtual ranks on one device, dims 2x4
 * (= {4, 2} innermost first), an int32 all-reduce checked against the closed form of
 * rank-indexed inputs, then an fp32 avg all-reduce checked for replica consistency.
 *
 *   gcc -std=c99 -I include examples/loopback_allreduce.c -L paper_1811_12174_b200 -lddl \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,paper_1811_12174_b200 -o /tmp/lb && /tmp/lb
 */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ddl.h"

#define P 8
#define N 1000003 /* ragged on purpose */

static int fail(const char* what, int code) {
  fprintf(stderr, "%s failed: %s (%d)\n", what, ddl_result_string((ddl_result_t)code), code);
  return 1;
}

int main(void) {
  const int dims[2] = {4, 2};
  ddl_comm_t comm;
  int r = ddl_loopback_init(&comm, P, dims, 2, 0);
  if (r != DDL_SUCCESS) return fail("ddl_loopback_init", r);

  void* bufs[P];
  int* host = (int*)malloc(sizeof(int) * N);
  for (int k = 0; k < P; ++k) {
    if (cudaMalloc(&bufs[k], sizeof(int) * N) != cudaSuccess) return fail("cudaMalloc", 4);
    for (int i = 0; i < N; ++i) host[i] = (1 << k) | ((i % (1 << 20)) << 8); /* rank bitmask */
    cudaMemcpy(bufs[k], host, sizeof(int) * N, cudaMemcpyHostToDevice);
  }
  r = ddl_group_allreduce(comm, bufs, N, DDL_INT32, DDL_SUM, NULL);
  if (r != DDL_SUCCESS) return fail("ddl_group_allreduce(int32)", r);
  cudaDeviceSynchronize();
  if ((r = ddl_async_error(comm)) != DDL_SUCCESS) return fail("async", r);
  for (int k = 0; k < P; ++k) {
    cudaMemcpy(host, bufs[k], sizeof(int) * N, cudaMemcpyDeviceToHost);
    for (int i = 0; i < N; ++i) {
      const unsigned want = (unsigned)((1 << P) - 1) + (unsigned)P * ((unsigned)(i % (1 << 20)) << 8);
      if ((unsigned)host[i] != want) {
        fprintf(stderr, "rank %d element %d: %u != %u\n", k, i, (unsigned)host[i], want);
        return 1;
      }
    }
  }

  /* fp32 avg: every virtual rank must end bit-identical */
  float* hf = (float*)host;
  for (int k = 0; k < P; ++k) {
    for (int i = 0; i < N; ++i) hf[i] = (float)((i * 7 + k * 13) % 101) / 3.0f;
    cudaMemcpy(bufs[k], hf, sizeof(float) * N, cudaMemcpyHostToDevice);
  }
  r = ddl_group_allreduce(comm, bufs, N, DDL_FLOAT32, DDL_AVG, NULL);
  if (r != DDL_SUCCESS) return fail("ddl_group_allreduce(fp32)", r);
  cudaDeviceSynchronize();
  float* ref = (float*)malloc(sizeof(float) * N);
  cudaMemcpy(ref, bufs[0], sizeof(float) * N, cudaMemcpyDeviceToHost);
  for (int k = 1; k < P; ++k) {
    cudaMemcpy(hf, bufs[k], sizeof(float) * N, cudaMemcpyDeviceToHost);
    if (memcmp(hf, ref, sizeof(float) * N)) {
      fprintf(stderr, "rank %d differs from rank 0\n", k);
      return 1;
    }
  }
  for (int k = 0; k < P; ++k) cudaFree(bufs[k]);
  ddl_finalize(comm);
  free(host);
  free(ref);
  printf("loopback_allreduce ok: 8 virtual ranks, dims 2x4, int32 closed form + fp32 replicas identical\n");
  return 0;
}
