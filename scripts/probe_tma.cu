// Access-pattern probe (MEASUREMENT ONLY, not the product): the loopback all-reduce's compulsory
// traffic -- P = 8 virtual ranks, every column read once from each rank and the result written
// once to each rank -- moved by different mechanisms, to find the HBM floor of each:
//   A  ldg   : one thread per 16-B column, 8 x LDG.128 + fold + 8 x STG.128
//   B  tmald : a producer warp bulk-loads (cp.async.bulk) the 8 ranks' segments of a tile into a
//              shared-memory ring; 512 consumer threads fold from smem and STG.128 x 8
//   C  tmaall: as B, and the result goes to smem and out by 8 bulk stores per tile
//   D  copy  : 1 read + 1 write stream of the same total bytes (LDG/STG), the copy-peak pattern
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/probe_tma.cu -o scripts/probe_tma.bin
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int P = 8;
constexpr int kCons = 512;          // consumer threads (one column of the tile each)
constexpr int kTileB = kCons * 16;  // bytes per rank segment per tile
#ifndef STAGES
#define STAGES 3
#endif

struct Bufs { char* r[P]; };

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(su32(b)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_ld(void* s, const void* g, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(s)),
               "l"(g), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bulk_st(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(n) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

__global__ void __launch_bounds__(256) k_ldg(Bufs b, size_t ncol) {
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < ncol; c += (size_t)gridDim.x * blockDim.x) {
    float4 v[P];
#pragma unroll
    for (int i = 0; i < P; ++i) v[i] = __ldcg(reinterpret_cast<const float4*>(b.r[i]) + c);
    float4 s0 = add4(add4(add4(v[0], v[1]), v[2]), v[3]), s1 = add4(add4(add4(v[4], v[5]), v[6]), v[7]);
    float4 f = add4(s0, s1);
#pragma unroll
    for (int i = 0; i < P; ++i) reinterpret_cast<float4*>(b.r[i])[c] = f;
  }
}

template <bool TMA_ST>
__global__ void __launch_bounds__(kCons + 32, 1) k_tma(Bufs b, size_t ntiles) {
  extern __shared__ __align__(128) char sm[];
  char* ring = sm;                                             // STAGES x P x kTileB
  char* outs = sm + (size_t)STAGES * P * kTileB;               // STAGES x kTileB (TMA_ST)
  uint64_t* full = reinterpret_cast<uint64_t*>(outs + (TMA_ST ? (size_t)STAGES * kTileB : 0));
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == kCons / 32) {  // producer warp
    if (lane == 0) {
      uint32_t i = 0;
      for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        if (TMA_ST && i >= STAGES) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arm(&full[s], P * kTileB);
        for (int r = 0; r < P; ++r) bulk_ld(ring + ((size_t)s * P + r) * kTileB, b.r[r] + t * kTileB, kTileB, &full[s]);
      }
    }
    return;
  }
  uint32_t i = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    float4 v[P];
#pragma unroll
    for (int r = 0; r < P; ++r) v[r] = reinterpret_cast<const float4*>(ring + ((size_t)s * P + r) * kTileB)[threadIdx.x];
    float4 s0 = add4(add4(add4(v[0], v[1]), v[2]), v[3]), s1 = add4(add4(add4(v[4], v[5]), v[6]), v[7]);
    float4 f = add4(s0, s1);
    if (!TMA_ST) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
      for (int r = 0; r < P; ++r) reinterpret_cast<float4*>(b.r[r] + t * kTileB)[threadIdx.x] = f;
    } else {
      reinterpret_cast<float4*>(outs + (size_t)s * kTileB)[threadIdx.x] = f;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // the whole tile's result in smem, then one thread per rank bulk-stores it
      asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
      if (threadIdx.x < P) bulk_st(b.r[threadIdx.x] + t * kTileB, outs + (size_t)s * kTileB, kTileB);
      if (threadIdx.x < P) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (TMA_ST && threadIdx.x < P) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_copy(const float4* a, float4* o, size_t n) {
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < n; c += (size_t)gridDim.x * blockDim.x) o[c] = __ldcg(a + c);
}

int main() {
  const size_t per = 102228128;  // bytes per rank (the ResNet-50 gradient set)
  const size_t bytes = per / kTileB * kTileB;
  Bufs b;
  for (int r = 0; r < P; ++r) {
    cudaMalloc(&b.r[r], bytes);
    cudaMemset(b.r[r], 0, bytes);
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double comp = 2.0 * P * bytes;
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int reps = 20;
    for (int k = 0; k < reps; ++k) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-10s %.4f ms  %.0f GB/s (compulsory %.3f GB)  err=%s\n", name, ms, comp / ms / 1e6, comp / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  const size_t ncol = bytes / 16, ntiles = bytes / kTileB;
  for (int blocks : {4, 8})
    timeit(blocks == 4 ? "ldg(4/SM)" : "ldg(8/SM)", [&] { k_ldg<<<sms * blocks, 256>>>(b, ncol); });
  const size_t sm_ld = (size_t)STAGES * P * kTileB + 2 * STAGES * 8;
  const size_t sm_all = sm_ld + (size_t)STAGES * kTileB;
  cudaFuncSetAttribute(k_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_ld);
  cudaFuncSetAttribute(k_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_all);
  timeit("tmald", [&] { k_tma<false><<<sms, kCons + 32, sm_ld>>>(b, ntiles); });
  timeit("tmaall", [&] { k_tma<true><<<sms, kCons + 32, sm_all>>>(b, ntiles); });
  float4 *a, *o;
  cudaMalloc(&a, P * bytes);
  cudaMalloc(&o, P * bytes);
  timeit("copy", [&] { k_copy<<<sms * 8, 256>>>(a, o, P * bytes / 16); });
  return 0;
}
