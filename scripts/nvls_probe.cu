// NVLS feasibility probe: can this box build an NVSwitch multicast
// object, bind HBM to it, and run multimem.ld_reduce / multimem.st through it?  With one
// visible GPU the team has one member, so ld_reduce returns the single bound value -- the
// probe checks the mechanism and times traffic that goes GPU -> NVSwitch -> GPU.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/nvls_probe.cu -lcuda -o /tmp/nvls_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CU(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_ = nullptr; cuGetErrorString(r_, &s_); \
  printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?"); return 1; } } while (0)
#define RT(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void ld_reduce_f32(const float* mc, float* out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
    reinterpret_cast<float4*>(out)[i] = make_float4(a, b, c, d);
  }
}
__global__ void ld_reduce_s32(const int* mc, int* out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    int v[4];   // integer ld_reduce has no vector form
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v[j]) : "l"(mc + 4 * i + j) : "memory");
    reinterpret_cast<int4*>(out)[i] = make_int4(v[0], v[1], v[2], v[3]);
  }
}
__global__ void ld_reduce_bf16(const unsigned* mc, unsigned* out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    unsigned a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc + 4 * i) : "memory");
    reinterpret_cast<uint4*>(out)[i] = make_uint4(a, b, c, d);
  }
}
__global__ void mc_store(float* mc, const float* in, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(in)[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
}

int main() {
  CU(cuInit(0));
  RT(cudaSetDevice(0));
  RT(cudaFree(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  int mcs = -1, ndev = 0;
  CU(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  RT(cudaGetDeviceCount(&ndev));
  printf("visible devices %d, MULTICAST_SUPPORTED %d\n", ndev, mcs);
  if (!mcs) { printf("RESULT no-multicast\n"); return 0; }

  const size_t bytes = 512ull << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gmin = 0, grec = 0;
  CU(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CU(cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("mc granularity min %zu rec %zu\n", gmin, grec);
  CUmemGenericAllocationHandle mc;
  // which object properties does the driver accept for a one-GPU team?
  for (unsigned long long ht : {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC})
    for (size_t sz : {gmin, (size_t)(256ull << 20), grec}) {
      CUmulticastObjectProp t = {};
      t.numDevices = 1; t.size = sz; t.handleTypes = ht;
      CUmemGenericAllocationHandle h;
      CUresult r = cuMulticastCreate(&h, &t);
      printf("cuMulticastCreate(numDevices 1, size %zu, handleTypes %llu) -> %d\n", sz, ht, (int)r);
      if (r == CUDA_SUCCESS) cuMemRelease(h);
    }
  {
    CUmulticastObjectProp t = {};
    t.numDevices = 2; t.size = grec; t.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle h;
    CUresult r = cuMulticastCreate(&h, &t);
    printf("cuMulticastCreate(numDevices 2) -> %d\n", (int)r);
    if (r == CUDA_SUCCESS) cuMemRelease(h);
  }
  CU(cuMulticastCreate(&mc, &mp));
  CU(cuMulticastAddDevice(mc, dev));

  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t ag = 0;
  CU(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("alloc granularity %zu\n", ag);
  CUmemGenericAllocationHandle mem;
  CU(cuMemCreate(&mem, bytes, &ap, 0));
  CU(cuMulticastBindMem(mc, 0, mem, 0, bytes, 0));

  CUdeviceptr uc = 0, mcp = 0;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemAddressReserve(&uc, bytes, grec, 0, 0));
  CU(cuMemMap(uc, bytes, 0, mem, 0));
  CU(cuMemSetAccess(uc, bytes, &acc, 1));
  CU(cuMemAddressReserve(&mcp, bytes, grec, 0, 0));
  CU(cuMemMap(mcp, bytes, 0, mc, 0));
  CU(cuMemSetAccess(mcp, bytes, &acc, 1));

  const size_t n = bytes / 4, n4 = n / 4;
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761ull) % 1000003) * 0.001f - 500.f;
  RT(cudaMemcpy((void*)uc, h.data(), bytes, cudaMemcpyHostToDevice));
  float* out;
  RT(cudaMalloc(&out, bytes));
  int sms = 0;
  RT(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  ld_reduce_f32<<<sms * 4, 512>>>((const float*)mcp, out, n4);
  RT(cudaGetLastError());
  RT(cudaDeviceSynchronize());
  std::vector<float> o(n);
  RT(cudaMemcpy(o.data(), out, bytes, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += (o[i] != h[i]);
  printf("ld_reduce.f32 1-member team: %zu mismatches of %zu\n", bad, n);

  cudaEvent_t e0, e1;
  RT(cudaEventCreate(&e0));
  RT(cudaEventCreate(&e1));
  for (int grid_mult : {1, 2, 4, 8}) {
    for (int it = 0; it < 3; ++it) ld_reduce_f32<<<sms * grid_mult, 512>>>((const float*)mcp, out, n4);
    RT(cudaEventRecord(e0));
    for (int it = 0; it < 20; ++it) ld_reduce_f32<<<sms * grid_mult, 512>>>((const float*)mcp, out, n4);
    RT(cudaEventRecord(e1));
    RT(cudaEventSynchronize(e1));
    float ms;
    RT(cudaEventElapsedTime(&ms, e0, e1));
    printf("ld_reduce.f32 512MiB grid %dx%d: %.1f us/launch, %.0f GB/s read through the switch\n",
           sms * grid_mult, 512, ms * 1e3 / 20, bytes / (ms / 20 * 1e-3) / 1e9);
  }
  // multimem.st broadcast (to the one member) and read back through the unicast mapping
  RT(cudaMemset(out, 0, bytes));
  float* src;
  RT(cudaMalloc(&src, bytes));
  RT(cudaMemcpy(src, h.data(), bytes, cudaMemcpyHostToDevice));
  RT(cudaMemset((void*)uc, 0, bytes));
  mc_store<<<sms * 4, 512>>>((float*)mcp, src, n4);
  RT(cudaDeviceSynchronize());
  RT(cudaMemcpy(o.data(), (void*)uc, bytes, cudaMemcpyDeviceToHost));
  bad = 0;
  for (size_t i = 0; i < n; ++i) bad += (o[i] != h[i]);
  printf("multimem.st.v4.f32 1-member team: %zu mismatches\n", bad);
  for (int it = 0; it < 3; ++it) mc_store<<<sms * 4, 512>>>((float*)mcp, src, n4);
  RT(cudaEventRecord(e0));
  for (int it = 0; it < 20; ++it) mc_store<<<sms * 4, 512>>>((float*)mcp, src, n4);
  RT(cudaEventRecord(e1));
  RT(cudaEventSynchronize(e1));
  float ms;
  RT(cudaEventElapsedTime(&ms, e0, e1));
  printf("multimem.st.f32 512MiB: %.1f us/launch, %.0f GB/s written through the switch\n", ms * 1e3 / 20,
         bytes / (ms / 20 * 1e-3) / 1e9);
  // int32 and bf16 reductions
  RT(cudaMemcpy((void*)uc, h.data(), bytes, cudaMemcpyHostToDevice));
  ld_reduce_s32<<<sms * 4, 512>>>((const int*)mcp, (int*)out, n4);
  ld_reduce_bf16<<<sms * 4, 512>>>((const unsigned*)mcp, (unsigned*)src, n4);
  RT(cudaDeviceSynchronize());
  std::vector<float> o2(n);
  RT(cudaMemcpy(o.data(), out, bytes, cudaMemcpyDeviceToHost));
  RT(cudaMemcpy(o2.data(), src, bytes, cudaMemcpyDeviceToHost));
  size_t bad_i = 0, bad_b = 0;
  for (size_t i = 0; i < n; ++i) { bad_i += (o[i] != h[i]); bad_b += (o2[i] != h[i]); }
  printf("ld_reduce.s32 mismatches %zu, ld_reduce.bf16x2(acc f32) mismatches %zu (bitwise identity expected)\n", bad_i, bad_b);
  printf("RESULT ok\n");
  return 0;
}
