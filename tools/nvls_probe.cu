// NVLS (NVSwitch multicast) probe: one process, all visible GPUs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/nvls_probe tools/nvls_probe.cu -lcuda
//   gpurun_out/nvls_probe [MiB] [ctas]
// Creates a multicast object over every GPU, binds one physical buffer per GPU,
// and times GPU0 reading its local HBM and storing it through the multicast
// address (multimem.st) so the switch replicates it into every GPU's buffer.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s: %s (line %d)\n", #x, s_, __LINE__); exit(1); } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r_)); exit(1); } } while (0)

__global__ void fill(uint4* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = (uint32_t)i * 2654435761u ^ seed;
    p[i] = make_uint4(a, a * 3u + 1u, a ^ 0x7fc00001u, 0xffc00000u | (a & 0xff));  // NaN patterns included
  }
}

__global__ void mc_store(const uint4* __restrict__ src, uint4* mc, size_t n) {
  constexpr int U = 4;
  size_t T = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * T < n; i += U * T) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i + u * T), "r"(v[u].x),
                   "r"(v[u].y), "r"(v[u].z), "r"(v[u].w) : "memory");
  }
  for (; i < n; i += T)
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(src[i].x),
                 "r"(src[i].y), "r"(src[i].z), "r"(src[i].w) : "memory");
}

__global__ void cmp(const uint4* a, const uint4* b, size_t n, unsigned long long* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = a[i], y = b[i];
    if (x.x != y.x || x.y != y.y || x.z != y.z || x.w != y.w) atomicAdd(bad, 1ull);
  }
}

int main(int argc, char** argv) {
  size_t mib = argc > 1 ? atol(argv[1]) : 4096;
  int ctas = argc > 2 ? atoi(argv[2]) : 132;
  CK(cuInit(0));
  int ndev = 0;
  RK(cudaGetDeviceCount(&ndev));
  for (int d = 0; d < ndev; ++d) {
    int mc = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
    printf("device %d multicast_supported=%d\n", d, mc);
  }
  if (ndev < 2) { printf("need >= 2 GPUs\n"); return 0; }
  CUmulticastObjectProp prop = {};
  prop.numDevices = ndev;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, mgran = 0;
  prop.size = 1 << 21;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CK(cuMulticastGetGranularity(&mgran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM));
  size_t bytes = (mib << 20);
  bytes = (bytes + gran - 1) / gran * gran;
  prop.size = bytes;
  printf("granularity recommended=%zu minimum=%zu bytes=%zu\n", gran, mgran, bytes);
  CUmemGenericAllocationHandle mch;
  CK(cuMulticastCreate(&mch, &prop));
  for (int d = 0; d < ndev; ++d) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    CK(cuMulticastAddDevice(mch, dev));
  }
  std::vector<CUdeviceptr> uni(ndev), mcva(ndev);
  std::vector<CUmemGenericAllocationHandle> ph(ndev);
  for (int d = 0; d < ndev; ++d) {
    RK(cudaSetDevice(d));
    RK(cudaFree(0));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ug = 0;
    CK(cuMemGetAllocationGranularity(&ug, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CK(cuMemCreate(&ph[d], bytes, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph[d], 0, bytes, 0));
    CK(cuMemAddressReserve(&uni[d], bytes, gran, 0, 0));
    CK(cuMemMap(uni[d], bytes, 0, ph[d], 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uni[d], bytes, &acc, 1));
    CK(cuMemAddressReserve(&mcva[d], bytes, gran, 0, 0));
    CK(cuMemMap(mcva[d], bytes, 0, mch, 0));
    CK(cuMemSetAccess(mcva[d], bytes, &acc, 1));
    RK(cudaMemset((void*)uni[d], 0, bytes));
  }
  RK(cudaSetDevice(0));
  uint4* src;
  RK(cudaMalloc(&src, bytes));
  size_t n = bytes / 16;
  fill<<<1184, 256>>>(src, n, 12345u);
  RK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  for (int c : {ctas, 74, 148, 296}) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      RK(cudaEventRecord(e0));
      mc_store<<<c, 512>>>(src, (uint4*)mcva[0], n);
      RK(cudaEventRecord(e1));
      RK(cudaEventSynchronize(e1));
      float ms;
      RK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf("multimem.st %zu MiB to %d GPUs, %d CTAs: %.3f ms, %.1f GB/s per receiver\n", mib, ndev, c, best,
           bytes / (best * 1e-3) / 1e9);
  }
  // verify every GPU's unicast buffer against the source (peer reads from GPU0)
  for (int d = 0; d < ndev; ++d) {
    RK(cudaSetDevice(d));
    uint4* copy;
    RK(cudaMalloc(&copy, bytes));
    RK(cudaMemcpyPeer(copy, d, src, 0, bytes));
    unsigned long long* bad;
    RK(cudaMalloc(&bad, 8));
    RK(cudaMemset(bad, 0, 8));
    cmp<<<1184, 256>>>((const uint4*)uni[d], copy, n, bad);
    unsigned long long h = 0;
    RK(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost));
    printf("device %d mismatched 16B words: %llu\n", d, h);
    RK(cudaFree(copy));
    RK(cudaFree(bad));
  }
  return 0;
}
