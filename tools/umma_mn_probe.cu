// Probe: one CTA computes D[128 x N] = A[128 x 64] * B[64 x N] with
// tcgen05.mma kind::f16 (fp16 in, fp32 out), A K-major SW128 (rows of 64
// elements = one 128 B swizzle atom), B MN-major SW128 (B[k][n] with n
// contiguous: N/64 atoms of [64 k rows][64 n] each, loaded like a TMA box of
// 64 n x 64 k with 128B swizzle), for the descriptor variants listed below,
// and prints the max error vs a host fp32 reference.  Validates the layout
// the tcgen05 attention kernel uses for P.V (V stored [key][hd]).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_mn tools/umma_mn_probe.cu && /tmp/umma_mn
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, K = 64, N = 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// byte offset of element (row, col) in a [rows][64] 128B-swizzled atom block
__device__ __host__ inline int sw(int row, int col) {
  return (row / 8) * 1024 + (row % 8) * 128 + ((((col / 8) ^ (row % 8)) & 7) * 16) + (col % 8) * 2;
}

__global__ void probe(const __half* A, const __half* B, float* D, uint32_t lbo, uint32_t sbo, int kstep_mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sb = sa + M * 128;                       // A: 128 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  // A: K-major [M][K]
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    int r = i / K, c = i % K;
    *(__half*)(sa + sw(r, c)) = A[r * K + c];
  }
  // B: MN-major: atom a holds n in [64a, 64a+64): [K rows][64 n]
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    int k = i / N, n = i % N;
    *(__half*)(sb + (n / 64) * (K * 128) + sw(k, n % 64)) = B[k * N + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    // c F32, a F16 (0), b F16 (0), a K-major, b MN-major (bit 16), N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t da = desc(su32(sa) + kk * 32, 16, 1024);
      uint32_t boff = kstep_mode == 0 ? kk * 16 * 128 : kk * 2 * sbo;
      uint64_t db = desc(su32(sb) + boff, lbo, sbo);
      uint32_t acc = kk > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  // wait
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = threadIdx.x;      // 4 warps: lanes 0..127
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + ((uint32_t)((threadIdx.x / 32) * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(N));
}

int main() {
  std::vector<__half> hA(M * K), hB(K * N);
  std::vector<float> fA(M * K), fB(K * N), ref(M * N, 0.f);
  srand(1);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 8.f; hA[i] = __float2half(v); fA[i] = v; }
  for (int i = 0; i < K * N; ++i) { float v = (rand() % 13 - 6) / 4.f; hB[i] = __float2half(v); fB[i] = v; }
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += fA[m * K + k] * fB[k * N + n];
      ref[m * N + n] = s;
    }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, K * N * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), K * N * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  struct V { uint32_t lbo, sbo; int mode; const char* name; } vs[] = {
      {K * 128, 1024, 0, "LBO=atom stride(MN) SBO=1024(K 8-row) kstep=16 rows"},
      {1024, K * 128, 0, "LBO=1024 SBO=atom stride"},
      {K * 128, 1024, 1, "LBO=atom SBO=1024 kstep=2*SBO"},
  };
  for (auto& v : vs) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128, 64 * 1024>>>(dA, dB, dD, v.lbo, v.sbo, v.mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(M * N);
    cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("%-55s err %.4g (%s)\n", v.name, err, cudaGetErrorString(e));
  }
  return 0;
}
