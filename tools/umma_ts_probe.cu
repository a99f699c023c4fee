// Probe: tcgen05.mma kind::f16 with the A operand in TMEM ("TS" form), the
// layout the FA4-style attention kernel needs for O += P V with P kept in
// TMEM: D[128 x N] = A[128 x 64] * B[64 x N], A (fp16) written by tcgen05.st
// as row = lane, column c = packed half2 of k = 2c, 2c + 1; B MN-major SW128
// in smem (B[k][n], n contiguous: V's [key][hd] layout).  Prints the max
// error vs a host fp32 reference for the A-address step variants below.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_ts tools/umma_ts_probe.cu && /tmp/umma_ts
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
__device__ __host__ inline int sw(int row, int col) {
  return (row / 8) * 1024 + (row % 8) * 128 + ((((col / 8) ^ (row % 8)) & 7) * 16) + (col % 8) * 2;
}

__global__ void probe(const __half* A, const __half* B, float* D, int astep) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sb = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;           // D: columns [0, N); A: columns [N, N + K / 2)
  const int row = threadIdx.x;
  const uint32_t lane_off = (uint32_t)((threadIdx.x / 32) * 32) << 16;
  {  // A row -> TMEM (32 columns of half2)
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) {
      __half2 h = __halves2half2(A[row * K + 2 * c], A[row * K + 2 * c + 1]);
      v[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + lane_off + N),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
        "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
        "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    // c F32 (bit 4), a F16 / b F16 (0), a K-major (0), b MN-major (bit 16), N >> 3, M >> 4
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t db = desc(su32(sb) + kk * 2048, K * 128, 1024);
      const uint32_t ta = tm + N + kk * astep;
      const uint32_t acc = kk > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
          "r"(ta), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + lane_off + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  std::vector<__half> hA(M * K), hB(K * N);
  std::vector<float> fA(M * K), fB(K * N), ref(M * N, 0.f);
  srand(3);
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
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int astep : {8, 16, 4}) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, astep);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(M * N);
    cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("A in TMEM, +%2d columns per 16-key step: max err %.4g (%s)\n", astep, err, cudaGetErrorString(e));
  }
  return 0;
}
