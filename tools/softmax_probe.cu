// Probe: throughput of the prefill attention's softmax inner loop in
// isolation (64 scores per thread: FFMA2 scale, MUFU.EX2 / FMA-pipe exp2 for
// one pair in four, FADD2 row sum, F2FP pack, swizzled STS.128 of fp16 P,
// FMNMX3 raw max) at W warps per SM, scores re-read from smem each pass.
// Prints cycles per pass per warp-pair (compare with the ~1,300-cycle exp
// phase of attention_tc_kernel's chunk trace).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smx tools/softmax_probe.cu && /tmp/smx
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}" : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  constexpr float MAGIC = 12582912.0f;
  x.x = fmaxf(x.x, -100.f);
  x.y = fmaxf(x.y, -100.f);
  const float2 t = fadd2(x, make_float2(MAGIC, MAGIC));
  const float2 n = fadd2(t, make_float2(-MAGIC, -MAGIC));
  const float2 f = fadd2(x, make_float2(-n.x, -n.y));
  float2 q = ffma2(f, make_float2(0.05517166f, 0.05517166f), make_float2(0.24261116f, 0.24261116f));
  q = ffma2(q, f, make_float2(0.69326099f, 0.69326099f));
  q = ffma2(q, f, make_float2(0.99992807f, 0.99992807f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

template <int POLY, int KW>
__global__ void k(float* out, long long* clk, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* S = reinterpret_cast<float*>(sm);                       // [threads][KW] scores
  uint8_t* P = sm + blockDim.x * KW * 4;                           // [threads / 128][128 rows][128 B] fp16 P
  const int r = threadIdx.x & 127;
  for (int i = threadIdx.x; i < blockDim.x * KW; i += blockDim.x) S[i] = -0.01f * (i % 97);
  __syncthreads();
  float l = 0.f, mraw = -INFINITY;
  const float2 sl = make_float2(0.125f, 0.125f);
  float nm = 0.5f;
  uint8_t* prow = P + (threadIdx.x >> 7) * 16384 + (r >> 3) * 1024 + (r & 7) * 128;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[KW];
#pragma unroll
    for (int q = 0; q < KW / 4; ++q) {
      const float4 w = reinterpret_cast<const float4*>(S + threadIdx.x * KW)[q ^ (threadIdx.x & 7)];
      v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
    }
    float2 ls2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    float mx4[4] = {mraw, mraw, mraw, mraw};
    const float2 nm2 = make_float2(-nm, -nm);
#pragma unroll
    for (int q = 0; q < KW / 8; ++q) {
      uint32_t pk[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const float2 sv = make_float2(v[q * 8 + e], v[q * 8 + e + 1]);
        mx4[e >> 1] = fmax3(mx4[e >> 1], sv.x, sv.y);
        const float2 x = ffma2(sv, sl, nm2);
        float2 p;
        if ((e >> 1) >= 4 - POLY) p = exp2_poly2(x);
        else { p.x = ex2(x.x); p.y = ex2(x.y); }
        ls2[e >> 1] = fadd2(ls2[e >> 1], p);
        const __half2 hv = __floats2half2_rn(p.x, p.y);
        pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&hv);
      }
      *reinterpret_cast<uint4*>(prow + ((q ^ (r & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    const float2 s01 = fadd2(ls2[0], ls2[1]), s23 = fadd2(ls2[2], ls2[3]);
    l += (s01.x + s01.y) + (s23.x + s23.y);
    mraw = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
    nm += 1e-7f;
    __syncwarp();
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + mraw;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* clk;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&clk, sms * 8);
  const int iters = 2000;
  auto run = [&](auto kern, int KW, int warps, const char* name) {
    const int smem = warps * 32 * KW * 4 + ((warps * 32 + 127) / 128) * 16384;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, warps * 32, smem>>>(out, clk, iters);
    kern<<<sms, warps * 32, smem>>>(out, clk, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double per_pass = (double)c / iters;
    const double exps_per_clk = (double)warps * 32 * KW * iters / c;
    printf("%-28s KW %3d warps/SM %2d: %7.1f cycles per pass, %.2f exp per clock per SM (%s)\n", name, KW, warps,
           per_pass, exps_per_clk, cudaGetErrorString(e));
  };
  for (int w : {4, 8, 12, 16}) {
    run(k<0, 64>, 64, w, "SFU only");
    run(k<1, 64>, 64, w, "1 pair in 4 on FMA pipe");
    run(k<2, 64>, 64, w, "2 pairs in 4 on FMA pipe");
  }
  return 0;
}
