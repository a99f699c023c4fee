// Probe: MUFU.EX2 and FMA-polynomial exp2 throughput per SM per clock on
// this GPU (the softmax of the tensor-core attention is bound by one of
// them).  One CTA per SM, W warps, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sfu tools/sfu_probe.cu && /tmp/sfu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for x <= 0 on the FMA pipe: split x = n + f (f in [0,1)), degree-3
// minimax polynomial for 2^f, exponent add on the integer pipe
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = fmaf(f, 0.0555041086648216f, 0.2402264923172690f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)fl << 23));
}

template <int MODE>
__global__ void k(float* out, long long* clk, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = -0.001f * (threadIdx.x + j);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) a[j] = ex2(a[j]) - 1.0f;
      else if (MODE == 1) a[j] = ex2_poly(a[j]) - 1.0f;
      else if (MODE == 2) a[j] = (j & 1 ? ex2_poly(a[j]) : ex2(a[j])) - 1.0f;
      else if (MODE == 3) {       // F2FP pack (fp32 pair -> half2) + unpack-free feedback
        const __half2 h = __floats2half2_rn(a[j], a[j ^ 1]);
        a[j] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&h)) * 1e-30f - 0.5f;
      } else {                    // MUFU.EX2 then F2FP (the softmax's per-pair work)
        const float e0 = ex2(a[j]);
        const __half2 h = __floats2half2_rn(e0, e0);
        a[j] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&h)) * 1e-30f - 0.5f;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* clk;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&clk, sms * 8);
  const int iters = 4096;
  const char* names[5] = {"MUFU.EX2", "FMA poly exp2", "half MUFU / half poly", "F2FP pack (+FMUL/FADD)",
                          "MUFU.EX2 + F2FP"};
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : k<4>;
      fn<<<sms, warps * 32>>>(out, clk, iters);
      fn<<<sms, warps * 32>>>(out, clk, iters);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)warps * 32 * 8 * iters;
      printf("%-24s warps/SM %2d: %.2f ops per clock per SM\n", names[mode], warps, ops / c);
    }
  return 0;
}
