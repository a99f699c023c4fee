// Synthetic packed-image fill and per-block checksums.
//
// The generator and checksum are restated bit-for-bit in C by the oracle
// (oracle/dataplane.c: lp_ref_fill / lp_ref_checksum), which is how the tests
// prove that every receiver holds exactly the source's bytes.
#include "lp_common.cuh"
#include "../../include/lambdapipe.h"
#include <vector>

namespace {

struct TensorDesc {
  int64_t off;    // byte offset in the image (16-byte aligned)
  int64_t numel;  // bf16 elements
  int32_t kind;   // 0 random, 1 ones, 2 zeros
  int32_t scale_exp;
};

__device__ __forceinline__ uint16_t gen_bf16(uint64_t seed, int t, int64_t i, int kind, int scale_exp) {
  if (kind == 1) return 0x3F80;  // 1.0
  if (kind == 2) return 0;
  uint64_t z = lp::mix64(seed + ((uint64_t)(t + 1) << 40) + (uint64_t)i);
  int v = (int)(z >> 48) - 32768;
  float f = ldexpf((float)v, scale_exp - 15);  // exact: |v| < 2^16
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&b);
}

// one CTA row per tensor (blockIdx.y); grid-stride over 8-element groups
__global__ void fill_kernel(char* base, const TensorDesc* td, uint64_t seed) {
  const TensorDesc d = td[blockIdx.y];
  uint16_t* out = reinterpret_cast<uint16_t*>(base + d.off);
  const int64_t groups = d.numel / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t lo = gen_bf16(seed, blockIdx.y, g * 8 + 2 * j, d.kind, d.scale_exp);
      uint32_t hi = gen_bf16(seed, blockIdx.y, g * 8 + 2 * j + 1, d.kind, d.scale_exp);
      w[j] = lo | (hi << 16);
    }
    *reinterpret_cast<int4*>(out + g * 8) = make_int4(w[0], w[1], w[2], w[3]);
  }
  if (blockIdx.x == 0) {
    for (int64_t i = groups * 8 + threadIdx.x; i < d.numel; i += blockDim.x)
      out[i] = gen_bf16(seed, blockIdx.y, i, d.kind, d.scale_exp);
  }
}

struct BlockDesc {
  int64_t off;
  int64_t len;
};

__global__ void checksum_kernel(const char* base, const BlockDesc* bd, unsigned long long* out) {
  const BlockDesc d = bd[blockIdx.y];
  const uint64_t* w = reinterpret_cast<const uint64_t*>(base + d.off);
  const int64_t nw = d.len / 8;
  uint64_t acc = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nw;
       k += (int64_t)gridDim.x * blockDim.x) {
    acc += lp::mix64(w[k] ^ ((uint64_t)k * 0x9E3779B97F4A7C15ull));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ uint64_t part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += part[i];
    atomicAdd(out + blockIdx.y, (unsigned long long)s);
  }
}

}  // namespace

extern "C" {

int lp_fill_tensors(void* base, int n_tensors, const int64_t* off, const int64_t* numel,
                    const int32_t* kind, const int32_t* scale_exp, uint64_t seed, void* stream) {
  LP_CHECK(n_tensors > 0 && n_tensors < 65536, "lp_fill_tensors: bad tensor count %d", n_tensors);
  std::vector<TensorDesc> h(n_tensors);
  int64_t biggest = 0;
  for (int i = 0; i < n_tensors; ++i) {
    LP_CHECK(off[i] % 16 == 0, "lp_fill_tensors: tensor %d offset not 16-byte aligned", i);
    h[i] = {off[i], numel[i], kind[i], scale_exp[i]};
    if (numel[i] > biggest) biggest = numel[i];
  }
  cudaStream_t s = (cudaStream_t)stream;
  TensorDesc* d = nullptr;
  LP_CUDA(cudaMallocAsync(&d, sizeof(TensorDesc) * n_tensors, s));
  LP_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(TensorDesc) * n_tensors, cudaMemcpyHostToDevice, s));
  int64_t want = (biggest / 8 + 255) / 256;
  int gx = (int)(want < 1 ? 1 : (want > 1184 ? 1184 : want));
  fill_kernel<<<dim3(gx, n_tensors), 256, 0, s>>>((char*)base, d, seed);
  LP_CUDA(cudaGetLastError());
  LP_CUDA(cudaFreeAsync(d, s));
  LP_CUDA(cudaStreamSynchronize(s));
  return 0;
}

int lp_block_checksums(const void* base, int n_blocks, const int64_t* off, const int64_t* len,
                       uint64_t* out_host, void* stream) {
  LP_CHECK(n_blocks > 0 && n_blocks < 65536, "lp_block_checksums: bad block count");
  std::vector<BlockDesc> h(n_blocks);
  for (int i = 0; i < n_blocks; ++i) {
    LP_CHECK(off[i] % 8 == 0 && len[i] % 8 == 0, "lp_block_checksums: block %d not 8-byte aligned", i);
    h[i] = {off[i], len[i]};
  }
  cudaStream_t s = (cudaStream_t)stream;
  BlockDesc* d = nullptr;
  unsigned long long* acc = nullptr;
  LP_CUDA(cudaMallocAsync(&d, sizeof(BlockDesc) * n_blocks, s));
  LP_CUDA(cudaMallocAsync(&acc, sizeof(unsigned long long) * n_blocks, s));
  LP_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(BlockDesc) * n_blocks, cudaMemcpyHostToDevice, s));
  LP_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * n_blocks, s));
  checksum_kernel<<<dim3(148, n_blocks), 512, 0, s>>>((const char*)base, d, acc);
  LP_CUDA(cudaGetLastError());
  LP_CUDA(cudaMemcpyAsync(out_host, acc, sizeof(uint64_t) * n_blocks, cudaMemcpyDeviceToHost, s));
  LP_CUDA(cudaFreeAsync(d, s));
  LP_CUDA(cudaFreeAsync(acc, s));
  LP_CUDA(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"
