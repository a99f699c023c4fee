// Llama decoder-layer kernels around the tensor-core GEMMs (lp_gemm.cu):
// embedding gather, RMSNorm, RoPE + KV-cache append, ragged causal attention
// (prefill and decode share one kernel: every token attends to positions
// 0..pos of its own sequence), and greedy argmax.
//
// Numerics: weights bf16, residual stream fp32, GEMM inputs bf16, fp32
// accumulation everywhere (the oracle, oracle/llama.py, is the same network
// in fp32 on the same bf16 weights).
#include "lp_common.cuh"
#include "../../include/lambdapipe.h"

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// x[t, :] = float(table[tokens[t], :])
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ table, int64_t d, const int32_t* __restrict__ tokens,
                             float* __restrict__ x) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  const __nv_bfloat16* row = table + (int64_t)tokens[t] * d;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) x[(int64_t)t * d + i] = __bfloat162float(row[i]);
}

// y[t, :] = bf16(x * rsqrt(mean(x^2) + eps) * w)
__global__ void rmsnorm_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w, int64_t d,
                               float eps, __nv_bfloat16* __restrict__ y) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  const float* xr = x + (int64_t)t * d;
  float ss = 0.f;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
  __shared__ float part[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[0] = v;
  }
  __syncthreads();
  const float r = rsqrtf(part[0] / (float)d + eps);
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x)
    y[(int64_t)t * d + i] = __float2bfloat16_rn(xr[i] * r * __bfloat162float(w[i]));
}

// qkv: [T, (H + 2*KV) * hd] fp32.  HF Llama rotate_half RoPE: element j < hd/2
// pairs with j + hd/2 at angle pos * theta^(-2j/hd).
// q_out [T, H*hd] bf16; k/v appended to cache[seq][kv][pos][hd] bf16.
__global__ void rope_kv_kernel(const float* __restrict__ qkv, int H, int KV, int hd, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ seq, float theta, __nv_bfloat16* __restrict__ q_out,
                               __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache,
                               int64_t max_len) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  const int p = pos[t];
  const int sq = seq[t];
  const int half = hd / 2;
  const float* row = qkv + (int64_t)t * (H + 2 * KV) * hd;
  for (int idx = threadIdx.x; idx < (H + KV) * half; idx += blockDim.x) {
    const int head = idx / half;
    const int j = idx % half;
    const float inv = powf(theta, -2.0f * (float)j / (float)hd);
    float sn, cs;
    sincosf((float)p * inv, &sn, &cs);
    const float* src = row + head * hd;
    const float a = src[j], b = src[j + half];
    const float ra = a * cs - b * sn;
    const float rb = b * cs + a * sn;
    if (head < H) {
      __nv_bfloat16* dst = q_out + ((int64_t)t * H + head) * hd;
      dst[j] = __float2bfloat16_rn(ra);
      dst[j + half] = __float2bfloat16_rn(rb);
    } else {
      const int kh = head - H;
      __nv_bfloat16* dst = k_cache + (((int64_t)sq * KV + kh) * max_len + p) * hd;
      dst[j] = __float2bfloat16_rn(ra);
      dst[j + half] = __float2bfloat16_rn(rb);
    }
  }
  for (int idx = threadIdx.x; idx < KV * hd; idx += blockDim.x) {
    const int kh = idx / hd;
    const int j = idx % hd;
    v_cache[(((int64_t)sq * KV + kh) * max_len + p) * hd + j] =
        __float2bfloat16_rn(row[(H + KV) * hd + kh * hd + j]);
  }
}

// One CTA per (token, kv head); its G = H/KV query heads attend over keys
// 0..pos of the token's sequence.  Warps split the keys (online softmax per
// warp, merged through smem).  head_dim <= 128 (lanes hold hd/32 dims).
constexpr int ATT_WARPS = 8;
constexpr int MAX_G = 8;
__global__ void __launch_bounds__(ATT_WARPS * 32) attention_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __nv_bfloat16* __restrict__ v_cache, const int32_t* __restrict__ pos, const int32_t* __restrict__ seq,
    int H, int KV, int hd, int64_t max_len, float scale, __nv_bfloat16* __restrict__ out) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  const int kh = blockIdx.y;
  const int G = H / KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = pos[t] + 1;
  const int per = hd / 32;  // dims per lane (<= 4)
  const __nv_bfloat16* kb = k_cache + ((int64_t)seq[t] * KV + kh) * max_len * hd;
  const __nv_bfloat16* vb = v_cache + ((int64_t)seq[t] * KV + kh) * max_len * hd;
  float qr[MAX_G][4], acc[MAX_G][4], m[MAX_G], l[MAX_G];
  for (int g = 0; g < G; ++g) {
    const __nv_bfloat16* qh = q + ((int64_t)t * H + kh * G + g) * hd;
    for (int i = 0; i < per; ++i) {
      qr[g][i] = __bfloat162float(qh[lane * per + i]) * scale;
      acc[g][i] = 0.f;
    }
    m[g] = -INFINITY;
    l[g] = 0.f;
  }
  for (int j = warp; j < L; j += ATT_WARPS) {
    float kv[4], vv[4];
    for (int i = 0; i < per; ++i) {
      kv[i] = __bfloat162float(kb[(int64_t)j * hd + lane * per + i]);
      vv[i] = __bfloat162float(vb[(int64_t)j * hd + lane * per + i]);
    }
    for (int g = 0; g < G; ++g) {
      float s = 0.f;
      for (int i = 0; i < per; ++i) s += qr[g][i] * kv[i];
      s = warp_sum(s);
      const float mn = fmaxf(m[g], s);
      const float corr = __expf(m[g] - mn);
      const float pexp = __expf(s - mn);
      l[g] = l[g] * corr + pexp;
      for (int i = 0; i < per; ++i) acc[g][i] = acc[g][i] * corr + pexp * vv[i];
      m[g] = mn;
    }
  }
  __shared__ float sm_m[ATT_WARPS][MAX_G], sm_l[ATT_WARPS][MAX_G];
  __shared__ float sm_acc[ATT_WARPS][MAX_G][128];
  for (int g = 0; g < G; ++g) {
    if (lane == 0) {
      sm_m[warp][g] = m[g];
      sm_l[warp][g] = l[g];
    }
    for (int i = 0; i < per; ++i) sm_acc[warp][g][lane * per + i] = acc[g][i];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * hd; idx += blockDim.x) {
    const int g = idx / hd, dcol = idx % hd;
    float mx = -INFINITY;
    for (int w = 0; w < ATT_WARPS; ++w) mx = fmaxf(mx, sm_m[w][g]);
    float den = 0.f, num = 0.f;
    for (int w = 0; w < ATT_WARPS; ++w) {
      if (sm_m[w][g] == -INFINITY) continue;
      const float f = __expf(sm_m[w][g] - mx);
      den += sm_l[w][g] * f;
      num += sm_acc[w][g][dcol] * f;
    }
    out[((int64_t)t * H + kh * G + g) * hd + dcol] = __float2bfloat16_rn(num / den);
  }
}

// greedy next token: argmax over logits[t, :] (lowest index wins ties)
__global__ void argmax_kernel(const float* __restrict__ logits, int64_t V, int32_t* __restrict__ out,
                              float* __restrict__ top2 /* optional [T,2]: best, runner-up */) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  const float* row = logits + (int64_t)t * V;
  float best = -INFINITY, second = -INFINITY;
  int64_t bi = V;
  for (int64_t i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (v > best || (v == best && i < bi)) {
      second = fmaxf(second, best);
      best = v;
      bi = i;
    } else {
      second = fmaxf(second, v);
    }
  }
  __shared__ float sb[1024], s2[1024];
  __shared__ int64_t si[1024];
  sb[threadIdx.x] = best;
  s2[threadIdx.x] = second;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const int o = threadIdx.x + st;
      float b1 = sb[threadIdx.x], b2 = sb[o];
      int64_t i1 = si[threadIdx.x], i2 = si[o];
      float sec = fmaxf(s2[threadIdx.x], s2[o]);
      if (b2 > b1 || (b2 == b1 && i2 < i1)) {
        sec = fmaxf(sec, b1);
        b1 = b2;
        i1 = i2;
      } else {
        sec = fmaxf(sec, b2);
      }
      sb[threadIdx.x] = b1;
      si[threadIdx.x] = i1;
      s2[threadIdx.x] = sec;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[t] = (int32_t)si[0];
    if (top2) {
      top2[2 * t] = sb[0];
      top2[2 * t + 1] = s2[0];
    }
  }
}

// Stage -> stage hand-off of the hidden state: 16-byte vector stores from
// the producing GPU straight into the consumer's receive buffer over NVLink,
// then (optional) a .sys release of a flag in the consumer's memory that its
// stream waits on (cuStreamWaitValue32), so no host round trip sits between
// pipeline stages.
__global__ void handoff_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16, uint32_t* flag,
                               uint32_t value, unsigned int* done_ctas) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    lp::st16(dst + i, src[i]);
  if (flag == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    lp::fence_sys();
    const unsigned int prev = atomicAdd(done_ctas, 1u);
    if (prev + 1 == gridDim.x) {  // last CTA: every CTA's stores are fenced
      *done_ctas = 0;
      lp::fence_sys();
      lp::st_release_sys(flag, value);
    }
  }
}

}  // namespace

extern "C" {

int lp_handoff(const void* src, void* dst, int64_t bytes, uint32_t* flag, uint32_t value, uint32_t* scratch,
               void* stream) {
  LP_CHECK(src && dst && bytes > 0 && bytes % 16 == 0, "lp_handoff: bad arguments (bytes %% 16 == 0)");
  LP_CHECK(!flag || scratch, "lp_handoff: a flag needs a zeroed u32 scratch counter on the producer");
  const int64_t n16 = bytes / 16;
  int blocks = (int)((n16 + 255) / 256);
  if (blocks > 32) blocks = 32;
  handoff_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const int4*)src, (int4*)dst, n16, flag, value,
                                                           scratch);
  LP_CUDA(cudaGetLastError());
  return 0;
}


int lp_embed(const void* table, int64_t d, const int32_t* tokens, int64_t T, float* x, void* stream) {
  LP_CHECK(table && tokens && x && T > 0 && d > 0, "lp_embed: bad arguments");
  LP_CUDA(lp::launch(embed_kernel, dim3((unsigned)T), dim3(256), 0, (cudaStream_t)stream,
                     (const __nv_bfloat16*)table, d, tokens, x));
  return 0;
}

int lp_rmsnorm(const float* x, const void* w, int64_t T, int64_t d, float eps, void* y, void* stream) {
  LP_CHECK(x && w && y && T > 0 && d > 0, "lp_rmsnorm: bad arguments");
  LP_CUDA(lp::launch(rmsnorm_kernel, dim3((unsigned)T), dim3(512), 0, (cudaStream_t)stream, x,
                     (const __nv_bfloat16*)w, d, eps, (__nv_bfloat16*)y));
  return 0;
}

int lp_rope_kv(const float* qkv, int64_t T, int n_heads, int n_kv, int head_dim, const int32_t* pos,
               const int32_t* seq, float theta, void* q_out, void* k_cache, void* v_cache, int64_t max_len,
               void* stream) {
  LP_CHECK(qkv && pos && seq && q_out && k_cache && v_cache && T > 0, "lp_rope_kv: bad arguments");
  LP_CHECK(n_kv > 0 && n_heads % n_kv == 0 && head_dim % 2 == 0, "lp_rope_kv: bad head shape");
  LP_CUDA(lp::launch(rope_kv_kernel, dim3((unsigned)T), dim3(256), 0, (cudaStream_t)stream, qkv, n_heads, n_kv,
                     head_dim, pos, seq, theta, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_cache,
                     (__nv_bfloat16*)v_cache, max_len));
  return 0;
}

int lp_attention(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos, const int32_t* seq,
                 int64_t T, int n_heads, int n_kv, int head_dim, int64_t max_len, float scale, void* out,
                 void* stream) {
  LP_CHECK(q && k_cache && v_cache && pos && seq && out && T > 0, "lp_attention: bad arguments");
  LP_CHECK(n_kv > 0 && n_heads % n_kv == 0 && n_heads / n_kv <= MAX_G, "lp_attention: GQA group > %d", MAX_G);
  LP_CHECK(head_dim % 32 == 0 && head_dim <= 128, "lp_attention: head_dim must be 32..128, multiple of 32");
  dim3 grid((unsigned)T, (unsigned)n_kv);
  LP_CUDA(lp::launch(attention_kernel, grid, dim3(ATT_WARPS * 32), 0, (cudaStream_t)stream,
                     (const __nv_bfloat16*)q, (const __nv_bfloat16*)k_cache, (const __nv_bfloat16*)v_cache, pos, seq,
                     n_heads, n_kv, head_dim, max_len, scale, (__nv_bfloat16*)out));
  return 0;
}

int lp_argmax(const float* logits, int64_t T, int64_t V, int32_t* out, float* top2, void* stream) {
  LP_CHECK(logits && out && T > 0 && V > 0, "lp_argmax: bad arguments");
  LP_CUDA(lp::launch(argmax_kernel, dim3((unsigned)T), dim3(1024), 0, (cudaStream_t)stream, logits, V, out, top2));
  return 0;
}

}  // extern "C"
