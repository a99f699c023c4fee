// Llama decoder-layer kernels around the tensor-core GEMMs (lp_gemm.cu):
// embedding gather, RMSNorm, RoPE + KV-cache append, ragged causal attention
// (prefill and decode share one kernel: every token attends to positions
// 0..pos of its own sequence), and greedy argmax.
//
// Numerics: weights bf16, residual stream fp32, GEMM inputs bf16, fp32
// accumulation everywhere; the V cache and the softmax probabilities of P V
// are fp16 (oracle/llama.py bf16=True rounds at the same points).
#include "lp_common.cuh"
#include <cooperative_groups.h>
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

// y[t, :] = bf16(x * rsqrt(mean(x^2) + eps) * w); d % 4 == 0.  16-byte
// loads, the row kept in registers between the reduction and the scaling
// (one HBM read of x instead of two: prefill rows are 16-32 KB).
constexpr int RMS_THREADS = 512;
constexpr int RMS_CACHE = 4;     // float4 per thread held in registers (d <= 8192)
//
// zero (optional): also clear row t of an fp32 [T, zero_cols] buffer — the
// accumulator the next (split-K, red.add) GEMM adds into — so no separate
// fill kernel sits between the norm and the GEMM (a non-PDL fill would also
// break the programmatic-launch chain inside captured graphs).
__global__ void __launch_bounds__(RMS_THREADS) rmsnorm_kernel(const float* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ w, int64_t d,
                                                              float eps, __nv_bfloat16* __restrict__ y,
                                                              float* __restrict__ zero, int64_t zero_cols) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  if (zero) {
    float* zr = zero + (int64_t)t * zero_cols;
    if ((zero_cols & 3) == 0 && (((uintptr_t)zr) & 15) == 0) {
      for (int64_t i = threadIdx.x; i < zero_cols / 4; i += RMS_THREADS)
        reinterpret_cast<float4*>(zr)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int64_t i = threadIdx.x; i < zero_cols; i += RMS_THREADS) zr[i] = 0.f;
    }
  }
  const int n4 = (int)(d / 4);
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)t * d);
  const uint2* wr = reinterpret_cast<const uint2*>(w);
  uint2* yr = reinterpret_cast<uint2*>(y + (int64_t)t * d);
  float4 c[RMS_CACHE];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < RMS_CACHE; ++k) {
    const int i = threadIdx.x + k * RMS_THREADS;
    c[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += c[k].x * c[k].x + c[k].y * c[k].y + c[k].z * c[k].z + c[k].w * c[k].w;
  }
  for (int i = threadIdx.x + RMS_CACHE * RMS_THREADS; i < n4; i += RMS_THREADS) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float part[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (RMS_THREADS >> 5) ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[0] = v;
  }
  __syncthreads();
  const float r = rsqrtf(part[0] / (float)d + eps);
  auto emit = [&](int i, const float4& v) {
    const uint2 wv = wr[i];
    const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.x));
    const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.y));
    __nv_bfloat162 o[2] = {__floats2bfloat162_rn(v.x * r * w01.x, v.y * r * w01.y),
                           __floats2bfloat162_rn(v.z * r * w23.x, v.w * r * w23.y)};
    yr[i] = *reinterpret_cast<const uint2*>(o);
  };
#pragma unroll
  for (int k = 0; k < RMS_CACHE; ++k) {
    const int i = threadIdx.x + k * RMS_THREADS;
    if (i < n4) emit(i, c[k]);
  }
  for (int i = threadIdx.x + RMS_CACHE * RMS_THREADS; i < n4; i += RMS_THREADS) emit(i, xr[i]);
}

// qkv: [T, (H + 2*KV) * hd] fp32.  HF Llama rotate_half RoPE: element j < hd/2
// pairs with j + hd/2 at angle pos * theta^(-2j/hd).
// q_out [T, H*hd] bf16; k appended to k_cache[seq][kv][pos][hd] bf16, v to
// v_cache (same layout) fp16 -- the P V product runs in fp16.
//
// One CTA per (token, group of 8 heads): the angle table (cos, sin of
// pos * theta^(-2j/hd), j < hd/2) depends only on the token's position, so it
// is computed once into smem and shared by the group's rotated heads (a CTA
// per (token, head) recomputed it per head: 87 us per 70B prefill layer at
// T = 1024); one more CTA per token copies the v heads.
constexpr int ROPE_THREADS = 256;
constexpr int ROPE_MAX_HALF = 128;
constexpr int ROPE_HEADS = 8;      // rotated heads per CTA
__global__ void __launch_bounds__(ROPE_THREADS) rope_kv_kernel(
    const float* __restrict__ qkv, int H, int KV, int hd, const int32_t* __restrict__ pos,
    const int32_t* __restrict__ seq, float theta, __nv_bfloat16* __restrict__ q_out,
    __nv_bfloat16* __restrict__ k_cache, __half* __restrict__ v_cache, int64_t max_len) {
  lp::pdl_wait();
  lp::pdl_trigger();
  const int t = blockIdx.x;
  const int p = pos[t];
  const int sq = seq[t];
  const int half = hd / 2;
  __shared__ float s_cos[ROPE_MAX_HALF], s_sin[ROPE_MAX_HALF];
  const float l2t = log2f(theta);
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    const float inv = exp2f(-2.0f * (float)j / (float)hd * l2t);
    float sn, cs;
    sincosf((float)p * inv, &sn, &cs);
    s_cos[j] = cs;
    s_sin[j] = sn;
  }
  __syncthreads();
  // grid.y splits the token's heads over CTAs (decode has only a handful of
  // tokens): y < groups rotates ROPE_HEADS q/k heads, y == groups copies v
  const float* row = qkv + (int64_t)t * (H + 2 * KV) * hd;
  const int groups = (H + KV + ROPE_HEADS - 1) / ROPE_HEADS;
  if ((int)blockIdx.y < groups) {
    const int h0 = blockIdx.y * ROPE_HEADS;
    const int h1 = min(H + KV, h0 + ROPE_HEADS);
    for (int i = threadIdx.x; i < (h1 - h0) * half; i += blockDim.x) {
      const int head = h0 + i / half, j = i % half;
      const float* src = row + (int64_t)head * hd;
      __nv_bfloat16* dst = head < H ? q_out + ((int64_t)t * H + head) * hd
                                    : k_cache + (((int64_t)sq * KV + (head - H)) * max_len + p) * hd;
      const float a = src[j], b = src[j + half], cs = s_cos[j], sn = s_sin[j];
      dst[j] = __float2bfloat16_rn(a * cs - b * sn);
      dst[j + half] = __float2bfloat16_rn(b * cs + a * sn);
    }
  } else {
    const float* vsrc = row + (int64_t)(H + KV) * hd;
    for (int i = threadIdx.x; i < KV * hd; i += blockDim.x) {
      const int kh = i / hd, j = i % hd;
      v_cache[(((int64_t)sq * KV + kh) * max_len + p) * hd + j] = __float2half_rn(vsrc[i]);
    }
  }
}

// One CTA per (token, kv head); its G = H/KV query heads attend over keys
// 0..pos of the token's sequence.  Lane-per-key: each warp takes chunks of 32
// keys, every lane computes its key's G dot products from 16-byte K loads
// against q in smem (no per-key shuffles), one max/sum reduction per chunk,
// then P.V with the chunk's probabilities broadcast lane by lane while each
// lane accumulates its HD/32 output dims.  Warps merge through smem.
// HD is a template parameter so both phases issue their loads in batches
// (all HD/8 K vectors of a key, then V rows 8 keys at a time) before using
// them: a decode CTA is latency bound, and a load -> FMA chain per key was
// 45 us per layer at B = 16 (profiles/decode_step_launches_r01.csv).
constexpr int ATT_WARPS = 4;
constexpr int MAX_G = 8;
constexpr int PV_BATCH = 8;

template <int PER>
__device__ __forceinline__ void load_v(const __half* p, float (&f)[4]) {
  if constexpr (PER == 4) {
    const uint2 raw = *reinterpret_cast<const uint2*>(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
    f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
  } else if constexpr (PER == 2) {
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(p));
    f[0] = a.x; f[1] = a.y;
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) f[i] = __half2float(p[i]);
  }
}

// Online-softmax attention of one query row (G heads, q pre-scaled in sq)
// over keys c_begin, c_begin + c_step, ... (32-key chunks, lane per key) of
// K/V rows at kb / vb with the given row strides (global cache or smem copy).
template <int HD>
__device__ __forceinline__ void att_chunks(const float (&sq)[MAX_G][HD], const __nv_bfloat16* kb, int kstride,
                                           const __half* vb, int vstride, int G, int L, int c_begin,
                                           int c_step, int lane, float (&m)[MAX_G], float (&l)[MAX_G],
                                           float (&acc)[MAX_G][HD / 32]) {
  constexpr int PER = HD / 32;
  for (int c0 = c_begin; c0 < L; c0 += c_step) {
    const int j = c0 + lane;
    const bool live = j < L;
    float s[MAX_G];
#pragma unroll
    for (int g = 0; g < MAX_G; ++g) s[g] = 0.f;
    if (live) {
      const int4* kr = reinterpret_cast<const int4*>(kb + (int64_t)j * kstride);
      int4 raw[HD / 8];
#pragma unroll
      for (int v8 = 0; v8 < HD / 8; ++v8) raw[v8] = kr[v8];
#pragma unroll
      for (int v8 = 0; v8 < HD / 8; ++v8) {
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw[v8]);
        float kf[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          kf[2 * e] = f.x;
          kf[2 * e + 1] = f.y;
        }
#pragma unroll
        for (int g = 0; g < MAX_G; ++g) {
          if (g < G) {
#pragma unroll
            for (int e = 0; e < 8; ++e) s[g] += sq[g][v8 * 8 + e] * kf[e];
          }
        }
      }
    }
    float p[MAX_G];
#pragma unroll
    for (int g = 0; g < MAX_G; ++g) {
      p[g] = 0.f;
      if (g >= G) continue;
      const float cm = warp_max(live ? s[g] : -INFINITY);
      const float mn = fmaxf(m[g], cm);
      const float corr = __expf(m[g] - mn);
      p[g] = live ? __expf(s[g] - mn) : 0.f;
      l[g] = l[g] * corr + warp_sum(p[g]);
#pragma unroll
      for (int i = 0; i < PER; ++i) acc[g][i] *= corr;
      m[g] = mn;
    }
    const int nk = min(32, L - c0);
    for (int j0 = 0; j0 < nk; j0 += PV_BATCH) {
      float vf[PV_BATCH][4];
#pragma unroll
      for (int b = 0; b < PV_BATCH; ++b) {
        const int key = c0 + min(j0 + b, nk - 1);     // clamped: dead keys have p = 0
        load_v<PER>(vb + (int64_t)key * vstride + lane * PER, vf[b]);
      }
#pragma unroll
      for (int b = 0; b < PV_BATCH; ++b) {
#pragma unroll
        for (int g = 0; g < MAX_G; ++g) {
          if (g >= G) break;
          const float pj = __shfl_sync(0xffffffffu, p[g], (j0 + b) & 31);
          const float w = (j0 + b < nk) ? pj : 0.f;
#pragma unroll
          for (int i = 0; i < PER; ++i) acc[g][i] += w * vf[b][i];
        }
      }
    }
  }
}

//
// ROW_PER_WARP (many rows, e.g. prefill): each warp owns one row and walks all
// of its key chunks — no idle warps on short contexts, no cross-warp merge;
// otherwise (decode: few rows, long contexts) the CTA's warps split one row's
// keys and merge through smem.
template <int HD, bool ROW_PER_WARP>
__global__ void __launch_bounds__(ATT_WARPS * 32) attention_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __half* __restrict__ v_cache, const int32_t* __restrict__ pos, const int32_t* __restrict__ seq,
    int T, int H, int KV, int64_t max_len, float scale, __nv_bfloat16* __restrict__ out) {
  constexpr int PER = HD / 32;   // output dims per lane
  lp::pdl_wait();
  lp::pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = ROW_PER_WARP ? blockIdx.x * ATT_WARPS + warp : blockIdx.x;
  if (ROW_PER_WARP && t >= T) return;
  const int kh = blockIdx.y;
  const int G = H / KV;
  const int L = pos[t] + 1;
  const __nv_bfloat16* kb = k_cache + ((int64_t)seq[t] * KV + kh) * max_len * HD;
  const __half* vb = v_cache + ((int64_t)seq[t] * KV + kh) * max_len * HD;
  __shared__ float sq_all[ROW_PER_WARP ? ATT_WARPS : 1][MAX_G][HD];
  float (&sq)[MAX_G][HD] = sq_all[ROW_PER_WARP ? warp : 0];
  if (ROW_PER_WARP) {
    for (int i = lane; i < G * HD; i += 32) {
      const int g = i / HD, dd = i % HD;
      sq[g][dd] = __bfloat162float(q[((int64_t)t * H + kh * G + g) * HD + dd]) * scale;
    }
    __syncwarp();
  } else {
    for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
      const int g = i / HD, dd = i % HD;
      sq[g][dd] = __bfloat162float(q[((int64_t)t * H + kh * G + g) * HD + dd]) * scale;
    }
    __syncthreads();
  }
  float m[MAX_G], l[MAX_G], acc[MAX_G][PER];
#pragma unroll
  for (int g = 0; g < MAX_G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) acc[g][i] = 0.f;
  }
  att_chunks<HD>(sq, kb, HD, vb, HD, G, L, ROW_PER_WARP ? 0 : warp * 32, ROW_PER_WARP ? 32 : ATT_WARPS * 32, lane,
                 m, l, acc);
  if constexpr (ROW_PER_WARP) {
#pragma unroll
    for (int g = 0; g < MAX_G; ++g) {
      if (g >= G) break;
      const float inv = 1.0f / l[g];
#pragma unroll
      for (int i = 0; i < PER; ++i)
        out[((int64_t)t * H + kh * G + g) * HD + lane * PER + i] = __float2bfloat16_rn(acc[g][i] * inv);
    }
    return;
  }
  __shared__ float sm_m[ATT_WARPS][MAX_G], sm_l[ATT_WARPS][MAX_G];
  __shared__ float sm_acc[ATT_WARPS][MAX_G][HD];
#pragma unroll
  for (int g = 0; g < MAX_G; ++g) {
    if (g >= G) break;
    if (lane == 0) {
      sm_m[warp][g] = m[g];
      sm_l[warp][g] = l[g];
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) sm_acc[warp][g][lane * PER + i] = acc[g][i];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
    const int g = idx / HD, dcol = idx % HD;
    float mx = -INFINITY;
    for (int w = 0; w < ATT_WARPS; ++w) mx = fmaxf(mx, sm_m[w][g]);
    float den = 0.f, num = 0.f;
    for (int w = 0; w < ATT_WARPS; ++w) {
      if (sm_m[w][g] == -INFINITY) continue;
      const float f = __expf(sm_m[w][g] - mx);
      den += sm_l[w][g] * f;
      num += sm_acc[w][g][dcol] * f;
    }
    out[((int64_t)t * H + kh * G + g) * HD + dcol] = __float2bfloat16_rn(num / den);
  }
}

// Prefill on the tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate):
// FlashAttention-2 style.  A CTA takes 16 consecutive rows and one kv head;
// each of its 4 warps one query head of the GQA group (grid z covers groups
// > 4).  When the 16 rows share one sequence (a request's prompt tokens are
// consecutive rows), that sequence's keys are streamed through smem in
// 64-key chunks: S = Q K^T (Q fragments in registers, K fragments straight
// from padded smem rows), per-row causal mask pos[row], online softmax in
// registers, P reused as the A operand of P V (V fragments via
// ldmatrix.trans).  Tiles mixing sequences fall back to the CUDA-core row
// path.  Replaces a lane-per-key CUDA-core loop that ran at ~9 % of FMA
// peak (8B prefill, 2048 rows: 340 us per layer).
constexpr int MMA_ROWS = 16;
constexpr int MMA_KEYS = 64;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// P V runs in fp16 (P in [0, 1] keeps 3 more mantissa bits than bf16; V is
// stored fp16 in the cache, exact for its activations' range)
__device__ __forceinline__ void mma_f16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  const __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// NST = 2: K/V chunk j + 1 is fetched with cp.async into a second stage
// (dynamic smem) while chunk j is on the tensor cores.
template <int HD, int NST>
__global__ void __launch_bounds__(ATT_WARPS * 32) attention_mma_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __half* __restrict__ v_cache, const int32_t* __restrict__ pos, const int32_t* __restrict__ seq,
    int T, int H, int KV, int64_t max_len, float scale, __nv_bfloat16* __restrict__ out) {
  constexpr int KS = HD + 8;                 // padded smem row (elements): conflict-free fragments
  constexpr int KSTEPS = HD / 16;            // QK^T k-steps
  constexpr int DT = HD / 8;                 // PV n-tiles
  __shared__ __align__(16) __nv_bfloat16 Ks[MMA_KEYS][KS];
  __shared__ __align__(16) __nv_bfloat16 Vs[MMA_KEYS][KS];
  extern __shared__ __align__(16) uint8_t att_dyn[];  // NST = 2: stage 1 (K then V)
  __shared__ int s_same, s_len, s_pos[MMA_ROWS];
  lp::pdl_wait();
  lp::pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh = blockIdx.y;
  const int G = H / KV;
  const int t0 = blockIdx.x * MMA_ROWS;
  const int t1 = min(T, t0 + MMA_ROWS);
  if (threadIdx.x == 0) {
    const int s0 = seq[t0];
    int same = 1, len = 0;
    for (int t = t0; t < t1; ++t) {
      same &= seq[t] == s0;
      len = max(len, pos[t] + 1);
    }
    s_same = same;
    s_len = len;
  }
  if (threadIdx.x < MMA_ROWS) s_pos[threadIdx.x] = (t0 + (int)threadIdx.x < T) ? pos[t0 + threadIdx.x] : -1;
  __syncthreads();
  if (!s_same) {
    // mixed sequences: CUDA-core rows (all G heads per row), z == 0 CTAs only
    if (blockIdx.z != 0) return;
    constexpr int PER = HD / 32;
    static_assert(sizeof(float) * ATT_WARPS * MAX_G * HD <= sizeof(__nv_bfloat16) * MMA_KEYS * KS,
                  "fallback q staging must fit the K tile");
    float (&sq)[MAX_G][HD] = reinterpret_cast<float (*)[MAX_G][HD]>(&Ks[0][0])[warp];
    for (int t = t0 + warp; t < t1; t += ATT_WARPS) {
      for (int i = lane; i < G * HD; i += 32) {
        const int g = i / HD, dd = i % HD;
        sq[g][dd] = __bfloat162float(q[((int64_t)t * H + kh * G + g) * HD + dd]) * scale;
      }
      __syncwarp();
      float m[MAX_G], l[MAX_G], acc[MAX_G][PER];
#pragma unroll
      for (int g = 0; g < MAX_G; ++g) {
        m[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[g][i] = 0.f;
      }
      const __nv_bfloat16* kb = k_cache + ((int64_t)seq[t] * KV + kh) * max_len * HD;
      const __half* vb = v_cache + ((int64_t)seq[t] * KV + kh) * max_len * HD;
      att_chunks<HD>(sq, kb, HD, vb, HD, G, pos[t] + 1, 0, 32, lane, m, l, acc);
#pragma unroll
      for (int g = 0; g < MAX_G; ++g) {
        if (g >= G) break;
        const float inv = 1.0f / l[g];
#pragma unroll
        for (int i = 0; i < PER; ++i)
          out[((int64_t)t * H + kh * G + g) * HD + lane * PER + i] = __float2bfloat16_rn(acc[g][i] * inv);
      }
      __syncwarp();
    }
    return;
  }
  const int g = blockIdx.z * ATT_WARPS + warp;    // this warp's query head within the group
  const bool active = g < G;
  const int head = kh * G + (active ? g : 0);
  const int r0 = lane >> 2, cq = (lane & 3) * 2;  // fragment row / column pair
  // Q fragments (A operand, 16 rows x HD), rows past T are zero
  uint32_t qa[KSTEPS][4];
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {              // h: row r0 / r0 + 8
      const int t = t0 + r0 + 8 * h;
      const __nv_bfloat16* qr = q + ((int64_t)t * H + head) * HD + ks * 16 + cq;
      qa[ks][h] = t < T ? *reinterpret_cast<const uint32_t*>(qr) : 0u;
      qa[ks][2 + h] = t < T ? *reinterpret_cast<const uint32_t*>(qr + 8) : 0u;
    }
  }
  const int prow[2] = {s_pos[r0], s_pos[r0 + 8]};
  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const float sl2 = scale * 1.4426950408889634f;  // softmax in base 2
  const int len = s_len;
  const __nv_bfloat16* kg = k_cache + ((int64_t)seq[t0] * KV + kh) * max_len * HD;
  const __half* vg = v_cache + ((int64_t)seq[t0] * KV + kh) * max_len * HD;
  constexpr int V8 = HD / 8;
  using Row = __nv_bfloat16[KS];
  Row* const dynK = reinterpret_cast<Row*>(att_dyn);
  Row* const dynV = dynK + MMA_KEYS;
  auto fetch = [&](int c, int st) {   // zero-filled past len
    Row* const dK = st ? dynK : Ks;
    Row* const dV = st ? dynV : Vs;
    for (int i = threadIdx.x; i < MMA_KEYS * V8; i += blockDim.x) {
      const int r = i / V8, cc = i % V8;
      const bool in = c + r < len;
      const int64_t src = (in ? (int64_t)(c + r) : 0) * HD + cc * 8;
      const uint32_t nb = in ? 16u : 0u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(lp::smem_u32(&dK[r][cc * 8])),
                   "l"(kg + src), "r"(nb) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(lp::smem_u32(&dV[r][cc * 8])),
                   "l"(vg + src), "r"(nb) : "memory");
    }
  };
  if constexpr (NST == 2) {
    fetch(0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int jc = 0;
  for (int c0 = 0; c0 < len; c0 += MMA_KEYS, ++jc) {
    const int nk = min(MMA_KEYS, len - c0);
    Row* const Kc = (NST == 2 && (jc & 1)) ? dynK : Ks;
    Row* const Vc = (NST == 2 && (jc & 1)) ? dynV : Vs;
    if constexpr (NST == 2) {
      if (c0 + MMA_KEYS < len) fetch(c0 + MMA_KEYS, (jc + 1) & 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      for (int i = threadIdx.x; i < MMA_KEYS * V8; i += blockDim.x) {
        const int r = i / V8, c = i % V8;
        int4 kv = make_int4(0, 0, 0, 0), vv = kv;
        if (r < nk) {
          kv = reinterpret_cast<const int4*>(kg + (int64_t)(c0 + r) * HD)[c];
          vv = reinterpret_cast<const int4*>(vg + (int64_t)(c0 + r) * HD)[c];
        }
        reinterpret_cast<int4*>(&Kc[r][0])[c] = kv;
        reinterpret_cast<int4*>(&Vc[r][0])[c] = vv;
      }
    }
    __syncthreads();
    if (active) {
      // S = Q K^T over this chunk: 8 n-tiles of 8 keys
      float sc[MMA_KEYS / 8][4];
#pragma unroll
      for (int nt = 0; nt < MMA_KEYS / 8; ++nt) {
        sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
        const __nv_bfloat16* kr = &Kc[nt * 8 + r0][cq];
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + ks * 16);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + ks * 16 + 8);
          mma_bf16_16816(sc[nt], qa[ks], b0, b1);
        }
      }
      // causal mask + online softmax (each thread: rows r0, r0 + 8; a quad shares a row)
      float mnew[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float mx = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < MMA_KEYS / 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int key = c0 + nt * 8 + cq + e;
            float v = sc[nt][2 * h + e] * sl2;
            if (key > prow[h]) v = -INFINITY;
            sc[nt][2 * h + e] = v;
            mx = fmaxf(mx, v);
          }
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mnew[h] = fmaxf(mrow[h], mx);
        const float corr = mnew[h] == -INFINITY ? 1.f : exp2f(mrow[h] - mnew[h]);
        lrow[h] *= corr;
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          o[dt][2 * h] *= corr;
          o[dt][2 * h + 1] *= corr;
        }
        mrow[h] = mnew[h];
      }
      uint32_t pa[MMA_KEYS / 16][4];
#pragma unroll
      for (int nt = 0; nt < MMA_KEYS / 8; ++nt) {
        float pv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int h = i >> 1;
          pv[i] = mnew[h] == -INFINITY ? 0.f : exp2f(sc[nt][i] - mnew[h]);
          lrow[h] += pv[i];
        }
        // C fragment of S -> A fragment of P (keys 16 kk .. 16 kk + 15)
        const int kk = nt >> 1, hi = nt & 1;
        pa[kk][2 * hi] = pack_f16(pv[0], pv[1]);
        pa[kk][2 * hi + 1] = pack_f16(pv[2], pv[3]);
      }
      // O += P V: V fragments (k = keys, n = dims) via ldmatrix.trans
#pragma unroll
      for (int kk = 0; kk < MMA_KEYS / 16; ++kk) {
        if (c0 + kk * 16 >= len) break;
        const uint32_t row_addr = lp::smem_u32(&Vc[kk * 16 + (lane & 15)][0]);
#pragma unroll
        for (int dt = 0; dt < DT; ++dt) {
          uint32_t b0, b1;
          asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                       : "=r"(b0), "=r"(b1)
                       : "r"(row_addr + dt * 16));
          mma_f16_16816(o[dt], pa[kk], b0, b1);
        }
      }
    }
    __syncthreads();
  }
  if (!active) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float lsum = lrow[h];
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    const int t = t0 + r0 + 8 * h;
    if (t >= T) continue;
    const float inv = 1.0f / lsum;
    __nv_bfloat16* orow = out + ((int64_t)t * H + head) * HD + cq;
#pragma unroll
    for (int dt = 0; dt < DT; ++dt)
      *reinterpret_cast<__nv_bfloat162*>(orow + dt * 8) =
          __floats2bfloat162_rn(o[dt][2 * h] * inv, o[dt][2 * h + 1] * inv);
  }
}

// Decode on the tensor cores: one CTA per (token, kv head).  The G query
// heads of the GQA group share the token's K/V, so they form the rows of an
// m16n8k16 tile (rows >= G are zero); each warp takes 32-key chunks
// (warp w: keys 32w, 32w + 128, ...), stages them in its own padded smem
// slice, runs S = QKᵀ, online softmax and PV on the tensor cores, and the
// four warps merge (m, l, O) through smem at the end.  The CUDA-core
// lane-per-key loop took 28.7 us per 8B layer at B = 16, ctx 160
// (tools/attn_perf.py): a chain of dependent loads per 32 keys.
// Long contexts with few rows (flash-decoding): gridDim.z CTAs of one
// thread-block cluster split a row's keys (CTA z takes the chunks of warps
// z * ATT_WARPS ..), and each CTA merges a slice of the output from every
// CTA's (m, l, O) through distributed shared memory -- no workspace, no
// second kernel.
constexpr int DEC_KEYS = 32;

// NST = 2 (the split path): each warp double-buffers its chunks, cp.async
// fetches chunk j + 1 into the other smem stage while the MMAs run on chunk j.
template <int HD, int NST>
__global__ void __launch_bounds__(ATT_WARPS * 32) attention_mma_decode_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __half* __restrict__ v_cache, const int32_t* __restrict__ pos, const int32_t* __restrict__ seq,
    int H, int KV, int64_t max_len, float scale, __nv_bfloat16* __restrict__ out) {
  constexpr int KS = HD + 8;
  constexpr int KSTEPS = HD / 16;
  constexpr int DT = HD / 8;
  extern __shared__ __align__(16) uint8_t dec_smem[];
  __shared__ float sm_m[ATT_WARPS][16], sm_l[ATT_WARPS][16];
  lp::pdl_wait();
  lp::pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x, kh = blockIdx.y;
  const int S = gridDim.z, split = blockIdx.z;       // key split over the cluster
  const int G = H / KV;
  const int L = pos[t] + 1;
  const int r0 = lane >> 2, cq = (lane & 3) * 2;
  const __nv_bfloat16* kg = k_cache + ((int64_t)seq[t] * KV + kh) * max_len * HD;
  const __half* vg = v_cache + ((int64_t)seq[t] * KV + kh) * max_len * HD;
  __nv_bfloat16 (*Kbase)[KS] = reinterpret_cast<__nv_bfloat16 (*)[KS]>(dec_smem) + warp * NST * 2 * DEC_KEYS;
  const int cstep = S * ATT_WARPS * DEC_KEYS;
  const int cstart = (split * ATT_WARPS + warp) * DEC_KEYS;
  // chunk c -> stage st, coalesced: a warp instruction covers 512 contiguous
  // bytes (HD = 128: two key rows), rows past the context are zero-filled
  auto fetch = [&](int c, int st) {
    constexpr int R = HD / 8;                          // 16-byte units per key row
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int u = i * 32 + lane, row = u / R, col = u % R;
      const bool in = c + row < L;
      const int64_t src = (in ? (int64_t)(c + row) : 0) * HD + col * 8;
      const uint32_t nb = in ? 16u : 0u;
      const uint32_t kd = lp::smem_u32(&Kbase[st * 2 * DEC_KEYS + row][col * 8]);
      const uint32_t vd = lp::smem_u32(&Kbase[st * 2 * DEC_KEYS + DEC_KEYS + row][col * 8]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(kd), "l"(kg + src), "r"(nb) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(vd), "l"(vg + src), "r"(nb) : "memory");
    }
  };
  if constexpr (NST == 2) {
    if (cstart < L) fetch(cstart, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  uint32_t qa[KSTEPS][4];
#pragma unroll
  for (int ks = 0; ks < KSTEPS; ++ks) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = r0 + 8 * h;
      const __nv_bfloat16* qr = q + ((int64_t)t * H + kh * G + (row < G ? row : 0)) * HD + ks * 16 + cq;
      qa[ks][h] = row < G ? *reinterpret_cast<const uint32_t*>(qr) : 0u;
      qa[ks][2 + h] = row < G ? *reinterpret_cast<const uint32_t*>(qr + 8) : 0u;
    }
  }
  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const float sl2 = scale * 1.4426950408889634f;
  int jc = 0;
  for (int c0 = cstart; c0 < L; c0 += cstep, ++jc) {
    const int nk = min(DEC_KEYS, L - c0);
    __nv_bfloat16 (*Kw)[KS] = Kbase + (NST == 2 ? (jc & 1) : 0) * 2 * DEC_KEYS;
    __nv_bfloat16 (*Vw)[KS] = Kw + DEC_KEYS;
    if constexpr (NST == 2) {
      if (c0 + cstep < L) fetch(c0 + cstep, (jc + 1) & 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");   // chunk jc has landed
    } else {   // coalesced register staging (zero past the context), same unit map as fetch()
      constexpr int R = HD / 8;
      int4 kv[R], vv[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int u = i * 32 + lane, row = u / R, col = u % R;
        const int64_t src = (int64_t)(c0 + row) * HD + col * 8;
        kv[i] = row < nk ? *reinterpret_cast<const int4*>(kg + src) : make_int4(0, 0, 0, 0);
        vv[i] = row < nk ? *reinterpret_cast<const int4*>(vg + src) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int u = i * 32 + lane, row = u / R, col = u % R;
        *reinterpret_cast<int4*>(&Kw[row][col * 8]) = kv[i];
        *reinterpret_cast<int4*>(&Vw[row][col * 8]) = vv[i];
      }
    }
    __syncwarp();
    float sc[DEC_KEYS / 8][4];
#pragma unroll
    for (int nt = 0; nt < DEC_KEYS / 8; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
      const __nv_bfloat16* kr = &Kw[nt * 8 + r0][cq];
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + ks * 16);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + ks * 16 + 8);
        mma_bf16_16816(sc[nt], qa[ks], b0, b1);
      }
    }
    float mnew[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < DEC_KEYS / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = c0 + nt * 8 + cq + e;
          float v = sc[nt][2 * h + e] * sl2;
          if (key >= L) v = -INFINITY;
          sc[nt][2 * h + e] = v;
          mx = fmaxf(mx, v);
        }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mnew[h] = fmaxf(mrow[h], mx);
      const float corr = mnew[h] == -INFINITY ? 1.f : exp2f(mrow[h] - mnew[h]);
      lrow[h] *= corr;
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        o[dt][2 * h] *= corr;
        o[dt][2 * h + 1] *= corr;
      }
      mrow[h] = mnew[h];
    }
    uint32_t pa[DEC_KEYS / 16][4];
#pragma unroll
    for (int nt = 0; nt < DEC_KEYS / 8; ++nt) {
      float pv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int h = i >> 1;
        pv[i] = mnew[h] == -INFINITY ? 0.f : exp2f(sc[nt][i] - mnew[h]);
        lrow[h] += pv[i];
      }
      const int kk = nt >> 1, hi = nt & 1;
      pa[kk][2 * hi] = pack_f16(pv[0], pv[1]);
      pa[kk][2 * hi + 1] = pack_f16(pv[2], pv[3]);
    }
#pragma unroll
    for (int kk = 0; kk < DEC_KEYS / 16; ++kk) {
      if (kk * 16 >= nk) break;
      const uint32_t row_addr = lp::smem_u32(&Vw[kk * 16 + (lane & 15)][0]);
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        uint32_t b0, b1;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                     : "=r"(b0), "=r"(b1)
                     : "r"(row_addr + dt * 16));
        mma_f16_16816(o[dt], pa[kk], b0, b1);
      }
    }
    __syncwarp();   // this warp's K/V slice is restaged for its next chunk
  }
  // merge the warps' partial softmax states (rows = heads of the group)
  __syncthreads();
  constexpr int OP = HD + 4;                          // padded row: the fragment stores hit 32 banks
  float* Om = reinterpret_cast<float*>(dec_smem);    // [ATT_WARPS][16][OP], reuses the K/V slices
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float lsum = lrow[h];
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    if (cq == 0) {
      sm_m[warp][r0 + 8 * h] = mrow[h];
      sm_l[warp][r0 + 8 * h] = lsum;
    }
    float* orow = Om + ((size_t)warp * 16 + r0 + 8 * h) * OP + cq;
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      orow[dt * 8] = o[dt][2 * h];
      orow[dt * 8 + 1] = o[dt][2 * h + 1];
    }
  }
  __syncthreads();
  if (S > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();                                   // every CTA's partial state is in its smem
    for (int idx = split * blockDim.x + threadIdx.x; idx < G * HD; idx += S * blockDim.x) {
      const int row = idx / HD, d = idx % HD;
      float mx = -INFINITY;
      for (int r = 0; r < S; ++r) {
        const float (*rm)[16] = cluster.map_shared_rank(sm_m, r);
#pragma unroll
        for (int w = 0; w < ATT_WARPS; ++w) mx = fmaxf(mx, rm[w][row]);
      }
      float den = 0.f, num = 0.f;
      for (int r = 0; r < S; ++r) {
        const float (*rm)[16] = cluster.map_shared_rank(sm_m, r);
        const float (*rl)[16] = cluster.map_shared_rank(sm_l, r);
        const float* rO = cluster.map_shared_rank(Om, r);
#pragma unroll
        for (int w = 0; w < ATT_WARPS; ++w) {
          const float mw = rm[w][row];
          if (mw == -INFINITY) continue;
          const float f = exp2f(mw - mx);
          den += rl[w][row] * f;
          num += rO[((size_t)w * 16 + row) * OP + d] * f;
        }
      }
      out[((int64_t)t * H + kh * G + row) * HD + d] = __float2bfloat16_rn(num / den);
    }
    cluster.sync();                                   // peers stay resident until their smem is read
    return;
  }
  for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
    const int row = idx / HD, d = idx % HD;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) mx = fmaxf(mx, sm_m[w][row]);
    float den = 0.f, num = 0.f;
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) {
      if (sm_m[w][row] == -INFINITY) continue;
      const float f = exp2f(sm_m[w][row] - mx);
      den += sm_l[w][row] * f;
      num += Om[((size_t)w * 16 + row) * OP + d] * f;
    }
    out[((int64_t)t * H + kh * G + row) * HD + d] = __float2bfloat16_rn(num / den);
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

template <int HD>
constexpr size_t prefill_stage_bytes() { return (size_t)2 * MMA_KEYS * (HD + 8) * 2; }

template <int HD, int NST = 1>
constexpr size_t decode_smem() { return (size_t)ATT_WARPS * NST * 2 * DEC_KEYS * (HD + 8) * 2; }

// Per device, once: the smem opt-in, and the largest key-split cluster the
// decode kernel may use -- 16 CTAs (non-portable) when the occupancy query
// says such a cluster fits, else the portable 8.  -1 on a CUDA error.
template <int HD>
int decode_max_split(int dev) {
  static int cached[64] = {};
  if (dev < 64 && cached[dev]) return cached[dev];
  if (cudaFuncSetAttribute(attention_mma_decode_kernel<HD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)decode_smem<HD>()) != cudaSuccess)
    return -1;
  auto kern = attention_mma_decode_kernel<HD, 2>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)decode_smem<HD, 2>()) !=
      cudaSuccess)
    return -1;
  int best = 8;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, 16);
    cfg.blockDim = dim3(ATT_WARPS * 32);
    cfg.dynamicSmemBytes = decode_smem<HD, 2>();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 16;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) best = 16;
  }
  cudaGetLastError();   // a refused query leaves no sticky error
  if (dev < 64) cached[dev] = best;
  return best;
}

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
  return lp_rmsnorm_zero(x, w, T, d, eps, y, nullptr, 0, stream);
}

int lp_rmsnorm_zero(const float* x, const void* w, int64_t T, int64_t d, float eps, void* y, float* zero,
                    int64_t zero_cols, void* stream) {
  LP_CHECK(x && w && y && T > 0 && d > 0, "lp_rmsnorm: bad arguments");
  LP_CHECK(d % 4 == 0, "lp_rmsnorm: d must be a multiple of 4");
  LP_CHECK(!zero || zero_cols > 0, "lp_rmsnorm_zero: zero_cols must be positive");
  LP_CUDA(lp::launch(rmsnorm_kernel, dim3((unsigned)T), dim3(RMS_THREADS), 0, (cudaStream_t)stream, x,
                     (const __nv_bfloat16*)w, d, eps, (__nv_bfloat16*)y, zero, zero_cols));
  return 0;
}

int lp_rope_kv(const float* qkv, int64_t T, int n_heads, int n_kv, int head_dim, const int32_t* pos,
               const int32_t* seq, float theta, void* q_out, void* k_cache, void* v_cache, int64_t max_len,
               void* stream) {
  LP_CHECK(qkv && pos && seq && q_out && k_cache && v_cache && T > 0, "lp_rope_kv: bad arguments");
  LP_CHECK(n_kv > 0 && n_heads % n_kv == 0 && head_dim % 2 == 0, "lp_rope_kv: bad head shape");
  LP_CHECK(head_dim / 2 <= ROPE_MAX_HALF, "lp_rope_kv: head_dim > %d", 2 * ROPE_MAX_HALF);
  const unsigned groups = (unsigned)((n_heads + n_kv + ROPE_HEADS - 1) / ROPE_HEADS);
  LP_CUDA(lp::launch(rope_kv_kernel, dim3((unsigned)T, groups + 1), dim3(ROPE_THREADS), 0, (cudaStream_t)stream, qkv, n_heads, n_kv,
                     head_dim, pos, seq, theta, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_cache,
                     (__half*)v_cache, max_len));
  return 0;
}

int lp_attention(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos, const int32_t* seq,
                 int64_t T, int n_heads, int n_kv, int head_dim, int64_t max_len, float scale, void* out,
                 void* stream) {
  LP_CHECK(q && k_cache && v_cache && pos && seq && out && T > 0, "lp_attention: bad arguments");
  LP_CHECK(n_kv > 0 && n_heads % n_kv == 0 && n_heads / n_kv <= MAX_G, "lp_attention: GQA group > %d", MAX_G);
  LP_CHECK(head_dim % 32 == 0 && head_dim <= 128, "lp_attention: head_dim must be 32..128, multiple of 32");
  const __nv_bfloat16 *qq = (const __nv_bfloat16*)q, *kk = (const __nv_bfloat16*)k_cache;
  const __half* vv = (const __half*)v_cache;
  __nv_bfloat16* oo = (__nv_bfloat16*)out;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 blk(ATT_WARPS * 32);
  // many rows (prefill): tensor-core row tiles (head_dim 64 / 128); few rows
  // (decode): a CTA per row with warps splitting the keys
  const bool many = T * n_kv >= 1024;
  if (many && (head_dim == 64 || head_dim == 128)) {
    // tcgen05 / TMEM kernel (lp_attn_tc.cu); LP_ATTN_TC=0 keeps the mma.sync one
    static const int tc_env = [] {
      const char* e = getenv("LP_ATTN_TC");
      return e ? atoi(e) : 1;
    }();
    // caches of at most ~one 128-key chunk of MHA models stay on the mma.sync
    // kernel (16 x 128-token prompts: 76 vs 78 us); longer ones take tcgen05
    // (16 x 200: 365 -> 148 us for 13B heads); GQA groups of >= 4 heads take
    // tcgen05 at any length (8B 29.3 -> 27.3 us, 70B 51.4 -> 44.7 us,
    // profiles/r02/attn_prefill_short_ab.txt, attn_prefill_mha_short.txt)
    static const int64_t tc_min_len = [] {   // LP_ATTN_TC_MIN_LEN: caches longer than this take tcgen05
      const char* e = getenv("LP_ATTN_TC_MIN_LEN");
      return e ? (int64_t)atoll(e) : (int64_t)160;
    }();
    if (tc_env && (max_len > tc_min_len || n_heads / n_kv >= 4)) {
      const int r = lp::attention_tc(q, k_cache, v_cache, pos, seq, T, n_heads, n_kv, head_dim, max_len, scale,
                                     out, s);
      if (r <= 0) return r;
    }
    const int G = n_heads / n_kv;
    const dim3 mgrid((unsigned)((T + MMA_ROWS - 1) / MMA_ROWS), (unsigned)n_kv,
                     (unsigned)((G + ATT_WARPS - 1) / ATT_WARPS));
    const int Ti = (int)T;
    static const int pdb = [] {
      const char* e = getenv("LP_PREFILL_DBUF");
      return e ? atoi(e) : 1;
    }();
    if (pdb) {
      int dev = 0;
      LP_CUDA(cudaGetDevice(&dev));
      static uint64_t pattr = 0;
      if (!(pattr >> dev & 1)) {
        LP_CUDA(cudaFuncSetAttribute(attention_mma_kernel<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)prefill_stage_bytes<64>()));
        LP_CUDA(cudaFuncSetAttribute(attention_mma_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)prefill_stage_bytes<128>()));
        pattr |= 1ull << dev;
      }
      if (head_dim == 64)
        LP_CUDA(lp::launch(attention_mma_kernel<64, 2>, mgrid, blk, prefill_stage_bytes<64>(), s, qq, kk, vv, pos,
                           seq, Ti, n_heads, n_kv, max_len, scale, oo));
      else
        LP_CUDA(lp::launch(attention_mma_kernel<128, 2>, mgrid, blk, prefill_stage_bytes<128>(), s, qq, kk, vv, pos,
                           seq, Ti, n_heads, n_kv, max_len, scale, oo));
      return 0;
    }
    if (head_dim == 64)
      LP_CUDA(lp::launch(attention_mma_kernel<64, 1>, mgrid, blk, 0, s, qq, kk, vv, pos, seq, Ti, n_heads, n_kv,
                         max_len, scale, oo));
    else
      LP_CUDA(lp::launch(attention_mma_kernel<128, 1>, mgrid, blk, 0, s, qq, kk, vv, pos, seq, Ti, n_heads, n_kv,
                         max_len, scale, oo));
    return 0;
  }
  if (!many && (head_dim == 64 || head_dim == 128) && n_heads / n_kv <= 16) {
    // key split over a cluster when the rows alone cannot fill the SMs and
    // the cache can hold long contexts (short-context serving keeps S = 1)
    static const int64_t split_ctas = [] {
      const char* e = getenv("LP_DEC_SPLIT_CTAS");   // tuning knob: grid size the split may grow to
      return e ? (int64_t)atoll(e) : (int64_t)148;
    }();
    int dev = 0;
    LP_CUDA(cudaGetDevice(&dev));
    int max_split = head_dim == 64 ? decode_max_split<64>(dev) : decode_max_split<128>(dev);
    LP_CHECK(max_split > 0, "lp_attention: decode kernel attribute setup failed");
    // 16-CTA clusters pay only for very long caches (1 x 32768 keys 136 -> 125 us;
    // 1 x 4096 keys 20.5 -> 22.6 us, the 64-way merge outweighs the keys)
    if (max_len < 16384 && max_split > 8) max_split = 8;
    unsigned S = 1;
    if (max_len >= 1024)
      while ((int)S < max_split && (int64_t)T * n_kv * S * 2 <= split_ctas &&
             (int64_t)S * 2 * ATT_WARPS * DEC_KEYS <= max_len)
        S *= 2;
    const dim3 dgrid((unsigned)T, (unsigned)n_kv, S);
    // the double-buffered variant holds one CTA per SM: only while the grid is
    // one wave, and only for long caches -- in a short-context graph step its
    // 139 KB of smem keeps the next kernel's PDL prologue off the SMs
    // (8B B = 16 step 3.09 -> 3.12 ms with it, profiles/attn_decode_coalesced_ab_r01.txt)
    static const int dbuf_env = [] {
      const char* e = getenv("LP_DEC_DBUF");
      return e ? atoi(e) : 1;
    }();
    const bool dbuf = S > 1 || (dbuf_env && (int64_t)T * n_kv <= 148 && max_len >= 1024);
#define LP_DEC(HDV)                                                                                                 \
  (S > 1 ? lp::launch_cluster_z(attention_mma_decode_kernel<HDV, 2>, dgrid, blk, S, decode_smem<HDV, 2>(), s, qq, \
                                kk, vv, pos, seq, n_heads, n_kv, max_len, scale, oo)                                 \
   : dbuf ? lp::launch(attention_mma_decode_kernel<HDV, 2>, dgrid, blk, decode_smem<HDV, 2>(), s, qq, kk, vv, pos,   \
                       seq, n_heads, n_kv, max_len, scale, oo)                                                      \
          : lp::launch(attention_mma_decode_kernel<HDV, 1>, dgrid, blk, decode_smem<HDV>(), s, qq, kk, vv, pos, seq, \
                       n_heads, n_kv, max_len, scale, oo))
    if (head_dim == 64) LP_CUDA(LP_DEC(64));
    else LP_CUDA(LP_DEC(128));
#undef LP_DEC
    return 0;
  }
  const bool rpw = many;
  const dim3 grid(rpw ? (unsigned)((T + ATT_WARPS - 1) / ATT_WARPS) : (unsigned)T, (unsigned)n_kv);
  const int Ti = (int)T;
#define LP_ATT(HDV)                                                                                              \
  (rpw ? lp::launch(attention_kernel<HDV, true>, grid, blk, 0, s, qq, kk, vv, pos, seq, Ti, n_heads, n_kv, max_len, \
                    scale, oo)                                                                                   \
       : lp::launch(attention_kernel<HDV, false>, grid, blk, 0, s, qq, kk, vv, pos, seq, Ti, n_heads, n_kv,        \
                    max_len, scale, oo))
  switch (head_dim) {
    case 32: LP_CUDA(LP_ATT(32)); break;
    case 64: LP_CUDA(LP_ATT(64)); break;
    case 96: LP_CUDA(LP_ATT(96)); break;
    default: LP_CUDA(LP_ATT(128)); break;
  }
#undef LP_ATT
  return 0;
}

int lp_argmax(const float* logits, int64_t T, int64_t V, int32_t* out, float* top2, void* stream) {
  LP_CHECK(logits && out && T > 0 && V > 0, "lp_argmax: bad arguments");
  LP_CUDA(lp::launch(argmax_kernel, dim3((unsigned)T), dim3(1024), 0, (cudaStream_t)stream, logits, V, out, top2));
  return 0;
}

}  // extern "C"
