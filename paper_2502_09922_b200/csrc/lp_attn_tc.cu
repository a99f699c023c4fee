// Causal GQA prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM +
// TMA), FlashAttention-style online softmax.
//
// Tile: one CTA owns 128 TMEM lanes = R tokens x G query heads of one kv head
// (R = 128 / G; Llama-3-8B G = 4 -> 32 tokens, 70B G = 8 -> 16, MHA -> 128),
// so the heads of a GQA group share every K/V chunk the CTA streams.  Rows
// are token-major (row = i * G + g), which is exactly what a 3-D TMA box
// {64 dims, G heads, R tokens} of q [T, H, hd] lands in shared memory.
//
// Per 128-key chunk j of the tile's sequence:
//   S_j  = Q K_j^T      tcgen05.mma kind::f16, A = Q (smem, K-major, bf16),
//                       B = K_j (smem, K-major, bf16), D = S in TMEM (fp32)
//   P_j  = exp2(S_j * scale * log2e - m_j)   softmax warps: TMEM -> regs,
//                       causal mask from pos[], fp16 P written to smem
//   O_j  = P_j V_j      tcgen05.mma kind::f16, A = P (smem, K-major, fp16),
//                       B = V_j (smem, MN-major: the fp16 V cache is [key][hd]),
//                       D = O_j in TMEM (fp32, a fresh buffer per chunk)
//   O   <- O * 2^(m_{j-1} - m_j) + O_j       softmax warps, in registers
// S and O are double-buffered in TMEM (2 x 128 + 2 x hd columns), K/V in two
// smem stages and P in two smem buffers, so the MMAs of chunk j + 1 run
// while the softmax warps work on chunk j.
//
//   warp 0   : TMA producer (Q once, then K/V chunks)
//   warp 1   : TMEM allocator + MMA issuer (one thread)
//   warps 2-5: softmax / output (thread = one TMEM lane = one row)
//
// A tile whose tokens belong to several sequences (ragged batches) walks the
// chunks of each sequence run in turn with the other rows masked.
#include "lp_common.cuh"
#include <cuda.h>

namespace {

constexpr int TC_M = 128;       // rows per tile (TMEM lanes)
constexpr int TC_KEYS = 128;    // keys per chunk
constexpr int TC_THREADS = 192;
constexpr int ATOM = TC_M * 128;   // bytes of one 128-row x 128-byte swizzle column block

template <int HD>
struct TcCfg {
  static constexpr int ATOMS = HD / 64;                 // 64-element (128 B) column blocks along hd
  static constexpr int Q_BYTES = TC_M * HD * 2;
  static constexpr int KV_BYTES = TC_KEYS * HD * 2;     // K (bf16) or V (fp16) chunk
  static constexpr int P_BYTES = TC_M * TC_KEYS * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;         // 2 stages
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;    // 2 stages
  static constexpr int OFF_P = OFF_V + 2 * KV_BYTES;    // 2 buffers
  static constexpr int SMEM = OFF_P + 2 * P_BYTES + 1024;
  static constexpr int S_COL = 0;                       // S buffers: [0, 128), [128, 256)
  static constexpr int O_COL = 2 * TC_KEYS;             // O buffers: [256, 256 + HD), [256 + HD, 256 + 2 HD)
};

struct TcArgs {
  const int32_t* pos;
  const int32_t* seq;
  __nv_bfloat16* out;
  int T, H, KV, G, R;
  float sl2;   // softmax scale * log2(e)
};

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;          // 128-byte swizzle
  return d;
}

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(lp::smem_u32(dst)),
      "l"(m), "r"(lp::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   lp::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lp::smem_u32(bar)) : "memory");
}

template <int HD>
__global__ void __launch_bounds__(TC_THREADS, 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const TcArgs a) {
  using C = TcCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], s_empty[2], p_full[2], o_full[2],
      o_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ int s_pos[TC_M], s_seq[TC_M], s_run_of[TC_M];
  __shared__ int s_run_seq[TC_M], s_run_chunks[TC_M], s_nrun;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = gridDim.x - 1 - blockIdx.x;          // later (longer) tiles first: causal balance
  const int kh = blockIdx.y;
  const int t0 = tile * a.R;

  if (threadIdx.x == 0) {
    lp::mbar_init(&q_full, 1);
    for (int b = 0; b < 2; ++b) {
      lp::mbar_init(&kv_full[b], 1);
      lp::mbar_init(&kv_empty[b], 1);
      lp::mbar_init(&s_full[b], 1);
      lp::mbar_init(&s_empty[b], 4);
      lp::mbar_init(&p_full[b], 4);
      lp::mbar_init(&o_full[b], 1);
      lp::mbar_init(&o_empty[b], 4);
    }
    lp::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     lp::smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
  }
  lp::pdl_wait();
  lp::pdl_trigger();
  // token table and sequence runs of the tile
  for (int i = threadIdx.x; i < a.R; i += blockDim.x) {
    const bool v = t0 + i < a.T;
    s_pos[i] = v ? a.pos[t0 + i] : -1;
    s_seq[i] = v ? a.seq[t0 + i] : -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int i = 0; i < a.R; ++i) {
      if (s_seq[i] < 0) {
        s_run_of[i] = -1;
        continue;
      }
      if (n == 0 || s_run_seq[n - 1] != s_seq[i] || s_run_of[i - 1] != n - 1) {
        s_run_seq[n] = s_seq[i];
        s_run_chunks[n] = 0;
        ++n;
      }
      s_run_of[i] = n - 1;
      const int need = (s_pos[i] + TC_KEYS) / TC_KEYS;   // chunks covering keys 0..pos
      if (need > s_run_chunks[n - 1]) s_run_chunks[n - 1] = need;
    }
    s_nrun = n;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;
  const int nrun = s_nrun;

  if (warp == 0) {
    if (lane == 0 && nrun > 0) {
      // ---------------- TMA producer ----------------
      lp::mbar_expect_tx(&q_full, C::Q_BYTES);
      for (int at = 0; at < C::ATOMS; ++at)
        tma3d(sm + C::OFF_Q + at * ATOM, &tmQ, &q_full, at * 64, kh * a.G, t0);
      int it = 0;
      for (int ri = 0; ri < nrun; ++ri) {
        const int row = s_run_seq[ri] * a.KV + kh;
        for (int c = 0; c < s_run_chunks[ri]; ++c, ++it) {
          const int st = it & 1;
          if (it >= 2) lp::mbar_wait(&kv_empty[st], ((it >> 1) - 1) & 1);
          lp::mbar_expect_tx(&kv_full[st], 2 * C::KV_BYTES);
          for (int at = 0; at < C::ATOMS; ++at) {
            tma3d(sm + C::OFF_K + st * C::KV_BYTES + at * (TC_KEYS * 128), &tmK, &kv_full[st], at * 64,
                  c * TC_KEYS, row);
            tma3d(sm + C::OFF_V + st * C::KV_BYTES + at * (TC_KEYS * 128), &tmV, &kv_full[st], at * 64,
                  c * TC_KEYS, row);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nrun > 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_KEYS >> 3) << 17) |
                                   ((uint32_t)(TC_M >> 4) << 24);          // bf16 x bf16, both K-major
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) |
                                    ((uint32_t)(TC_M >> 4) << 24);         // fp16 x fp16, B MN-major
      const uint32_t sq = lp::smem_u32(sm + C::OFF_Q);
      int total = 0;
      for (int ri = 0; ri < nrun; ++ri) total += s_run_chunks[ri];
      auto issue_pv = [&](int j) {
        const int b = j & 1;
        lp::mbar_wait(&p_full[b], (j >> 1) & 1);
        if (j >= 2) lp::mbar_wait(&o_empty[b], ((j >> 1) - 1) & 1);
        fence_after();
        const uint32_t sp = lp::smem_u32(sm + C::OFF_P + b * C::P_BYTES);
        const uint32_t sv = lp::smem_u32(sm + C::OFF_V + b * C::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < TC_KEYS / 16; ++kk)
          umma(tmem + C::O_COL + b * HD, desc_sw128(sp + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024),
               desc_sw128(sv + kk * 2048, TC_KEYS * 128, 1024), idesc_pv, kk > 0);
        commit(&o_full[b]);
        commit(&kv_empty[b]);     // K_j (S_j done earlier) and V_j are free
      };
      lp::mbar_wait(&q_full, 0);
      for (int it = 0; it < total; ++it) {
        const int st = it & 1;
        lp::mbar_wait(&kv_full[st], (it >> 1) & 1);
        if (it >= 2) lp::mbar_wait(&s_empty[st], ((it >> 1) - 1) & 1);
        fence_after();
        const uint32_t sk = lp::smem_u32(sm + C::OFF_K + st * C::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma(tmem + C::S_COL + st * TC_KEYS, desc_sw128(sq + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024),
               desc_sw128(sk + (kk >> 2) * (TC_KEYS * 128) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
        commit(&s_full[st]);
        if (it > 0) issue_pv(it - 1);
      }
      if (total > 0) issue_pv(total - 1);
    }
  } else {
    // ---------------- softmax / output: thread = row ----------------
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int i = r / a.G, g = r % a.G;
    const int prow = i < a.R ? s_pos[i] : -1;
    const int myrun = i < a.R ? s_run_of[i] : -1;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    float o[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) o[d] = 0.f;
    float m_run = -INFINITY, l_run = 0.f, m_acc = -INFINITY;
    float m_hist[2] = {-INFINITY, -INFINITY};
    auto merge = [&](int j) {
      const int b = j & 1;
      lp::mbar_wait(&o_full[b], (j >> 1) & 1);
      fence_after();
      const float mj = m_hist[b];
      const float sc = m_acc == -INFINITY ? 0.f : exp2f(m_acc - mj);
#pragma unroll
      for (int cg = 0; cg < HD / 32; ++cg) {
        uint32_t v[32];
        ld32(trow + C::O_COL + b * HD + cg * 32, v);
        wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[cg * 32 + e] = o[cg * 32 + e] * sc + __uint_as_float(v[e]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[b]);
      m_acc = mj;
    };
    int it = 0;
    for (int ri = 0; ri < nrun; ++ri) {
      const bool mine = myrun == ri;
      for (int c = 0; c < s_run_chunks[ri]; ++c, ++it) {
        const int b = it & 1;
        lp::mbar_wait(&s_full[b], (it >> 1) & 1);
        fence_after();
        const int lim = mine ? prow - c * TC_KEYS : -1;     // keys 0..lim of this chunk are visible
        float cmax = -INFINITY;
#pragma unroll
        for (int cg = 0; cg < TC_KEYS / 32; ++cg) {
          uint32_t v[32];
          ld32(trow + C::S_COL + b * TC_KEYS + cg * 32, v);
          wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (cg * 32 + e <= lim) cmax = fmaxf(cmax, __uint_as_float(v[e]) * a.sl2);
        }
        const float m_new = fmaxf(m_run, cmax);
        float lsum = 0.f;
        uint8_t* prow_s = sm + C::OFF_P + b * C::P_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int cg = 0; cg < TC_KEYS / 32; ++cg) {
          uint32_t v[32];
          ld32(trow + C::S_COL + b * TC_KEYS + cg * 32, v);
          wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int k = cg * 32 + e;
            const float p0 = (k <= lim) ? exp2f(__uint_as_float(v[e]) * a.sl2 - m_new) : 0.f;
            const float p1 = (k + 1 <= lim) ? exp2f(__uint_as_float(v[e + 1]) * a.sl2 - m_new) : 0.f;
            const __half2 h = __floats2half2_rn(p0, p1);
            const float2 hf = __half22float2(h);
            lsum += hf.x + hf.y;                       // the fp16 values P V multiplies
            pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&h);
          }
          uint8_t* atom = prow_s + (cg >> 1) * ATOM;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = ((cg & 1) * 4 + q) ^ (r & 7);
            *reinterpret_cast<uint4*>(atom + chunk * 16) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
        fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P stores -> visible to the MMA
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&s_empty[b]);
          mbar_arrive(&p_full[b]);
        }
        const float al = m_run == -INFINITY ? 0.f : exp2f(m_run - m_new);
        l_run = l_run * al + lsum;
        m_run = m_new;
        m_hist[b] = m_new;
        if (it > 0) merge(it - 1);
      }
    }
    if (it > 0) merge(it - 1);
    if (i < a.R && t0 + i < a.T && l_run > 0.f) {
      const float inv = 1.0f / l_run;
      __nv_bfloat16* orow = a.out + ((int64_t)(t0 + i) * a.H + kh * a.G + g) * HD;
#pragma unroll
      for (int d = 0; d < HD; d += 8) {
        __nv_bfloat162 w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) w[e] = __floats2bfloat162_rn(o[d + 2 * e] * inv, o[d + 2 * e + 1] * inv);
        *reinterpret_cast<uint4*>(orow + d) = *reinterpret_cast<const uint4*>(w);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encode g_enc = nullptr;

int map3d(CUtensorMap* m, CUtensorMapDataType ty, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
          uint64_t s1_bytes, uint64_t s2_bytes, uint32_t b1, uint32_t b2) {
  if (!g_enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    LP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    LP_CHECK(q == cudaDriverEntryPointSuccess && fn, "cuTensorMapEncodeTiled unavailable");
    g_enc = (PFN_encode)fn;
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_bytes, s2_bytes};
  cuuint32_t box[3] = {64, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_enc(m, ty, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LP_CHECK(r == CUDA_SUCCESS, "attention_tc: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

template <int HD>
int launch_tc(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos, const int32_t* seq,
              int T, int H, int KV, int64_t max_len, float scale, void* out, cudaStream_t s) {
  using C = TcCfg<HD>;
  const int G = H / KV;
  const int R = TC_M / G;
  CUtensorMap mq, mk, mv;
  const uint64_t rows = (uint64_t)1 << 24;   // sequence x kv-head rows of the caches (unbounded here)
  if (map3d(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, q, HD, H, T, (uint64_t)HD * 2, (uint64_t)H * HD * 2, G, R)) return -1;
  if (map3d(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, k_cache, HD, max_len, rows, (uint64_t)HD * 2,
            (uint64_t)max_len * HD * 2, TC_KEYS, 1))
    return -1;
  if (map3d(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, v_cache, HD, max_len, rows, (uint64_t)HD * 2,
            (uint64_t)max_len * HD * 2, TC_KEYS, 1))
    return -1;
  static uint64_t attr = 0;
  int dev = 0;
  LP_CUDA(cudaGetDevice(&dev));
  if (!(attr >> dev & 1)) {
    LP_CUDA(cudaFuncSetAttribute(attention_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr |= 1ull << dev;
  }
  TcArgs args{pos, seq, (__nv_bfloat16*)out, T, H, KV, G, R, scale * 1.4426950408889634f};
  const dim3 grid((unsigned)((T + R - 1) / R), (unsigned)KV);
  LP_CUDA(lp::launch(attention_tc_kernel<HD>, grid, dim3(TC_THREADS), C::SMEM, s, mq, mk, mv, args));
  return 0;
}

}  // namespace

namespace lp {
// Causal GQA attention over the KV cache on tcgen05 (see file head).  Returns
// 1 when the shape is not covered (caller falls back), 0 on launch, < 0 on error.
int attention_tc(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos, const int32_t* seq,
                 int64_t T, int n_heads, int n_kv, int head_dim, int64_t max_len, float scale, void* out,
                 cudaStream_t s) {
  const int G = n_heads / n_kv;
  if (G < 1 || G > TC_M || TC_M % G != 0) return 1;
  if (max_len % 8 != 0 || T > (1 << 30)) return 1;
  if (head_dim == 128) return launch_tc<128>(q, k_cache, v_cache, pos, seq, (int)T, n_heads, n_kv, max_len, scale,
                                             out, s);
  if (head_dim == 64) return launch_tc<64>(q, k_cache, v_cache, pos, seq, (int)T, n_heads, n_kv, max_len, scale,
                                           out, s);
  return 1;
}
}  // namespace lp
