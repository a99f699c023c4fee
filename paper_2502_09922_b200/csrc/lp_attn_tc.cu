// Causal GQA prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM +
// TMA), FlashAttention-style online softmax.
//
// Default: attention_fa_kernel (FA4 layout, below the one-tile kernel): two
// Q tiles per CTA, P kept in TMEM as the P V MMA's A operand, one softmax
// thread per row.  The one-tile kernel described first stays selectable
// (LP_ATTN_TC=1/3, launch_tc) and shares the tiling, TMA boxes and the
// MN-major V operand.
//
// Tile: one CTA owns 128 TMEM lanes = R tokens x G query heads of one kv head
// (R = 128 / G; Llama-3-8B G = 4 -> 32 tokens, 70B G = 8 -> 16, MHA -> 128),
// so the heads of a GQA group share every K/V chunk the CTA streams.  Rows
// are token-major (row = i * G + g), which is exactly what a 3-D TMA box
// {64 dims, G heads, R tokens} of q [T, H, hd] lands in shared memory.
//
// Per 128-key chunk j of the tile's sequence:
//   S_j  = Q K_j^T      tcgen05.mma kind::f16, A = Q (smem, K-major, bf16),
//                       B = K_j (smem, K-major, bf16), D = S in TMEM (fp32,
//                       three buffers)
//   P_j  = exp2(S_j * scale * log2e - m)     softmax warps: TMEM -> regs,
//                       causal mask from pos[], fp16 P written to smem
//   O   += P_j V_j      tcgen05.mma kind::f16, A = P (smem, K-major, fp16),
//                       B = V_j (smem, MN-major: the fp16 V cache is [key][hd]),
//                       D = O, accumulated in TMEM across all chunks
// The row max m used for P only moves when the running max exceeds it by
// more than 2^8 (P then stays <= 256, exact enough in fp16; the row sum l
// uses the same m), so O almost never needs rescaling: when it does, the
// row's softmax threads rescale it in TMEM (after the previous P V) before
// releasing P_j.  Final: O / l.  Its lazy variant (LP_ATTN_TC=3) computes
// P_j with the current m first and only then combines the halves' raw maxima
// (one atomicMax slot + a 64-thread named barrier per chunk), recomputing P_j
// from the S values still in registers when m has to move.
//
//   warp 0   : TMA producer (Q once, then K chunks)      warp 10: TMA (V chunks)
//   warp 1   : TMEM allocator + MMA issuer (one thread)
//   warps 2-9: softmax (two threads per row: key / dim halves)
//
// A tile whose tokens belong to several sequences (ragged batches) walks the
// chunks of each sequence run in turn with the other rows masked.
#include "lp_common.cuh"
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

namespace {

constexpr int TC_M = 128;       // rows per tile (TMEM lanes)
constexpr int TC_KEYS = 128;    // keys per chunk
// threads: warp 0 TMA (Q, K), warp 1 MMA, 4 NS softmax warps, then one TMA (V) warp: (3 + 4 NS) x 32
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
  static constexpr int BODY = OFF_P + 2 * P_BYTES;
  // + the pad that aligns the body to 1024 B after the kernel's static smem
  // (launch_tc computes it; the full 1024 B slack would not fit in 227 KB)

  static constexpr int S_COL = 0;                       // S buffers: [0, 128), [128, 256), [256, 384)
  static constexpr int O_COL = 3 * TC_KEYS;             // O accumulator: [384, 384 + HD)
};

struct TcArgs {
  const int32_t* pos;
  const int32_t* seq;
  __nv_bfloat16* out;
  int T, H, KV, G, R;
  float sl2;   // softmax scale * log2(e)
  long long* trace;   // debug (LP_ATTN_TRACE): per-chunk clock64 stamps of the last CTA, else null
};
// trace slots per chunk: 0 S issued, 1 PV issued, 2 softmax S ready, 3 S loaded, 4 P written, 5 p_full arrive
#define TRACE(slot, it)                                                                    \
  do {                                                                                     \
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && (it) < 64)            \
      a.trace[(it) * 16 + (slot)] = clock64();                                              \
  } while (0)

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
// wait for outstanding tcgen05.ld with v's registers as in-out operands: the
// compiler cannot read, move or reuse them before the loads have landed
// (needed when a load stays in flight across other code)
__device__ __forceinline__ void wait_ld32(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 2^x on the SFU without exp2f's denormal-range fix-ups (P underflowing to 0
// instead of a denormal is harmless): one MUFU.EX2
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Packed fp32 pairs (Blackwell FFMA2 / FADD2: one issue slot for two lanes'
// worth of math) and the 3-input max (FMNMX3)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// 2^x for a pair on the FMA pipe (offloads the SFU, 16 ex2 / clock / SM on
// B200 = the MMA time of a chunk): x = n + f with n = rint(x) via the
// 1.5 * 2^23 magic add, f in [-0.5, 0.5], 2^f by a degree-3 fit (max relative
// error 7.5e-5, below fp16 P's half ulp), n added to the exponent with one
// IMAD.  x is clamped at -100 (2^-100 is 0 in fp16 P and in the row sum).
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
// order-preserving int image of a float (atomicMax on floats of any sign)
constexpr int ORD_NEG_INF = (int)0x807FFFFF;   // ord_f32(-inf)
__device__ __forceinline__ int ord_f32(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float unord_f32(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }
// One thread's share of a softmax chunk: KW raw scores v (keys 0..lim of
// them visible) -> fp16 P = exp2(v * sl2 - mu) into its 128-B swizzled smem
// row (16-B chunks cb .. cb + KW / 8 - 1, XOR-swizzled by r & 7); returns the
// row sum, and with WM the raw max over the visible keys in mraw.  Warp-
// collective (the unmasked test is a vote).  Unmasked chunks use packed
// FFMA2 / FADD2 / FMNMX3 and one key pair in four on the FMA-pipe exp2.
template <int KW, bool WM, int POLY = 1>
__device__ __forceinline__ float softmax_write_p(const uint32_t (&v)[KW], int lim, float sl2, float mu,
                                                 uint8_t* prow_s, int cb, int r, float& mraw) {
  const bool unmasked = __all_sync(0xffffffffu, lim >= KW - 1);   // before any lane returns
  if (lim < 0) {
#pragma unroll
    for (int q = 0; q < KW / 8; ++q)
      *reinterpret_cast<uint4*>(prow_s + (((cb + q) ^ (r & 7)) * 16)) = make_uint4(0, 0, 0, 0);
    return 0.f;
  }
  const float nm = -mu;
  if (unmasked) {
    float2 ls2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    const float2 sl = make_float2(sl2, sl2), nm2 = make_float2(nm, nm);
#pragma unroll
    for (int q = 0; q < KW / 8; ++q) {
      uint32_t pk[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const int k = q * 8 + e;
        const float2 sv = make_float2(__uint_as_float(v[k]), __uint_as_float(v[k + 1]));
        if (WM) mx4[e >> 1] = fmax3(mx4[e >> 1], sv.x, sv.y);
        const float2 x = ffma2(sv, sl, nm2);
        float2 p;
        if ((e >> 1) >= 4 - POLY) {      // POLY of every 4 key pairs on the FMA pipe
          p = exp2_poly2(x);
        } else {
          p.x = fast_exp2(x.x);
          p.y = fast_exp2(x.y);
        }
        ls2[e >> 1] = fadd2(ls2[e >> 1], p);
        const __half2 hv = __floats2half2_rn(p.x, p.y);
        pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&hv);
      }
      *reinterpret_cast<uint4*>(prow_s + (((cb + q) ^ (r & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    if (WM) mraw = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
    const float2 s01 = fadd2(ls2[0], ls2[1]), s23 = fadd2(ls2[2], ls2[3]);
    return (s01.x + s01.y) + (s23.x + s23.y);
  }
  float ls[4] = {0.f, 0.f, 0.f, 0.f};
  float mx8[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) mx8[q] = -INFINITY;
#pragma unroll
  for (int q = 0; q < KW / 8; ++q) {
    uint32_t pk[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const int k = q * 8 + e;
      const float s0 = __uint_as_float(v[k]), s1 = __uint_as_float(v[k + 1]);
      const float p0 = k <= lim ? fast_exp2(fmaf(s0, sl2, nm)) : 0.f;
      const float p1 = k + 1 <= lim ? fast_exp2(fmaf(s1, sl2, nm)) : 0.f;
      if (WM) {
        mx8[e] = k <= lim ? fmaxf(mx8[e], s0) : mx8[e];
        mx8[e + 1] = k + 1 <= lim ? fmaxf(mx8[e + 1], s1) : mx8[e + 1];
      }
      ls[e >> 1] += p0 + p1;
      const __half2 hv = __floats2half2_rn(p0, p1);
      pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    *reinterpret_cast<uint4*>(prow_s + (((cb + q) ^ (r & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  if (WM)
    mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                 fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
  return (ls[0] + ls[1]) + (ls[2] + ls[3]);
}
// raw max over the visible keys 0..lim of v
template <int KW>
__device__ __forceinline__ float softmax_row_max(const uint32_t (&v)[KW], int lim) {
  float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  if (lim >= KW - 1) {
#pragma unroll
    for (int e = 0; e < KW; e += 2)
      mx4[(e >> 1) & 3] = fmax3(mx4[(e >> 1) & 3], __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
  } else if (lim >= 0) {
#pragma unroll
    for (int e = 0; e < KW; ++e)
      if (e <= lim) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(v[e]));
  }
  return fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lp::smem_u32(bar)) : "memory");
}

template <int HD, int NS, bool LAZY, int POLY = 1>
__global__ void __launch_bounds__((3 + 4 * NS) * 32, 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const TcArgs a) {
  using C = TcCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if ((uint32_t)(sm - smem_raw) + C::BODY > dyn) __trap();   // launch_tc's pad assumption broken
  }
  __shared__ __align__(8) uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[3], s_empty[3],
      p_full[2], o_done, o_final;
  __shared__ uint32_t tmem_base;
  __shared__ int s_pos[TC_M];                 // per token of the tile (-1 past T)
  __shared__ int16_t s_seq[TC_M];
  __shared__ int s_cmx[3][TC_M];               // lazy path: joint raw row max per chunk (it % 3)
  static_assert(NS == 2 || (LAZY && HD % (32 * NS) == 0), "4-way key split: lazy path, 32 O columns per warp");
  constexpr int VW = 2 + 4 * NS;               // the V producer warp (after the softmax warps)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 1-D grid over (tile, kv head), longest tiles of EVERY head first: the
  // block scheduler then fills the SMs in LPT order (a [tiles, heads] grid
  // launched head 0's short tiles before head 7's long ones)
  const int tile = (int)(gridDim.x / a.KV) - 1 - (int)(blockIdx.x / a.KV);
  const int kh = (int)(blockIdx.x % a.KV);
  const int t0 = tile * a.R;

  if (threadIdx.x == 0) {
    lp::mbar_init(&q_full, 1);
    for (int b = 0; b < 2; ++b) {
      lp::mbar_init(&k_full[b], 1);
      lp::mbar_init(&k_empty[b], 1);
      lp::mbar_init(&v_full[b], 1);
      lp::mbar_init(&v_empty[b], 1);
      lp::mbar_init(&p_full[b], 4 * NS);
    }
    for (int b = 0; b < 3; ++b) {
      lp::mbar_init(&s_full[b], 1);
      lp::mbar_init(&s_empty[b], 4 * NS);
    }
    lp::mbar_init(&o_done, 1);
    lp::mbar_init(&o_final, 1);
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
  for (int i = threadIdx.x; i < 3 * TC_M; i += blockDim.x) (&s_cmx[0][0])[i] = ORD_NEG_INF;
  for (int i = threadIdx.x; i < a.R; i += blockDim.x) {
    const bool v = t0 + i < a.T;
    s_pos[i] = v ? a.pos[t0 + i] : -1;
    s_seq[i] = v ? (int16_t)a.seq[t0 + i] : (int16_t)-1;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;
  // runs of consecutive tokens of one sequence; every role walks them with
  // run(): [lo, hi) tokens, sequence, chunks covering keys 0..max pos
  auto run = [&](int lo, int& hi, int& sq, int& chunks) {
    sq = s_seq[lo];
    chunks = 0;
    for (hi = lo; hi < a.R && s_seq[hi] == sq; ++hi) chunks = max(chunks, (s_pos[hi] + TC_KEYS) / TC_KEYS);
  };
  const int nvalid = min(a.R, a.T - t0);

  if (warp == 0 || warp == VW) {
    if (lane == 0) {
      // ---------------- TMA producers: warp 0 Q + K, warp 10 V ----------------
      // K_j's stage frees when S_j is done, V_j's when P_j V_j is: separate
      // rings let K_{j+2} stream in while chunk j is still in softmax / P V
      const bool is_k = warp == 0;
      if (is_k) {
        lp::mbar_expect_tx(&q_full, C::Q_BYTES);
        for (int at = 0; at < C::ATOMS; ++at)
          tma3d(sm + C::OFF_Q + at * ATOM, &tmQ, &q_full, at * 64, kh * a.G, t0);
      }
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      const CUtensorMap* map = is_k ? &tmK : &tmV;
      uint8_t* base = sm + (is_k ? C::OFF_K : C::OFF_V);
      int it = 0;
      for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
        run(lo, hi, sq, nch);
        const int row = sq * a.KV + kh;
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it & 1;
          if (it >= 2) lp::mbar_wait(&empty[st], ((it >> 1) - 1) & 1);
          TRACE(is_k ? 7 : 8, it);
          lp::mbar_expect_tx(&full[st], C::KV_BYTES);
          for (int at = 0; at < C::ATOMS; ++at)
            tma3d(base + st * C::KV_BYTES + at * (TC_KEYS * 128), map, &full[st], at * 64, c * TC_KEYS, row);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_KEYS >> 3) << 17) |
                                   ((uint32_t)(TC_M >> 4) << 24);          // bf16 x bf16, both K-major
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) |
                                    ((uint32_t)(TC_M >> 4) << 24);         // fp16 x fp16, B MN-major
      const uint32_t sq = lp::smem_u32(sm + C::OFF_Q);
      int total = 0;
      for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
        run(lo, hi, sq, nch);
        total += nch;
      }
      auto issue_pv = [&](int j) {
        const int b = j & 1;
        lp::mbar_wait(&p_full[b], (j >> 1) & 1);     // P_j written (and O rescaled if its rows needed it)
        lp::mbar_wait(&v_full[b], (j >> 1) & 1);
        fence_after();
        TRACE(1, j);
        const uint32_t sp = lp::smem_u32(sm + C::OFF_P + b * C::P_BYTES);
        const uint32_t sv = lp::smem_u32(sm + C::OFF_V + b * C::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < TC_KEYS / 16; ++kk)
          umma(tmem + C::O_COL, desc_sw128(sp + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024),
               desc_sw128(sv + kk * 2048, TC_KEYS * 128, 1024), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        commit(&o_done);
        commit(&v_empty[b]);
      };
      lp::mbar_wait(&q_full, 0);
      for (int it = 0; it < total; ++it) {
        const int st = it & 1, sb = it % 3;
        lp::mbar_wait(&k_full[st], (it >> 1) & 1);
        TRACE(9, it);
        if (it >= 3) lp::mbar_wait(&s_empty[sb], (it / 3 - 1) & 1);
        fence_after();
        const uint32_t sk = lp::smem_u32(sm + C::OFF_K + st * C::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma(tmem + C::S_COL + sb * TC_KEYS, desc_sw128(sq + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024),
               desc_sw128(sk + (kk >> 2) * (TC_KEYS * 128) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
        commit(&s_full[sb]);
        TRACE(0, it);
        commit(&k_empty[st]);
        if (it > 0) issue_pv(it - 1);
      }
      if (total > 0) {
        issue_pv(total - 1);
        commit(&o_final);      // every MMA done: o_done's parity cannot tell phase it-1 from it-3
      }
    }
  } else if (warp < VW) {
    // ---------------- softmax ----------------
    // two warps per TMEM lane quarter: thread (row r, half h) owns keys
    // [64h, 64h + 64) of every S chunk (= P atom h) and O columns
    // [h HD/2, (h + 1) HD/2); the row max is exchanged through smem once per
    // chunk (named barrier over the 256 softmax threads), the row sums only
    // at the end (both halves use the same m).
    constexpr int HH = HD / NS;                  // O columns per warp
    constexpr float RESCALE = 8.0f;              // log2 headroom before m moves (P <= 2^8 in fp16)
    const int quarter = warp & 3;
    const int hq = (warp - 2) >> 2;              // which NS-th of the keys / O columns
    const int h = hq;
    const int r = quarter * 32 + lane;
    const int i = r / a.G, g = r % a.G;
    const int prow = i < nvalid ? s_pos[i] : -1;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    float m_use = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
      run(lo, hi, sq, nch);
      const bool mine = i >= lo && i < hi;
      for (int c = 0; c < nch; ++c, ++it) {
        const int b = it & 1, sb = it % 3;
        lp::mbar_wait(&s_full[sb], (it / 3) & 1);
        fence_after();
        if (warp == 2 && lane == 0) TRACE(2, it);
        if constexpr (LAZY) {
          // Lazy max: P is computed with the current m first, the row max
          // (own keys, fused into the exp pass) is combined across the NS
          // warps of the row through a shared atomicMax slot and one named
          // barrier; only when the joint max moves m by more than RESCALE
          // (first visible chunk, rare after) is P recomputed from the S
          // values still in registers.
          constexpr int KW = TC_KEYS / NS;             // keys of each chunk this warp owns
          const int lim = mine ? prow - c * TC_KEYS - hq * KW : -1;
          uint32_t v[KW];
#pragma unroll
          for (int cg = 0; cg < KW / 32; ++cg)
            ld32(trow + C::S_COL + sb * TC_KEYS + hq * KW + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(v + cg * 32));
          wait_ld();
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[sb]);
          if (warp == 2 && lane == 0) TRACE(3, it);
          uint8_t* prow_s = sm + C::OFF_P + b * C::P_BYTES + ((hq * KW) >> 6) * ATOM + (r >> 3) * 1024 + (r & 7) * 128;
          const int cb = ((hq * KW) & 63) >> 3;       // my first 16-B chunk of the 128-B P row
          auto write_p = [&](float mu, float& mraw, auto want_max) -> float {
            return softmax_write_p<KW, decltype(want_max)::value, POLY>(v, lim, a.sl2, mu, prow_s, cb, r, mraw);
          };
          auto own_max = [&]() -> float { return softmax_row_max<KW>(v, lim); };
          // joint raw max of the row: atomicMax on an order-preserving int
          // image of the float into slot it % 3, one barrier over the row's
          // NS warps; slot (it + 2) % 3 (last read before this barrier, next
          // written after the following one) is reset here
          auto exchange = [&](float mraw) -> float {
            atomicMax(&s_cmx[it % 3][r], ord_f32(mraw));
            switch (quarter) {                  // literal ids: a register id reserves all 16 barriers
              case 0: asm volatile("bar.sync 2, %0;" ::"n"(NS * 32) : "memory"); break;
              case 1: asm volatile("bar.sync 3, %0;" ::"n"(NS * 32) : "memory"); break;
              case 2: asm volatile("bar.sync 4, %0;" ::"n"(NS * 32) : "memory"); break;
              default: asm volatile("bar.sync 5, %0;" ::"n"(NS * 32) : "memory"); break;
            }
            const float m = a.sl2 * unord_f32(s_cmx[it % 3][r]);
            if (hq == 0) s_cmx[(it + 2) % 3][r] = ORD_NEG_INF;
            return m;
          };
          // m moves: rescale O (after P_{it-1} V_{it-1}) and the running sum
          auto move_m = [&](float m_row) {
            const bool move = m_row > m_use + RESCALE || (m_use == -INFINITY && m_row > -INFINITY);
            const float sc = (move && m_use != -INFINITY) ? exp2f(m_use - m_row) : 1.f;
            const bool resc = move && m_use != -INFINITY && it > 0;
            if (move) {
              l_run *= m_use == -INFINITY ? 0.f : sc;
              m_use = m_row;
            }
            if (__any_sync(0xffffffffu, resc)) {
              lp::mbar_wait(&o_done, (it - 1) & 1);
              fence_after();
              uint32_t o[HH];
#pragma unroll
              for (int cg = 0; cg < HH / 32; ++cg)
                ld32(trow + C::O_COL + hq * HH + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o + cg * 32));
              wait_ld();
#pragma unroll
              for (int e = 0; e < HH; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * sc);
#pragma unroll
              for (int cg = 0; cg < HH / 32; ++cg)
                st32(trow + C::O_COL + hq * HH + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o + cg * 32));
              wait_st();
            }
            return move;
          };
          float ls, mraw = -INFINITY;
          if (__any_sync(0xffffffffu, m_use == -INFINITY && lim >= 0)) {
            // a row of the warp has no m yet: max first, then P
            const float m_row = exchange(own_max());
            if (warp == 2 && lane == 0) TRACE(6, it);
            move_m(m_row);
            ls = write_p(m_use, mraw, std::false_type{});
          } else {
            ls = write_p(m_use, mraw, std::true_type{});
            if (warp == 2 && lane == 0) TRACE(6, it);
            const bool moved = move_m(exchange(mraw));
            if (__any_sync(0xffffffffu, moved)) {      // write_p is warp-collective; rewrites are idempotent
              const float ls_new = write_p(m_use, mraw, std::false_type{});
              if (moved) ls = ls_new;
            }
          }
          l_run += ls;
          fence_before();
          if (warp == 2 && lane == 0) TRACE(4, it);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[b]);
          if (warp == 2 && lane == 0) TRACE(5, it);
          continue;
        }
        const int lim = mine ? prow - c * TC_KEYS - h * 64 : -1;   // my keys 0..lim are visible
        const int limp = mine ? prow - c * TC_KEYS - (h ^ 1) * 64 : -1;   // the partner half's
        // the row max over all 128 keys: own half kept in registers, the
        // partner half streamed through 32 registers (TMEM reads are cheap;
        // exchanging halves through smem cost two 256-thread barriers a chunk)
        uint32_t v[64];
        float mx8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = -INFINITY;
#pragma unroll
        for (int cg = 0; cg < 2; ++cg) {
          uint32_t w[32];
          ld32(trow + C::S_COL + sb * TC_KEYS + (h ^ 1) * 64 + cg * 32, w);
          wait_ld();
          if (limp >= 63) {
#pragma unroll
            for (int e = 0; e < 32; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(w[e]));
          } else if (limp >= 0) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (cg * 32 + e <= limp) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(w[e]));
          }
        }
        ld32(trow + C::S_COL + sb * TC_KEYS + h * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
        ld32(trow + C::S_COL + sb * TC_KEYS + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);  // S buffer may be overwritten (S_{it+3})
        if (warp == 2 && lane == 0) TRACE(3, it);
        // raw scores; the scale (> 0) is applied to the max and inside the exp FFMA
        if (lim >= 63) {                             // whole half below the diagonal: no mask
#pragma unroll
          for (int e = 0; e < 64; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(v[e]));
        } else if (lim >= 0) {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (e <= lim) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(v[e]));
        }
        const float m_row = a.sl2 * fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                          fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        if (warp == 2 && lane == 0) TRACE(6, it);
        // both halves take the same decision from the same inputs; a row whose
        // m was -inf has P = 0 so far, i.e. O = 0: nothing to rescale
        const bool move = m_row > m_use + RESCALE || (m_use == -INFINITY && m_row > -INFINITY);
        const float sc = (move && m_use != -INFINITY) ? exp2f(m_use - m_row) : 1.f;
        const bool resc = move && m_use != -INFINITY && it > 0;
        if (move) {
          l_run *= m_use == -INFINITY ? 0.f : sc;
          m_use = m_row;
        }
        if (__any_sync(0xffffffffu, resc)) {           // tcgen05.ld/st are warp-collective
          lp::mbar_wait(&o_done, (it - 1) & 1);        // P_{it-1} V_{it-1} has landed
          fence_after();
          uint32_t o[HH];
#pragma unroll
          for (int cg = 0; cg < HH / 32; ++cg)
            ld32(trow + C::O_COL + h * HH + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o + cg * 32));
          wait_ld();
#pragma unroll
          for (int e = 0; e < HH; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * sc);
#pragma unroll
          for (int cg = 0; cg < HH / 32; ++cg)
            st32(trow + C::O_COL + h * HH + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o + cg * 32));
          wait_st();
        }
        float ls[4] = {0.f, 0.f, 0.f, 0.f};          // independent sum chains
        uint8_t* prow_s = sm + C::OFF_P + b * C::P_BYTES + h * ATOM + (r >> 3) * 1024 + (r & 7) * 128;
        if (lim < 0) {                               // nothing visible: P = 0
#pragma unroll
          for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(prow_s + q * 16) = make_uint4(0, 0, 0, 0);
        } else {
          const float nm = -m_use;
#pragma unroll
          for (int q = 0; q < 8; ++q) {               // 8 x 16 B: keys 8q .. 8q + 7 of my 64
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const int k = q * 8 + e;
              float p0 = fast_exp2(fmaf(__uint_as_float(v[k]), a.sl2, nm));
              float p1 = fast_exp2(fmaf(__uint_as_float(v[k + 1]), a.sl2, nm));
              if (lim < 63) {
                p0 = k <= lim ? p0 : 0.f;
                p1 = k + 1 <= lim ? p1 : 0.f;
              }
              ls[e >> 1] += p0 + p1;
              const __half2 hv = __floats2half2_rn(p0, p1);
              pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&hv);
            }
            *reinterpret_cast<uint4*>(prow_s + ((q ^ (r & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
        l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        fence_before();                              // TMEM stores (rescale) before the MMA reads O
        if (warp == 2 && lane == 0) TRACE(4, it);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P stores -> visible to the MMA
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (warp == 2 && lane == 0) TRACE(5, it);
      }
    }
    if (it > 0) {
      lp::mbar_wait(&o_final, 0);                    // the last P V has landed
      fence_after();
    }
    // row sums across the NS warps through the P buffers (free once the
    // last P V has landed), summed in a fixed order
    float* lsum = reinterpret_cast<float*>(sm + C::OFF_P);
    lsum[hq * TC_M + r] = l_run;
    asm volatile("bar.sync 1, %0;" ::"n"(NS * 128) : "memory");
    float l_tot = 0.f;
#pragma unroll
    for (int j = 0; j < NS; ++j) l_tot += lsum[j * TC_M + r];
    uint32_t o[HH];
#pragma unroll
    for (int cg = 0; cg < HH / 32; ++cg)
      ld32(trow + C::O_COL + h * HH + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o + cg * 32));
    wait_ld();
    if (i < a.R && t0 + i < a.T && l_tot > 0.f) {
      const float inv = 1.0f / l_tot;
      __nv_bfloat16* orow = a.out + ((int64_t)(t0 + i) * a.H + kh * a.G + g) * HD + h * HH;
#pragma unroll
      for (int d = 0; d < HH; d += 8) {
        __nv_bfloat162 w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          w[e] = __floats2bfloat162_rn(__uint_as_float(o[d + 2 * e]) * inv, __uint_as_float(o[d + 2 * e + 1]) * inv);
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

// ---------------------------------------------------------------------------
// Ping-pong variant: TWO Q tiles per CTA (tokens [t0, t0 + R) and
// [t0 + R, t0 + 2R) of one kv head) over 64-key chunks.  Each tile has its own
// softmax warpgroup (warps 2-5: tile 0, warps 6-9: tile 1; one thread per row
// holds the chunk's whole 64-key row, so no max exchange), its own two S
// buffers and O accumulator in TMEM (2 x (2 x 64 + 128) = 512 columns), and
// two P buffers; K/V chunks are shared.  While one tile's warps sit in TMEM
// loads / max / P stores the other's use the SFU, and the MMAs of one tile run
// under the other's softmax (FA4-style), which the one-tile kernel's lock-step
// half-row warps could not do (its measured chunk: ~2,300 softmax cycles vs
// ~1,100 MMA cycles, profiles/r02/attn_tc_chunk_trace_8b_1x2048.txt).
constexpr int PP_KEYS = 64;
constexpr int PP_THREADS = 352;

template <int HD>
struct PpCfg {
  static constexpr int ATOMS = HD / 64;
  static constexpr int Q_BYTES = TC_M * HD * 2;          // one tile
  static constexpr int KV_BYTES = PP_KEYS * HD * 2;      // one chunk
  static constexpr int P_BYTES = TC_M * PP_KEYS * 2;     // one tile's chunk = one 128B-swizzle atom
  static constexpr int OFF_Q = 0;                        // 2 tiles
  static constexpr int OFF_K = 2 * Q_BYTES;              // 2 stages
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;     // 2 stages
  static constexpr int OFF_P = OFF_V + 2 * KV_BYTES;     // [tile][2]
  static constexpr int BODY = OFF_P + 4 * P_BYTES;
  static constexpr int SMEM = BODY + 1024;
  static constexpr int TILE_COLS = 256;                  // per tile: S0 [0,64), S1 [64,128), O [128, 128 + HD)
};

template <int HD>
__global__ void __launch_bounds__(PP_THREADS, 1)
    attention_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const TcArgs a) {
  using C = PpCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if ((uint32_t)(sm - smem_raw) + C::BODY > dyn) __trap();   // launch_tc's pad assumption broken
  }
  __shared__ __align__(8) uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2][2], s_empty[2][2],
      p_full[2][2], o_done[2], o_final;
  __shared__ uint32_t tmem_base;
  __shared__ int s_pos[2 * TC_M];
  __shared__ int16_t s_seq[2 * TC_M];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 1-D grid over (tile, kv head), longest tiles of EVERY head first: the
  // block scheduler then fills the SMs in LPT order (a [tiles, heads] grid
  // launched head 0's short tiles before head 7's long ones)
  const int tile = (int)(gridDim.x / a.KV) - 1 - (int)(blockIdx.x / a.KV);
  const int kh = (int)(blockIdx.x % a.KV);
  const int R2 = 2 * a.R;
  const int t0 = tile * R2;

  if (threadIdx.x == 0) {
    lp::mbar_init(&q_full, 1);
    for (int b = 0; b < 2; ++b) {
      lp::mbar_init(&k_full[b], 1);
      lp::mbar_init(&k_empty[b], 1);
      lp::mbar_init(&v_full[b], 1);
      lp::mbar_init(&v_empty[b], 1);
      for (int t = 0; t < 2; ++t) {
        lp::mbar_init(&s_full[t][b], 1);
        lp::mbar_init(&s_empty[t][b], 4);
        lp::mbar_init(&p_full[t][b], 4);
      }
      lp::mbar_init(&o_done[b], 1);
    }
    lp::mbar_init(&o_final, 1);
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
  for (int i = threadIdx.x; i < R2; i += blockDim.x) {
    const bool v = t0 + i < a.T;
    s_pos[i] = v ? a.pos[t0 + i] : -1;
    s_seq[i] = v ? (int16_t)a.seq[t0 + i] : (int16_t)-1;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;
  auto run = [&](int lo, int& hi, int& sq, int& chunks) {
    sq = s_seq[lo];
    chunks = 0;
    for (hi = lo; hi < R2 && s_seq[hi] == sq; ++hi) chunks = max(chunks, (s_pos[hi] + PP_KEYS) / PP_KEYS);
  };
  const int nvalid = min(R2, a.T - t0);

  if (warp == 0 || warp == 10) {
    if (lane == 0) {
      const bool is_k = warp == 0;
      if (is_k) {
        lp::mbar_expect_tx(&q_full, 2 * C::Q_BYTES);
        for (int t = 0; t < 2; ++t)
          for (int at = 0; at < C::ATOMS; ++at)
            tma3d(sm + C::OFF_Q + t * C::Q_BYTES + at * ATOM, &tmQ, &q_full, at * 64, kh * a.G, t0 + t * a.R);
      }
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      const CUtensorMap* map = is_k ? &tmK : &tmV;
      uint8_t* base = sm + (is_k ? C::OFF_K : C::OFF_V);
      int it = 0;
      for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
        run(lo, hi, sq, nch);
        const int row = sq * a.KV + kh;
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it & 1;
          if (it >= 2) lp::mbar_wait(&empty[st], ((it >> 1) - 1) & 1);
          lp::mbar_expect_tx(&full[st], C::KV_BYTES);
          for (int at = 0; at < C::ATOMS; ++at)
            tma3d(base + st * C::KV_BYTES + at * (PP_KEYS * 128), map, &full[st], at * 64, c * PP_KEYS, row);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(PP_KEYS >> 3) << 17) |
                                   ((uint32_t)(TC_M >> 4) << 24);
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) |
                                    ((uint32_t)(TC_M >> 4) << 24);
      int total = 0;
      for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
        run(lo, hi, sq, nch);
        total += nch;
      }
      auto issue_pv = [&](int t, int j) {
        const int b = j & 1;
        if (t == 0) lp::mbar_wait(&v_full[b], (j >> 1) & 1);
        lp::mbar_wait(&p_full[t][b], (j >> 1) & 1);
        fence_after();
        const uint32_t sv = lp::smem_u32(sm + C::OFF_V + b * C::KV_BYTES);
        const uint32_t sp = lp::smem_u32(sm + C::OFF_P + (t * 2 + b) * C::P_BYTES);
#pragma unroll
        for (int kk = 0; kk < PP_KEYS / 16; ++kk)
          umma(tmem + t * C::TILE_COLS + 128, desc_sw128(sp + kk * 32, 16, 1024),
               desc_sw128(sv + kk * 2048, PP_KEYS * 128, 1024), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        commit(&o_done[t]);
        if (t == 1) commit(&v_empty[b]);
      };
      auto issue_s = [&](int t, int it) {
        const int st = it & 1;
        if (it >= 2) lp::mbar_wait(&s_empty[t][st], ((it >> 1) - 1) & 1);
        fence_after();
        const uint32_t sk = lp::smem_u32(sm + C::OFF_K + st * C::KV_BYTES);
        const uint32_t sq = lp::smem_u32(sm + C::OFF_Q + t * C::Q_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma(tmem + t * C::TILE_COLS + st * PP_KEYS, desc_sw128(sq + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024),
               desc_sw128(sk + (kk >> 2) * (PP_KEYS * 128) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
        commit(&s_full[t][st]);
        if (t == 1) commit(&k_empty[st]);
      };
      // both tiles' S of chunk it + 1 go into the in-order tensor pipe before
      // the P V of chunk it (S is double-buffered per tile): each softmax
      // warpgroup finds its next S computed when it finishes a chunk, and the
      // two warpgroups never wait on each other (an earlier order, S1(it)
      // after P0(it - 1), chained them: ~2,870 cycles per chunk)
      lp::mbar_wait(&q_full, 0);
      if (total > 0) {
        lp::mbar_wait(&k_full[0], 0);
        TRACE(0, 0);
        issue_s(0, 0);
        issue_s(1, 0);
      }
      for (int it = 0; it < total; ++it) {
        if (it + 1 < total) {
          TRACE(10, it + 1);
          lp::mbar_wait(&k_full[(it + 1) & 1], ((it + 1) >> 1) & 1);
          TRACE(0, it + 1);
          issue_s(0, it + 1);
          issue_s(1, it + 1);
        }
        issue_pv(0, it);
        issue_pv(1, it);
      }
      if (total > 0) commit(&o_final);
    }
  } else if (warp <= 9) {
    // ---------------- softmax: warpgroup t owns Q tile t, thread = row ----------------
    constexpr float RESCALE = 8.0f;
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int i = t * a.R + r / a.G, g = r % a.G;    // token index within the CTA's 2R tokens
    const int prow = i < nvalid ? s_pos[i] : -1;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16) + t * C::TILE_COLS;
    float m_use = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
      run(lo, hi, sq, nch);
      const bool mine = i >= lo && i < hi;
      for (int c = 0; c < nch; ++c, ++it) {
        const int b = it & 1;
        lp::mbar_wait(&s_full[t][b], (it >> 1) & 1);
        fence_after();
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(2 + 4 * t, it);
        const int lim = mine ? prow - c * PP_KEYS : -1;     // keys 0..lim of this chunk are visible
        uint32_t v[64];
        ld32(trow + b * PP_KEYS, *reinterpret_cast<uint32_t(*)[32]>(v));
        ld32(trow + b * PP_KEYS + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[t][b]);
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(3 + 4 * t, it);
        // lazy row max (one thread owns the row: no exchange): P with the
        // current m and the raw max in one pass; only a move of m by more
        // than RESCALE (first visible chunk, rare after) recomputes P
        uint8_t* prow_s = sm + C::OFF_P + (t * 2 + b) * C::P_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
        auto move_m = [&](float m_row) {
          const bool move = m_row > m_use + RESCALE || (m_use == -INFINITY && m_row > -INFINITY);
          const float sc = (move && m_use != -INFINITY) ? exp2f(m_use - m_row) : 1.f;
          const bool resc = move && m_use != -INFINITY && it > 0;
          if (move) {
            l_run *= m_use == -INFINITY ? 0.f : sc;
            m_use = m_row;
          }
          if (__any_sync(0xffffffffu, resc)) {         // rescale O in TMEM (warp-collective ld/st)
            lp::mbar_wait(&o_done[t], (it - 1) & 1);   // P V of chunk it - 1 has landed
            fence_after();
#pragma unroll
            for (int cg = 0; cg < HD / 32; ++cg) {
              uint32_t o[32];
              ld32(trow + 128 + cg * 32, o);
              wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * sc);
              st32(trow + 128 + cg * 32, o);
            }
            wait_st();
          }
          return move;
        };
        float ls, mraw = -INFINITY;
        if (__any_sync(0xffffffffu, m_use == -INFINITY && lim >= 0)) {
          move_m(a.sl2 * softmax_row_max<PP_KEYS>(v, lim));
          if ((warp == 2 || warp == 6) && lane == 0) TRACE(4 + 4 * t, it);
          ls = softmax_write_p<PP_KEYS, false>(v, lim, a.sl2, m_use, prow_s, 0, r, mraw);
        } else {
          ls = softmax_write_p<PP_KEYS, true>(v, lim, a.sl2, m_use, prow_s, 0, r, mraw);
          if ((warp == 2 || warp == 6) && lane == 0) TRACE(4 + 4 * t, it);
          const bool moved = move_m(a.sl2 * mraw);
          if (__any_sync(0xffffffffu, moved)) {        // warp-collective rewrite, idempotent where m stayed
            const float ls_new = softmax_write_p<PP_KEYS, false>(v, lim, a.sl2, m_use, prow_s, 0, r, mraw);
            if (moved) ls = ls_new;
          }
        }
        l_run += ls;
        fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t][b]);
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(5 + 4 * t, it);
      }
    }
    if (it > 0) {
      lp::mbar_wait(&o_final, 0);
      fence_after();
    }
    const bool live = i < nvalid && l_run > 0.f;
    const float inv = live ? 1.0f / l_run : 0.f;
    __nv_bfloat16* orow = a.out + ((int64_t)(t0 + i) * a.H + kh * a.G + g) * HD;
#pragma unroll
    for (int cg = 0; cg < HD / 32; ++cg) {
      uint32_t o[32];
      ld32(trow + 128 + cg * 32, o);
      wait_ld();
      if (live) {
#pragma unroll
        for (int d = 0; d < 32; d += 8) {
          __nv_bfloat162 w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            w[e] = __floats2bfloat162_rn(__uint_as_float(o[d + 2 * e]) * inv, __uint_as_float(o[d + 2 * e + 1]) * inv);
          *reinterpret_cast<uint4*>(orow + cg * 32 + d) = *reinterpret_cast<const uint4*>(w);
        }
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

// ---------------------------------------------------------------------------
// FA4-layout variant (LP_ATTN_TC=7): two Q tiles per CTA over 128-key chunks
// with P kept in TMEM.  Tile t owns TMEM columns [256 t, 256 t + 256): S_t at
// [0, 128) (fp32), O_t at [128, 128 + HD); P_t (fp16 pairs) overwrites S_t's
// first 64 columns once the softmax has read them, and O_t += P_t V is a
// tcgen05.mma with the A operand read from TMEM (row = lane, 16 keys = 8
// columns per k-step; layout validated by tools/umma_ts_probe.cu), so the
// P V MMA moves only V through smem.  Smem: Q 2 x 32 KB + K / V rings 2 x 2 x
// 32 KB.  Per tile the chain is S_t(j) -> softmax_t(j) -> P_t(j) V -> S_t(j+1)
// (single S buffer: the in-order tensor pipe issues S_t(j+1) after the P V
// that reads P_t(j) from the same columns), and the other tile's MMAs run
// under each softmax.  Softmax: one thread per row, a max pass and an exp
// pass over the S columns (no exchange, no recompute); O is rescaled in TMEM
// without waiting (S_t(j) complete implies P_t(j-1) V complete).
constexpr int FA_THREADS = 352;   // warp 0 TMA Q + K, 1 MMA, 2-5 softmax tile 0, 6-9 tile 1, 10 TMA V

template <int HD>
struct FaCfg {
  static constexpr int ATOMS = HD / 64;
  static constexpr int Q_BYTES = TC_M * HD * 2;          // one tile
  static constexpr int KV_BYTES = TC_KEYS * HD * 2;      // one chunk
  static constexpr int OFF_Q = 0;                        // 2 tiles
  static constexpr int OFF_K = 2 * Q_BYTES;              // 2 stages
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;     // 2 stages
  static constexpr int BODY = OFF_V + 2 * KV_BYTES;
  static constexpr int TILE_COLS = 256;
};

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 32 scores -> 16 packed fp16 pairs of P (keys 0..lim visible); returns the sum
template <int POLY>
__device__ __forceinline__ float fa_exp32(const uint32_t (&v)[32], int lim, float sl2, float nm, uint32_t (&pk)[16]) {
  if (lim >= 31) {
    float2 ls2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    const float2 sl = make_float2(sl2, sl2), nm2 = make_float2(nm, nm);
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 x = ffma2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), sl, nm2);
      float2 p;
      if (((e >> 1) & 3) >= 4 - POLY) {      // POLY of every 4 key pairs on the FMA pipe
        p = exp2_poly2(x);
      } else {
        p.x = fast_exp2(x.x);
        p.y = fast_exp2(x.y);
      }
      ls2[(e >> 1) & 3] = fadd2(ls2[(e >> 1) & 3], p);
      const __half2 hv = __floats2half2_rn(p.x, p.y);
      pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    const float2 s01 = fadd2(ls2[0], ls2[1]), s23 = fadd2(ls2[2], ls2[3]);
    return (s01.x + s01.y) + (s23.x + s23.y);
  }
  float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    const float p0 = e <= lim ? fast_exp2(fmaf(__uint_as_float(v[e]), sl2, nm)) : 0.f;
    const float p1 = e + 1 <= lim ? fast_exp2(fmaf(__uint_as_float(v[e + 1]), sl2, nm)) : 0.f;
    ls[(e >> 1) & 3] += p0 + p1;
    const __half2 hv = __floats2half2_rn(p0, p1);
    pk[e >> 1] = *reinterpret_cast<const uint32_t*>(&hv);
  }
  return (ls[0] + ls[1]) + (ls[2] + ls[3]);
}

template <int HD, int POLY = 1>
__global__ void __launch_bounds__(FA_THREADS, 1)
    attention_fa_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const TcArgs a) {
  using C = FaCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  if (threadIdx.x == 0) {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if ((uint32_t)(sm - smem_raw) + C::BODY > dyn) __trap();   // launch_tc's pad assumption broken
  }
  __shared__ __align__(8) uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[2],
      o_final;
  __shared__ uint32_t tmem_base;
  __shared__ int s_pos[2 * TC_M];
  __shared__ int16_t s_seq[2 * TC_M];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 1-D grid over (tile, kv head), longest tiles of EVERY head first: the
  // block scheduler then fills the SMs in LPT order (a [tiles, heads] grid
  // launched head 0's short tiles before head 7's long ones)
  const int tile = (int)(gridDim.x / a.KV) - 1 - (int)(blockIdx.x / a.KV);
  const int kh = (int)(blockIdx.x % a.KV);
  const int R2 = 2 * a.R;
  const int t0 = tile * R2;

  if (threadIdx.x == 0) {
    lp::mbar_init(&q_full, 1);
    for (int b = 0; b < 2; ++b) {
      lp::mbar_init(&k_full[b], 1);
      lp::mbar_init(&k_empty[b], 1);
      lp::mbar_init(&v_full[b], 1);
      lp::mbar_init(&v_empty[b], 1);
      lp::mbar_init(&s_full[b], 1);
      lp::mbar_init(&p_full[b], 4);
    }
    lp::mbar_init(&o_final, 1);
    lp::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
    // Q and the first K / V chunk (chunk 0 of the tile's first sequence)
    // go out before the token table and the CTA barrier: the first S MMA's
    // operand latency overlaps the rest of the prologue
    lp::pdl_wait();
    lp::mbar_expect_tx(&q_full, 2 * C::Q_BYTES);
    for (int t = 0; t < 2; ++t)
      for (int at = 0; at < C::ATOMS; ++at)
        tma3d(sm + C::OFF_Q + t * C::Q_BYTES + at * ATOM, &tmQ, &q_full, at * 64, kh * a.G, t0 + t * a.R);
    const int row0 = a.seq[t0] * a.KV + kh;
    lp::mbar_expect_tx(&k_full[0], C::KV_BYTES);
    lp::mbar_expect_tx(&v_full[0], C::KV_BYTES);
    for (int at = 0; at < C::ATOMS; ++at) {
      tma3d(sm + C::OFF_K + at * (TC_KEYS * 128), &tmK, &k_full[0], at * 64, 0, row0);
      tma3d(sm + C::OFF_V + at * (TC_KEYS * 128), &tmV, &v_full[0], at * 64, 0, row0);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     lp::smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  lp::pdl_wait();
  lp::pdl_trigger();
  for (int i = threadIdx.x; i < R2; i += blockDim.x) {
    const bool v = t0 + i < a.T;
    s_pos[i] = v ? a.pos[t0 + i] : -1;
    s_seq[i] = v ? (int16_t)a.seq[t0 + i] : (int16_t)-1;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;
  auto run = [&](int lo, int& hi, int& sq, int& chunks) {
    sq = s_seq[lo];
    chunks = 0;
    for (hi = lo; hi < R2 && s_seq[hi] == sq; ++hi) chunks = max(chunks, (s_pos[hi] + TC_KEYS) / TC_KEYS);
  };
  const int nvalid = min(R2, a.T - t0);

  if (warp == 0 || warp == 10) {
    if (lane == 0) {
      const bool is_k = warp == 0;     // Q, K(0) and V(0) were issued in the prologue
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      const CUtensorMap* map = is_k ? &tmK : &tmV;
      uint8_t* base = sm + (is_k ? C::OFF_K : C::OFF_V);
      int it = 0;
      for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
        run(lo, hi, sq, nch);
        const int row = sq * a.KV + kh;
        for (int c = 0; c < nch; ++c, ++it) {
          if (it == 0) continue;
          const int st = it & 1;
          if (it >= 2) lp::mbar_wait(&empty[st], ((it >> 1) - 1) & 1);
          lp::mbar_expect_tx(&full[st], C::KV_BYTES);
          for (int at = 0; at < C::ATOMS; ++at)
            tma3d(base + st * C::KV_BYTES + at * (TC_KEYS * 128), map, &full[st], at * 64, c * TC_KEYS, row);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_KEYS >> 3) << 17) |
                                   ((uint32_t)(TC_M >> 4) << 24);          // bf16 x bf16, both K-major
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) |
                                    ((uint32_t)(TC_M >> 4) << 24);         // fp16: A (TMEM) K-major, B MN-major
      int total = 0;
      for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
        run(lo, hi, sq, nch);
        total += nch;
      }
      auto issue_s = [&](int t, int j) {
        const int st = j & 1;
        const uint32_t sk = lp::smem_u32(sm + C::OFF_K + st * C::KV_BYTES);
        const uint32_t sq = lp::smem_u32(sm + C::OFF_Q + t * C::Q_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma(tmem + t * C::TILE_COLS, desc_sw128(sq + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024),
               desc_sw128(sk + (kk >> 2) * (TC_KEYS * 128) + (kk & 3) * 32, 16, 1024), idesc_s, kk > 0);
        commit(&s_full[t]);
        if (t == 1) commit(&k_empty[st]);
      };
      auto issue_pv = [&](int t, int j) {
        const int b = j & 1;
        if (t == 0) lp::mbar_wait(&v_full[b], (j >> 1) & 1);
        lp::mbar_wait(&p_full[t], j & 1);
        fence_after();
        TRACE(1, j);
        const uint32_t sv = lp::smem_u32(sm + C::OFF_V + b * C::KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < TC_KEYS / 16; ++kk)
          umma_ts(tmem + t * C::TILE_COLS + 128, tmem + t * C::TILE_COLS + kk * 8,
                  desc_sw128(sv + kk * 2048, TC_KEYS * 128, 1024), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        if (t == 1) commit(&v_empty[b]);
      };
      lp::mbar_wait(&q_full, 0);
      if (total > 0) {
        lp::mbar_wait(&k_full[0], 0);
        fence_after();
        TRACE(0, 0);
        issue_s(0, 0);
        issue_s(1, 0);
      }
      for (int j = 0; j < total; ++j) {
        issue_pv(0, j);
        if (j + 1 < total) {
          lp::mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
          fence_after();
          TRACE(0, j + 1);
          issue_s(0, j + 1);           // after P_0(j) V in the in-order pipe: S_0 may overwrite P_0
        }
        issue_pv(1, j);
        if (j + 1 < total) issue_s(1, j + 1);
      }
      if (total > 0) commit(&o_final);
    }
  } else if (warp <= 9) {
    // ---------------- softmax: warpgroup t owns Q tile t, thread = row ----------------
    constexpr float RESCALE = 8.0f;
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int i = t * a.R + r / a.G, g = r % a.G;    // token index within the CTA's 2R tokens
    const int prow = i < nvalid ? s_pos[i] : -1;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16) + t * C::TILE_COLS;
    float m_use = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int lo = 0, hi, sq, nch; lo < nvalid; lo = hi) {
      run(lo, hi, sq, nch);
      const bool mine = i >= lo && i < hi;
      for (int c = 0; c < nch; ++c, ++it) {
        lp::mbar_wait(&s_full[t], it & 1);
        fence_after();
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(2 + 4 * t, it);
        const int lim = mine ? prow - c * TC_KEYS : -1;     // keys 0..lim of this chunk are visible
        // pass 1: the row max over the visible keys (one TMEM round trip)
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        {
          uint32_t v[128];
#pragma unroll
          for (int q = 0; q < 4; ++q) ld32(trow + q * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * q));
          wait_ld();
          if (lim >= 127) {
#pragma unroll
            for (int e = 0; e < 128; e += 2)
              mx4[(e >> 1) & 3] = fmax3(mx4[(e >> 1) & 3], __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
          } else if (lim >= 0) {
#pragma unroll
            for (int e = 0; e < 128; ++e)
              if (e <= lim) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(v[e]));
          }
        }
        const float m_row = a.sl2 * fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(3 + 4 * t, it);
        const bool move = m_row > m_use + RESCALE || (m_use == -INFINITY && m_row > -INFINITY);
        const float sc = (move && m_use != -INFINITY) ? exp2f(m_use - m_row) : 1.f;
        const bool resc = move && m_use != -INFINITY && it > 0;
        if (move) {
          l_run *= m_use == -INFINITY ? 0.f : sc;
          m_use = m_row;
        }
        if (__any_sync(0xffffffffu, resc)) {   // O_t is stable here: S_t(it) done => P_t(it-1) V done
#pragma unroll
          for (int cg = 0; cg < HD / 32; ++cg) {
            uint32_t o[32];
            ld32(trow + 128 + cg * 32, o);
            wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * sc);
            st32(trow + 128 + cg * 32, o);
          }
        }
        // pass 2: P = exp2(S sl2 - m) in fp16 over S's first 64 columns (each
        // 32-key quarter's P lands on columns already read); the load of
        // quarter q + 1 is in flight while quarter q computes
        const float nm = -m_use;
        float ls = 0.f;
        uint32_t va[32], vb[32], pk[32];
        // P of quarter q into pk[16 h .. 16 h + 15]
        auto quarter_p = [&](const uint32_t (&vq)[32], int q, int h) {
          uint32_t (&ph)[16] = *reinterpret_cast<uint32_t(*)[16]>(pk + 16 * h);
          if (lim - q * 32 < 0) {
#pragma unroll
            for (int e = 0; e < 16; ++e) ph[e] = 0u;
          } else {
            ls += fa_exp32<POLY>(vq, lim - q * 32, a.sl2, nm, ph);
          }
        };
        ld32(trow, va);
        ld32(trow + 32, vb);
        wait_ld32(va);
        wait_ld32(vb);
        quarter_p(va, 0, 0);
        ld32(trow + 64, va);
        quarter_p(vb, 1, 1);
        st32(trow, pk);                  // P keys 0..63 -> columns 0..31 (S keys 0..31, read)
        wait_ld32(va);
        ld32(trow + 96, vb);
        quarter_p(va, 2, 0);
        wait_ld32(vb);
        quarter_p(vb, 3, 1);
        st32(trow + 32, pk);             // P keys 64..127 -> columns 32..63 (S keys 32..63, read)
        l_run += ls;
        wait_st();
        fence_before();
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(4 + 4 * t, it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        if ((warp == 2 || warp == 6) && lane == 0) TRACE(5 + 4 * t, it);
      }
    }
    if (it > 0) {
      lp::mbar_wait(&o_final, 0);
      fence_after();
    }
    const bool live = i < nvalid && l_run > 0.f;
    const float inv = live ? 1.0f / l_run : 0.f;
    __nv_bfloat16* orow = a.out + ((int64_t)(t0 + i) * a.H + kh * a.G + g) * HD;
#pragma unroll
    for (int cg = 0; cg < HD / 32; ++cg) {
      uint32_t o[32];
      ld32(trow + 128 + cg * 32, o);
      wait_ld();
      if (live) {
#pragma unroll
        for (int d = 0; d < 32; d += 8) {
          __nv_bfloat162 w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            w[e] = __floats2bfloat162_rn(__uint_as_float(o[d + 2 * e]) * inv, __uint_as_float(o[d + 2 * e + 1]) * inv);
          *reinterpret_cast<uint4*>(orow + cg * 32 + d) = *reinterpret_cast<const uint4*>(w);
        }
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

template <int HD>
int launch_tc(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos, const int32_t* seq,
              int T, int H, int KV, int64_t max_len, float scale, void* out, cudaStream_t s) {
  using C = TcCfg<HD>;
  const int G = H / KV;
  const int R = TC_M / G;
  // LP_ATTN_TC selects the variant (A/B tables: profiles/r02/attn_prefill_*):
  //   7 (default) FA4 layout: two Q tiles per CTA, 128-key chunks, P kept in
  //     TMEM as the P V MMA's A operand, one softmax thread per row, LPT
  //     launch order: 8B 1 x 2048 rows 82.5 -> 57 us, 2 x 4096 439 -> 335 us,
  //     8 x 512 84 -> 66 us; 70B 2 x 4096 847 -> 644 us (vs the eager kernel);
  //   3 one Q tile per CTA, lazy row max (exchanged after the exp pass),
  //     packed FFMA2/FADD2/FMNMX3 math, one key pair in four on the FMA-pipe
  //     exp2 (80.2 / 418 / 86 us);
  //   1 the eager one-tile kernel (row max first, partner half streamed);
  //   (measured and dropped: variant 3 with four warps per row quarter, or
  //   with 0 / 2 of 4 key pairs on the FMA pipe: attn_prefill_lazy_ab.txt)
  //   2 the 64-key ping-pong kernel (P in smem; its N = 64 S MMAs are
  //     smem-bound).
  static const int variant_env = [] {
    const char* e = getenv("LP_ATTN_TC");
    return e ? atoi(e) : 7;
  }();
  // groups of <= 2 heads (R >= 64 tokens per tile) with short caches: the FA
  // kernel's 2R-token CTAs would span several prompts (each walking the
  // others' chunks masked), so the one-tile kernel runs them (MHA 16 x 128
  // tokens: 78 vs 103 us, profiles/r02/attn_prefill_mha_short.txt)
  const int variant = (variant_env == 7 && G <= 2 && max_len <= 512) ? 1 : variant_env;
  const uint32_t kbox = variant == 2 ? PP_KEYS : TC_KEYS;   // 7 and the one-tile kernels: 128-key chunks
  CUtensorMap mq, mk, mv;
  const uint64_t rows = (uint64_t)1 << 24;   // sequence x kv-head rows of the caches (unbounded here)
  if (map3d(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, q, HD, H, T, (uint64_t)HD * 2, (uint64_t)H * HD * 2, G, R)) return -1;
  if (map3d(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, k_cache, HD, max_len, rows, (uint64_t)HD * 2,
            (uint64_t)max_len * HD * 2, kbox, 1))
    return -1;
  if (map3d(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, v_cache, HD, max_len, rows, (uint64_t)HD * 2,
            (uint64_t)max_len * HD * 2, kbox, 1))
    return -1;
  static uint64_t attr = 0;
  int dev = 0;
  LP_CUDA(cudaGetDevice(&dev));
  // dynamic bytes per instantiation: body + 1024-B alignment pad after the static smem
  auto smem_for = [](auto kern) -> int {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return -1;
    const int bytes = C::BODY + (int)((1024 - fa.sharedSizeBytes % 1024) % 1024);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return -1;
    return bytes;
  };
  static int tc_smem[2] = {0, 0};
  if (!(attr >> dev & 1)) {
    tc_smem[0] = smem_for(attention_tc_kernel<HD, 2, false>);
    tc_smem[1] = smem_for(attention_tc_kernel<HD, 2, true>);
    LP_CHECK(tc_smem[0] > 0 && tc_smem[1] > 0, "attention_tc: smem attributes: %s",
             cudaGetErrorString(cudaGetLastError()));
    attr |= 1ull << dev;
  }
  static long long* trace = [] {     // device memory: a managed buffer's page faults distort the stamps
    long long* t = nullptr;
    if (getenv("LP_ATTN_TRACE")) {
      cudaMalloc(&t, 64 * 16 * sizeof(long long));
      cudaMemset(t, 0, 64 * 16 * sizeof(long long));
    }
    return t;
  }();
  TcArgs args{pos, seq, (__nv_bfloat16*)out, T, H, KV, G, R, scale * 1.4426950408889634f, trace};
  if (variant == 7) {
    using F = FaCfg<HD>;
    if (trace) LP_CUDA(cudaMemset(trace, 0, 64 * 16 * sizeof(long long)));
    static int fa_smem[3] = {0, 0, 0};
    static uint64_t fattr = 0;
    auto fa_attr = [](auto kern) -> int {
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return -1;
      const int bytes = F::BODY + (int)((1024 - fa.sharedSizeBytes % 1024) % 1024);
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return -1;
      return bytes;
    };
    if (!(fattr >> dev & 1)) {
      fa_smem[0] = fa_attr(attention_fa_kernel<HD, 1>);
      fa_smem[1] = fa_attr(attention_fa_kernel<HD, 0>);
      fa_smem[2] = fa_attr(attention_fa_kernel<HD, 2>);
      LP_CHECK(fa_smem[0] > 0 && fa_smem[1] > 0 && fa_smem[2] > 0, "attention_fa: smem attributes: %s",
               cudaGetErrorString(cudaGetLastError()));
      fattr |= 1ull << dev;
    }
    // LP_ATTN_FA_POLY: key pairs in four on the FMA-pipe exp2 (1 default; 0, 2 for A/B)
    static const int poly = [] {
      const char* e = getenv("LP_ATTN_FA_POLY");
      return e ? atoi(e) : 1;
    }();
    const dim3 grid((unsigned)((T + 2 * R - 1) / (2 * R) * KV));
    if (poly == 0)
      LP_CUDA(lp::launch(attention_fa_kernel<HD, 0>, grid, dim3(FA_THREADS), fa_smem[1], s, mq, mk, mv, args));
    else if (poly == 2)
      LP_CUDA(lp::launch(attention_fa_kernel<HD, 2>, grid, dim3(FA_THREADS), fa_smem[2], s, mq, mk, mv, args));
    else
      LP_CUDA(lp::launch(attention_fa_kernel<HD, 1>, grid, dim3(FA_THREADS), fa_smem[0], s, mq, mk, mv, args));
    if (trace) {
      static long long h[64 * 16];
      LP_CUDA(cudaStreamSynchronize(s));
      LP_CUDA(cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost));
      for (int it = 0; it < 64 && (it == 0 || h[it * 16 + 2]); ++it) {
        const long long* t = h + it * 16;
        fprintf(stderr, "fa chunk %2d: K_ready %7lld PV1_issue %7lld | tile0 S_ready %7lld max %+5lld exp %+5lld arrive "
                "%+5lld | tile1 S_ready %7lld max %+5lld exp %+5lld arrive %+5lld\n", it, t[0] - h[0],
                t[1] ? t[1] - h[0] : 0, t[2] - h[0], t[3] - t[2], t[4] - t[3], t[5] - t[4], t[6] - h[0], t[7] - t[6],
                t[8] - t[7], t[9] - t[8]);
      }
    }
    return 0;
  }
  if (variant == 2) {
    using P = PpCfg<HD>;
    if (trace) LP_CUDA(cudaMemset(trace, 0, 64 * 16 * sizeof(long long)));
    static uint64_t pattr = 0;
    if (!(pattr >> dev & 1)) {
      LP_CUDA(cudaFuncSetAttribute(attention_pp_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM));
      pattr |= 1ull << dev;
    }
    const dim3 grid((unsigned)((T + 2 * R - 1) / (2 * R) * KV));
    LP_CUDA(lp::launch(attention_pp_kernel<HD>, grid, dim3(PP_THREADS), P::SMEM, s, mq, mk, mv, args));
    if (trace) {
      static long long h[64 * 16];
      LP_CUDA(cudaStreamSynchronize(s));
      LP_CUDA(cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost));
      for (int it = 0; it < 64 && h[it * 16]; ++it) {
        const long long* t = h + it * 16;
        fprintf(stderr, "pp chunk %2d: mma_at %7lld K_ready %7lld | tile0 S_ready %7lld ld %+5lld exp %+5lld P %+5lld | "
                "tile1 S_ready %7lld ld %+5lld exp %+5lld P %+5lld\n", it, t[10] ? t[10] - h[0] : 0, t[0] - h[0],
                t[2] - h[0], t[3] - t[2], t[4] - t[3], t[5] - t[4], t[6] - h[0], t[7] - t[6], t[8] - t[7], t[9] - t[8]);
      }
    }
    return 0;
  }
  const dim3 grid((unsigned)((T + R - 1) / R * KV));
  if (variant == 1)
    LP_CUDA(lp::launch(attention_tc_kernel<HD, 2, false>, grid, dim3(11 * 32), tc_smem[0], s, mq, mk, mv, args));
  else
    LP_CUDA(lp::launch(attention_tc_kernel<HD, 2, true>, grid, dim3(11 * 32), tc_smem[1], s, mq, mk, mv, args));
  if (trace) {
    static long long h[64 * 16];
    LP_CUDA(cudaStreamSynchronize(s));
    LP_CUDA(cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost));
    const long long* tr0 = h;
    for (int it = 0; it < 64 && h[it * 16]; ++it) {
      const long long* t = h + it * 16;
      fprintf(stderr, "chunk %2d: S_issue %7lld PV_issue %7lld | sm: S_ready %7lld S_loaded %+6lld max %+6lld "
              "P_written %+6lld arrive %+6lld | K_issue %7lld V_issue %7lld K_landed %7lld\n", it, t[0] - tr0[0],
              t[1] - tr0[0], t[2] - tr0[0], t[3] - t[2], t[6] - t[3], t[4] - t[6], t[5] - t[4], t[7] - tr0[0],
              t[8] - tr0[0], t[9] - tr0[0]);
    }
    LP_CUDA(cudaMemset(trace, 0, sizeof(h)));
  }
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
