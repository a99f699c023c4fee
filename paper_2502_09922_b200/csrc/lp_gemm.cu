// Llama linear layers on the 5th-gen tensor cores: tcgen05.mma with the
// accumulator in TMEM, operands staged by TMA (128B swizzle), warp-specialised.
//
//   Y[t, n] (epilogue) = sum_k X[t, k] * W[n, k]        X: [T, K] bf16, W: [N, K] bf16
//
// "Swap-AB": the weight tile (128 output features x 64 k) is the MMA's A
// operand (M = 128 TMEM lanes) and the token tile is B (N = BT tokens), so the
// same kernel serves decode (T = a few tokens, weight streaming bound) and
// prefill (T = hundreds, tensor bound).  Both operands are K-major, loaded by
// TMA boxes of 64 bf16 (= one 128-byte swizzle atom) into a STAGES-deep smem
// ring guarded by full/empty mbarriers.
//
//   warp 0  : TMA producer (one elected lane)
//   warp 1  : TMEM allocator + MMA issuer (one elected lane issues
//             tcgen05.mma.cta_group::1.kind::f16, commits to mbarriers)
//   warps 2-5: epilogue — tcgen05.ld 32x32b -> registers -> global, fused:
//             EPI_ADD_F32   out_f32[t,n] += acc    (residual add; split-K safe)
//             EPI_STORE_F32 out_f32[t,n]  = acc    (logits)
//             EPI_SWIGLU    out_bf16[t,n] = silu(acc_gate) * acc_up  (two
//                           accumulators: gate and up weights share the B tile)
//
// Grid: x = 128-row weight tiles, y = token tiles, z = K splits.
#include "lp_common.cuh"
#include "../../include/lambdapipe.h"
#include <cuda.h>
#include <stdlib.h>
#include <mutex>
#include <unordered_map>

namespace {

constexpr int BM = 128;       // weight rows per CTA (TMEM lanes)
constexpr int BK = 64;        // k per stage = one 128B swizzle atom of bf16
constexpr int UMMA_K = 16;    // k per tcgen05.mma (kind::f16)
constexpr int THREADS = 192;  // 6 warps

enum { EPI_ADD_F32 = 0, EPI_STORE_F32 = 1, EPI_SWIGLU = 2 };

struct GemmArgs {
  void* out;
  int64_t ldo;        // elements between consecutive tokens in out
  int n_rows;         // N (valid weight rows)
  int tokens;         // T (valid tokens)
  int k_blocks;       // ceil(K / BK)
  int kb_per_split;   // k blocks per z-split
  int atomic;         // EPI_ADD with split-K: red.add; without: plain read-modify-write
  int tiles_n, tiles_t, splits;   // persistent kernel tile space
  int streamk;        // CTA-pair kernel: equal k-block spans per cluster (EPI_ADD only, splits = 1)
};

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B canonical layout: 8-row groups 1024 B apart (SBO),
  // LBO unused (1), descriptor version 1 (sm_100), layout type 2 (128B swizzle)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N>
__host__ __device__ constexpr uint32_t idesc_bf16_f32() {
  // c_format F32 [4,6), a/b format BF16 [7,10)/[10,13), K-major A/B, N>>3 at 17, M>>4 at 24
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(lp::smem_u32(smem_dst)),
      "l"(map), "r"(lp::smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   lp::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int BT, int EPI>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;              // 16 KiB
  static constexpr int B_BYTES = BT * BK * 2;
  static constexpr int NA = (EPI == EPI_SWIGLU) ? 2 : 1;   // weight tiles per stage
  static constexpr int STAGE_BYTES = NA * A_BYTES + B_BYTES;
  // <= 6 stages: small decode tiles (18-34 KiB/stage) then fit two CTAs per SM,
  // which overlaps one CTA's prologue/epilogue with the other's streaming —
  // measured faster than a single 12-stage CTA (profiles/gemm_split_sweep_r01.txt)
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int ACC_COLS = NA * BT;
  static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128
                                   : ACC_COLS <= 256 ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;  // + alignment slack
};

template <int BT, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmW2,
                const __grid_constant__ CUtensorMap tmX, const GemmArgs args) {
  using C = Cfg<BT, EPI>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[C::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[C::STAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base_smem;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BM;
  const int t0 = blockIdx.y * BT;
  const int kb0 = blockIdx.z * args.kb_per_split;
  const int kb1 = min(args.k_blocks, kb0 + args.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      lp::mbar_init(&full_bar[s], 1);
      lp::mbar_init(&empty_bar[s], 1);
    }
    lp::mbar_init(&done_bar, 1);
    lp::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     lp::smem_u32(&tmem_base_smem)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    if (EPI == EPI_SWIGLU) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW2) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;

  if (threadIdx.x == 0) lp::pdl_trigger();
  if (warp == 0 && lane == 0 && nkb > 0) {
    // ---------------- TMA producer ----------------
    // weights do not depend on the previous kernel: the first ring's worth of
    // weight tiles is requested before waiting for it (PDL), activations after
    const int pre = nkb < C::STAGES ? nkb : C::STAGES;
    for (int i = 0; i < pre; ++i) {
      uint8_t* st = smem + i * C::STAGE_BYTES;
      lp::mbar_expect_tx(&full_bar[i], C::STAGE_BYTES);
      const int kc = (kb0 + i) * BK;
      tma_load_2d(st, &tmW, &full_bar[i], kc, n0);
      if (EPI == EPI_SWIGLU) tma_load_2d(st + C::A_BYTES, &tmW2, &full_bar[i], kc, n0);
    }
    lp::pdl_wait();
    for (int i = 0; i < pre; ++i)
      tma_load_2d(smem + i * C::STAGE_BYTES + C::NA * C::A_BYTES, &tmX, &full_bar[i], (kb0 + i) * BK, t0);
    for (int i = pre; i < nkb; ++i) {
      const int s = i % C::STAGES;
      lp::mbar_wait(&empty_bar[s], ((i / C::STAGES) & 1) ^ 1);
      uint8_t* st = smem + s * C::STAGE_BYTES;
      lp::mbar_expect_tx(&full_bar[s], C::STAGE_BYTES);
      const int kc = (kb0 + i) * BK;
      tma_load_2d(st, &tmW, &full_bar[s], kc, n0);
      if (EPI == EPI_SWIGLU) tma_load_2d(st + C::A_BYTES, &tmW2, &full_bar[s], kc, n0);
      tma_load_2d(st + C::NA * C::A_BYTES, &tmX, &full_bar[s], kc, t0);
    }
  } else if (warp == 1 && lane == 0 && nkb > 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_bf16_f32<BT>();
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::STAGES;
      lp::mbar_wait(&full_bar[s], (i / C::STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = lp::smem_u32(smem + s * C::STAGE_BYTES);
      const uint32_t sb = sa + C::NA * C::A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / UMMA_K; ++kk) {
        const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
        // +32 bytes per 16-element k step inside the 128B swizzle atom
        umma_bf16(tmem, smem_desc_sw128(sa + kk * 32), smem_desc_sw128(sb + kk * 32), idesc, acc);
        if (EPI == EPI_SWIGLU)
          umma_bf16(tmem + BT, smem_desc_sw128(sa + C::A_BYTES + kk * 32), smem_desc_sw128(sb + kk * 32), idesc,
                    acc);
      }
      umma_commit(&empty_bar[s]);   // smem slot free once these MMAs have read it
    }
    umma_commit(&done_bar);         // accumulator complete
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int n = n0 + row;
    if (nkb > 0) {
      lp::mbar_wait(&done_bar, 0);
      tc_fence_after();
    } else {
      lp::pdl_wait();
    }
    constexpr int CH = BT < 32 ? BT : 32;
    for (int c = 0; c < BT; c += CH) {
      uint32_t v[32], u[32];
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + c;
      if (nkb > 0) {
        if (CH == 32) tmem_ld32(taddr, v); else tmem_ld16(taddr, v);
        if (EPI == EPI_SWIGLU) {
          if (CH == 32) tmem_ld32(taddr + BT, u); else tmem_ld16(taddr + BT, u);
        }
        tmem_wait_ld();
      } else {
        for (int j = 0; j < 32; ++j) v[j] = u[j] = 0;
      }
      if (n < args.n_rows) {
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int t = t0 + c + j;
          if (t >= args.tokens) break;
          const float a = __uint_as_float(v[j]);
          if (EPI == EPI_ADD_F32) {
            float* o = (float*)args.out + (int64_t)t * args.ldo + n;
            if (args.atomic) atomicAdd(o, a); else *o += a;
          } else if (EPI == EPI_STORE_F32) {
            ((float*)args.out)[(int64_t)t * args.ldo + n] = a;
          } else {
            const float up = __uint_as_float(u[j]);
            const float act = a / (1.0f + __expf(-a)) * up;
            ((__nv_bfloat16*)args.out)[(int64_t)t * args.ldo + n] = __float2bfloat16_rn(act);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Persistent variant (prefill, T > 64): grid = #SMs, each CTA walks output
// tiles (weight tile fastest, so neighbouring CTAs share the token tile in
// L2).  Two TMEM accumulators: the MMA warp fills buffer (i & 1) while the
// epilogue warps drain buffer ((i - 1) & 1), so the epilogue of one tile
// overlaps the MMAs of the next; the smem ring runs across tile boundaries.

template <int BT, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_persistent_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmW2,
                           const __grid_constant__ CUtensorMap tmX, const GemmArgs args) {
  using C = Cfg<BT, EPI>;
  // two TMEM accumulator buffers (epilogue of tile i overlaps the MMAs of
  // tile i+1) when they fit the 512 columns; SwiGLU at BT = 256 holds gate and
  // up accumulators of 256 columns each, so it runs single-buffered — still
  // faster than BT = 128, whose 128x128x16 MMAs need 128 B/clk of smem operand
  // reads (the SM's whole smem bandwidth) against 96 B/clk at N = 256
  constexpr int NBUF = 2 * C::ACC_COLS <= 512 ? 2 : 1;
  constexpr int TC = NBUF * C::ACC_COLS;
  constexpr int TCOLS = TC <= 32 ? 32 : TC <= 64 ? 64 : TC <= 128 ? 128 : TC <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[C::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[C::STAGES];
  __shared__ __align__(8) uint64_t tfull[2];
  __shared__ __align__(8) uint64_t tempty[2];
  __shared__ uint32_t tmem_base_smem;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total = args.tiles_n * args.tiles_t * args.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      lp::mbar_init(&full_bar[s], 1);
      lp::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      lp::mbar_init(&tfull[a], 1);
      lp::mbar_init(&tempty[a], 4);     // one arrive per epilogue warp
    }
    lp::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     lp::smem_u32(&tmem_base_smem)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    if (EPI == EPI_SWIGLU) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW2) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;

  auto tile_coords = [&](int tile, int& n0, int& t0, int& kb0, int& nkb) {
    const int nt = tile % args.tiles_n;
    const int rest = tile / args.tiles_n;
    const int tt = rest % args.tiles_t;
    const int z = rest / args.tiles_t;
    n0 = nt * BM;
    t0 = tt * BT;
    kb0 = z * args.kb_per_split;
    nkb = min(args.k_blocks, kb0 + args.kb_per_split) - kb0;
  };

  if (threadIdx.x == 0) lp::pdl_trigger();
  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    lp::pdl_wait();
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int n0, t0, kb0, nkb;
      tile_coords(tile, n0, t0, kb0, nkb);
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % C::STAGES;
        lp::mbar_wait(&empty_bar[s], ((it / C::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        lp::mbar_expect_tx(&full_bar[s], C::STAGE_BYTES);
        const int kc = (kb0 + i) * BK;
        tma_load_2d(st, &tmW, &full_bar[s], kc, n0);
        if (EPI == EPI_SWIGLU) tma_load_2d(st + C::A_BYTES, &tmW2, &full_bar[s], kc, n0);
        tma_load_2d(st + C::NA * C::A_BYTES, &tmX, &full_bar[s], kc, t0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_bf16_f32<BT>();
    int it = 0, li = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++li) {
      int n0, t0, kb0, nkb;
      tile_coords(tile, n0, t0, kb0, nkb);
      const int a = li % NBUF;
      lp::mbar_wait(&tempty[a], ((li / NBUF) & 1) ^ 1);  // epilogue drained this accumulator
      tc_fence_after();
      const uint32_t acc_base = tmem + a * C::ACC_COLS;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % C::STAGES;
        lp::mbar_wait(&full_bar[s], (it / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = lp::smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t sb = sa + C::NA * C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          umma_bf16(acc_base, smem_desc_sw128(sa + kk * 32), smem_desc_sw128(sb + kk * 32), idesc, acc);
          if (EPI == EPI_SWIGLU)
            umma_bf16(acc_base + BT, smem_desc_sw128(sa + C::A_BYTES + kk * 32), smem_desc_sw128(sb + kk * 32),
                      idesc, acc);
        }
        umma_commit(&empty_bar[s]);
      }
      umma_commit(&tfull[a]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int li = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++li) {
      int n0, t0, kb0, nkb;
      tile_coords(tile, n0, t0, kb0, nkb);
      const int a = li % NBUF;
      lp::mbar_wait(&tfull[a], (li / NBUF) & 1);
      tc_fence_after();
      const int n = n0 + row;
      constexpr int CH = BT < 32 ? BT : 32;
      for (int c = 0; c < BT; c += CH) {
        uint32_t v[32], u[32];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + a * C::ACC_COLS + c;
        if (CH == 32) tmem_ld32(taddr, v); else tmem_ld16(taddr, v);
        if (EPI == EPI_SWIGLU) {
          if (CH == 32) tmem_ld32(taddr + BT, u); else tmem_ld16(taddr + BT, u);
        }
        tmem_wait_ld();
        if (n < args.n_rows) {
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = t0 + c + j;
            if (t >= args.tokens) break;
            const float x = __uint_as_float(v[j]);
            if (EPI == EPI_ADD_F32) {
              float* o = (float*)args.out + (int64_t)t * args.ldo + n;
              if (args.atomic) atomicAdd(o, x); else *o += x;
            } else if (EPI == EPI_STORE_F32) {
              ((float*)args.out)[(int64_t)t * args.ldo + n] = x;
            } else {
              const float up = __uint_as_float(u[j]);
              ((__nv_bfloat16*)args.out)[(int64_t)t * args.ldo + n] =
                  __float2bfloat16_rn(x / (1.0f + __expf(-x)) * up);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lp::smem_u32(&tempty[a])) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant for prefill (tcgen05.mma.cta_group::2).  At 128 x BT x 16
// per CTA the MMA reads 96 B/clk of smem operands while TMA writes another
// 96 B/clk into the same smem — more than the SM's smem bandwidth, which is
// what held the single-CTA kernel's tensor pipe at ~65 % (ncu,
// gemm_prefill_qkv_T4096_full_r01.csv).  A cluster of two CTAs on one TPC
// computes a 256 x BT tile: each CTA stages its own 128 weight rows and HALF
// of the token tile (BT/2 rows); the leader's single thread issues
// M = 256 MMAs that read both CTAs' smem, and every CTA's TMEM receives its
// 128 rows x BT accumulator — per-SM smem traffic per MMA is halved for B.
//   * both CTAs' TMA loads complete on the LEADER's full barrier
//     (.cta_group::2 TMA, barrier address mapped to rank 0); the leader
//     expects the pair's bytes;
//   * the leader's commits arrive on both CTAs' empty / accumulator-full
//     barriers (multicast::cluster, mask 0b11);
//   * both CTAs' epilogue warps release the accumulator on the leader's
//     tempty barrier (remote mbarrier.arrive.release.cluster).
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(lp::smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(lp::smem_u32(smem_dst)),
      "l"(map), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                           uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          lp::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
template <int N>
__host__ __device__ constexpr uint32_t idesc2_bf16_f32() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

template <int BT, int EPI>
struct Cfg2 {
  static constexpr int A_BYTES = BM * BK * 2;                 // this CTA's 128 weight rows
  static constexpr int B_BYTES = (BT / 2) * BK * 2;           // this CTA's half of the token tile
  static constexpr int NA = (EPI == EPI_SWIGLU) ? 2 : 1;
  static constexpr int STAGE_BYTES = NA * A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int ACC_COLS = NA * BT;
  static constexpr int NBUF = 2 * ACC_COLS <= 512 ? 2 : 1;
  static constexpr int TC = NBUF * ACC_COLS;
  static constexpr int TCOLS = TC <= 32 ? 32 : TC <= 64 ? 64 : TC <= 128 ? 128 : TC <= 256 ? 256 : 512;
  // SwiGLU epilogue transpose tiles: per epilogue warp 32 tokens x 32 rows
  // bf16, rows padded to 80 B (conflict-free 16-byte reads)
  static constexpr int XPOSE_PITCH = 40;                      // bf16 elements per token row
  static constexpr int XPOSE_BYTES = (EPI == EPI_SWIGLU) ? 8 * 32 * XPOSE_PITCH * 2 : 0;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + XPOSE_BYTES;
};

// 8 epilogue warps (two per TMEM lane quarter, alternating 32-token chunks):
// the single-buffered SwiGLU accumulator's drain is on the critical path, and
// one warp per SM sub-partition could not hide its TMEM-load and exp latency
constexpr int PAIR_THREADS = 320;

template <int BT, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PAIR_THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmW2,
                     const __grid_constant__ CUtensorMap tmXh, const GemmArgs args) {
  using C = Cfg2<BT, EPI>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[C::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[C::STAGES];
  __shared__ __align__(8) uint64_t tfull[2];
  __shared__ __align__(8) uint64_t tempty[2];
  __shared__ uint32_t tmem_base_smem;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int tiles_n2 = (args.tiles_n + 1) >> 1;            // 256-row pair tiles
  const int total = tiles_n2 * args.tiles_t * args.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      lp::mbar_init(&full_bar[s], 1);
      lp::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      lp::mbar_init(&tfull[a], 1);
      lp::mbar_init(&tempty[a], 16);    // 8 epilogue warps x 2 CTAs
    }
    lp::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     lp::smem_u32(&tmem_base_smem)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmXh) : "memory");
    if (EPI == EPI_SWIGLU) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW2) : "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;

  auto tile_coords = [&](int tile, int& n0, int& t0, int& kb0, int& nkb) {
    const int nt = tile % tiles_n2;
    const int rest = tile / tiles_n2;
    const int tt = rest % args.tiles_t;
    const int z = rest / args.tiles_t;
    n0 = nt * 2 * BM + (int)rank * BM;
    t0 = tt * BT;
    kb0 = z * args.kb_per_split;
    nkb = min(args.k_blocks, kb0 + args.kb_per_split) - kb0;
  };

  // work items of this cluster.  Default: whole tiles (x K splits) dealt
  // round-robin.  Stream-K tail (args.streamk; accumulating epilogue only):
  // the full waves stay round-robin (neighbouring clusters share operand
  // tiles in L2), and only the k-blocks of the last partial wave's tiles are
  // laid end to end and cut into nclusters equal spans (QKV T = 4096: 384
  // pair tiles = 5 waves of 74 + 14 tiles, i.e. 12 k-blocks per cluster
  // instead of a sixth round); a tile cut between clusters is summed by the
  // red.add epilogue.  Positions p are k-block indices (tile * KB + kb).
  const int64_t KB = args.k_blocks;
  const int full = args.streamk ? (total / nclusters) * nclusters : total;
  const int64_t p_full = (int64_t)full * KB;
  const int64_t w_tail = (int64_t)(total - full) * KB;
  const int64_t sk_beg = p_full + w_tail * cid / nclusters, sk_end = p_full + w_tail * (cid + 1) / nclusters;
  const int64_t p_first = !args.streamk ? (int64_t)cid : (cid < full ? (int64_t)cid * KB : sk_beg);
  auto valid = [&](int64_t p) { return args.streamk ? p < sk_end : p < (int64_t)total; };
  auto decode = [&](int64_t p, int& n0, int& t0, int& kb0, int& nkb) {
    if (args.streamk) {
      int d0, d1;
      tile_coords((int)(p / KB), n0, t0, d0, d1);
      kb0 = (int)(p % KB);
      nkb = p < p_full ? (int)KB : (int)min((int64_t)(KB - kb0), sk_end - p);
    } else {
      tile_coords((int)p, n0, t0, kb0, nkb);
    }
  };
  auto advance = [&](int64_t p, int nkb) -> int64_t {
    if (!args.streamk) return p + nclusters;
    if (p < p_full) {
      const int64_t q = p + (int64_t)nclusters * KB;
      return q < p_full ? q : sk_beg;
    }
    return p + nkb;
  };

  if (threadIdx.x == 0) lp::pdl_trigger();
  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    lp::pdl_wait();
    int it = 0;
    for (int64_t p = p_first; valid(p);) {
      int n0, t0, kb0, nkb;
      decode(p, n0, t0, kb0, nkb);
      p = advance(p, nkb);
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % C::STAGES;
        lp::mbar_wait(&empty_bar[s], ((it / C::STAGES) & 1) ^ 1);
        if (rank == 0) lp::mbar_expect_tx(&full_bar[s], 2 * C::STAGE_BYTES);
        const uint32_t lbar = mapa_rank(lp::smem_u32(&full_bar[s]), 0);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        const int kc = (kb0 + i) * BK;
        tma_load_2d_pair(st, &tmW, lbar, kc, n0);
        if (EPI == EPI_SWIGLU) tma_load_2d_pair(st + C::A_BYTES, &tmW2, lbar, kc, n0);
        tma_load_2d_pair(st + C::NA * C::A_BYTES, &tmXh, lbar, kc, t0 + (int)rank * (BT / 2));
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    constexpr uint32_t idesc = idesc2_bf16_f32<BT>();
    int it = 0, li = 0;
    for (int64_t p = p_first; valid(p); ++li) {
      int n0, t0, kb0, nkb;
      decode(p, n0, t0, kb0, nkb);
      p = advance(p, nkb);
      const int a = li % C::NBUF;
      mbar_wait_cluster(&tempty[a], ((li / C::NBUF) & 1) ^ 1);   // both CTAs drained this accumulator
      tc_fence_after();
      const uint32_t acc_base = tmem + a * C::ACC_COLS;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % C::STAGES;
        lp::mbar_wait(&full_bar[s], (it / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = lp::smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t sb = sa + C::NA * C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          umma2_bf16(acc_base, smem_desc_sw128(sa + kk * 32), smem_desc_sw128(sb + kk * 32), idesc, acc);
          if (EPI == EPI_SWIGLU)
            umma2_bf16(acc_base + BT, smem_desc_sw128(sa + C::A_BYTES + kk * 32), smem_desc_sw128(sb + kk * 32),
                       idesc, acc);
        }
        umma2_commit_both(&empty_bar[s]);
      }
      umma2_commit_both(&tfull[a]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    const int quarter = warp & 3;
    const int ehalf = (warp - 2) >> 2;         // which 32-token chunks of the tile this warp drains
    const int row = quarter * 32 + lane;
    const uint32_t leader_tempty0 = mapa_rank(lp::smem_u32(&tempty[0]), 0);
    const uint32_t leader_tempty1 = mapa_rank(lp::smem_u32(&tempty[1]), 0);
    int li = 0;
    for (int64_t p = p_first; valid(p); ++li) {
      int n0, t0, kb0, nkb;
      decode(p, n0, t0, kb0, nkb);
      p = advance(p, nkb);
      const int a = li % C::NBUF;
      lp::mbar_wait(&tfull[a], (li / C::NBUF) & 1);
      tc_fence_after();
      const int n = n0 + row;
      constexpr int CH = BT < 32 ? BT : 32;
      for (int c = ehalf * CH; c < BT; c += 2 * CH) {
        uint32_t v[32], u[32];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + a * C::ACC_COLS + c;
        if (CH == 32) tmem_ld32(taddr, v); else tmem_ld16(taddr, v);
        if (EPI == EPI_SWIGLU) {
          if (CH == 32) tmem_ld32(taddr + BT, u); else tmem_ld16(taddr + BT, u);
        }
        tmem_wait_ld();
        if constexpr (EPI == EPI_SWIGLU && CH == 32) {
          // transpose through smem so each lane stores one token's 32
          // consecutive outputs as 4 x 16 B (a warp writes whole 128 B lines
          // instead of 64 B per token) — the SwiGLU tile is single-buffered,
          // so its epilogue is on the critical path
          __nv_bfloat16* xt = reinterpret_cast<__nv_bfloat16*>(smem + C::STAGES * C::STAGE_BYTES) +
                              (size_t)(warp - 2) * 32 * C::XPOSE_PITCH;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = __uint_as_float(v[j]), up = __uint_as_float(u[j]);
            xt[j * C::XPOSE_PITCH + lane] = __float2bfloat16_rn(__fdividef(x, 1.0f + __expf(-x)) * up);
          }
          __syncwarp();
          const int t = t0 + c + lane;
          const int nb = n0 + quarter * 32;                        // this warp's first row
          if (t < args.tokens) {
            __nv_bfloat16* orow = (__nv_bfloat16*)args.out + (int64_t)t * args.ldo + nb;
            const int4* src = reinterpret_cast<const int4*>(xt + lane * C::XPOSE_PITCH);
            if (nb + 32 <= args.n_rows && ((((uintptr_t)orow) & 15) == 0)) {
#pragma unroll
              for (int q = 0; q < 4; ++q) reinterpret_cast<int4*>(orow)[q] = src[q];
            } else {
              for (int r = 0; r < 32 && nb + r < args.n_rows; ++r) orow[r] = xt[lane * C::XPOSE_PITCH + r];
            }
          }
          __syncwarp();                                            // xt is rewritten for the next chunk
        } else if (n < args.n_rows) {
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = t0 + c + j;
            if (t >= args.tokens) break;
            const float x = __uint_as_float(v[j]);
            if (EPI == EPI_ADD_F32) {
              float* o = (float*)args.out + (int64_t)t * args.ldo + n;
              if (args.atomic) atomicAdd(o, x); else *o += x;
            } else if (EPI == EPI_STORE_F32) {
              ((float*)args.out)[(int64_t)t * args.ldo + n] = x;
            } else {
              const float up = __uint_as_float(u[j]);
              ((__nv_bfloat16*)args.out)[(int64_t)t * args.ldo + n] =
                  __float2bfloat16_rn(x / (1.0f + __expf(-x)) * up);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(a == 0 ? leader_tempty0 : leader_tempty1);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps (driver entry point via the runtime) + dispatch

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled g_encode = nullptr;

int get_encode() {
  if (g_encode) return 0;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  LP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  LP_CHECK(q == cudaDriverEntryPointSuccess && fn, "cuTensorMapEncodeTiled unavailable");
  g_encode = (PFN_encodeTiled)fn;
  return 0;
}

// row-major [rows, cols] bf16 matrix, box = box_rows x 64 cols, 128B swizzle
int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
  if (get_encode() != 0) return -1;
  LP_CHECK(((uintptr_t)base & 15) == 0 && (cols * 2) % 16 == 0, "tensor map: base/row stride not 16B aligned");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LP_CHECK(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

template <int BT, int EPI>
int launch(const void* W, const void* W2, int64_t N, int64_t K, const void* X, int64_t T, void* out, int64_t ldo,
           int split_k, cudaStream_t s) {
  using C = Cfg<BT, EPI>;
  CUtensorMap mw, mw2, mx;
  if (make_map(&mw, W, N, K, BM) != 0) return -1;
  if (make_map(&mw2, EPI == EPI_SWIGLU ? W2 : W, N, K, BM) != 0) return -1;
  if (make_map(&mx, X, T, K, BT) != 0) return -1;
  // persistent (grid-stride over (tile, split) work items) for prefill; for
  // decode when LP_GEMM_STREAMK=1 (experiment: split-K items balanced over
  // 2 CTAs per SM instead of one wave of fixed tiles)
  static int streamk = -1;
  if (streamk < 0) {
    const char* e = getenv("LP_GEMM_STREAMK");
    streamk = (e && e[0] == '1') ? 1 : 0;
  }
  const bool persistent = T > 64 || streamk;
  // CTA pairs for prefill (LP_GEMM_PAIR=0 selects the single-CTA kernel)
  static int pair_env = -1;
  if (pair_env < 0) {
    const char* e = getenv("LP_GEMM_PAIR");
    pair_env = (e && e[0] == '0') ? 0 : 1;
  }
  const bool pair = T > 64 && pair_env;
  static uint64_t attr_set = 0;   // per-device bit: the smem opt-in is a per-device function attribute
  int dev = 0;
  LP_CUDA(cudaGetDevice(&dev));
  if (!(attr_set >> dev & 1)) {
    LP_CUDA(cudaFuncSetAttribute(gemm_kernel<BT, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    LP_CUDA(cudaFuncSetAttribute(gemm_persistent_kernel<BT, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM));
    if constexpr (BT >= 32)
      LP_CUDA(cudaFuncSetAttribute(gemm_pair_kernel<BT, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   Cfg2<BT, EPI>::SMEM));
    attr_set |= 1ull << dev;
  }
  GemmArgs a;
  a.out = out;
  a.ldo = ldo;
  a.n_rows = (int)N;
  a.tokens = (int)T;
  a.k_blocks = (int)((K + BK - 1) / BK);
  const int splits = split_k < 1 ? 1 : (split_k > a.k_blocks ? a.k_blocks : split_k);
  a.kb_per_split = (a.k_blocks + splits - 1) / splits;
  // fire-and-forget red.add even without split-K: a plain read-modify-write
  // stalls the epilogue on every load (measured 4x slower at T=4096)
  a.atomic = 1;
  a.tiles_n = (int)((N + BM - 1) / BM);
  a.tiles_t = (int)((T + BT - 1) / BT);
  a.splits = splits;
  a.streamk = 0;
  if constexpr (BT >= 32) {
    if (pair) {
      CUtensorMap mxh;
      if (make_map(&mxh, X, T, K, BT / 2) != 0) return -1;
      static int sms2 = 0;
      if (!sms2) LP_CUDA(cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev));
      const int total = ((a.tiles_n + 1) / 2) * a.tiles_t * a.splits;
      const int slots = sms2 / 2;
      // stream-K tail for the accumulating epilogue when whole tiles leave a
      // partial last wave (LP_GEMM_PAIR_STREAMK=0: round-robin tiles only);
      // below one wave the caller's split-K policy balances instead
      static int sk_env = -1;
      if (sk_env < 0) {
        const char* e = getenv("LP_GEMM_PAIR_STREAMK");
        sk_env = (e && e[0] == '0') ? 0 : 1;
      }
      // (a tail above 80 % of a wave measured faster as a plain last round:
      // 70B down T = 4096, 68 of 74 slots: 1332 vs 1407 us)
      a.streamk = (EPI == EPI_ADD_F32 && sk_env && a.splits == 1 && total > slots && total % slots != 0 &&
                   (total % slots) * 10 <= 8 * slots) ? 1 : 0;
      const int clusters = total < slots ? total : slots;
      LP_CUDA(lp::launch(gemm_pair_kernel<BT, EPI>, dim3(2 * clusters), dim3(PAIR_THREADS), Cfg2<BT, EPI>::SMEM, s, mw,
                         mw2, mxh, a));
      return 0;
    }
  }
  if (persistent) {
    static int sms = 0;
    if (!sms) LP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int total = a.tiles_n * a.tiles_t * a.splits;
    const int slots = (T > 64 ? 1 : 2) * sms;      // small decode rings fit two CTAs per SM
    LP_CUDA(lp::launch(gemm_persistent_kernel<BT, EPI>, dim3(total < slots ? total : slots), dim3(THREADS), C::SMEM,
                       s, mw, mw2, mx, a));
  } else {
    dim3 grid((unsigned)a.tiles_n, (unsigned)a.tiles_t, (unsigned)splits);
    LP_CUDA(lp::launch(gemm_kernel<BT, EPI>, grid, dim3(THREADS), C::SMEM, s, mw, mw2, mx, a));
  }
  return 0;
}

template <int EPI>
int dispatch(const void* W, const void* W2, int64_t N, int64_t K, const void* X, int64_t T, void* out, int64_t ldo,
             int split_k, cudaStream_t s) {
  if (T <= 16) return launch<16, EPI>(W, W2, N, K, X, T, out, ldo, split_k, s);
  if (T <= 32) return launch<32, EPI>(W, W2, N, K, X, T, out, ldo, split_k, s);
  if (T <= 64) return launch<64, EPI>(W, W2, N, K, X, T, out, ldo, split_k, s);
  if (T <= 128) return launch<128, EPI>(W, W2, N, K, X, T, out, ldo, split_k, s);
  if constexpr (EPI == EPI_SWIGLU) {
    // experiment switch: 128-token SwiGLU tiles (double-buffered TMEM, more
    // tiles per wave) instead of 256 (single-buffered)
    static int bt128 = -1;
    if (bt128 < 0) {
      const char* e = getenv("LP_SWIGLU_BT128");
      bt128 = (e && e[0] == '1') ? 1 : 0;
    }
    if (bt128) return launch<128, EPI>(W, W2, N, K, X, T, out, ldo, split_k, s);
    // the non-linear epilogue cannot take the stream-K tail: when 256-row x
    // 256-token pair tiles leave a partial last wave, the rows that would
    // fill it go to a second launch in 64-token tiles (a quarter-size round
    // instead of a full one; T = 2048 / 1024: 448 / 224 pair tiles = 6.05 /
    // 3.03 waves of 74).  LP_SWIGLU_TAIL=0 keeps one launch.
    static int tail_env = -1;
    static int sms = 0;
    if (tail_env < 0) {
      const char* e = getenv("LP_SWIGLU_TAIL");
      tail_env = (e && e[0] == '0') ? 0 : 1;
    }
    if (!sms) {
      int dev = 0;
      LP_CUDA(cudaGetDevice(&dev));
      LP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (tail_env && sms >= 2) {
      const int64_t slots = sms / 2;
      const int64_t tt = (T + 255) / 256, n2 = (N + 255) / 256, total = n2 * tt;
      const int64_t rounds = (total + slots - 1) / slots;
      const int64_t n_main2 = rounds >= 2 ? (rounds - 1) * slots / tt : 0;
      const int64_t n_tail2 = n2 - n_main2;
      if (n_main2 >= 1 && n_tail2 >= 1 && n_tail2 * ((T + 63) / 64) <= slots) {
        const int64_t n_main = n_main2 * 256;
        const int r = launch<256, EPI>(W, W2, n_main, K, X, T, out, ldo, split_k, s);
        if (r) return r;
        const size_t off = (size_t)n_main * (size_t)K * 2;
        return launch<64, EPI>((const char*)W + off, (const char*)W2 + off, N - n_main, K, X, T,
                               (__nv_bfloat16*)out + n_main, ldo, split_k, s);
      }
    }
  }
  return launch<256, EPI>(W, W2, N, K, X, T, out, ldo, split_k, s);
}

}  // namespace

extern "C" {

int lp_gemm_bf16(const void* W, int64_t n_rows, int64_t k, const void* X, int64_t tokens, void* out,
                 int64_t ldo, int epilogue, int split_k, void* stream) {
  LP_CHECK(W && X && out && n_rows > 0 && k > 0 && tokens > 0, "lp_gemm_bf16: bad arguments");
  LP_CHECK(epilogue == EPI_ADD_F32 || epilogue == EPI_STORE_F32, "lp_gemm_bf16: epilogue must be 0 (add) or 1 (store)");
  LP_CHECK(epilogue == EPI_ADD_F32 || split_k <= 1, "lp_gemm_bf16: split-K needs the accumulating epilogue");
  cudaStream_t s = (cudaStream_t)stream;
  return epilogue == EPI_ADD_F32 ? dispatch<EPI_ADD_F32>(W, nullptr, n_rows, k, X, tokens, out, ldo, split_k, s)
                                 : dispatch<EPI_STORE_F32>(W, nullptr, n_rows, k, X, tokens, out, ldo, 1, s);
}

int lp_gemm_swiglu(const void* W_gate, const void* W_up, int64_t n_rows, int64_t k, const void* X, int64_t tokens,
                   void* out_bf16, int64_t ldo, void* stream) {
  LP_CHECK(W_gate && W_up && X && out_bf16 && n_rows > 0 && k > 0 && tokens > 0, "lp_gemm_swiglu: bad arguments");
  return dispatch<EPI_SWIGLU>(W_gate, W_up, n_rows, k, X, tokens, out_bf16, ldo, 1, (cudaStream_t)stream);
}

}  // extern "C"
