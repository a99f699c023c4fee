// λPipe multicast engine: executes a reference binomial/k-way schedule as a
// tile-granular dataflow over NVLink peer stores and PCIe host pulls.
//
// Reference semantics replaced: the lockstep "transfer_step_done" events of
// simengine.py:594-596 / :628-644, whose cost is the formula at
// simengine.py:95-103.  Here every transfer (step, sender, receiver, block)
// of schedule_to_lines (multicast.py:546-551) moves the block's real bytes:
//
//   * GPU sender  -> the sender's CTAs read the block tile by tile from local
//                    HBM and store it with 16-byte vector stores straight into
//                    the receiver's image (a CUDA-IPC / peer pointer), then
//                    publish a per-tile flag in the receiver's memory with a
//                    .sys release;
//   * HOST sender -> the receiver's CTAs pull the tiles from mapped pinned host
//                    memory over PCIe into local HBM and publish local flags.
//
// A relay forwards tile t of block j as soon as its own flag for (j, t) holds
// the current epoch (cut-through).  Each executing node's sends run in
// schedule step order; no flag is ever polled across NVLink (all waits are on
// local memory).  Flags carry the run's epoch so they never need resetting.
#include "lp_common.cuh"
#include "../../include/lambdapipe.h"
#include <cuda.h>
#include <algorithm>
#include <string.h>
#include <stdlib.h>
#include <vector>

#define LP_MAX_EXEC 32
#define LP_MC_THREADS 512

namespace {

struct NodeDev {
  char* image;
  uint32_t* flags;    // [total_tiles]
  uint32_t* counts;   // [n_blocks] cumulative tiles delivered (epoch * ntiles when complete)
  uint64_t* arrival;  // [n_blocks] globaltimer ns when the block completed (last run)
  uint32_t* ready;    // optional mapped-host [n_blocks] = epoch when complete
  int32_t kind;
  int32_t pad;
};
struct BlockDev {
  int64_t off;
  int64_t len;
  int64_t tile;       // bytes per tile of this block (uniform unless lp_mc_create_tiled)
  int32_t tile_base;
  int32_t ntiles;
};
struct OpDev {
  int32_t block, src, dst, wait, step, pad;
};
struct ExecDesc {
  int32_t node, push_b, push_e, pull_b, pull_e, recv_b, recv_e, dma_b, dma_e, pad;
};
struct McParams {
  const NodeDev* nodes;
  const BlockDev* blocks;
  const OpDev* ops;
  const int32_t* recv_blocks;
  int* err;
  int64_t tile_bytes;
  uint64_t timeout_ns;
  uint32_t epoch;
  uint32_t chunk_bytes;
  int push_ctas, pull_ctas, n_exec;
  int push_mode, pull_mode;   // 0 = LDG/STG vectors, 1 = TMA bulk pipeline
  int window;                 // ops a CTA may interleave (ldg role)
  int wide_loads;             // 256 B L2 fetch granule on LDG-role loads
  ExecDesc exec[LP_MAX_EXEC];
};

__device__ __forceinline__ bool wait_flag(const uint32_t* f, uint32_t epoch, uint64_t t0,
                                          uint64_t timeout_ns, int* err, int code = 1) {
  uint32_t spins = 0;
  while (lp::ld_acquire_sys(f) != epoch) {
    if (++spins > 64) {
      lp::nanosleep(200);
      if ((spins & 1023) == 0 && lp::globaltimer() - t0 > timeout_ns) {
        atomicExch(err, code);
        return false;
      }
    }
  }
  return true;
}

template <bool WIDE>
__device__ __forceinline__ int4 ld16(const int4* p) {
  return WIDE ? lp::ld_stream16_l2_256(p) : lp::ld_stream16(p);
}

template <bool WIDE>
__device__ __forceinline__ void copy_tile_t(const char* __restrict__ s, char* __restrict__ d, int64_t n) {
  constexpr int U = 8;
  const int4* s4 = reinterpret_cast<const int4*>(s);
  int4* d4 = reinterpret_cast<int4*>(d);
  const int64_t n16 = n >> 4;
  const int T = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + (int64_t)(U - 1) * T < n16; i += (int64_t)U * T) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld16<WIDE>(s4 + i + (int64_t)u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) lp::st16(d4 + i + (int64_t)u * T, v[u]);
  }
  for (; i < n16; i += T) lp::st16(d4 + i, ld16<WIDE>(s4 + i));
}

__device__ __forceinline__ void copy_tile(const char* __restrict__ s, char* __restrict__ d, int64_t n, bool wide) {
  if (wide)
    copy_tile_t<true>(s, d, n);
  else
    copy_tile_t<false>(s, d, n);
}

// ---------------------------------------------------------------------------
// Role A: LDG/STG copy.  All 512 threads move 16-byte vectors; one thread
// waits for the tile's flag before, and publishes the receiver's flag after.

__device__ __forceinline__ void publish_tile(const NodeDev& dst, const BlockDev& bl, int block, int t,
                                             uint32_t epoch) {
  lp::st_release_sys(dst.flags + bl.tile_base + t, epoch);
  const uint32_t old = lp::atom_add_release_sys(dst.counts + block, 1u);
  if (old + 1u == epoch * (uint32_t)bl.ntiles) {
    dst.arrival[block] = lp::globaltimer();
    if (dst.ready) lp::st_release_sys(dst.ready + block, epoch);
  }
}

// Ops of one role are consumed through a window of `window` consecutive ops:
// each op's tiles are taken in order, but when the next tile of the oldest op
// is not ready yet (its sender is a relay still receiving it), the CTA moves
// on to the first op in the window whose next tile IS ready.  That keeps the
// node's NVLink ingress busy instead of idling behind one slow upstream; the
// transfer set and each op's bytes are unchanged.
constexpr int kMaxWindow = 8;

__device__ void ldg_role(const McParams& p, int ob, int oe, int lane, int lanes, uint64_t t0, int* s_ok) {
  const uint32_t epoch = p.epoch;
  const int W = p.window < 1 ? 1 : (p.window > kMaxWindow ? kMaxWindow : p.window);
  __shared__ int cur[kMaxWindow];
  __shared__ int s_base, s_pick, s_tile;
  if (threadIdx.x == 0) {
    for (int w = 0; w < kMaxWindow; ++w) cur[w] = lane;
    s_base = ob;
  }
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) {
      int base = s_base;
      while (base < oe && cur[0] >= p.blocks[p.ops[base].block].ntiles) {
        for (int w = 0; w + 1 < W; ++w) cur[w] = cur[w + 1];
        cur[W - 1] = lane;
        ++base;
      }
      s_base = base;
      int pick = -1;
      for (int w = 0; w < W && base + w < oe; ++w) {
        const OpDev op = p.ops[base + w];
        const BlockDev bl = p.blocks[op.block];
        if (cur[w] >= bl.ntiles) continue;
        if (!op.wait || lp::ld_acquire_sys(p.nodes[op.src].flags + bl.tile_base + cur[w]) == epoch) {
          pick = w;
          break;
        }
      }
      if (pick < 0 && base < oe) {  // nothing ready: block on the oldest op's next tile
        for (int w = 0; w < W && base + w < oe; ++w) {
          const OpDev op = p.ops[base + w];
          const BlockDev bl = p.blocks[op.block];
          if (cur[w] >= bl.ntiles) continue;
          if (!wait_flag(p.nodes[op.src].flags + bl.tile_base + cur[w], epoch, t0, p.timeout_ns, p.err))
            *s_ok = 0;
          pick = w;
          break;
        }
      }
      s_pick = pick < 0 ? -1 : base + pick;
      s_tile = pick < 0 ? 0 : cur[pick];
      if (pick >= 0) cur[pick] += lanes;
    }
    __syncthreads();
    const int oi = s_pick;
    const int t = s_tile;
    if (oi < 0 || !*s_ok) return;
    const OpDev op = p.ops[oi];
    const BlockDev bl = p.blocks[op.block];
    const NodeDev src = p.nodes[op.src];
    const NodeDev dst = p.nodes[op.dst];
    const int64_t lo = (int64_t)t * bl.tile;
    const int64_t n = min(bl.tile, bl.len - lo);
    copy_tile(src.image + bl.off + lo, dst.image + bl.off + lo, n, p.wide_loads != 0);
    __syncthreads();  // every thread's stores of this tile precede the flag
    if (threadIdx.x == 0) {
      lp::fence_sys();
      publish_tile(dst, bl, op.block, t, epoch);
    }
  }
}

// ---------------------------------------------------------------------------
// Role B: TMA bulk-copy pipeline driven by ONE thread.  Tiles are cut into
// chunks; chunk q is loaded HBM(or host)->smem ring slot q % S with
// cp.async.bulk (mbarrier completion) and stored smem->destination with a
// bulk_group store (the destination is the peer's image over NVLink).  Loads
// run LA = 3 chunks ahead of stores, leaving S - LA slots to stores in flight
// (a slot is reusable once its store has READ it, which over NVLink takes
// about the write latency, so in-flight stores set the per-CTA rate); a tile's flag is published once its
// last store group completed (bulk wait_group), a few groups after issue, so
// the pipeline never drains between tiles.

constexpr int kStages = 12;
constexpr int kLookaheadPush = 3;   // local HBM reads: short latency, many stores in flight
constexpr int kLookaheadPull = 9;   // remote NVLink / PCIe reads: long latency, local stores
constexpr int kPendTiles = 16;

struct ChunkDesc {
  const char* src;
  char* dst;
  uint32_t bytes;
  int32_t last;      // last chunk of its tile
  int32_t op;        // op index (for publishing)
  int32_t tile;
};

struct TileGen {  // walks (op, my tiles, chunks) in order
  int oi, oe, t, lane, lanes;
  int64_t c;         // byte offset within the tile
};

__device__ void tma_role(const McParams& p, int ob, int oe, int lane, int lanes, uint64_t t0, int* s_ok,
                         char* ring, uint64_t* bars, const int lookahead) {
  if (threadIdx.x != 0) return;
  const uint32_t epoch = p.epoch;
  const uint32_t chunk = p.chunk_bytes;
  ChunkDesc desc[kStages];
  int pend_op[kPendTiles], pend_tile[kPendTiles];
  int64_t pend_group[kPendTiles];
  int pend_head = 0, pend_tail = 0;
  int64_t q_load = 0, q_store = 0;

  TileGen g{ob, oe, lane, lane, lanes, 0};
  // skip ops with no tile for this lane
  auto settle = [&]() {
    while (g.oi < g.oe && g.t >= p.blocks[p.ops[g.oi].block].ntiles) {
      ++g.oi;
      g.t = g.lane;
      g.c = 0;
    }
  };
  settle();

  auto publish_ready = [&](bool force) {
    while (pend_head != pend_tail) {
      const int i = pend_head % kPendTiles;
      const int64_t after = q_store - 1 - pend_group[i];  // groups issued after the tile's last one
      if (!force && after < kStages - 1) break;
      lp::bulk_wait_n((int)(after < 0 ? 0 : after));
      lp::fence_proxy_async_global();
      lp::fence_sys();
      const OpDev op = p.ops[pend_op[i]];
      publish_tile(p.nodes[op.dst], p.blocks[op.block], op.block, pend_tile[i], epoch);
      ++pend_head;
    }
  };

  auto store_one = [&]() {
    const int slot = (int)(q_store % kStages);
    lp::mbar_wait(&bars[slot], (uint32_t)((q_store / kStages) & 1));
    const ChunkDesc d = desc[slot];
    lp::bulk_s2g(d.dst, ring + (size_t)slot * chunk, d.bytes);
    lp::bulk_commit();
    if (d.last) {
      if (pend_tail - pend_head == kPendTiles) publish_ready(true);
      const int i = pend_tail % kPendTiles;
      pend_op[i] = d.op;
      pend_tile[i] = d.tile;
      pend_group[i] = q_store;
      ++pend_tail;
    }
    ++q_store;
    publish_ready(false);
  };

  while (true) {
    const bool have_next = g.oi < g.oe;
    if (!have_next && q_store == q_load) break;
    if (have_next && q_load - q_store < lookahead) {
      const OpDev op = p.ops[g.oi];
      const BlockDev bl = p.blocks[op.block];
      const NodeDev src = p.nodes[op.src];
      const NodeDev dst = p.nodes[op.dst];
      if (g.c == 0 && op.wait) {
        const uint32_t* f = src.flags + bl.tile_base + g.t;
        if (lp::ld_acquire_sys(f) != epoch) {
          if (q_store < q_load) {  // keep the pipe moving while the tile is in flight upstream
            store_one();
            continue;
          }
          publish_ready(true);
          if (!wait_flag(f, epoch, t0, p.timeout_ns, p.err)) {
            *s_ok = 0;
            lp::bulk_wait<0>();
            return;
          }
        }
        lp::fence_proxy_async_global();  // order the acquire before async-proxy reads
      }
      const int64_t tlo = (int64_t)g.t * bl.tile;
      const int64_t tlen = min(bl.tile, bl.len - tlo);
      const uint32_t nb = (uint32_t)min((int64_t)chunk, tlen - g.c);
      const int slot = (int)(q_load % kStages);
      if (q_load >= kStages) lp::bulk_wait_read_n((int)(q_store - 1 - (q_load - kStages)));
      ChunkDesc d;
      d.src = src.image + bl.off + tlo + g.c;
      d.dst = dst.image + bl.off + tlo + g.c;
      d.bytes = nb;
      d.last = (g.c + nb >= tlen) ? 1 : 0;
      d.op = g.oi;
      d.tile = g.t;
      desc[slot] = d;
      lp::mbar_expect_tx(&bars[slot], nb);
      lp::bulk_g2s(ring + (size_t)slot * chunk, d.src, nb, &bars[slot]);
      ++q_load;
      g.c += nb;
      if (g.c >= tlen) {
        g.c = 0;
        g.t += g.lanes;
        settle();
      }
    } else {
      store_one();
    }
  }
  lp::bulk_wait<0>();
  publish_ready(true);
}

__global__ void __launch_bounds__(LP_MC_THREADS) mc_kernel(const McParams p) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t bars[kStages];
  __shared__ int s_ok;
  const int per = p.push_ctas + p.pull_ctas;
  const int e = blockIdx.x / per;
  const int local = blockIdx.x % per;
  const ExecDesc ex = p.exec[e];
  const bool pusher = local < p.push_ctas;
  const int lane = pusher ? local : local - p.push_ctas;
  const int lanes = pusher ? p.push_ctas : p.pull_ctas;
  const int ob = pusher ? ex.push_b : ex.pull_b;
  const int oe = pusher ? ex.push_e : ex.pull_e;
  const bool tma = pusher ? (p.push_mode == 1) : (p.pull_mode == 1);
  uint64_t t0 = 0;
  if (threadIdx.x == 0) {
    t0 = lp::globaltimer();
    s_ok = 1;
    if (tma) {
      for (int i = 0; i < kStages; ++i) lp::mbar_init(&bars[i], 1);
      lp::fence_mbar_init();
    }
  }
  __syncthreads();
  if (tma)
    tma_role(p, ob, oe, lane, lanes, t0, &s_ok, ring, bars, pusher ? kLookaheadPush : kLookaheadPull);
  else
    ldg_role(p, ob, oe, lane, lanes, t0, &s_ok);

  // the node is complete when every tile it receives this epoch has landed
  if (pusher && threadIdx.x == 0 && s_ok) {
    const NodeDev me = p.nodes[ex.node];
    for (int r = ex.recv_b; r < ex.recv_e; ++r) {
      const BlockDev bl = p.blocks[p.recv_blocks[r]];
      for (int t = lane; t < bl.ntiles; t += lanes) {
        if (!wait_flag(me.flags + bl.tile_base + t, p.epoch, t0, p.timeout_ns, p.err)) return;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Verify-as-it-lands: per-block checksums (the lp_block_checksums function,
// sum of mix64(word ^ k * golden) over the block's 8-byte words, k = word
// index in the block) of what a receiver holds, computed while the scale-out
// is still running.  Nothing spins on a flag: the verify stream parks in a
// stream-ordered wait (cuStreamWaitValue32 on the node's own block counter,
// handled by the GPU front end, no SM held) and then launches this kernel over
// the one block that just completed.
__global__ void __launch_bounds__(512) block_sum_kernel(const char* __restrict__ base, int64_t len,
                                                        unsigned long long* __restrict__ sum) {
  __shared__ uint64_t part[16];
  constexpr uint64_t G = 0x9E3779B97F4A7C15ull;
  const ulonglong2* w = reinterpret_cast<const ulonglong2*>(base);
  const int64_t n16 = len >> 4;                        // blocks are 16-byte multiples
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  uint64_t acc = 0;
  constexpr int U = 8;                                 // 128 B in flight per thread
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * T < n16; i += U * T) {
    ulonglong2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(w + i + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = 2 * (uint64_t)(i + u * T);
      acc += lp::mix64(v[u].x ^ (k * G)) + lp::mix64(v[u].y ^ ((k + 1) * G));
    }
  }
  for (; i < n16; i += T) {
    const ulonglong2 v = __ldcs(w + i);
    const uint64_t k = 2 * (uint64_t)i;
    acc += lp::mix64(v.x ^ (k * G)) + lp::mix64(v.y ^ ((k + 1) * G));
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += part[j];
    atomicAdd(sum, (unsigned long long)t);
  }
}

// Start-of-run block counters of the blocks a node PULLS in-kernel: (epoch-1)
// x ntiles, so completion (old + 1 == epoch x ntiles in publish_tile) holds for
// this run whatever an earlier, aborted run left behind.  Only the receiver's
// own kernel increments these counters, and it runs after this on the stream.
struct CountReset {
  uint32_t* counts[LP_MAX_EXEC];
  int op_b[LP_MAX_EXEC], op_e[LP_MAX_EXEC];
  const OpDev* ops;
  const BlockDev* blocks;
  uint32_t epoch;
};
__global__ void count_reset_kernel(const CountReset r) {
  const int e = blockIdx.x;
  for (int i = r.op_b[e] + threadIdx.x; i < r.op_e[e]; i += blockDim.x) {
    const OpDev op = r.ops[i];
    r.counts[e][op.block] = (r.epoch - 1u) * (uint32_t)r.blocks[op.block].ntiles;
  }
}

}  // namespace

struct lp_mc {
  int n_nodes = 0, n_blocks = 0;
  int64_t tile_bytes = 0;
  int64_t total_tiles = 0;
  int64_t off_counts = 0, off_arrival = 0, signal_bytes = 0;
  std::vector<BlockDev> blocks;
  std::vector<NodeDev> nodes;
  std::vector<int32_t> xfers;   // rows of 4
  std::vector<int32_t> sources;
  bool dirty = true;
  // compiled per-node op ranges
  std::vector<ExecDesc> per_node;
  std::vector<OpDev> h_ops;         // host copy of the compiled op lists (copy-engine executor)
  std::vector<int32_t> vr_off;      // [N+1] offsets of each node's receive order in h_vorder
  std::vector<int32_t> h_vorder;    // blocks each node receives, in step order (verify)
  int dev = 0;
  NodeDev* d_nodes = nullptr;
  BlockDev* d_blocks = nullptr;
  OpDev* d_ops = nullptr;
  int32_t* d_recv = nullptr;
  int* d_err = nullptr;
  int max_resident = 0;
  int direction = 1;                  // 0 push (sender executes), 1 pull (receiver executes)
  int push_mode = 1, pull_mode = 1;   // 0 LDG/STG, 1 TMA
  int64_t chunk_bytes = 16384;
  int window = 3;
  int wide_loads = 0;
  int host_dma = 0;                   // HOST-sourced transfers run on the copy engines (lp_mc_run_host_dma)
  int ce_split = 0;                   // > 0: GPU-sourced transfers of blocks b % ce_split == 0 run there too
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;   // flag-wait watchdog
  uint32_t last_epoch = 0;            // last epoch launched on this handle
  bool failed = false;                // a watchdog expired: signals must be reset before the next run
  cudaStream_t poll = nullptr;   // private non-blocking stream for host polls
};

static int poll_stream(lp_mc* mc) {
  lp::DeviceGuard g(mc->dev);
  if (!mc->poll) LP_CUDA(cudaStreamCreateWithFlags(&mc->poll, cudaStreamNonBlocking));
  return 0;
}

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

static int compile(lp_mc* mc) {
  const int N = mc->n_nodes;
  std::vector<char> is_src(N, 0);
  for (int s : mc->sources) {
    LP_CHECK(s >= 0 && s < N, "lp_mc: source %d out of range", s);
    is_src[s] = 1;
  }
  for (int i = 0; i < N; ++i)
    LP_CHECK(mc->nodes[i].kind == LP_NODE_HOST || mc->nodes[i].image != nullptr,
             "lp_mc: node %d has no image (call lp_mc_set_node)", i);
  struct Row { int step, snd, rcv, blk; };
  std::vector<Row> rows;
  const int T = (int)mc->xfers.size() / 4;
  std::vector<char> got((size_t)N * mc->n_blocks, 0);
  for (int i = 0; i < T; ++i) {
    Row r{mc->xfers[4 * i], mc->xfers[4 * i + 1], mc->xfers[4 * i + 2], mc->xfers[4 * i + 3]};
    LP_CHECK(r.snd >= 0 && r.snd < N && r.rcv >= 0 && r.rcv < N && r.snd != r.rcv,
             "lp_mc: transfer %d has bad endpoints %d->%d", i, r.snd, r.rcv);
    LP_CHECK(r.blk >= 0 && r.blk < mc->n_blocks, "lp_mc: transfer %d block %d out of range", i, r.blk);
    LP_CHECK(mc->nodes[r.rcv].kind == LP_NODE_GPU, "lp_mc: receiver %d is not a GPU node", r.rcv);
    LP_CHECK(mc->nodes[r.snd].kind == LP_NODE_GPU || is_src[r.snd],
             "lp_mc: host node %d sends but is not a source", r.snd);
    char& g = got[(size_t)r.rcv * mc->n_blocks + r.blk];
    LP_CHECK(!g && !is_src[r.rcv], "lp_mc: node %d receives block %d twice", r.rcv, r.blk);
    g = 1;
    rows.push_back(r);
  }
  std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
    return a.step != b.step ? a.step < b.step : (a.snd != b.snd ? a.snd < b.snd : a.rcv < b.rcv);
  });
  // causality (multicast.py:507-509): a sender holds the block at step start,
  // otherwise its flag wait could never be satisfied
  {
    std::vector<int> held_at((size_t)N * mc->n_blocks, -2);  // step the block landed, -1 = source
    for (int n = 0; n < N; ++n)
      if (is_src[n])
        for (int b = 0; b < mc->n_blocks; ++b) held_at[(size_t)n * mc->n_blocks + b] = -1;
    for (const Row& r : rows) {  // rows are step-sorted; same-step arrivals do not count
      int h = held_at[(size_t)r.snd * mc->n_blocks + r.blk];
      LP_CHECK(h != -2 && h < r.step, "lp_mc: step %d: node %d sends block %d it does not hold", r.step,
               r.snd, r.blk);
      held_at[(size_t)r.rcv * mc->n_blocks + r.blk] = r.step;
    }
  }
  // executor of a transfer: its sender pushes (direction 0) unless the sender
  // is a HOST node; with direction 1 every transfer is pulled by its receiver
  auto from_host = [&](const Row& r) { return mc->nodes[r.snd].kind == LP_NODE_HOST; };
  auto pulled = [&](const Row& r) { return mc->direction == 1 || from_host(r); };
  // with host_dma the receiver's copy engine performs the PCIe hop and the
  // kernel only relays over NVLink (waiting on the flags the DMA publishes)
  // with ce_split = m, GPU->GPU transfers of every m-th block also go to the
  // copy engines, so DMA engines and SMs share each link's traffic
  auto dma = [&](const Row& r) {
    return (mc->host_dma && from_host(r)) || (mc->ce_split > 0 && !from_host(r) && r.blk % mc->ce_split == 0);
  };
  std::vector<OpDev> ops;
  std::vector<int32_t> recv;
  mc->per_node.assign(N, ExecDesc{});
  for (int n = 0; n < N; ++n) {
    ExecDesc& d = mc->per_node[n];
    d.node = n;
    d.push_b = (int)ops.size();
    for (const Row& r : rows)
      if (r.snd == n && !pulled(r) && !dma(r))
        ops.push_back(OpDev{r.blk, r.snd, r.rcv, is_src[r.snd] ? 0 : 1, r.step, 0});
    d.push_e = (int)ops.size();
    d.pull_b = (int)ops.size();
    for (const Row& r : rows)
      if (r.rcv == n && pulled(r) && !dma(r))
        ops.push_back(OpDev{r.blk, r.snd, r.rcv, is_src[r.snd] ? 0 : 1, r.step, 0});
    d.pull_e = (int)ops.size();
    d.dma_b = (int)ops.size();
    for (const Row& r : rows)
      if (r.rcv == n && dma(r)) ops.push_back(OpDev{r.blk, r.snd, r.rcv, is_src[r.snd] ? 0 : 1, r.step, 0});
    d.dma_e = (int)ops.size();
    // tiles other nodes push into n: waited for before n's kernel completes
    d.recv_b = (int)recv.size();
    for (const Row& r : rows)
      if (r.rcv == n && !pulled(r) && !dma(r)) recv.push_back(r.blk);
    d.recv_e = (int)recv.size();
  }
  // receive order per node (verify kernel): blocks in the step order they land
  std::vector<int32_t> vorder;
  mc->vr_off.assign(N + 1, 0);
  for (int n = 0; n < N; ++n) {
    mc->vr_off[n] = (int)vorder.size();
    for (const Row& r : rows)
      if (r.rcv == n) vorder.push_back(r.blk);
  }
  mc->vr_off[N] = (int)vorder.size();
  mc->h_vorder = vorder;
  lp::DeviceGuard g(mc->dev);
  if (mc->d_ops) cudaFree(mc->d_ops);
  if (mc->d_recv) cudaFree(mc->d_recv);
  mc->d_ops = nullptr;
  mc->d_recv = nullptr;
  mc->h_ops = ops;
  LP_CUDA(cudaMalloc(&mc->d_ops, sizeof(OpDev) * std::max<size_t>(1, ops.size())));
  LP_CUDA(cudaMalloc(&mc->d_recv, sizeof(int32_t) * std::max<size_t>(1, recv.size())));
  if (!ops.empty()) LP_CUDA(cudaMemcpy(mc->d_ops, ops.data(), sizeof(OpDev) * ops.size(), cudaMemcpyHostToDevice));
  if (!recv.empty())
    LP_CUDA(cudaMemcpy(mc->d_recv, recv.data(), sizeof(int32_t) * recv.size(), cudaMemcpyHostToDevice));
  LP_CUDA(cudaMemcpy(mc->d_nodes, mc->nodes.data(), sizeof(NodeDev) * N, cudaMemcpyHostToDevice));
  mc->dirty = false;
  return 0;
}

extern "C" {

int lp_mc_create_tiled(lp_mc** out, int n_nodes, int n_blocks, const int64_t* block_off,
                       const int64_t* block_len, const int64_t* block_tile) {
  LP_CHECK(out && n_nodes >= 1 && n_nodes <= 4096 && n_blocks >= 1 && block_tile, "lp_mc_create: bad arguments");
  int64_t min_tile = INT64_MAX;
  for (int i = 0; i < n_blocks; ++i) {
    LP_CHECK(block_tile[i] >= 4096 && block_tile[i] % 16 == 0,
             "lp_mc_create: tile bytes must be >= 4096 and a multiple of 16 (block %d)", i);
    min_tile = std::min(min_tile, block_tile[i]);
  }
  lp_mc* mc = new lp_mc();
  mc->n_nodes = n_nodes;
  mc->n_blocks = n_blocks;
  mc->tile_bytes = min_tile;         // the smallest tile bounds the kernel's chunk size
  int64_t tiles = 0;
  for (int i = 0; i < n_blocks; ++i) {
    if (block_off[i] % 16 || block_len[i] % 16 || block_len[i] <= 0) {
      delete mc;
      lp::set_error("lp_mc_create: block %d offset/length must be positive multiples of 16", i);
      return -2;
    }
    int64_t nt = (block_len[i] + block_tile[i] - 1) / block_tile[i];
    mc->blocks.push_back(BlockDev{block_off[i], block_len[i], block_tile[i], (int32_t)tiles, (int32_t)nt});
    tiles += nt;
  }
  mc->total_tiles = tiles;
  mc->off_counts = align_up(tiles * 4, 256);
  mc->off_arrival = align_up(mc->off_counts + (int64_t)n_blocks * 4, 256);
  mc->signal_bytes = align_up(mc->off_arrival + (int64_t)n_blocks * 8, 256);
  mc->nodes.assign(n_nodes, NodeDev{});
  cudaGetDevice(&mc->dev);
  if (cudaMalloc(&mc->d_nodes, sizeof(NodeDev) * n_nodes) != cudaSuccess ||
      cudaMalloc(&mc->d_blocks, sizeof(BlockDev) * n_blocks) != cudaSuccess ||
      cudaMalloc(&mc->d_err, sizeof(int)) != cudaSuccess) {
    lp::set_error("lp_mc_create: device allocation failed");
    delete mc;
    return -1;
  }
  cudaMemcpy(mc->d_blocks, mc->blocks.data(), sizeof(BlockDev) * n_blocks, cudaMemcpyHostToDevice);
  cudaMemset(mc->d_err, 0, sizeof(int));
  // force-load the engine's kernels now: under lazy module loading, loading a
  // kernel while the multicast kernel spins on a peer's (or a copy engine's)
  // flags would wait for that kernel to finish
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, mc_kernel);
  cudaFuncGetAttributes(&fa, block_sum_kernel);
  cudaFuncGetAttributes(&fa, count_reset_kernel);
  *out = mc;
  return 0;
}

int lp_mc_create(lp_mc** out, int n_nodes, int n_blocks, const int64_t* block_off,
                 const int64_t* block_len, int64_t tile_bytes) {
  LP_CHECK(n_blocks >= 1, "lp_mc_create: bad arguments");
  std::vector<int64_t> tiles((size_t)n_blocks, tile_bytes);
  return lp_mc_create_tiled(out, n_nodes, n_blocks, block_off, block_len, tiles.data());
}

int lp_mc_destroy(lp_mc* mc) {
  if (!mc) return 0;
  lp::DeviceGuard g(mc->dev);
  cudaFree(mc->d_nodes);
  cudaFree(mc->d_blocks);
  cudaFree(mc->d_ops);
  cudaFree(mc->d_recv);
  cudaFree(mc->d_err);
  if (mc->poll) cudaStreamDestroy(mc->poll);
  delete mc;
  return 0;
}

int lp_mc_signal_bytes(const lp_mc* mc, int64_t* bytes) {
  LP_CHECK(mc && bytes, "lp_mc_signal_bytes: null argument");
  *bytes = mc->signal_bytes;
  return 0;
}

int lp_mc_set_node(lp_mc* mc, int node, int kind, void* image, void* signals, void* ready_host) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes, "lp_mc_set_node: node %d out of range", node);
  LP_CHECK(kind == LP_NODE_GPU || kind == LP_NODE_HOST, "lp_mc_set_node: bad kind %d", kind);
  LP_CHECK(image != nullptr, "lp_mc_set_node: node %d image is null", node);
  LP_CHECK(kind == LP_NODE_HOST || signals != nullptr, "lp_mc_set_node: GPU node %d needs a signal area", node);
  NodeDev& d = mc->nodes[node];
  d.image = (char*)image;
  d.kind = kind;
  d.ready = (uint32_t*)ready_host;
  char* s = (char*)signals;
  d.flags = s ? (uint32_t*)s : nullptr;
  d.counts = s ? (uint32_t*)(s + mc->off_counts) : nullptr;
  d.arrival = s ? (uint64_t*)(s + mc->off_arrival) : nullptr;
  mc->dirty = true;
  return 0;
}

int lp_mc_set_schedule(lp_mc* mc, const int32_t* xfers, int n_xfers, const int32_t* sources, int n_sources) {
  LP_CHECK(mc && n_xfers >= 0 && n_sources >= 1, "lp_mc_set_schedule: bad arguments");
  mc->xfers.assign(xfers, xfers + 4 * (size_t)n_xfers);
  mc->sources.assign(sources, sources + n_sources);
  mc->dirty = true;
  return 0;
}

int lp_mc_reset_signals(lp_mc* mc, int node, void* stream) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes, "lp_mc_reset_signals: bad node");
  LP_CHECK(mc->nodes[node].flags, "lp_mc_reset_signals: node %d has no signal area", node);
  LP_CUDA(cudaMemsetAsync(mc->nodes[node].flags, 0, (size_t)mc->signal_bytes, (cudaStream_t)stream));
  mc->failed = false;
  mc->last_epoch = 0;
  return 0;
}

int lp_mc_configure(lp_mc* mc, int direction, int push_mode, int pull_mode, int64_t chunk_bytes,
                    int window) {
  LP_CHECK(mc, "lp_mc_configure: null handle");
  LP_CHECK(direction == 0 || direction == 1, "lp_mc_configure: direction is 0 (push) or 1 (pull)");
  LP_CHECK((push_mode == 0 || push_mode == 1) && (pull_mode == 0 || pull_mode == 1),
           "lp_mc_configure: modes are 0 (ldg) or 1 (tma)");
  LP_CHECK(chunk_bytes >= 1024 && chunk_bytes % 16 == 0 && chunk_bytes * kStages <= 216 * 1024,
           "lp_mc_configure: chunk_bytes must be a multiple of 16 in [1024, %d]", 216 * 1024 / kStages);
  LP_CHECK(chunk_bytes <= mc->tile_bytes, "lp_mc_configure: chunk larger than a tile");
  if (direction != mc->direction) mc->dirty = true;
  if (window >= 1) mc->window = window < kMaxWindow ? window : kMaxWindow;

  mc->direction = direction;
  mc->push_mode = push_mode;
  mc->pull_mode = pull_mode;
  mc->chunk_bytes = chunk_bytes;
  return 0;
}

int lp_mc_set_option(lp_mc* mc, const char* name, int64_t value) {
  LP_CHECK(mc && name, "lp_mc_set_option: null argument");
  if (!strcmp(name, "wide_loads")) {
    mc->wide_loads = value != 0;
  } else if (!strcmp(name, "window")) {
    LP_CHECK(value >= 1 && value <= kMaxWindow, "lp_mc_set_option: window must be in [1, %d]", kMaxWindow);
    mc->window = (int)value;
  } else if (!strcmp(name, "ce_split")) {
    LP_CHECK(value >= 0 && value <= 64, "lp_mc_set_option: ce_split must be in [0, 64]");
    if (value != mc->ce_split) mc->dirty = true;
    mc->ce_split = (int)value;
  } else if (!strcmp(name, "host_dma")) {
    if ((value != 0) != (mc->host_dma != 0)) mc->dirty = true;
    mc->host_dma = value != 0;
  } else if (!strcmp(name, "timeout_ms")) {
    LP_CHECK(value > 0, "lp_mc_set_option: timeout_ms must be positive");
    mc->timeout_ns = (uint64_t)value * 1000000ull;
  } else {
    LP_CHECK(false, "lp_mc_set_option: unknown option '%s'", name);
  }
  return 0;
}

int lp_mc_run(lp_mc* mc, const int32_t* exec_nodes, int n_exec, uint32_t epoch, int push_ctas,
              int pull_ctas, void* stream) {
  LP_CHECK(mc && n_exec >= 1 && n_exec <= LP_MAX_EXEC, "lp_mc_run: n_exec must be in [1, %d]", LP_MAX_EXEC);
  LP_CHECK(epoch >= 1, "lp_mc_run: epoch must be >= 1");
  LP_CHECK(push_ctas >= 0 && pull_ctas >= 0 && push_ctas + pull_ctas >= 1, "lp_mc_run: bad CTA counts");
  const int per = push_ctas + pull_ctas;
  const bool any_tma = (push_ctas > 0 && mc->push_mode == 1) || (pull_ctas > 0 && mc->pull_mode == 1);
  const int smem = any_tma ? (int)(kStages * mc->chunk_bytes) : 0;
  LP_CUDA(cudaFuncSetAttribute(mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 0 ? smem : 0));
  int occ = 0, sms = 0;
  LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mc_kernel, LP_MC_THREADS, smem));
  LP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, mc->dev));
  LP_CHECK(per * n_exec <= occ * sms,
           "lp_mc_run: %d CTAs exceed the %d co-resident CTAs the dataflow needs", per * n_exec, occ * sms);
  LP_CHECK(!mc->failed, "lp_mc_run: an earlier run timed out; call lp_mc_reset_signals on every node "
                        "(then restart at epoch 1)");
  // pushed tiles are counted in the receiver's memory by remote senders, so
  // their block counters cannot be re-based here: pushes need every earlier
  // epoch complete, i.e. consecutive epochs on this handle
  LP_CHECK(push_ctas == 0 || epoch == mc->last_epoch + 1 || epoch == mc->last_epoch,
           "lp_mc_run: push runs need consecutive epochs (last %u, got %u)", mc->last_epoch, epoch);
  if (mc->dirty && compile(mc) != 0) return -2;
  McParams p{};
  p.nodes = mc->d_nodes;
  p.blocks = mc->d_blocks;
  p.ops = mc->d_ops;
  p.recv_blocks = mc->d_recv;
  p.err = mc->d_err;
  p.tile_bytes = mc->tile_bytes;
  p.timeout_ns = mc->timeout_ns;
  p.epoch = epoch;
  p.chunk_bytes = (uint32_t)mc->chunk_bytes;
  p.push_ctas = push_ctas;
  p.pull_ctas = pull_ctas;
  p.push_mode = mc->push_mode;
  p.pull_mode = mc->pull_mode;
  p.n_exec = n_exec;
  p.window = mc->window;
  p.wide_loads = mc->wide_loads;
  for (int i = 0; i < n_exec; ++i) {
    int n = exec_nodes[i];
    LP_CHECK(n >= 0 && n < mc->n_nodes, "lp_mc_run: exec node %d out of range", n);
    LP_CHECK(mc->nodes[n].kind == LP_NODE_GPU, "lp_mc_run: exec node %d is not a GPU node", n);
    p.exec[i] = mc->per_node[n];
  }
  if (pull_ctas > 0) {   // re-base the counters of the blocks this run pulls in-kernel
    CountReset r{};
    for (int i = 0; i < n_exec; ++i) {
      r.counts[i] = mc->nodes[exec_nodes[i]].counts;
      r.op_b[i] = p.exec[i].pull_b;
      r.op_e[i] = p.exec[i].pull_e;
    }
    r.ops = mc->d_ops;
    r.blocks = mc->d_blocks;
    r.epoch = epoch;
    count_reset_kernel<<<n_exec, 128, 0, (cudaStream_t)stream>>>(r);
    LP_CUDA(cudaGetLastError());
  }
  mc_kernel<<<per * n_exec, LP_MC_THREADS, smem, (cudaStream_t)stream>>>(p);
  LP_CUDA(cudaGetLastError());
  mc->last_epoch = epoch;
  return 0;
}

// ---------------------------------------------------------------------------
// Copy-engine executor.  Same transfer set, same tile flags, but every tile is
// moved by a DMA copy engine: the receiver's stream waits (cuStreamWaitValue32)
// until the sender's flag for the tile holds the epoch, issues a
// cudaMemcpyAsync of the tile (peer NVLink read, or PCIe from pinned host
// memory) and then publishes its own flag with a fenced cuStreamWriteValue32.
// Copy engines keep ~778 GB/s per direction while a GPU both sends and
// receives, where SM-issued peer traffic drops to ~673 GB/s
// (tools/p2p_micro.cu, profiles/), and they leave every SM free for
// execute-while-load serving.  Ops are dealt round-robin over `n_streams`
// streams so one slow upstream does not idle the node's ingress.
// driver entry points resolved through the runtime (no link-time libcuda
// dependency, so the library loads on CPU-only hosts for the ABI checks)
typedef CUresult (*PFN_waitv32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writev32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_waitv32 g_wait32 = nullptr;
static PFN_writev32 g_write32 = nullptr;

static int resolve_stream_memops() {
  if (g_wait32 && g_write32) return 0;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  LP_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q));
  LP_CHECK(q == cudaDriverEntryPointSuccess && fn, "cuStreamWaitValue32 unavailable");
  g_wait32 = (PFN_waitv32)fn;
  LP_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q));
  LP_CHECK(q == cudaDriverEntryPointSuccess && fn, "cuStreamWriteValue32 unavailable");
  g_write32 = (PFN_writev32)fn;
  return 0;
}
#define cuStreamWaitValue32 g_wait32
#define cuStreamWriteValue32 g_write32

// Enqueue ops `seq` (indices into h_ops) of `node` on the copy engines.
static int enqueue_ce(lp_mc* mc, int node, uint32_t epoch, const std::vector<int>& seq, int n_streams,
                      void* const* streams, void* const* block_events) {
  int k = 0;
  const bool dbg = getenv("LP_DEBUG_CE") != nullptr;
  for (int oi : seq) {
    const OpDev op = mc->h_ops[oi];
    if (dbg)
      fprintf(stderr, "lp_mc ce node %d: op %d step %d %d->%d block %d wait %d stream %d\n", node, oi, op.step,
              op.src, op.dst, op.block, op.wait, k % n_streams);
    const BlockDev bl = mc->blocks[op.block];
    const NodeDev src = mc->nodes[op.src];
    const NodeDev dst = mc->nodes[op.dst];
    CUstream s = (CUstream)streams[k % n_streams];
    for (int t = 0; t < bl.ntiles; ++t) {
      const int64_t lo = (int64_t)t * bl.tile;
      const int64_t n = std::min<int64_t>(bl.tile, bl.len - lo);
      if (op.wait) {
        CUresult r = cuStreamWaitValue32(s, (CUdeviceptr)(src.flags + bl.tile_base + t), epoch,
                                         CU_STREAM_WAIT_VALUE_GEQ);
        LP_CHECK(r == CUDA_SUCCESS, "lp_mc_run_ce: cuStreamWaitValue32 failed (%d)", (int)r);
      }
      LP_CUDA(cudaMemcpyAsync(dst.image + bl.off + lo, src.image + bl.off + lo, (size_t)n, cudaMemcpyDefault,
                              (cudaStream_t)s));
      CUresult r = cuStreamWriteValue32(s, (CUdeviceptr)(dst.flags + bl.tile_base + t), epoch,
                                        CU_STREAM_WRITE_VALUE_DEFAULT);
      LP_CHECK(r == CUDA_SUCCESS, "lp_mc_run_ce: cuStreamWriteValue32 failed (%d)", (int)r);
    }
    CUresult r = cuStreamWriteValue32(s, (CUdeviceptr)(dst.counts + op.block), epoch * (uint32_t)bl.ntiles,
                                      CU_STREAM_WRITE_VALUE_DEFAULT);
    LP_CHECK(r == CUDA_SUCCESS, "lp_mc_run_ce: cuStreamWriteValue32 failed (%d)", (int)r);
    if (dst.ready) {
      r = cuStreamWriteValue32(s, (CUdeviceptr)(dst.ready + op.block), epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
      LP_CHECK(r == CUDA_SUCCESS, "lp_mc_run_ce: ready write failed (%d)", (int)r);
    }
    if (block_events && block_events[op.block] && op.dst == node)
      LP_CUDA(cudaEventRecord((cudaEvent_t)block_events[op.block], (cudaStream_t)s));
    ++k;
  }
  return 0;
}

int lp_mc_run_ce(lp_mc* mc, int node, uint32_t epoch, int n_streams, void* const* streams,
                 void* const* block_events) {
  if (resolve_stream_memops() != 0) return -1;
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes, "lp_mc_run_ce: bad node");
  LP_CHECK(epoch >= 1 && n_streams >= 1 && streams, "lp_mc_run_ce: bad arguments");
  LP_CHECK(mc->nodes[node].kind == LP_NODE_GPU, "lp_mc_run_ce: node %d is not a GPU node", node);
  if (mc->dirty && compile(mc) != 0) return -2;
  const ExecDesc ex = mc->per_node[node];
  // direction 1: this node's copy engine pulls every block it receives;
  // direction 0: its copy engine pushes every block it sends (waits are then
  // on its OWN flags, flag writes land in the receiver's memory) and it still
  // pulls host-sourced blocks.  One step-ordered sequence of this node's
  // pushes and pulls: a push of a block this node itself pulls (e.g. from the
  // host) must be enqueued after that pull, or a single stream would wait on
  // itself.
  std::vector<int> seq;
  for (int oi = ex.push_b; oi < ex.push_e; ++oi) seq.push_back(oi);
  for (int oi = ex.pull_b; oi < ex.pull_e; ++oi) seq.push_back(oi);
  for (int oi = ex.dma_b; oi < ex.dma_e; ++oi) seq.push_back(oi);
  std::stable_sort(seq.begin(), seq.end(),
                   [&](int a, int b) { return mc->h_ops[a].step < mc->h_ops[b].step; });
  return enqueue_ce(mc, node, epoch, seq, n_streams, streams, block_events);
}

// Hybrid executor, PCIe half: with option host_dma=1 the transfers whose
// sender is a HOST node are left out of the kernel's op lists; this enqueues
// them (this node's host pulls, in step order) on the copy engines, while
// lp_mc_run on another stream relays the landed tiles over NVLink.
int lp_mc_run_host_dma(lp_mc* mc, int node, uint32_t epoch, int n_streams, void* const* streams,
                       void* const* block_events) {
  if (resolve_stream_memops() != 0) return -1;
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes, "lp_mc_run_host_dma: bad node");
  LP_CHECK(epoch >= 1 && n_streams >= 1 && streams, "lp_mc_run_host_dma: bad arguments");
  LP_CHECK(mc->host_dma || mc->ce_split, "lp_mc_run_host_dma: enable option host_dma or ce_split first");
  if (mc->dirty && compile(mc) != 0) return -2;
  const ExecDesc ex = mc->per_node[node];
  std::vector<int> seq;
  for (int oi = ex.dma_b; oi < ex.dma_e; ++oi) seq.push_back(oi);
  return enqueue_ce(mc, node, epoch, seq, n_streams, streams, block_events);
}

int lp_mc_landing_events(lp_mc* mc, int node, uint32_t epoch, void* stream, void* const* block_events) {
  if (resolve_stream_memops() != 0) return -1;
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && block_events && epoch >= 1,
           "lp_mc_landing_events: bad arguments");
  LP_CHECK(mc->nodes[node].kind == LP_NODE_GPU && mc->nodes[node].counts,
           "lp_mc_landing_events: node %d is not a GPU node with signals", node);
  if (mc->dirty && compile(mc) != 0) return -2;
  std::vector<char> recv(mc->n_blocks, 0);
  for (const OpDev& op : mc->h_ops)
    if (op.dst == node) recv[op.block] = 1;
  for (int b = 0; b < mc->n_blocks; ++b) {
    if (!recv[b] || !block_events[b]) continue;
    CUresult r = cuStreamWaitValue32((CUstream)stream, (CUdeviceptr)(mc->nodes[node].counts + b),
                                     epoch * (uint32_t)mc->blocks[b].ntiles, CU_STREAM_WAIT_VALUE_GEQ);
    LP_CHECK(r == CUDA_SUCCESS, "lp_mc_landing_events: cuStreamWaitValue32 failed (%d)", (int)r);
    LP_CUDA(cudaEventRecord((cudaEvent_t)block_events[b], (cudaStream_t)stream));
  }
  return 0;
}

// Ops the kernel (push + pull roles) and the host DMA would execute for node.
int lp_mc_node_ops(lp_mc* mc, int node, int* kernel_ops, int* dma_ops) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && kernel_ops && dma_ops, "lp_mc_node_ops: bad arguments");
  if (mc->dirty && compile(mc) != 0) return -2;
  const ExecDesc ex = mc->per_node[node];
  *kernel_ops = (ex.push_e - ex.push_b) + (ex.pull_e - ex.pull_b);
  *dma_ops = ex.dma_e - ex.dma_b;
  return 0;
}

int lp_mc_verify(lp_mc* mc, int node, uint32_t epoch, int ctas, uint64_t* sums_dev, void* stream) {
  if (resolve_stream_memops() != 0) return -1;
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && sums_dev, "lp_mc_verify: bad arguments");
  LP_CHECK(epoch >= 1 && ctas >= 1 && ctas <= 1024, "lp_mc_verify: bad epoch / CTA count");
  LP_CHECK(mc->nodes[node].kind == LP_NODE_GPU && mc->nodes[node].counts,
           "lp_mc_verify: node %d is not a GPU node with signals", node);
  if (mc->dirty && compile(mc) != 0) return -2;
  cudaStream_t s = (cudaStream_t)stream;
  LP_CUDA(cudaMemsetAsync(sums_dev, 0, sizeof(uint64_t) * mc->n_blocks, s));
  const NodeDev me = mc->nodes[node];
  // blocks in the step order they land; each one: a stream-ordered wait on the
  // node's own counter, then one checksum launch over the landed block
  for (int i = mc->vr_off[node]; i < mc->vr_off[node + 1]; ++i) {
    const int blk = mc->h_vorder[i];
    const BlockDev bl = mc->blocks[blk];
    CUresult r = cuStreamWaitValue32((CUstream)s, (CUdeviceptr)(me.counts + blk), epoch * (uint32_t)bl.ntiles,
                                     CU_STREAM_WAIT_VALUE_GEQ);
    LP_CHECK(r == CUDA_SUCCESS, "lp_mc_verify: cuStreamWaitValue32 failed (%d)", (int)r);
    const int64_t want = (bl.len / 16 + 4095) / 4096;           // >= 8 x 16 B per thread
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, want));
    block_sum_kernel<<<grid, 512, 0, s>>>(me.image + bl.off, bl.len,
                                           reinterpret_cast<unsigned long long*>(sums_dev) + blk);
    LP_CUDA(cudaGetLastError());
  }
  return 0;
}

int lp_mc_status(lp_mc* mc, void* stream, int* code) {
  LP_CHECK(mc && code, "lp_mc_status: null argument");
  LP_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int h = 0;
  LP_CUDA(cudaMemcpy(&h, mc->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  *code = h;
  if (h) {
    cudaMemset(mc->d_err, 0, sizeof(int));
    mc->failed = true;
    lp::set_error("lp_mc: watchdog expired waiting for a tile flag (a peer never delivered; %s)",
                  "multicast kernel");
    return -3;
  }
  return 0;
}

int lp_mc_arrivals(lp_mc* mc, int node, uint64_t* out_ns) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && out_ns, "lp_mc_arrivals: bad arguments");
  LP_CHECK(mc->nodes[node].arrival, "lp_mc_arrivals: node %d has no signal area", node);
  if (poll_stream(mc) != 0) return -1;
  LP_CUDA(cudaMemcpyAsync(out_ns, mc->nodes[node].arrival, sizeof(uint64_t) * mc->n_blocks, cudaMemcpyDefault,
                          mc->poll));
  LP_CUDA(cudaStreamSynchronize(mc->poll));
  return 0;
}

int lp_mc_block_complete(lp_mc* mc, int node, uint32_t epoch, int32_t* out_flags) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && out_flags, "lp_mc_block_complete: bad arguments");
  LP_CHECK(mc->nodes[node].counts, "lp_mc_block_complete: node %d has no signal area", node);
  std::vector<uint32_t> c(mc->n_blocks);
  if (poll_stream(mc) != 0) return -1;
  LP_CUDA(cudaMemcpyAsync(c.data(), mc->nodes[node].counts, sizeof(uint32_t) * mc->n_blocks, cudaMemcpyDefault,
                          mc->poll));
  LP_CUDA(cudaStreamSynchronize(mc->poll));
  for (int i = 0; i < mc->n_blocks; ++i)
    out_flags[i] = c[i] >= epoch * (uint32_t)mc->blocks[i].ntiles ? 1 : 0;
  return 0;
}

}  // extern "C"
