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
#include <algorithm>
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
  int32_t tile_base;
  int32_t ntiles;
};
struct OpDev {
  int32_t block, src, dst, wait;
};
struct ExecDesc {
  int32_t node, push_b, push_e, pull_b, pull_e, recv_b, recv_e, pad;
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
  int push_ctas, pull_ctas, n_exec;
  ExecDesc exec[LP_MAX_EXEC];
};

__device__ __forceinline__ bool wait_flag(const uint32_t* f, uint32_t epoch, uint64_t t0,
                                          uint64_t timeout_ns, int* err) {
  uint32_t spins = 0;
  while (lp::ld_acquire_sys(f) != epoch) {
    if (++spins > 64) {
      lp::nanosleep(200);
      if ((spins & 1023) == 0 && lp::globaltimer() - t0 > timeout_ns) {
        atomicExch(err, 1);
        return false;
      }
    }
  }
  return true;
}

__device__ __forceinline__ void copy_tile(const char* __restrict__ s, char* __restrict__ d, int64_t n) {
  constexpr int U = 8;
  const int4* s4 = reinterpret_cast<const int4*>(s);
  int4* d4 = reinterpret_cast<int4*>(d);
  const int64_t n16 = n >> 4;
  const int T = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + (int64_t)(U - 1) * T < n16; i += (int64_t)U * T) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = lp::ld_stream16(s4 + i + (int64_t)u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) lp::st16(d4 + i + (int64_t)u * T, v[u]);
  }
  for (; i < n16; i += T) lp::st16(d4 + i, lp::ld_stream16(s4 + i));
}

__global__ void __launch_bounds__(LP_MC_THREADS) mc_kernel(const McParams p) {
  const int per = p.push_ctas + p.pull_ctas;
  const int e = blockIdx.x / per;
  const int local = blockIdx.x % per;
  const ExecDesc ex = p.exec[e];
  const bool pusher = local < p.push_ctas;
  const int lane = pusher ? local : local - p.push_ctas;
  const int lanes = pusher ? p.push_ctas : p.pull_ctas;
  const int ob = pusher ? ex.push_b : ex.pull_b;
  const int oe = pusher ? ex.push_e : ex.pull_e;
  const uint32_t epoch = p.epoch;
  __shared__ int s_ok;
  uint64_t t0 = 0;
  if (threadIdx.x == 0) {
    t0 = lp::globaltimer();
    s_ok = 1;
  }

  for (int oi = ob; oi < oe; ++oi) {
    const OpDev op = p.ops[oi];
    const BlockDev bl = p.blocks[op.block];
    const NodeDev src = p.nodes[op.src];
    const NodeDev dst = p.nodes[op.dst];
    for (int t = lane; t < bl.ntiles; t += lanes) {
      const int64_t lo = (int64_t)t * p.tile_bytes;
      const int64_t n = min(p.tile_bytes, bl.len - lo);
      if (op.wait) {
        if (threadIdx.x == 0 && !wait_flag(src.flags + bl.tile_base + t, epoch, t0, p.timeout_ns, p.err))
          s_ok = 0;
        __syncthreads();
        if (!s_ok) return;
      }
      copy_tile(src.image + bl.off + lo, dst.image + bl.off + lo, n);
      __syncthreads();  // every thread's stores of this tile precede the flag
      if (threadIdx.x == 0) {
        lp::fence_sys();
        lp::st_release_sys(dst.flags + bl.tile_base + t, epoch);
        const uint32_t old = lp::atom_add_release_sys(dst.counts + op.block, 1u);
        if (old + 1u == epoch * (uint32_t)bl.ntiles) {
          dst.arrival[op.block] = lp::globaltimer();
          if (dst.ready) lp::st_release_sys(dst.ready + op.block, epoch);
        }
      }
    }
  }

  // the node is complete when every tile it receives this epoch has landed
  if (pusher) {
    const NodeDev me = p.nodes[ex.node];
    for (int r = ex.recv_b; r < ex.recv_e; ++r) {
      const BlockDev bl = p.blocks[p.recv_blocks[r]];
      for (int t = lane; t < bl.ntiles; t += lanes) {
        if (threadIdx.x == 0 && s_ok &&
            !wait_flag(me.flags + bl.tile_base + t, epoch, t0, p.timeout_ns, p.err))
          s_ok = 0;
      }
    }
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
  int dev = 0;
  NodeDev* d_nodes = nullptr;
  BlockDev* d_blocks = nullptr;
  OpDev* d_ops = nullptr;
  int32_t* d_recv = nullptr;
  int* d_err = nullptr;
  int max_resident = 0;
};

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
  std::vector<OpDev> ops;
  std::vector<int32_t> recv;
  mc->per_node.assign(N, ExecDesc{});
  for (int n = 0; n < N; ++n) {
    ExecDesc& d = mc->per_node[n];
    d.node = n;
    d.push_b = (int)ops.size();
    for (const Row& r : rows)
      if (r.snd == n && mc->nodes[n].kind == LP_NODE_GPU)
        ops.push_back(OpDev{r.blk, r.snd, r.rcv, is_src[r.snd] ? 0 : 1});
    d.push_e = (int)ops.size();
    d.pull_b = (int)ops.size();
    for (const Row& r : rows)
      if (r.rcv == n && mc->nodes[r.snd].kind == LP_NODE_HOST) ops.push_back(OpDev{r.blk, r.snd, r.rcv, 0});
    d.pull_e = (int)ops.size();
    d.recv_b = (int)recv.size();
    for (const Row& r : rows)
      if (r.rcv == n) recv.push_back(r.blk);
    d.recv_e = (int)recv.size();
  }
  LP_CUDA(cudaSetDevice(mc->dev));
  if (mc->d_ops) cudaFree(mc->d_ops);
  if (mc->d_recv) cudaFree(mc->d_recv);
  mc->d_ops = nullptr;
  mc->d_recv = nullptr;
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

int lp_mc_create(lp_mc** out, int n_nodes, int n_blocks, const int64_t* block_off,
                 const int64_t* block_len, int64_t tile_bytes) {
  LP_CHECK(out && n_nodes >= 1 && n_nodes <= 4096 && n_blocks >= 1, "lp_mc_create: bad arguments");
  LP_CHECK(tile_bytes >= 4096 && tile_bytes % 16 == 0, "lp_mc_create: tile_bytes must be >=4096 and a multiple of 16");
  lp_mc* mc = new lp_mc();
  mc->n_nodes = n_nodes;
  mc->n_blocks = n_blocks;
  mc->tile_bytes = tile_bytes;
  int64_t tiles = 0;
  for (int i = 0; i < n_blocks; ++i) {
    if (block_off[i] % 16 || block_len[i] % 16 || block_len[i] <= 0) {
      delete mc;
      lp::set_error("lp_mc_create: block %d offset/length must be positive multiples of 16", i);
      return -2;
    }
    int64_t nt = (block_len[i] + tile_bytes - 1) / tile_bytes;
    mc->blocks.push_back(BlockDev{block_off[i], block_len[i], (int32_t)tiles, (int32_t)nt});
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
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mc_kernel, LP_MC_THREADS, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, mc->dev);
  mc->max_resident = occ * sms;
  *out = mc;
  return 0;
}

int lp_mc_destroy(lp_mc* mc) {
  if (!mc) return 0;
  cudaSetDevice(mc->dev);
  cudaFree(mc->d_nodes);
  cudaFree(mc->d_blocks);
  cudaFree(mc->d_ops);
  cudaFree(mc->d_recv);
  cudaFree(mc->d_err);
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
  return 0;
}

int lp_mc_run(lp_mc* mc, const int32_t* exec_nodes, int n_exec, uint32_t epoch, int push_ctas,
              int pull_ctas, void* stream) {
  LP_CHECK(mc && n_exec >= 1 && n_exec <= LP_MAX_EXEC, "lp_mc_run: n_exec must be in [1, %d]", LP_MAX_EXEC);
  LP_CHECK(epoch >= 1, "lp_mc_run: epoch must be >= 1");
  LP_CHECK(push_ctas >= 1 && pull_ctas >= 0, "lp_mc_run: need push_ctas >= 1, pull_ctas >= 0");
  const int per = push_ctas + pull_ctas;
  LP_CHECK(per * n_exec <= mc->max_resident,
           "lp_mc_run: %d CTAs exceed the %d co-resident CTAs the dataflow needs", per * n_exec,
           mc->max_resident);
  if (mc->dirty && compile(mc) != 0) return -2;
  McParams p{};
  p.nodes = mc->d_nodes;
  p.blocks = mc->d_blocks;
  p.ops = mc->d_ops;
  p.recv_blocks = mc->d_recv;
  p.err = mc->d_err;
  p.tile_bytes = mc->tile_bytes;
  p.timeout_ns = 20ull * 1000 * 1000 * 1000;
  p.epoch = epoch;
  p.push_ctas = push_ctas;
  p.pull_ctas = pull_ctas;
  p.n_exec = n_exec;
  for (int i = 0; i < n_exec; ++i) {
    int n = exec_nodes[i];
    LP_CHECK(n >= 0 && n < mc->n_nodes, "lp_mc_run: exec node %d out of range", n);
    LP_CHECK(mc->nodes[n].kind == LP_NODE_GPU, "lp_mc_run: exec node %d is not a GPU node", n);
    p.exec[i] = mc->per_node[n];
  }
  mc_kernel<<<per * n_exec, LP_MC_THREADS, 0, (cudaStream_t)stream>>>(p);
  LP_CUDA(cudaGetLastError());
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
    lp::set_error("lp_mc: watchdog expired waiting for a tile flag (a peer never delivered)");
    return -3;
  }
  return 0;
}

int lp_mc_arrivals(lp_mc* mc, int node, uint64_t* out_ns) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && out_ns, "lp_mc_arrivals: bad arguments");
  LP_CHECK(mc->nodes[node].arrival, "lp_mc_arrivals: node %d has no signal area", node);
  LP_CUDA(cudaMemcpy(out_ns, mc->nodes[node].arrival, sizeof(uint64_t) * mc->n_blocks, cudaMemcpyDefault));
  return 0;
}

int lp_mc_block_complete(lp_mc* mc, int node, uint32_t epoch, int32_t* out_flags) {
  LP_CHECK(mc && node >= 0 && node < mc->n_nodes && out_flags, "lp_mc_block_complete: bad arguments");
  LP_CHECK(mc->nodes[node].counts, "lp_mc_block_complete: node %d has no signal area", node);
  std::vector<uint32_t> c(mc->n_blocks);
  LP_CUDA(cudaMemcpy(c.data(), mc->nodes[node].counts, sizeof(uint32_t) * mc->n_blocks, cudaMemcpyDefault));
  for (int i = 0; i < mc->n_blocks; ++i)
    out_flags[i] = c[i] >= epoch * (uint32_t)mc->blocks[i].ntiles ? 1 : 0;
  return 0;
}

}  // extern "C"
