/* lambdapipe — C ABI of the B200-native λScale scaling hot path.
 *
 * The reference (blockcast, pkg/src/blockcast/) has no native layer: its data
 * plane is a cost formula (simengine.py:95-103) and an event that adds block
 * ids to a set (simengine.py:628-644).  This ABI is the bottom layer the
 * reference's planner would call to move real bytes and run real tokens; the
 * Python package paper_2502_09922_b200 wraps it with the reference's own
 * function names (INTEGRATION.md shows the ctypes binding a blockcast
 * maintainer would add).
 *
 * Conventions
 *   - every entry point returns 0 on success, <0 on failure; lp_last_error()
 *     returns a thread-local message for the last failure on this thread;
 *   - buffers are borrowed (device pointers in this process: local, CUDA-IPC
 *     mapped peers, or device aliases of registered pinned host memory);
 *     nothing allocated by the caller is freed by the library;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *   - work is asynchronous on the given stream unless stated otherwise.
 */
#ifndef LAMBDAPIPE_H
#define LAMBDAPIPE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library / device plumbing ----------------------------------------- */
int         lp_version(void);
const char* lp_last_error(void);
int lp_device_count(int* n);
int lp_set_device(int dev);
/* launch decoder kernels with programmatic dependent launch (this thread);
 * meant for CUDA-graph capture, where it overlaps each kernel's prologue and
 * weight prefetch with the previous kernel (env LP_PDL=0 forces it off) */
int lp_set_pdl(int on);
int lp_sync_device(int dev);
/* cudaDeviceEnablePeerAccess(dev -> peer); already-enabled is not an error */
int lp_enable_peer(int dev, int peer);
int lp_malloc(int dev, int64_t bytes, void** out);
int lp_free(int dev, void* ptr);
int lp_memset(void* dst, int value, int64_t bytes, void* stream);
int lp_memcpy(void* dst, const void* src, int64_t bytes, void* stream); /* cudaMemcpyDefault */
/* CUDA IPC: 64-byte opaque handle for a device allocation from lp_malloc */
int lp_ipc_get(void* dev_ptr, void* handle64);
int lp_ipc_open(int dev, const void* handle64, void** out);
int lp_ipc_close(void* ptr);
/* pin + map host memory (e.g. a shared-memory segment); returns device alias */
int lp_host_register(void* host, int64_t bytes, void** dev_alias);
int lp_host_unregister(void* host);
int lp_stream_create(int dev, void** stream);
int lp_stream_destroy(void* stream);
int lp_stream_sync(void* stream);
int lp_event_create(void** ev);
int lp_event_destroy(void* ev);
int lp_event_record(void* ev, void* stream);
int lp_event_elapsed_ms(void* start, void* end, float* ms);

/* ---- synthetic packed image + per-block checksums ----------------------
 * Replaces the reference's "bytes never move" block model
 * (multicast.py:153-173 block sizes; modelmgr.py:238-259 packing): the image
 * holds real tensors.  Tensor t occupies [off[t], off[t]+numel[t]*2) and is
 * filled with bf16 values from the counter-based generator (oracle/dataplane.c
 * lp_ref_fill restates it): kind 0 = random in [-2^scale_exp, 2^scale_exp),
 * kind 1 = ones, kind 2 = zeros. */
int lp_fill_tensors(void* base, int n_tensors, const int64_t* off, const int64_t* numel,
                    const int32_t* kind, const int32_t* scale_exp, uint64_t seed, void* stream);
/* out[i] = sum_w mix64(word_w ^ w*K) over 8-byte words of block i (wraps mod 2^64) */
int lp_block_checksums(const void* base, int n_blocks, const int64_t* off, const int64_t* len,
                       uint64_t* out_host, void* stream);

/* ---- λPipe multicast engine ----------------------------------------------
 * Executes a reference schedule (schedule_to_lines, multicast.py:546-551) as
 * a dataflow: each transfer (step, sender, receiver, block) becomes a push of
 * the block's tiles from sender to receiver over NVLink (in-kernel 16-byte
 * peer stores), or, when the sender is a HOST node, a pull of the tiles by
 * the receiver over PCIe from mapped pinned memory.  A relay forwards tile t
 * of a block as soon as tile t landed (chunk cut-through).  The transfer set,
 * each sender's send order and each receiver's delivered bytes are exactly
 * the schedule's (replaces simengine.py:594-596 + :628-644). */
typedef struct lp_mc lp_mc;
#define LP_NODE_GPU  0
#define LP_NODE_HOST 1
int lp_mc_create(lp_mc** out, int n_nodes, int n_blocks, const int64_t* block_off,
                 const int64_t* block_len, int64_t tile_bytes);
/* lp_mc_create with a tile size per block (the split executor: copy-engine
 * blocks in large tiles, in-kernel blocks in small ones); the smallest tile
 * bounds lp_mc_configure's chunk */
int lp_mc_create_tiled(lp_mc** out, int n_nodes, int n_blocks, const int64_t* block_off,
                       const int64_t* block_len, const int64_t* block_tile);
int lp_mc_destroy(lp_mc* mc);
/* bytes of the per-node signal area (tile flags, block counters, arrivals) */
int lp_mc_signal_bytes(const lp_mc* mc, int64_t* bytes);
/* image/signals: device-visible pointers in this process; host nodes pass
 * signals = NULL.  ready_host (optional) = device alias of pinned host words,
 * one u32 per block, set to the epoch when the block is complete. */
int lp_mc_set_node(lp_mc* mc, int node, int kind, void* image, void* signals, void* ready_host);
/* xfers = n_xfers x 4 int32 rows (step, sender, receiver, block), any order;
 * sources hold every block before step 0 (multicast.py:111-124). */
int lp_mc_set_schedule(lp_mc* mc, const int32_t* xfers, int n_xfers,
                       const int32_t* sources, int n_sources);
/* run every transfer whose executor is in exec_nodes (see lp_mc_configure);
 * push CTAs execute pushes, pull CTAs execute pulls; each exec node's kernel
 * also waits until every tile pushed into it this epoch landed.  Block
 * counters of in-kernel pulls are re-based to (epoch - 1) x tiles first, so
 * any later epoch works; runs with push CTAs need consecutive epochs.  After
 * a watchdog failure (lp_mc_status -3) the handle refuses runs until
 * lp_mc_reset_signals (then restart at epoch 1). */
int lp_mc_run(lp_mc* mc, const int32_t* exec_nodes, int n_exec, uint32_t epoch,
              int push_ctas, int pull_ctas, void* stream);
/* direction 0 = push: a GPU sender's CTAs store its blocks into the receiver
 * (NVLink writes); 1 = pull (default): every transfer is executed by its
 * receiver, which reads the sender's tiles (NVLink or PCIe reads) once the
 * sender's flag for the tile holds the epoch.  Host-sourced transfers are
 * always pulled.  push_mode/pull_mode pick the copy engine of each role:
 * 0 = LDG/STG 16-byte vectors on 512 threads, 1 = TMA bulk copies
 * (cp.async.bulk global->smem->global, one issuing thread, 12-slot smem ring
 * of chunk_bytes).  window (>= 1; 0 keeps the current value) = how many
 * consecutive ops of its list an LDG-role CTA may interleave when the oldest
 * op's next tile is not ready yet. */
int lp_mc_configure(lp_mc* mc, int direction, int push_mode, int pull_mode, int64_t chunk_bytes,
                    int window);
/* Copy-engine executor for one GPU node: enqueue, on the node's `n_streams`
 * streams, its ops as per-tile cuStreamWaitValue32(sender's flag) ->
 * cudaMemcpyAsync -> cuStreamWriteValue32(receiver's flag); no SM work.
 * direction 1 (lp_mc_configure): pulls everything it receives; direction 0:
 * pushes everything it sends (waits on its own flags) and pulls host-sourced
 * blocks.  block_events (optional, n_blocks entries, NULL to skip) are
 * recorded after each pulled block's last tile.  Every stream that may park a
 * wait needs its own hardware connection (CUDA_DEVICE_MAX_CONNECTIONS >=
 * streams on the device), else a parked wait stalls unrelated streams. */
int lp_mc_run_ce(lp_mc* mc, int node, uint32_t epoch, int n_streams, void* const* streams,
                 void* const* block_events);
/* Hybrid executor (option host_dma = 1): the transfers whose sender is a HOST
 * node leave the kernel's op lists and are enqueued here, per receiving GPU
 * node, on the copy engines (pinned-host DMA over PCIe, per-tile flag writes);
 * lp_mc_run on another stream of the same device relays the landed tiles over
 * NVLink, waiting on those flags.  Replaces the h2d leg of the reference's
 * step cost (simengine.py:95-103, h2d_Bps) with real pinned DMA overlapped
 * with the GPU->GPU relay. */
int lp_mc_run_host_dma(lp_mc* mc, int node, uint32_t epoch, int n_streams, void* const* streams,
                       void* const* block_events);
/* Landing events without touching peer memory: on `stream` (a stream of
 * `node`'s device), for every block `node` receives this epoch, wait until
 * its OWN block counter is complete (cuStreamWaitValue32 on local memory)
 * and record block_events[block] (created on that device).  Lets a caller
 * time per-block arrivals whichever executor/direction delivers them. */
int lp_mc_landing_events(lp_mc* mc, int node, uint32_t epoch, void* stream, void* const* block_events);
/* Verify-as-it-lands: zero sums_dev[n_blocks] (device memory), then for every
 * block `node` receives this epoch, in step order, enqueue on `stream` a
 * stream-ordered wait on the node's own block counter (cuStreamWaitValue32,
 * no SM held) followed by one checksum launch (<= `ctas` CTAs) over that
 * block (the lp_block_checksums function); entries of blocks the node does
 * not receive stay 0.  Enqueue it AFTER the epoch's producers (lp_mc_run /
 * _run_ce / _run_host_dma), on another stream of the node's device: nothing
 * then depends on cross-stream concurrency (runs under ncu's serialisation). */
int lp_mc_verify(lp_mc* mc, int node, uint32_t epoch, int ctas, uint64_t* sums_dev, void* stream);
/* number of ops node executes in-kernel (push + pull roles) and on the host
 * DMA path (0 unless host_dma) under the current configuration */
int lp_mc_node_ops(lp_mc* mc, int node, int* kernel_ops, int* dma_ops);
/* tunables: "wide_loads" (0/1: 256 B L2 fetch granule on LDG-role loads),
 * "window" (1..8), "timeout_ms" (flag-wait watchdog, default 20000),
 * "host_dma" (0/1: HOST-sourced transfers on the copy engines, see
 * lp_mc_run_host_dma), "ce_split" (m >= 0: GPU->GPU transfers of blocks with
 * block % m == 0 also leave the kernel for lp_mc_run_host_dma's copy-engine
 * list, so DMA engines and SMs share every link; 0 = off) */
int lp_mc_set_option(lp_mc* mc, const char* name, int64_t value);
/* synchronise `stream`; code = 1 (and return -3) if a flag wait timed out */
int lp_mc_status(lp_mc* mc, void* stream, int* code);
/* zero a node's signal area (call on every node, then barrier, before epoch 1) */
int lp_mc_reset_signals(lp_mc* mc, int node, void* stream);
/* synchronous: per-block arrival globaltimer (ns) at `node` for the last run,
 * and the executed-transfer count per node (sanity) */
int lp_mc_arrivals(lp_mc* mc, int node, uint64_t* out_ns);
int lp_mc_block_complete(lp_mc* mc, int node, uint32_t epoch, int32_t* out_flags);

/* ---- Llama decoder kernels (execute-while-load + local generate) --------
 * The reference models a token as `per_block_compute_ms` per block
 * (simengine.py:323-343) and prefill as `prompt x prefill_ms_per_token`
 * (:320-321); these compute the real thing on the packed image.  Weights
 * are bf16 [out, in] row-major, activations bf16, residual fp32.
 *
 * Tensor-core GEMM (tcgen05.mma + TMEM + TMA): Y[t,n] = sum_k X[t,k] W[n,k].
 * epilogue 0: out_f32[t*ldo+n] += Y (split_k >= 1 allowed)
 * epilogue 1: out_f32[t*ldo+n]  = Y (split_k must be 1) */
int lp_gemm_bf16(const void* W, int64_t n_rows, int64_t k, const void* X, int64_t tokens, void* out,
                 int64_t ldo, int epilogue, int split_k, void* stream);
/* fused gate/up + SwiGLU: out_bf16[t*ldo+n] = silu(X Wg^T)[t,n] * (X Wu^T)[t,n] */
int lp_gemm_swiglu(const void* W_gate, const void* W_up, int64_t n_rows, int64_t k, const void* X,
                   int64_t tokens, void* out_bf16, int64_t ldo, void* stream);
int lp_embed(const void* table, int64_t d, const int32_t* tokens, int64_t T, float* x, void* stream);
/* y_bf16[t,:] = x[t,:] * rsqrt(mean(x[t,:]^2) + eps) * w; d % 4 == 0 */
int lp_rmsnorm(const float* x, const void* w, int64_t T, int64_t d, float eps, void* y, void* stream);
/* lp_rmsnorm that also zeroes the fp32 [T, zero_cols] buffer `zero` (the
 * next split-K GEMM's accumulator) in the same launch */
int lp_rmsnorm_zero(const float* x, const void* w, int64_t T, int64_t d, float eps, void* y, float* zero,
                    int64_t zero_cols, void* stream);
/* RoPE (HF rotate_half) on q/k of qkv fp32 [T,(H+2KV)*hd]; q -> q_out bf16,
 * k appended to k_cache[seq][kv][pos][hd] bf16, v to v_cache (same layout)
 * fp16 (attention's P.V runs in fp16) */
int lp_rope_kv(const float* qkv, int64_t T, int n_heads, int n_kv, int head_dim, const int32_t* pos,
               const int32_t* seq, float theta, void* q_out, void* k_cache, void* v_cache, int64_t max_len,
               void* stream);
/* ragged causal GQA attention: token t attends to 0..pos[t] of seq[t]; k
 * cache bf16, v cache fp16 (lp_rope_kv), out bf16.  head_dim 32..128
 * (multiple of 32), H/KV <= 8.  T*KV >= 1024 (prefill), head_dim 64/128,
 * max_len > 160 or H/KV >= 4:
 * tcgen05/TMEM kernel (128-row tiles of R tokens x H/KV heads, TMA-fed,
 * two tiles per CTA, fp32 S and O in TMEM, fp16 P kept in TMEM as the P.V
 * MMA's A operand; LP_ATTN_TC selects the other variants, 0 = mma.sync);
 * decode:
 * mma.sync kernels (few rows, K/V streaming bound; long caches split keys
 * over a thread-block cluster); other head sizes: CUDA-core online softmax. */
int lp_attention(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos,
                 const int32_t* seq, int64_t T, int n_heads, int n_kv, int head_dim, int64_t max_len,
                 float scale, void* out, void* stream);
/* stage->stage activation hand-off: copy `bytes` (multiple of 16) into the
 * next stage's buffer (peer pointer, NVLink stores); if flag != NULL, release
 * *flag = value (sys scope) after all bytes landed (scratch: zeroed u32 on the
 * producer, reused) */
int lp_handoff(const void* src, void* dst, int64_t bytes, uint32_t* flag, uint32_t value, uint32_t* scratch,
               void* stream);
/* greedy argmax per row; top2 (optional, [T,2]) = best and runner-up logit */
int lp_argmax(const float* logits, int64_t T, int64_t V, int32_t* out, float* top2, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LAMBDAPIPE_H */
