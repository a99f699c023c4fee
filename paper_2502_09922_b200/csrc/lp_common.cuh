// Shared helpers for the lambdapipe C-ABI library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "lambdapipe is built for sm_100a only"
#endif

namespace lp {

// thread-local last error, surfaced by lp_last_error()
void set_error(const char* fmt, ...);

#define LP_CUDA(call)                                                             \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      lp::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #call,                  \
                    cudaGetErrorString(_e));                                      \
      return -1;                                                                  \
    }                                                                             \
  } while (0)

#define LP_CHECK(cond, ...)                                                       \
  do {                                                                            \
    if (!(cond)) {                                                                \
      lp::set_error(__VA_ARGS__);                                                 \
      return -2;                                                                  \
    }                                                                             \
  } while (0)

// The library shares the CUDA runtime (and so the calling thread's current
// device) with its host process: an entry point that needs a device switches
// to it for the call and restores the caller's device on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------------------
// PTX memory-model helpers.  Flags cross GPUs over NVLink, so release/acquire
// are .sys scoped; data moves with 16-byte vectors.

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_release_sys(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.release.sys.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void nanosleep(uint32_t ns) { asm volatile("nanosleep.u32 %0;" ::"r"(ns)); }

// streaming 16-byte load that does not allocate in L1 (data is read once)
__device__ __forceinline__ int4 ld_stream16(const int4* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// same, with a 256-byte L2 fetch granule: remote (NVLink) and host (PCIe)
// reads then go out as 256 B requests instead of 32-128 B sectors
__device__ __forceinline__ int4 ld_stream16_l2_256(const int4* p) {
  int4 r;
  asm volatile("ld.global.cg.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st16(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// splitmix64 finaliser: the mixing function shared by the synthetic weight
// generator and the block checksum (restated in C in oracle/dataplane.c).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}


// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Decoder kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so kernel i+1 is
// scheduled while kernel i drains: it does its prologue (barrier init, TMEM
// alloc, tensor-map prefetch, even the first weight TMA loads, which do not
// depend on kernel i) and then waits in pdl_wait() for kernel i's results.
// pdl_trigger() is issued by every CTA once it is running, so all of a grid's
// CTAs are resident before dependents can take resources (no starvation).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();   // lp_set_pdl(1) and env LP_PDL != 0

// tcgen05 prefill attention (lp_attn_tc.cu): 0 = launched, 1 = shape not
// covered (use another kernel), < 0 = error
int attention_tc(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos, const int32_t* seq,
                 int64_t T, int n_heads, int n_kv, int head_dim, int64_t max_len, float scale, void* out,
                 cudaStream_t s);

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // PDL pays off inside captured graphs (measured: decode step 3.90 -> 3.60 ms);
  // on eagerly launched streams it costs host time (prefill 39 -> 58 ms), so
  // the host side switches it on around graph captures (lp_set_pdl)
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// launch() with a thread-block cluster of `cz` CTAs along grid z
template <typename... KArgs, typename... Args>
cudaError_t launch_cluster_z(void (*kern)(KArgs...), dim3 grid, dim3 block, unsigned cz, size_t smem,
                             cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = cz;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA, non-tensor) helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking probe (try_wait may suspend the thread for a while)
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global bulk copy (destination may be a peer GPU's memory)
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// runtime-N dispatch (N clamped to [0, 15]); waits until <= N groups pending
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  switch (n <= 0 ? 0 : (n >= 15 ? 15 : n)) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    case 3: bulk_wait_read<3>(); break;
    case 4: bulk_wait_read<4>(); break;
    case 5: bulk_wait_read<5>(); break;
    case 6: bulk_wait_read<6>(); break;
    case 7: bulk_wait_read<7>(); break;
    case 8: bulk_wait_read<8>(); break;
    case 9: bulk_wait_read<9>(); break;
    case 10: bulk_wait_read<10>(); break;
    case 11: bulk_wait_read<11>(); break;
    case 12: bulk_wait_read<12>(); break;
    case 13: bulk_wait_read<13>(); break;
    case 14: bulk_wait_read<14>(); break;
    default: bulk_wait_read<15>(); break;
  }
}
__device__ __forceinline__ void bulk_wait_n(int n) {
  switch (n <= 0 ? 0 : (n >= 15 ? 15 : n)) {
    case 0: bulk_wait<0>(); break;
    case 1: bulk_wait<1>(); break;
    case 2: bulk_wait<2>(); break;
    case 3: bulk_wait<3>(); break;
    case 4: bulk_wait<4>(); break;
    case 5: bulk_wait<5>(); break;
    case 6: bulk_wait<6>(); break;
    case 7: bulk_wait<7>(); break;
    case 8: bulk_wait<8>(); break;
    case 9: bulk_wait<9>(); break;
    case 10: bulk_wait<10>(); break;
    case 11: bulk_wait<11>(); break;
    case 12: bulk_wait<12>(); break;
    case 13: bulk_wait<13>(); break;
    case 14: bulk_wait<14>(); break;
    default: bulk_wait<15>(); break;
  }
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

}  // namespace lp
