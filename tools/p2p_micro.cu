// NVLink peer-copy microbenchmark (dev tool): what rate can SM-issued peer
// traffic reach on B200, by mechanism and CTA count?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_micro tools/p2p_micro.cu
//   ./p2p_micro  (needs 2 GPUs)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <chrono>
#include "../paper_2502_09922_b200/csrc/lp_common.cuh"

namespace lp {
void set_error(const char*, ...) {}
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// mode 0: local-read, remote STG.128 (push); mode 1: remote LDG.128, local STG (pull)
template <int U>
__global__ void __launch_bounds__(512) vec_copy(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
  const int64_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n16, lo + per);
  int64_t i = lo + threadIdx.x;
  for (; i + (U - 1) * 512 < hi; i += U * 512) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = lp::ld_stream16(src + i + u * 512);
#pragma unroll
    for (int u = 0; u < U; ++u) lp::st16(dst + i + u * 512, v[u]);
  }
  for (; i < hi; i += 512) lp::st16(dst + i, lp::ld_stream16(src + i));
}

// TMA: g2s + s2g ring, one thread; S slots of CH bytes, LA loads ahead
template <int S, int LA>
__global__ void __launch_bounds__(32) tma_copy(const char* src, char* dst, int64_t bytes, int ch) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t bars[S];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i) lp::mbar_init(&bars[i], 1);
  lp::fence_mbar_init();
  const int64_t per = (bytes / gridDim.x) / ch * ch;
  const int64_t lo = blockIdx.x * per;
  const int64_t n = per / ch;
  int64_t ql = 0, qs = 0;
  while (qs < n) {
    if (ql < n && ql - qs < LA) {
      int slot = ql % S;
      if (ql >= S) lp::bulk_wait_read_n((int)(qs - 1 - (ql - S)));
      lp::mbar_expect_tx(&bars[slot], ch);
      lp::bulk_g2s(ring + slot * ch, src + lo + ql * ch, ch, &bars[slot]);
      ++ql;
    } else {
      int slot = qs % S;
      lp::mbar_wait(&bars[slot], (qs / S) & 1);
      lp::bulk_s2g(dst + lo + qs * ch, ring + slot * ch, ch);
      lp::bulk_commit();
      ++qs;
    }
  }
  lp::bulk_wait<0>();
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 3) { printf("need 3 GPUs\n"); return 0; }
  const int64_t bytes = 4ll << 30;
  char* buf[4][2];
  cudaStream_t st[4];
  for (int d = 0; d < n && d < 4; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&buf[d][0], bytes)); CK(cudaMalloc(&buf[d][1], bytes));
    CK(cudaMemset(buf[d][0], d + 1, bytes));
    CK(cudaStreamCreate(&st[d]));
    for (int pe = 0; pe < n && pe < 4; ++pe) if (pe != d) CK(cudaDeviceEnablePeerAccess(pe, 0));
  }
  int ng = n < 4 ? n : 4;
  auto run = [&](const char* name, auto body) {
    for (int w = 0; w < 2; ++w) body();
    for (int d = 0; d < ng; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int r = 0; r < 5; ++r) body();
    for (int d = 0; d < ng; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    double ms = std::chrono::duration<double, std::milli>(std::chrono::high_resolution_clock::now() - t0).count();
    printf("%-60s per-stream %7.1f GB/s\n", name, 5.0 * bytes / (ms * 1e-3) / 1e9);
  };
  const int C = 64;
  // dst device d pulls from src device s: kernel on d reads buf[s][0] writes buf[d][1]
  auto pull = [&](int d, int s) { CK(cudaSetDevice(d)); vec_copy<8><<<C, 512, 0, st[d]>>>((const int4*)buf[s][0], (int4*)buf[d][1], bytes / 16); };
  auto push = [&](int s, int d) { CK(cudaSetDevice(s)); vec_copy<8><<<C, 512, 0, st[s]>>>((const int4*)buf[s][0], (int4*)buf[d][1], bytes / 16); };
  auto ce = [&](int s, int d) { CK(cudaSetDevice(s)); CK(cudaMemcpyPeerAsync(buf[d][1], d, buf[s][0], s, bytes, st[s])); };
  auto tpull = [&](int d, int s, int c) { CK(cudaSetDevice(d)); CK(cudaFuncSetAttribute(tma_copy<12, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384)); tma_copy<12, 9><<<c, 32, 12 * 16384, st[d]>>>(buf[s][0], buf[d][1], bytes, 16384); };
  auto cepull = [&](int d, int s) { CK(cudaSetDevice(d)); CK(cudaMemcpyPeerAsync(buf[d][1], d, buf[s][0], s, bytes, st[d])); };
  run("CE pull 1<-0 alone (stream on dst)", [&] { cepull(1, 0); });
  run("CE pull chain 1<-0, 2<-1", [&] { cepull(1, 0); cepull(2, 1); });
  run("mixed: CE pull 1<-0 + SM pull 2<-1", [&] { cepull(1, 0); pull(2, 1); });
  run("mixed: SM pull 1<-0 + CE pull 2<-1", [&] { pull(1, 0); cepull(2, 1); });
  run("CE 0->1 alone", [&] { ce(0, 1); });
  run("CE 0->1 and 1->0", [&] { ce(0, 1); ce(1, 0); });
  run("CE chain 0->1, 1->2", [&] { ce(0, 1); ce(1, 2); });
  run("TMA pull(LA9) 1<-0 alone c=32", [&] { tpull(1, 0, 32); });
  run("TMA pull(LA9) 1<-0 and 0<-1 c=32", [&] { tpull(1, 0, 32); tpull(0, 1, 32); });
  run("TMA pull(LA9) 1<-0 and 0<-1 c=64", [&] { tpull(1, 0, 64); tpull(0, 1, 64); });
  run("pull 1<-0 alone", [&] { pull(1, 0); });
  run("pull 1<-0 and 0<-1 (bidirectional pair)", [&] { pull(1, 0); pull(0, 1); });
  run("chain: 1<-0 and 2<-1 (GPU1 reads+serves)", [&] { pull(1, 0); pull(2, 1); });
  run("push 0->1 alone", [&] { push(0, 1); });
  run("push 0->1 and 1->0 (bidirectional pair)", [&] { push(0, 1); push(1, 0); });
  run("chain: 0->1 and 1->2 push", [&] { push(0, 1); push(1, 2); });
  if (ng >= 4) {
    run("ring pull 1<-0,2<-1,3<-2,0<-3", [&] { pull(1, 0); pull(2, 1); pull(3, 2); pull(0, 3); });
    run("ring push 0->1,1->2,2->3,3->0", [&] { push(0, 1); push(1, 2); push(2, 3); push(3, 0); });
    run("pairs pull 1<-0,0<-1,3<-2,2<-3", [&] { pull(1, 0); pull(0, 1); pull(3, 2); pull(2, 3); });
  }
  return 0;
}
