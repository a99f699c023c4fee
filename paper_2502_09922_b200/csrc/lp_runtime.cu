// Device plumbing for the lambdapipe C ABI: errors, memory, IPC, streams,
// events, pinned-host registration.  No torch types cross this boundary.
#include "lp_common.cuh"
#include "../../include/lambdapipe.h"
#include <string.h>
#include <stdlib.h>

namespace lp {
static thread_local char g_err[1024] = "";
static thread_local int g_pdl = 0;
bool pdl_enabled() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("LP_PDL");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1 && g_pdl == 1;
}
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace lp

extern "C" {

int lp_version(void) { return 100; }
int lp_set_pdl(int on) {
  lp::g_pdl = on ? 1 : 0;
  return 0;
}
const char* lp_last_error(void) { return lp::g_err; }

int lp_device_count(int* n) {
  LP_CUDA(cudaGetDeviceCount(n));
  return 0;
}
int lp_set_device(int dev) {
  LP_CUDA(cudaSetDevice(dev));
  return 0;
}
int lp_sync_device(int dev) {
  lp::DeviceGuard g(dev);
  LP_CUDA(cudaDeviceSynchronize());
  return 0;
}
int lp_enable_peer(int dev, int peer) {
  lp::DeviceGuard g(dev);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  LP_CUDA(e);
  return 0;
}
int lp_malloc(int dev, int64_t bytes, void** out) {
  LP_CHECK(bytes > 0 && out, "lp_malloc: bad arguments");
  lp::DeviceGuard g(dev);
  LP_CUDA(cudaMalloc(out, (size_t)bytes));
  return 0;
}
int lp_free(int dev, void* ptr) {
  lp::DeviceGuard g(dev);
  LP_CUDA(cudaFree(ptr));
  return 0;
}
int lp_memset(void* dst, int value, int64_t bytes, void* stream) {
  LP_CUDA(cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream));
  return 0;
}
int lp_memcpy(void* dst, const void* src, int64_t bytes, void* stream) {
  LP_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return 0;
}
int lp_ipc_get(void* dev_ptr, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t h;
  LP_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle64, &h, 64);
  return 0;
}
int lp_ipc_open(int dev, const void* handle64, void** out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  lp::DeviceGuard g(dev);
  LP_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}
int lp_ipc_close(void* ptr) {
  LP_CUDA(cudaIpcCloseMemHandle(ptr));
  return 0;
}
int lp_host_register(void* host, int64_t bytes, void** dev_alias) {
  LP_CUDA(cudaHostRegister(host, (size_t)bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  LP_CUDA(cudaHostGetDevicePointer(dev_alias, host, 0));
  return 0;
}
int lp_host_unregister(void* host) {
  LP_CUDA(cudaHostUnregister(host));
  return 0;
}
int lp_stream_create(int dev, void** stream) {
  lp::DeviceGuard g(dev);
  cudaStream_t s;
  LP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = (void*)s;
  return 0;
}
int lp_stream_destroy(void* stream) {
  LP_CUDA(cudaStreamDestroy((cudaStream_t)stream));
  return 0;
}
int lp_stream_sync(void* stream) {
  LP_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}
int lp_event_create(void** ev) {
  cudaEvent_t e;
  LP_CUDA(cudaEventCreate(&e));
  *ev = (void*)e;
  return 0;
}
int lp_event_destroy(void* ev) {
  LP_CUDA(cudaEventDestroy((cudaEvent_t)ev));
  return 0;
}
int lp_event_record(void* ev, void* stream) {
  LP_CUDA(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream));
  return 0;
}
int lp_event_elapsed_ms(void* start, void* end, float* ms) {
  LP_CUDA(cudaEventSynchronize((cudaEvent_t)end));
  LP_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end));
  return 0;
}

}  // extern "C"
