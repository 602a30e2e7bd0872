// C-ABI plumbing: thread-local error messages, device queries.
#include "common.cuh"
#include "../../include/ringmix_b200.h"

#include <mutex>

namespace rm {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail_cuda(cudaError_t e, const char* where) {
  set_error("%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
  return static_cast<int>(e);
}

int sm_count(int device) {
  static int cache[64];
  if (device < 0) cudaGetDevice(&device);
  if (device < 0 || device >= 64) return 148;
  if (cache[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    cache[device] = n;
  }
  return cache[device];
}

}  // namespace rm

extern "C" const char* rm_last_error(void) { return rm::g_err; }

extern "C" int rm_version(void) { return 1; }

extern "C" int rm_device_info(int device, int* sms, int* major, int* minor) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return rm::fail_cuda(e, "cudaGetDeviceProperties");
  if (sms) *sms = p.multiProcessorCount;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  return 0;
}

// ---- helpers for FFI callers without a CUDA runtime of their own (e.g. the
// reference's numpy code through ctypes): device buffers and stream sync ----
extern "C" int rm_device_alloc(int64_t bytes, void** ptr) {
  if (ptr == nullptr || bytes < 0) {
    rm::set_error("invalid allocation arguments");
    return RM_EINVAL;
  }
  *ptr = nullptr;
  if (bytes == 0) return 0;
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e != cudaSuccess) return rm::fail_cuda(e, "cudaMalloc");
  return 0;
}

extern "C" int rm_device_free(void* ptr) {
  if (ptr == nullptr) return 0;
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) return rm::fail_cuda(e, "cudaFree");
  return 0;
}

extern "C" int rm_memcpy(void* dst, const void* src, int64_t bytes, void* stream) {
  if ((dst == nullptr || src == nullptr) && bytes > 0) {
    rm::set_error("null pointer");
    return RM_EINVAL;
  }
  if (bytes <= 0) return 0;
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return rm::fail_cuda(e, "cudaMemcpyAsync");
  return 0;
}

extern "C" int rm_stream_synchronize(void* stream) {
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return rm::fail_cuda(e, "cudaStreamSynchronize");
  return 0;
}

// single-process multi-GPU callers (one host thread driving several
// GPUs) enable peer access between every pair of the first ndev devices; the
// learner-sharded kernels then read / write peer rows through plain device
// pointers.  Already-enabled pairs are not an error.  The current device is
// restored.
extern "C" int rm_enable_peer_access(int ndev) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return rm::fail_cuda(e, "cudaGetDeviceCount");
  if (ndev < 1 || ndev > count) {
    rm::set_error("ndev=%d outside [1, %d]", ndev, count);
    return RM_EINVAL;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  for (int a = 0; a < ndev; a++) {
    e = cudaSetDevice(a);
    if (e != cudaSuccess) return rm::fail_cuda(e, "cudaSetDevice");
    for (int b = 0; b < ndev; b++) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can) {
        cudaSetDevice(cur);
        rm::set_error("device %d cannot access device %d", a, b);
        return RM_ENOSYS;
      }
      e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();  // clear the sticky-free status
      } else if (e != cudaSuccess) {
        cudaSetDevice(cur);
        return rm::fail_cuda(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
  cudaSetDevice(cur);
  return 0;
}
