// Host-buffer entry points: the same fused step with W/G/W' in HOST memory
// (the reference's calling convention — its arrays live in host RAM,
// simulation.py:263-268).  Coordinates are independent, so the step is cut into
// chunks (column chunks of the learner-major (L, d) layout, row chunks of the
// reference's own (d, L) layout) and pipelined over three streams:
//   H2D(chunk i+1) || mix kernel(chunk i) || D2H(chunk i-1)
// through a caller-provided device workspace of NSLOT chunk slots.  With
// pinned host memory the step costs max(H2D, D2H) PCIe time instead of the
// sum; pageable memory still works (the driver stages it).
//
// Each calling host thread has its own streams and events per device (a
// thread-local pipe), so calls from several threads on distinct streams and
// workspaces do not share completion events.
#include "common.cuh"

namespace rm {

constexpr int kSlots = 3;

template <typename T>
int dispatch_dL(const T* W, const T* G, T* out, const int32_t* left, const int32_t* right, int L,
                long long d, long long ldw, long long ldg, long long ldo, double lr,
                unsigned long long* absmax, void* stream);

struct HostPipe {
  int device = -1;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t loaded[kSlots], computed[kSlots], drained[kSlots], start;
  bool ok = false;
};

static thread_local HostPipe t_pipes[64];

static HostPipe* get_pipe(int* err) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) {
    *err = RM_EINVAL;
    return nullptr;
  }
  HostPipe& p = t_pipes[dev];
  if (!p.ok) {
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&p.comp, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking)) != cudaSuccess) {
      *err = fail_cuda(e, "cudaStreamCreate");
      return nullptr;
    }
    for (int s = 0; s < kSlots; s++) {
      if ((e = cudaEventCreateWithFlags(&p.loaded[s], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&p.computed[s], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&p.drained[s], cudaEventDisableTiming)) != cudaSuccess) {
        *err = fail_cuda(e, "cudaEventCreate");
        return nullptr;
      }
    }
    if ((e = cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming)) != cudaSuccess) {
      *err = fail_cuda(e, "cudaEventCreate");
      return nullptr;
    }
    p.device = dev;
    p.ok = true;
  }
  return &p;
}

}  // namespace rm

using namespace rm;

#define RM_TRY(call, where)                         \
  do {                                              \
    cudaError_t _e = (call);                        \
    if (_e != cudaSuccess) return fail_cuda(_e, where); \
  } while (0)

// Column chunk width so that NSLOT x (W, G, W') chunks of L rows fit the
// workspace (rounded down to 32 columns = 128 B rows).
extern "C" int rm_host_chunk_cols(int L, int64_t workspace_bytes, int64_t* chunk_cols) {
  if (L < 1 || workspace_bytes <= 4096 || chunk_cols == nullptr) {
    set_error("invalid workspace request");
    return RM_EINVAL;
  }
  int64_t avail = workspace_bytes - 4096;  // tables
  int64_t per_col = (int64_t)kSlots * 3 * L * (int64_t)sizeof(float);
  int64_t c = (avail / per_col) / 32 * 32;
  if (c < 32) {
    set_error("workspace too small for L=%d", L);
    return RM_ERANGE;
  }
  *chunk_cols = c;
  return 0;
}

extern "C" int rm_ring_mix_sgd_host_f32(const float* W_host, const float* G_host, float* out_host,
                                        const int32_t* left_host, const int32_t* right_host, int L,
                                        int64_t d, double lr, void* workspace,
                                        int64_t workspace_bytes, unsigned long long* absmax_bits,
                                        void* stream) {
  if (W_host == nullptr || out_host == nullptr || left_host == nullptr ||
      right_host == nullptr || workspace == nullptr || L < 3 || d < 0 || L > 4096) {
    set_error("invalid host mix arguments (L=%d)", L);
    return RM_EINVAL;
  }
  if (d == 0) return 0;
  int64_t cw = 0;
  int rc = rm_host_chunk_cols(L, workspace_bytes, &cw);
  if (rc) return rc;
  if (cw > d) cw = (d + 31) / 32 * 32;
  int err = 0;
  HostPipe* p = get_pipe(&err);
  if (p == nullptr) return err;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);

  char* ws = static_cast<char*>(workspace);
  int32_t* d_left = reinterpret_cast<int32_t*>(ws);
  int32_t* d_right = d_left + 512;
  if (L > 512) {
    set_error("host path supports L <= 512");
    return RM_EINVAL;
  }
  float* slots = reinterpret_cast<float*>(ws + 4096);
  const int64_t chunk = (int64_t)L * cw;  // elements per buffer per slot
  auto slotW = [&](int s) { return slots + (int64_t)s * 3 * chunk; };
  auto slotG = [&](int s) { return slots + (int64_t)s * 3 * chunk + chunk; };
  auto slotO = [&](int s) { return slots + (int64_t)s * 3 * chunk + 2 * chunk; };

  // order after whatever the caller queued on its stream
  cudaEvent_t start_ev = p->start;
  RM_TRY(cudaEventRecord(start_ev, caller), "cudaEventRecord");
  RM_TRY(cudaStreamWaitEvent(p->h2d, start_ev, 0), "cudaStreamWaitEvent");
  RM_TRY(cudaStreamWaitEvent(p->comp, start_ev, 0), "cudaStreamWaitEvent");
  RM_TRY(cudaStreamWaitEvent(p->d2h, start_ev, 0), "cudaStreamWaitEvent");
  RM_TRY(cudaMemcpyAsync(d_left, left_host, L * sizeof(int32_t), cudaMemcpyHostToDevice, p->h2d),
         "H2D tables");
  RM_TRY(cudaMemcpyAsync(d_right, right_host, L * sizeof(int32_t), cudaMemcpyHostToDevice,
                         p->h2d),
         "H2D tables");

  const int64_t nchunks = (d + cw - 1) / cw;
  for (int64_t i = 0; i < nchunks; i++) {
    const int s = (int)(i % kSlots);
    const int64_t c0 = i * cw;
    const int64_t w = (d - c0) < cw ? (d - c0) : cw;
    if (i >= kSlots) {
      // slot reuse: its previous kernel finished reading W/G
      RM_TRY(cudaStreamWaitEvent(p->h2d, p->computed[s], 0), "wait computed");
    }
    RM_TRY(cudaMemcpy2DAsync(slotW(s), cw * sizeof(float), W_host + c0, d * sizeof(float),
                             w * sizeof(float), L, cudaMemcpyHostToDevice, p->h2d),
           "H2D W");
    if (G_host)
      RM_TRY(cudaMemcpy2DAsync(slotG(s), cw * sizeof(float), G_host + c0, d * sizeof(float),
                               w * sizeof(float), L, cudaMemcpyHostToDevice, p->h2d),
             "H2D G");
    RM_TRY(cudaEventRecord(p->loaded[s], p->h2d), "record loaded");
    RM_TRY(cudaStreamWaitEvent(p->comp, p->loaded[s], 0), "wait loaded");
    if (i >= kSlots) RM_TRY(cudaStreamWaitEvent(p->comp, p->drained[s], 0), "wait drained");
    rc = rm_ring_mix_sgd_f32(slotW(s), G_host ? slotG(s) : nullptr, slotO(s), d_left, d_right, L,
                             w, cw, cw, cw, lr, absmax_bits, p->comp);
    if (rc) return rc;
    RM_TRY(cudaEventRecord(p->computed[s], p->comp), "record computed");
    RM_TRY(cudaStreamWaitEvent(p->d2h, p->computed[s], 0), "wait computed");
    RM_TRY(cudaMemcpy2DAsync(out_host + c0, d * sizeof(float), slotO(s), cw * sizeof(float),
                             w * sizeof(float), L, cudaMemcpyDeviceToHost, p->d2h),
           "D2H out");
    RM_TRY(cudaEventRecord(p->drained[s], p->d2h), "record drained");
  }
  // the caller's stream resumes after the last D2H
  RM_TRY(cudaEventRecord(p->drained[0], p->d2h), "record end");
  RM_TRY(cudaStreamWaitEvent(caller, p->drained[0], 0), "wait end");
  return 0;
}

// ---- the reference's own layout: (d, L) C-order host arrays ----
// Row chunks are contiguous in host memory (one memcpy per buffer per chunk);
// the device kernel works on the same layout (dl.cu), so nothing is transposed.
namespace rm {
template <typename T>
static int host_dL(const T* W_host, const T* G_host, T* out_host, const int32_t* left_host,
                   const int32_t* right_host, int L, int64_t d, double lr, void* workspace,
                   int64_t workspace_bytes, unsigned long long* absmax_bits, void* stream) {
  const bool mean = left_host == nullptr && right_host == nullptr;
  if (!mean && L < 3) {
    set_error("degenerate ring topology: need at least 3 learners, got %d", L);
    return RM_EINVAL;
  }
  if (W_host == nullptr || out_host == nullptr || workspace == nullptr || L < 1 || L > 512 ||
      d < 0 || (!mean && (left_host == nullptr || right_host == nullptr))) {
    set_error("invalid host (d, L) step arguments (L=%d)", L);
    return RM_EINVAL;
  }
  if (d == 0) return 0;
  const int64_t per_row = (int64_t)kSlots * 3 * L * (int64_t)sizeof(T);
  int64_t ch = (workspace_bytes - 4096) / per_row;
  if (ch < 1) {
    set_error("workspace too small for L=%d", L);
    return RM_ERANGE;
  }
  if (ch > d) ch = d;
  int err = 0;
  HostPipe* p = get_pipe(&err);
  if (p == nullptr) return err;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  int32_t* d_left = reinterpret_cast<int32_t*>(ws);
  int32_t* d_right = d_left + 512;
  T* slots = reinterpret_cast<T*>(ws + 4096);
  const int64_t chunk = ch * L;
  auto slotW = [&](int s) { return slots + (int64_t)s * 3 * chunk; };
  auto slotG = [&](int s) { return slots + (int64_t)s * 3 * chunk + chunk; };
  auto slotO = [&](int s) { return slots + (int64_t)s * 3 * chunk + 2 * chunk; };
  RM_TRY(cudaEventRecord(p->start, caller), "cudaEventRecord");
  RM_TRY(cudaStreamWaitEvent(p->h2d, p->start, 0), "cudaStreamWaitEvent");
  RM_TRY(cudaStreamWaitEvent(p->comp, p->start, 0), "cudaStreamWaitEvent");
  RM_TRY(cudaStreamWaitEvent(p->d2h, p->start, 0), "cudaStreamWaitEvent");
  if (!mean) {
    RM_TRY(cudaMemcpyAsync(d_left, left_host, L * sizeof(int32_t), cudaMemcpyHostToDevice,
                           p->h2d), "H2D tables");
    RM_TRY(cudaMemcpyAsync(d_right, right_host, L * sizeof(int32_t), cudaMemcpyHostToDevice,
                           p->h2d), "H2D tables");
  }
  const int64_t nchunks = (d + ch - 1) / ch;
  for (int64_t i = 0; i < nchunks; i++) {
    const int s = (int)(i % kSlots);
    const int64_t r0 = i * ch;
    const int64_t h = (d - r0) < ch ? (d - r0) : ch;
    const size_t bytes = (size_t)h * L * sizeof(T);
    if (i >= kSlots) RM_TRY(cudaStreamWaitEvent(p->h2d, p->computed[s], 0), "wait computed");
    RM_TRY(cudaMemcpyAsync(slotW(s), W_host + r0 * L, bytes, cudaMemcpyHostToDevice, p->h2d),
           "H2D W");
    if (G_host)
      RM_TRY(cudaMemcpyAsync(slotG(s), G_host + r0 * L, bytes, cudaMemcpyHostToDevice, p->h2d),
             "H2D G");
    RM_TRY(cudaEventRecord(p->loaded[s], p->h2d), "record loaded");
    RM_TRY(cudaStreamWaitEvent(p->comp, p->loaded[s], 0), "wait loaded");
    if (i >= kSlots) RM_TRY(cudaStreamWaitEvent(p->comp, p->drained[s], 0), "wait drained");
    int rc = dispatch_dL<T>(slotW(s), G_host ? slotG(s) : nullptr, slotO(s),
                            mean ? nullptr : d_left, mean ? nullptr : d_right, L, h, L, L, L, lr,
                            absmax_bits, p->comp);
    if (rc) return rc;
    RM_TRY(cudaEventRecord(p->computed[s], p->comp), "record computed");
    RM_TRY(cudaStreamWaitEvent(p->d2h, p->computed[s], 0), "wait computed");
    RM_TRY(cudaMemcpyAsync(out_host + r0 * L, slotO(s), bytes, cudaMemcpyDeviceToHost, p->d2h),
           "D2H out");
    RM_TRY(cudaEventRecord(p->drained[s], p->d2h), "record drained");
  }
  RM_TRY(cudaEventRecord(p->drained[0], p->d2h), "record end");
  RM_TRY(cudaStreamWaitEvent(caller, p->drained[0], 0), "wait end");
  return 0;
}
}  // namespace rm

extern "C" int rm_gossip_step_host_dL_f32(const float* W_host, const float* G_host,
                                          float* out_host, const int32_t* left_host,
                                          const int32_t* right_host, int L, int64_t d, double lr,
                                          void* workspace, int64_t workspace_bytes,
                                          unsigned long long* absmax_bits, void* stream) {
  return host_dL<float>(W_host, G_host, out_host, left_host, right_host, L, d, lr, workspace,
                        workspace_bytes, absmax_bits, stream);
}

extern "C" int rm_gossip_step_host_dL_f64(const double* W_host, const double* G_host,
                                          double* out_host, const int32_t* left_host,
                                          const int32_t* right_host, int L, int64_t d, double lr,
                                          void* workspace, int64_t workspace_bytes,
                                          unsigned long long* absmax_bits, void* stream) {
  return host_dL<double>(W_host, G_host, out_host, left_host, right_host, L, d, lr, workspace,
                         workspace_bytes, absmax_bits, stream);
}
