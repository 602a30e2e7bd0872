// Shared helpers for libringmix_b200: error plumbing and sm_100a PTX wrappers.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <stdlib.h>
#include <utility>

namespace rm {

// ---- error plumbing (thread-local message, see include/ringmix_b200.h) ----
void set_error(const char* fmt, ...);
int fail_cuda(cudaError_t e, const char* where);

#define RM_CHECK_LAUNCH(where)                                  \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::rm::fail_cuda(_e, where);   \
  } while (0)

#include "../../include/ringmix_b200.h"
constexpr int RM_OK = 0;

int sm_count(int device);

// ---- PTX wrappers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Bounded wait: a correct pipeline never waits more than microseconds; if the
// expected bytes never arrive (a bug), trap after ~4 s instead of hanging the
// GPU until the job's wall-clock limit.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > 8000000000LL) __trap();
  }
}

// TMA bulk copy global -> shared (1-D, bytes % 16 == 0, both ends 16B aligned),
// completion signalled on an mbarrier via complete_tx.
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 8-byte asynchronous global -> shared copy (LDGSTS; no register staging), grouped by
// cp_async_commit and waited for by the issuing thread with cp_async_wait<N>.
__device__ __forceinline__ void cp_async_8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc)
               : "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* sdst, const T* gsrc) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "cp.async element size");
  if constexpr (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 16-byte streaming store (evict-first; the output is not re-read this step).
__device__ __forceinline__ void st_cs_v4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// atomicMax on the bit pattern of |y| as a double: monotone for non-negative
// doubles, and every NaN pattern (> 0x7ff0...) sorts above +inf.
__device__ __forceinline__ void absmax_publish(unsigned long long* slot, unsigned long long bits) {
  // warp reduce then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = other > bits ? other : bits;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(slot, bits);
}

__device__ __forceinline__ unsigned long long abs_bits(double y) {
  return static_cast<unsigned long long>(__double_as_longlong(y)) & 0x7fffffffffffffffULL;
}


// Function attributes (e.g. the dynamic shared-memory opt-in) are per device: a
// bit per device ordinal records where one has been set (re-setting is harmless,
// so the unsynchronised update is benign).
__host__ inline bool attr_needed(unsigned long long* mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 64 || !((*mask >> dev) & 1ull);
}
__host__ inline void attr_done(unsigned long long* mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64) *mask |= 1ull << dev;
}

// ---- programmatic dependent launch (PDL) ----
// A kernel launched with launch_pdl may start while the previous kernel on the
// stream is still draining; it must call pdl_wait() before reading anything that
// kernel may have written.  pdl_launch_dependents() lets the next kernel start
// launching early (it still waits for this grid's completion in its pdl_wait).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// RINGMIX_PDL=1 launches with the programmatic-serialization attribute.  Off by
// default: measured on B200 it made consecutive mix launches slower (C1, CUDA graph:
// 39.9 vs 33.8 us per step; C2 3.31 vs 3.18 ms — profiles/r2_mix_ab2).
__host__ inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("RINGMIX_PDL");
    on = (env && env[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
__host__ inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                       size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- cross-GPU step ordering through flags in symmetric memory ----
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Cross-rank waits are bounded: a rank whose host falls behind (checkpoint,
// eval, module load, debugger) must not kill its peers' contexts, so the bound
// is long (RINGMIX_XGPU_TIMEOUT_S, default 600 s, set per device by the host
// launchers) and hitting it does not trap: the wait gives up, records the
// timeout in g_xgpu_status (rm_xgpu_status() reads and clears it) and the step
// completes with unspecified contents — the caller treats it as a failed step.
static __device__ unsigned long long g_xgpu_timeout_ns = 600ull * 1000000000ull;
static __device__ unsigned int g_xgpu_status = 0;

// Thread 0 spins (acquire, system scope) until *flag - target >= 0 (wraps), then
// the CTA proceeds.  The data guarded by the flag is read through another
// virtual alias (peer / multicast mapping), hence the alias fence.
__device__ __forceinline__ void xgpu_wait(const uint32_t* flag, uint32_t target) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = global_ns();
    const unsigned long long limit = g_xgpu_timeout_ns;
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(64);
      if (global_ns() - t0 > limit) {
        atomicOr(&g_xgpu_status, 1u);
        break;
      }
    }
    asm volatile("fence.proxy.alias;" ::: "memory");
    // the peers' generic-proxy stores are read next by TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
}

// A buffer that every rank of a learner-sharded job holds at the same offset
// (symmetric memory), seen from one rank: either its NVSwitch multicast address
// (mc != 0: one multimem instruction reaches every rank, reductions happen in
// the switch) or a table of every rank's address of it (peers: unicast loads and
// stores over NVLink P2P — or, with all "ranks" on one GPU, the single-device
// emulation the tests run).  Element i is at byte offset i * sizeof(element).
struct SymRef {
  unsigned long long mc;
  const unsigned long long* peers;  // device table [world] when mc == 0
  int world;
};

// +1 on element i of every rank (release, system scope)
__device__ __forceinline__ void sym_red_add_u32(const SymRef& s, long long i) {
  if (s.mc) {
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;" ::"l"(s.mc + 4 * i)
                 : "memory");
  } else {
    for (int r = 0; r < s.world; r++)
      asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(s.peers[r] + 4 * i)
                   : "memory");
  }
}

// sum over ranks of element i (multicast: in-switch reduction; unicast: ascending rank)
__device__ __forceinline__ double sym_ld_sum_f64(const SymRef& s, long long i) {
  double v;
  if (s.mc) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];"
                 : "=d"(v)
                 : "l"(s.mc + 8 * i)
                 : "memory");
  } else {
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(s.peers[0] + 8 * i)
                 : "memory");
    for (int r = 1; r < s.world; r++) {
      double x;
      asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(x) : "l"(s.peers[r] + 8 * i)
                   : "memory");
      v = __dadd_rn(v, x);
    }
  }
  return v;
}

// sum over ranks of element i in numpy's pairwise tree order: ((x0 + x1) + (x2 + x3)) + ...
// (world a power of two <= 8).  Multicast: the in-switch sum, exact for world <= 2 only (the
// switch's order of more addends is unspecified; callers use peer tables there).
__device__ __forceinline__ double sym_ld_sum_tree_f64(const SymRef& s, long long i) {
  if (s.mc || s.world <= 2) return sym_ld_sum_f64(s, i);
  double v[8];
#pragma unroll
  for (int r = 0; r < 8; r++)
    if (r < s.world)
      asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v[r]) : "l"(s.peers[r] + 8 * i)
                   : "memory");
#pragma unroll
  for (int w = 1; w < 8; w *= 2)
#pragma unroll
    for (int r = 0; r + w < 8; r += 2 * w)
      if (r + w < s.world) v[r] = __dadd_rn(v[r], v[r + w]);
  return v[0];
}

// element i := v on every rank
__device__ __forceinline__ void sym_st_f64(const SymRef& s, long long i, double v) {
  if (s.mc) {
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(s.mc + 8 * i), "d"(v)
                 : "memory");
  } else {
    for (int r = 0; r < s.world; r++)
      asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(s.peers[r] + 8 * i), "d"(v)
                   : "memory");
  }
}

// Every thread's writes so far are made visible system-wide; the CTA whose
// arrival completes `last` arrivals on `counter` adds 1 to element `i` of the
// flag buffer on every rank (multimem.red.release through the multicast address,
// or one red.release per rank in the peer-table form).
// reset: the last arriver zeroes the counter (for a counter private to one launch).
__device__ __forceinline__ void xgpu_arrive(uint32_t* counter, uint32_t last, const SymRef& flag,
                                            long long i, bool reset = false) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t old = atomicAdd(counter, 1u);
    if (old + 1u == last) {
      if (reset) atomicExch(counter, 0u);
      __threadfence_system();
      asm volatile("fence.proxy.alias;" ::: "memory");
      sym_red_add_u32(flag, i);
    }
  }
}

}  // namespace rm
