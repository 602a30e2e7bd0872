// NVLink peer-memory bandwidth probe (2 GPUs, one process): which access style
// reaches the link rate?  (1) 16-byte loads by all threads, (2) cp.async 16 B into
// shared memory, (3) TMA 1-D bulk copies peer -> shared, (4) 16-byte stores to
// the peer, (5) TMA 1-D bulk stores shared -> peer.  Build: make -C tools/p2p
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_ld(const uint4* __restrict__ src, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = acc;
}

__global__ void k_st(uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

// cp.async 16 B: each CTA copies chunks of CH bytes into a smem ring
template <int CH>
__global__ void k_cpasync(const char* __restrict__ src, size_t bytes, uint4* sink) {
  extern __shared__ __align__(128) char sm[];
  const size_t nch = bytes / CH;
  int slot = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    char* dst = sm + slot * CH;
    for (int o = threadIdx.x * 16; o < CH; o += blockDim.x * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(su32(dst + o)), "l"(src + c * CH + o) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 2;" ::: "memory");
    slot = (slot + 1) & 3;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (threadIdx.x == 0 && sm[0] == 123 && sm[1] == 45) sink[0] = make_uint4(1, 1, 1, 1);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"(su32(b)), "r"(ph) : "memory");
}

// TMA bulk loads peer -> smem, 4-stage ring of CH-byte chunks, one issuing thread per CTA
template <int CH>
__global__ void k_bulk_ld(const char* __restrict__ src, size_t bytes, uint4* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[4];
  const size_t nch = bytes / CH;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; i++) mbar_init(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int it = 0;
  size_t c = blockIdx.x;
  for (int s = 0; s < 4 && c + s * gridDim.x < nch; s++) {
    mbar_expect(&bar[s], CH);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(su32(sm + s * CH)), "l"(src + (c + s * gridDim.x) * CH), "r"(CH), "r"(su32(&bar[s])) : "memory");
  }
  for (; c < nch; c += gridDim.x, ++it) {
    const int s = it & 3;
    mbar_wait(&bar[s], (it >> 2) & 1);
    size_t cn = c + 4 * (size_t)gridDim.x;
    if (cn < nch) {
      mbar_expect(&bar[s], CH);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(sm + s * CH)), "l"(src + cn * CH), "r"(CH), "r"(su32(&bar[s])) : "memory");
    }
  }
  if (sm[0] == 123 && sm[1] == 45) sink[0] = make_uint4(1, 1, 1, 1);
}

// TMA bulk stores smem -> peer
template <int CH>
__global__ void k_bulk_st(char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char sm[];
  const size_t nch = bytes / CH;
  for (int o = threadIdx.x; o < CH; o += blockDim.x) sm[o] = (char)o;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + c * CH), "r"(su32(sm)), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n = 0; CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  int can = 0; CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("peer access 0->1: %d\n", can);
  const size_t bytes = 2ull << 30;
  char *b0, *b1; uint4* sink;
  CK(cudaSetDevice(1)); CK(cudaMalloc(&b1, bytes)); CK(cudaMemset(b1, 1, bytes));
  CK(cudaSetDevice(0)); CK(cudaMalloc(&b0, bytes)); CK(cudaMemset(b0, 1, bytes)); CK(cudaMalloc(&sink, 64));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto timeit = [&](const char* name, auto launch, size_t moved, const char* where) {
    for (int r = 0; r < 2; r++) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-28s %-6s %8.1f GB/s %s\n", name, where, moved * 5 / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int peer = 1; peer >= 0; peer--) {
    char* src = peer ? b1 : b0;
    const char* w = peer ? "peer" : "local";
    for (int cta : {1, 2, 4, 8}) {
      char nm[64]; snprintf(nm, 64, "ld16 x%d CTA/SM", cta);
      timeit(nm, [&] { k_ld<<<sms * cta, 256>>>((const uint4*)src, bytes / 16, sink); }, bytes, w);
    }
    timeit("cp.async 4KB x2", [&] { k_cpasync<4096><<<sms * 2, 256, 4 * 4096>>>(src, bytes, sink); }, bytes, w);
    timeit("cp.async 16KB x2", [&] { k_cpasync<16384><<<sms * 2, 256, 4 * 16384>>>(src, bytes, sink); }, bytes, w);
    cudaFuncSetAttribute(k_bulk_ld<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
    cudaFuncSetAttribute(k_bulk_ld<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    timeit("bulk ld 4KB x2", [&] { k_bulk_ld<4096><<<sms * 2, 32, 4 * 4096>>>(src, bytes, sink); }, bytes, w);
    timeit("bulk ld 16KB x1", [&] { k_bulk_ld<16384><<<sms, 32, 4 * 16384>>>(src, bytes, sink); }, bytes, w);
    timeit("bulk ld 32KB x1", [&] { k_bulk_ld<32768><<<sms, 32, 4 * 32768>>>(src, bytes, sink); }, bytes, w);
    timeit("bulk ld 512B x4", [&] { k_bulk_ld<512><<<sms * 4, 32, 4 * 512>>>(src, bytes, sink); }, bytes, w);
    for (int cta : {1, 4}) {
      char nm[64]; snprintf(nm, 64, "st16 x%d CTA/SM", cta);
      timeit(nm, [&] { k_st<<<sms * cta, 256>>>((uint4*)src, bytes / 16); }, bytes, w);
    }
    timeit("bulk st 4KB x2", [&] { k_bulk_st<4096><<<sms * 2, 32, 4096>>>(src, bytes); }, bytes, w);
    timeit("bulk st 16KB x2", [&] { k_bulk_st<16384><<<sms * 2, 32, 16384>>>(src, bytes); }, bytes, w);
    timeit("bulk st 512B x4", [&] { k_bulk_st<512><<<sms * 4, 32, 512>>>(src, bytes); }, bytes, w);
    timeit("cudaMemcpyPeer", [&] { cudaMemcpyPeerAsync(b0, 0, b1, 1, bytes); }, bytes, peer ? "peer" : "peer");
  }
  // bidirectional: each GPU reads the other's memory at the same time (what two ranks of
  // the learner-sharded pull kernel do), 16-byte loads, 4 CTAs/SM
  {
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    uint4* sink1; CK(cudaMalloc(&sink1, 64));
    cudaStream_t s1; CK(cudaStreamCreate(&s1));
    cudaEvent_t a1, b1e; CK(cudaEventCreate(&a1)); CK(cudaEventCreate(&b1e));
    CK(cudaSetDevice(0));
    cudaStream_t s0; CK(cudaStreamCreate(&s0));
    for (int rep = 0; rep < 3; rep++) {
      CK(cudaSetDevice(0));
      cudaEventRecord(a, s0);
      for (int r = 0; r < 5; r++) k_ld<<<sms * 4, 256, 0, s0>>>((const uint4*)b1, bytes / 16, sink);
      cudaEventRecord(b, s0);
      CK(cudaSetDevice(1));
      cudaEventRecord(a1, s1);
      for (int r = 0; r < 5; r++) k_ld<<<sms * 4, 256, 0, s1>>>((const uint4*)b0, bytes / 16, sink1);
      cudaEventRecord(b1e, s1);
      cudaEventSynchronize(b1e);
      CK(cudaSetDevice(0));
      cudaEventSynchronize(b);
      float m0 = 0, m1 = 0;
      cudaEventElapsedTime(&m0, a, b);
      cudaEventElapsedTime(&m1, a1, b1e);
      printf("%-28s %-6s %8.1f GB/s (GPU0 reads GPU1) %8.1f GB/s (GPU1 reads GPU0)\n",
             "bidirectional ld16 x4", "peer", bytes * 5 / (m0 * 1e-3) / 1e9,
             bytes * 5 / (m1 * 1e-3) / 1e9);
    }
    // bidirectional stores (what the ring-position layout's relabel stores do)
    for (int rep = 0; rep < 3; rep++) {
      CK(cudaSetDevice(0));
      cudaEventRecord(a, s0);
      for (int r = 0; r < 5; r++) k_st<<<sms * 4, 256, 0, s0>>>((uint4*)b1, bytes / 16);
      cudaEventRecord(b, s0);
      CK(cudaSetDevice(1));
      cudaEventRecord(a1, s1);
      for (int r = 0; r < 5; r++) k_st<<<sms * 4, 256, 0, s1>>>((uint4*)b0, bytes / 16);
      cudaEventRecord(b1e, s1);
      cudaEventSynchronize(b1e);
      CK(cudaSetDevice(0));
      cudaEventSynchronize(b);
      float m0 = 0, m1 = 0;
      cudaEventElapsedTime(&m0, a, b);
      cudaEventElapsedTime(&m1, a1, b1e);
      printf("%-28s %-6s %8.1f GB/s (GPU0 -> GPU1) %8.1f GB/s (GPU1 -> GPU0)\n",
             "bidirectional st16 x4", "peer", bytes * 5 / (m0 * 1e-3) / 1e9,
             bytes * 5 / (m1 * 1e-3) / 1e9);
    }
  }
  return 0;
}
