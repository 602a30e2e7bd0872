// On-device permutation generator, bit-exact with the reference's
// permutation_for_step (pkg/src/ringmix/mixing.py:79-86) and the sequential
// draws of monte_carlo_consensus (spectral.py:273-277).
//
// The reference draws through numpy: SeedSequence(entropy) -> PCG64 (XSL-RR
// 128/64) -> Generator.permutation(n) (Fisher-Yates, i = n-1..1, masked
// rejection on buffered 32-bit halves).  SURVEY.md Appendix A states the
// algorithm; this file is an independent CUDA implementation of it.
//
// Work decomposition: every (seed, tag, step) stream is independent, so one
// thread owns one stream.  A launch covers `nsteps` consecutive steps, which
// lets the step loop generate a whole block of future neighbour tables in one
// launch (each step is a pure function of (seed, step): SURVEY §8(a)).
#include "common.cuh"
#include "../../include/ringmix_b200.h"

namespace rm {

constexpr int kMaxPrefixWords = 24;

struct PermArgs {
  uint32_t prefix[kMaxPrefixWords];
  int nprefix;
};

// ---- SeedSequence (numpy bit_generator.pyx, pool_size = 4) ----
__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  return r ^ (r >> 16);
}

struct U128 {
  uint64_t hi, lo;
};

__device__ __forceinline__ U128 mul_add_128(U128 a, U128 m, U128 c) {
  // (a * m + c) mod 2^128
  uint64_t lo = a.lo * m.lo;
  uint64_t hi = __umul64hi(a.lo, m.lo) + a.lo * m.hi + a.hi * m.lo;
  uint64_t lo2 = lo + c.lo;
  hi += c.hi + (lo2 < lo ? 1ull : 0ull);
  return {hi, lo2};
}

struct Pcg64 {
  U128 state, inc;
  uint32_t buf;
  bool has32;

  __device__ __forceinline__ void step() {
    const U128 M = {2549297995355413924ull, 4865540595714422341ull};
    state = mul_add_128(state, M, inc);
  }
  __device__ __forceinline__ uint64_t next64() {
    step();
    uint64_t x = state.hi ^ state.lo;
    unsigned rot = static_cast<unsigned>(state.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf;
    }
    uint64_t n = next64();
    has32 = true;
    buf = static_cast<uint32_t>(n >> 32);
    return static_cast<uint32_t>(n);
  }
  // numpy random_interval: smallest all-ones mask >= max, reject > max.
  __device__ __forceinline__ uint32_t interval32(uint32_t max) {
    uint32_t mask = 0xffffffffu >> __clz(max | 1u);
    uint32_t v;
    do {
      v = next32() & mask;
    } while (v > max);
    return v;
  }
};

__device__ void seed_pcg(Pcg64& g, const uint32_t* ent, int n) {
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
#pragma unroll
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, hc);
#pragma unroll
  for (int s = 0; s < 4; s++)
#pragma unroll
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n; s++)
#pragma unroll
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
  uint32_t hb = 0x8b51f9ddu;
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  uint64_t v0 = w[0] | (uint64_t(w[1]) << 32), v1 = w[2] | (uint64_t(w[3]) << 32);
  uint64_t v2 = w[4] | (uint64_t(w[5]) << 32), v3 = w[6] | (uint64_t(w[7]) << 32);
  // pcg_setseq_128_srandom_r(initstate = v0:v1, initseq = v2:v3)
  g.inc = {(v2 << 1) | (v3 >> 63), (v3 << 1) | 1ull};
  g.state = {0, 0};
  g.step();
  uint64_t lo = g.state.lo + v1;
  g.state.hi += v0 + (lo < v1 ? 1ull : 0ull);
  g.state.lo = lo;
  g.step();
  g.has32 = false;
  g.buf = 0;
}

__device__ __forceinline__ int append_limbs(uint32_t* ent, int n, uint64_t v) {
  if (v == 0) {
    ent[n++] = 0;
    return n;
  }
  while (v) {
    ent[n++] = static_cast<uint32_t>(v);
    v >>= 32;
  }
  return n;
}

// Fisher-Yates over arange(L) into `a` (global scratch row, L1-resident).
__device__ __forceinline__ void shuffle_into(Pcg64& g, int32_t* a, int L) {
  for (int i = 0; i < L; i++) a[i] = i;
  for (int i = L - 1; i >= 1; i--) {
    int j = static_cast<int>(g.interval32(static_cast<uint32_t>(i)));
    int32_t t = a[i];
    a[i] = a[j];
    a[j] = t;
  }
}

__global__ void perm_tables_kernel(PermArgs args, uint64_t step0, int nsteps, int L,
                                   int32_t* __restrict__ perm, int32_t* __restrict__ inv,
                                   int32_t* __restrict__ left, int32_t* __restrict__ right) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsteps) return;
  uint32_t ent[kMaxPrefixWords + 2];
  for (int i = 0; i < args.nprefix; i++) ent[i] = args.prefix[i];
  int n = append_limbs(ent, args.nprefix, step0 + static_cast<uint64_t>(s));
  Pcg64 g;
  seed_pcg(g, ent, n);
  int32_t* p = perm + static_cast<int64_t>(s) * L;
  int32_t* q = inv + static_cast<int64_t>(s) * L;
  shuffle_into(g, p, L);
  for (int j = 0; j < L; j++) q[p[j]] = j;
  if (left != nullptr && right != nullptr) {
    int32_t* lf = left + static_cast<int64_t>(s) * L;
    int32_t* rt = right + static_cast<int64_t>(s) * L;
    for (int j = 0; j < L; j++) {
      int pj = p[j];
      lf[j] = q[pj == 0 ? L - 1 : pj - 1];
      rt[j] = q[pj == L - 1 ? 0 : pj + 1];
    }
  }
}

__global__ void perm_sequential_kernel(PermArgs args, uint64_t idx0, int nstreams, int count,
                                       int L, int32_t* __restrict__ perms) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nstreams) return;
  uint32_t ent[kMaxPrefixWords + 2];
  for (int i = 0; i < args.nprefix; i++) ent[i] = args.prefix[i];
  int n = append_limbs(ent, args.nprefix, idx0 + static_cast<uint64_t>(s));
  Pcg64 g;
  seed_pcg(g, ent, n);
  int32_t* base = perms + static_cast<int64_t>(s) * count * L;
  for (int c = 0; c < count; c++) shuffle_into(g, base + static_cast<int64_t>(c) * L, L);
}

// Stateful streams (seeding.stream objects): state = 6 x u64
// {state.hi, state.lo, inc.hi, inc.lo, has32, buf32}.
__device__ __forceinline__ void pcg_load(Pcg64& g, const uint64_t* s) {
  g.state = {s[0], s[1]};
  g.inc = {s[2], s[3]};
  g.has32 = s[4] != 0;
  g.buf = static_cast<uint32_t>(s[5]);
}
__device__ __forceinline__ void pcg_store(const Pcg64& g, uint64_t* s) {
  s[0] = g.state.hi;
  s[1] = g.state.lo;
  s[2] = g.inc.hi;
  s[3] = g.inc.lo;
  s[4] = g.has32 ? 1u : 0u;
  s[5] = g.buf;
}

__global__ void pcg_seed_kernel(PermArgs args, uint64_t idx0, int nstreams, int with_index,
                                uint64_t* __restrict__ states) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nstreams) return;
  uint32_t ent[kMaxPrefixWords + 2];
  for (int i = 0; i < args.nprefix; i++) ent[i] = args.prefix[i];
  int n = args.nprefix;
  if (with_index) n = append_limbs(ent, n, idx0 + static_cast<uint64_t>(s));
  Pcg64 g;
  seed_pcg(g, ent, n);
  pcg_store(g, states + 6 * static_cast<int64_t>(s));
}

__global__ void pcg_draw_kernel(uint64_t* __restrict__ states, int nstreams, int count, int L,
                                int32_t* __restrict__ perms) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nstreams) return;
  Pcg64 g;
  pcg_load(g, states + 6 * static_cast<int64_t>(s));
  int32_t* base = perms + static_cast<int64_t>(s) * count * L;
  for (int c = 0; c < count; c++) shuffle_into(g, base + static_cast<int64_t>(c) * L, L);
  pcg_store(g, states + 6 * static_cast<int64_t>(s));
}

// Raw next64 outputs (pins the generator core in tests).
__global__ void raw64_kernel(PermArgs args, int count, uint64_t* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  Pcg64 g;
  seed_pcg(g, args.prefix, args.nprefix);
  for (int c = 0; c < count; c++) out[c] = g.next64();
}

static int load_prefix(PermArgs& a, const uint32_t* prefix, int nprefix) {
  if (nprefix < 0 || nprefix > kMaxPrefixWords || (nprefix > 0 && prefix == nullptr)) {
    set_error("entropy prefix must have 0..%d words, got %d", kMaxPrefixWords, nprefix);
    return RM_EINVAL;
  }
  for (int i = 0; i < nprefix; i++) a.prefix[i] = prefix[i];
  a.nprefix = nprefix;
  return RM_OK;
}

}  // namespace rm

using namespace rm;

extern "C" int rm_perm_tables(const uint32_t* prefix_words, int n_prefix, uint64_t step0,
                              int nsteps, int L, int32_t* perm, int32_t* inv, int32_t* left,
                              int32_t* right, void* stream) {
  PermArgs a;
  int rc = load_prefix(a, prefix_words, n_prefix);
  if (rc) return rc;
  if (L < 1 || nsteps < 0) {
    set_error("need n >= 1, got %d", L);
    return RM_EINVAL;
  }
  if (perm == nullptr || inv == nullptr) {
    set_error("perm and inv buffers are required");
    return RM_EINVAL;
  }
  if (nsteps == 0) return RM_OK;
  int threads = 64;
  int blocks = (nsteps + threads - 1) / threads;
  perm_tables_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      a, step0, nsteps, L, perm, inv, left, right);
  RM_CHECK_LAUNCH("perm_tables_kernel");
  return RM_OK;
}

extern "C" int rm_perm_sequential(const uint32_t* prefix_words, int n_prefix, uint64_t idx0,
                                  int nstreams, int count, int L, int32_t* perms, void* stream) {
  PermArgs a;
  int rc = load_prefix(a, prefix_words, n_prefix);
  if (rc) return rc;
  if (L < 1 || nstreams < 0 || count < 0 || perms == nullptr) {
    set_error("invalid sequential permutation request (L=%d, nstreams=%d, count=%d)", L,
              nstreams, count);
    return RM_EINVAL;
  }
  if (nstreams == 0 || count == 0) return RM_OK;
  int threads = 64;
  int blocks = (nstreams + threads - 1) / threads;
  perm_sequential_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      a, idx0, nstreams, count, L, perms);
  RM_CHECK_LAUNCH("perm_sequential_kernel");
  return RM_OK;
}

extern "C" int rm_pcg64_raw(const uint32_t* entropy_words, int n_words, int count,
                            uint64_t* out, void* stream) {
  PermArgs a;
  int rc = load_prefix(a, entropy_words, n_words);
  if (rc) return rc;
  if (count < 0 || out == nullptr) {
    set_error("invalid raw request");
    return RM_EINVAL;
  }
  raw64_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(a, count, out);
  RM_CHECK_LAUNCH("raw64_kernel");
  return RM_OK;
}

extern "C" int rm_pcg_seed(const uint32_t* prefix_words, int n_prefix, int with_index,
                           uint64_t idx0, int nstreams, uint64_t* states, void* stream) {
  PermArgs a;
  int rc = load_prefix(a, prefix_words, n_prefix);
  if (rc) return rc;
  if (nstreams < 0 || states == nullptr) {
    set_error("invalid stream seeding request");
    return RM_EINVAL;
  }
  if (nstreams == 0) return RM_OK;
  int threads = 64;
  pcg_seed_kernel<<<(nstreams + threads - 1) / threads, threads, 0,
                    static_cast<cudaStream_t>(stream)>>>(a, idx0, nstreams, with_index, states);
  RM_CHECK_LAUNCH("pcg_seed_kernel");
  return RM_OK;
}

extern "C" int rm_pcg_permutations(uint64_t* states, int nstreams, int count, int L,
                                   int32_t* perms, void* stream) {
  if (L < 1 || nstreams < 0 || count < 0 || states == nullptr || perms == nullptr) {
    set_error("need n >= 1, got %d", L);
    return RM_EINVAL;
  }
  if (nstreams == 0 || count == 0) return RM_OK;
  int threads = 64;
  pcg_draw_kernel<<<(nstreams + threads - 1) / threads, threads, 0,
                    static_cast<cudaStream_t>(stream)>>>(states, nstreams, count, L, perms);
  RM_CHECK_LAUNCH("pcg_draw_kernel");
  return RM_OK;
}
