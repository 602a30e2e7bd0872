// Device gradient producer for the reference's quadratic oracle (SURVEY §8(f)
// next-1): G[l] = lambda * (Phi[l] - w*) + sd * z_l, where z_l is numpy's
// stream(seed, TAG_GRADIENT, k, l).standard_normal(d) — reference
// objectives.py:84-90 and simulation.py:226-238 — reproduced bit for bit.
//
// numpy draws a normal with a 256-layer ziggurat that consumes a VARIABLE
// number of 64-bit PCG64 outputs (1 in ~98 % of cases), so element c of the
// stream cannot be located without counting.  Parallel generation:
//   1. spec:  every raw block [b*B, (b+1)*B) of every stream is simulated from
//             its first draw as if an attempt started there (PCG64 jump-ahead
//             to the block start).  Record which of the first 32 draws start
//             attempts / produce outputs, the exit (first attempt >= next
//             block) and the output count.
//   2. merge: the true path enters block b at the exit of block b-1; if that
//             entry is an attempt start of b's speculative path the two paths
//             coincide from there (attempts are almost always single draws, so
//             paths merge within a couple of draws).  Blocks that fail are
//             re-simulated from the true entry (rare, sequential per stream).
//   3. scan:  per-stream prefix sums give every block's first output index.
//   4. gen:   each block regenerates its outputs from the true entry into
//             shared memory, then the CTA writes G for its contiguous output
//             range with coalesced loads of Phi / lambda / w* and stores of G.
// The ziggurat tables are numpy's own doubles (ziggurat_tables.h, generated
// from the installed libnpyrandom.a); fp arithmetic follows numpy's C code
// without FMA contraction.
#include "common.cuh"
#include "arith.cuh"
#include "ziggurat_tables.h"
#include "zsrc.cuh"
#include <math_constants.h>
#include "../../include/ringmix_b200.h"

namespace rm {

constexpr int kZBlock = 256;        // raw draws per speculative block
constexpr int kZGenThreads = 128;   // blocks (threads) per generation CTA
constexpr int kZMaxPrefix = 24;

struct U128d {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128d mul128(U128d a, U128d b) {
  return {__umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo, a.lo * b.lo};
}
__device__ __forceinline__ U128d add128(U128d a, U128d b) {
  uint64_t lo = a.lo + b.lo;
  return {a.hi + b.hi + (lo < a.lo ? 1ull : 0ull), lo};
}

// jump tables: state after r steps = M^r * s + inc * S_r (S_r = sum_{i<r} M^i)
__constant__ U128d c_jumpA[64];
__constant__ U128d c_jumpS[64];

struct ZStream {
  U128d state, inc;
};

struct ZArgs {
  uint32_t prefix[kZMaxPrefix];  // entropy words of (seed, tag)
  int nprefix;
  uint64_t k;                    // step index (entropy word after the prefix)
  int append;                    // trailing entropy ints: 0 none, 1 (k), 2 (k, stream)
  int nstreams;                  // learners
  long long n;                   // normals per stream (d)
  int nblocks;                   // raw blocks per stream
  long long stream0;             // stream s draws entropy stream0 + s (learner-sharded runs)
  int run;                       // > 0: stream0 + (s / run) * period + s % run (interleaved
  long long period;              //      learner sets, rm_set_shard_streams)
};

__device__ __forceinline__ uint32_t zs_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__device__ __forceinline__ uint32_t zs_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  return r ^ (r >> 16);
}

__device__ ZStream z_seed(const ZArgs& a, int stream) {
  uint32_t ent[kZMaxPrefix + 4];
  int n = 0;
  for (int i = 0; i < a.nprefix; i++) ent[n++] = a.prefix[i];
  auto limbs = [&](uint64_t v) {
    if (v == 0) {
      ent[n++] = 0;
      return;
    }
    while (v) {
      ent[n++] = (uint32_t)v;
      v >>= 32;
    }
  };
  if (a.append >= 1) limbs(a.k);
  if (a.append >= 2)
    limbs((uint64_t)(a.stream0 + (a.run > 0 ? (stream / a.run) * a.period + stream % a.run
                                             : (long long)stream)));
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; i++) pool[i] = zs_hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = zs_mix(pool[d], zs_hashmix(pool[s], hc));
  for (int s = 4; s < n; s++)
    for (int d = 0; d < 4; d++) pool[d] = zs_mix(pool[d], zs_hashmix(ent[s], hc));
  uint32_t hb = 0x8b51f9ddu, w[8];
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  uint64_t v0 = w[0] | ((uint64_t)w[1] << 32), v1 = w[2] | ((uint64_t)w[3] << 32);
  uint64_t v2 = w[4] | ((uint64_t)w[5] << 32), v3 = w[6] | ((uint64_t)w[7] << 32);
  const U128d M = {2549297995355413924ull, 4865540595714422341ull};
  ZStream z;
  z.inc = {(v2 << 1) | (v3 >> 63), (v3 << 1) | 1ull};
  U128d s = z.inc;                       // state = 0 * M + inc
  s = add128(s, U128d{v0, v1});          // += initstate
  s = add128(mul128(s, M), z.inc);       // step
  z.state = s;
  return z;
}

// state after r further steps
__device__ __forceinline__ U128d z_jump(const ZStream& z, uint64_t r) {
  U128d A = {0, 1}, S = {0, 0};
  for (int i = 0; r; i++, r >>= 1) {
    if (r & 1) {
      // compose current (A, S) with 2^i steps: A' = Ai*A, S' = Ai*S + Si
      S = add128(mul128(c_jumpA[i], S), c_jumpS[i]);
      A = mul128(c_jumpA[i], A);
    }
  }
  return add128(mul128(A, z.state), mul128(z.inc, S));
}

struct ZGen {
  U128d state, inc;
  __device__ __forceinline__ uint64_t next64() {
    const U128d M = {2549297995355413924ull, 4865540595714422341ull};
    state = add128(mul128(state, M), inc);
    // XSL-RR output: rotr64(hi ^ lo, hi >> 58), as two 32-bit funnel shifts after a
    // conditional half swap (a rotation by >= 32 is a swap plus a rotation by rot & 31)
    const uint64_t x = state.hi ^ state.lo;
    const unsigned rot = (unsigned)(state.hi >> 58);
    uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    const uint32_t sl = (rot & 32u) ? xh : xl, sh = (rot & 32u) ? xl : xh;
    xl = __funnelshift_r(sl, sh, rot);
    xh = __funnelshift_r(sh, sl, rot);
    return ((uint64_t)xh << 32) | xl;
  }
  __device__ __forceinline__ double next_double() {
    return __dmul_rn((double)(next64() >> 11), 1.0 / 9007199254740992.0);
  }
};

// log1p exactly as the host's libm computes it.  numpy calls libm log1p in the
// ziggurat tail; glibc 2.39 on x86-64 with FMA/AVX2 dispatches to the FMA build
// of sysdeps/ieee754/dbl-64/s_log1p.c (fdlibm algorithm, Estrin-style
// polynomial).  The operation sequence below follows that build instruction
// for instruction (fused multiply-adds where the compiler fused them), so the
// device value is bit-identical; CUDA's own log1p differs by 1 ulp in ~0.4 %
// of tail draws.  Only the domain (-1, 0] used by the ziggurat tail is needed,
// but the general cases are kept.
__device__ __noinline__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0, u;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec4) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return __dadd_rn(x, x);
  }
  if (k != 0) {
    if (hx < 0x43400000) {
      u = __dadd_rn(x, 1.0);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    }
    const double R = __dmul_rn(__fma_rn(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double v = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, v));
  const double t = __dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(dk, ln2_lo, c), v)), f);
  return __fma_rn(dk, ln2_hi, -t);
}

// numpy's ziggurat tables, staged in shared memory (indices are random per
// lane, which would serialise __constant__ reads)
struct ZigTables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};

__device__ __forceinline__ void load_tables(ZigTables* t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t->ki[i] = kZigKi[i];
    t->wi[i] = __longlong_as_double((long long)kZigWiBits[i]);
    t->fi[i] = __longlong_as_double((long long)kZigFiBits[i]);
  }
}

// Wedge test of a ziggurat attempt (strip idx >= 1, fast test failed) with its
// second draw u: accept iff (f[idx-1] - f[idx]) * u + f[idx] < exp(-x^2 / 2).  An
// fp32 exp (relative error < 2e-6 on the strips' range |x| < 3.66) decides unless
// lhs lies within 2^-16 of it; only then is the fp64 exp evaluated, so the outcome
// is that of the fp64 comparison.
#ifndef RM_ZWEDGE_FAST
#define RM_ZWEDGE_FAST 1
#endif
__device__ __forceinline__ bool z_wedge(const ZigTables& T, int idx, double x, uint64_t u) {
  const double f0 = T.fi[idx - 1], f1 = T.fi[idx];
  const double ud = __dmul_rn((double)(u >> 11), 1.0 / 9007199254740992.0);
  const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(f0, f1), ud), f1);
  const double t = __dmul_rn(__dmul_rn(-0.5, x), x);
#if RM_ZWEDGE_FAST
  const double e = (double)__expf((float)t);
  if (lhs < e * (1.0 - 1.0 / 65536.0)) return true;
  if (lhs > e * (1.0 + 1.0 / 65536.0)) return false;
#endif
  return lhs < exp(t);
}

// One ziggurat attempt starting with draw `r` (already taken).  Returns true
// and sets *x when it produces an output; `extra` = further draws consumed.
__device__ __forceinline__ bool z_attempt(const ZigTables& T, ZGen& g, uint64_t r, double* x,
                                          int* extra) {
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const int sign = (int)(r & 1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
  double v = __dmul_rn((double)rabs, T.wi[idx]);
  if (sign) v = -v;
  *extra = 0;
  if (rabs < T.ki[idx]) {
    *x = v;
    return true;
  }
  if (idx == 0) {
    const double R = 3.6541528853610087963519472518;
    const double INV_R = 0.27366123732975827203338247596;
    for (;;) {
      double xx = __dmul_rn(-INV_R, glibc_log1p(-g.next_double()));
      double yy = -glibc_log1p(-g.next_double());
      *extra += 2;
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        *x = ((rabs >> 8) & 1) ? -__dadd_rn(R, xx) : __dadd_rn(R, xx);
        return true;
      }
    }
  }
  *extra = 1;
  if (z_wedge(T, idx, v, g.next64())) {
    *x = v;
    return true;
  }
  return false;
}

// The slow part of a ziggurat attempt (the fast test `rabs < ki[idx]` failed):
// `u0` is the next draw of the stream (already taken), further draws come from
// g.  Same arithmetic as z_attempt; *extra = further draws consumed.
__device__ __forceinline__ bool z_slow(const ZigTables& T, ZGen& g, uint64_t u0, int idx,
                                    uint64_t rabs, double* x, int* extra) {
  const double v = *x;
  if (idx == 0) {
    const double R = 3.6541528853610087963519472518;
    const double INV_R = 0.27366123732975827203338247596;
    uint64_t u = u0;
    *extra = 0;
    for (;;) {
      const double d0 = __dmul_rn((double)(u >> 11), 1.0 / 9007199254740992.0);
      double xx = __dmul_rn(-INV_R, glibc_log1p(-d0));
      double yy = -glibc_log1p(-g.next_double());
      *extra += 2;
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        *x = ((rabs >> 8) & 1) ? -__dadd_rn(R, xx) : __dadd_rn(R, xx);
        return true;
      }
      u = g.next64();
    }
  }
  *extra = 1;
  return z_wedge(T, idx, v, u0);
}

__device__ __forceinline__ void st_v4_f64(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

struct BlockInfo {
  uint32_t att;    // bit i: draw b*B+i starts an attempt on the speculative path
  uint32_t outs;   // bit i: that attempt produced an output
  uint32_t exit;   // first speculative attempt start >= (b+1)*B, relative to b*B
  uint32_t count;  // outputs of attempts starting in [b*B, (b+1)*B)
};

// per-stream PCG64 state right after seeding (SeedSequence hashing done once)
__global__ void zig_seed_kernel(ZArgs a, ZStream* __restrict__ seeds) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < a.nstreams) seeds[s] = z_seed(a, s);
}

#ifndef RM_ZSPEC_MINB
#define RM_ZSPEC_MINB 1
#endif
// One speculative attempt at relative draw `pos` whose first draw is `cur`;
// `g` is positioned after draw pos+1 (= `nxt`, the one-draw lookahead).
struct ZStep {
  double x;
  uint32_t used;  // draws consumed
  bool ok;
};
__device__ __forceinline__ ZStep z_spec_step(const ZigTables& T, ZGen& g, uint64_t& cur) {
  const uint64_t nxt = g.next64();
  const int idx = (int)(cur & 0xff);
  const uint64_t rabs = (cur >> 9) & 0x000fffffffffffffull;
  const uint64_t ki = T.ki[idx];
  const double wi = T.wi[idx];
  // sign from bit 8: flip the product's sign bit (exact, as -x)
  double x = __dmul_rn((double)rabs, wi);
  x = __hiloint2double(__double2hiint(x) ^ (int)(((uint32_t)cur & 0x100u) << 23),
                       __double2loint(x));
  ZStep st;
  if (rabs < ki) {
    st.ok = true;
    st.used = 1;
    cur = nxt;
  } else {
    // slow path (about 1.2 % of draws): the further draws start at `nxt`
    int extra;
    st.ok = z_slow(T, g, nxt, idx, rabs, &x, &extra);
    st.used = 1 + extra;
    cur = g.next64();
  }
  st.x = x;
  return st;
}

#ifndef RM_ZKEEP
#define RM_ZKEEP 0
#endif
// RM_ZKEEP 0: quads buffered in registers, 32-byte stores; 1: pairs, 16-byte stores;
// 2: one 8-byte store per output
template <bool KEEP>
__device__ __forceinline__ void z_keep(double* slot, uint32_t count, double x, double& q0,
                                       double& q1, double& q2) {
  if (!KEEP) return;
#if RM_ZKEEP == 2
  slot[count] = x;
#elif RM_ZKEEP == 1
  if (count & 1u) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(slot + count - 1), "d"(q0), "d"(x)
                 : "memory");
  }
  q0 = x;
#else
  const uint32_t c = count & 3u;
  if (c == 3u) st_v4_f64(slot + count - 3, q0, q1, q2, x);
  q0 = c == 0u ? x : q0;
  q1 = c == 1u ? x : q1;
  q2 = c == 2u ? x : q2;
#endif
}


template <bool KEEP>
__global__ void __launch_bounds__(128, RM_ZSPEC_MINB)
    zig_spec_kernel(ZArgs a, const ZStream* __restrict__ seeds, BlockInfo* __restrict__ info,
                    double* __restrict__ scratch) {
  __shared__ ZigTables T;
  load_tables(&T);
  __syncthreads();
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)a.nstreams * a.nblocks) return;
  // stream-fastest block order keeps concurrent CTAs on the same columns
  const int stream = (int)(gid % a.nstreams);
  const int b = (int)(gid / a.nstreams);
  const ZStream zs = seeds[stream];
  ZGen g{z_jump(zs, (uint64_t)b * kZBlock), zs.inc};
  uint32_t att = 0, outs = 0, count = 0;
  uint32_t pos = 0;  // relative draw index of the next attempt
  // KEEP: speculative outputs are kept in the scratch, 32-byte stores of quads
  double* slot = KEEP ? scratch + ((long long)stream * a.nblocks + b) * kZBlock : nullptr;
  double q0 = 0.0, q1 = 0.0, q2 = 0.0;
  // one-draw lookahead: the PCG step for draw pos+1 is independent of the table
  // lookups for draw pos, so the two latencies overlap
  uint64_t cur = g.next64();
  while (pos < 32u) {  // attempts in the first 32 draws are recorded for the merge
    const ZStep st = z_spec_step(T, g, cur);
    att |= 1u << pos;
    outs |= (st.ok ? 1u : 0u) << pos;
    if (st.ok) z_keep<KEEP>(slot, count, st.x, q0, q1, q2);
    count += st.ok ? 1u : 0u;
    pos += st.used;
  }
  while (pos < (uint32_t)kZBlock) {
    const ZStep st = z_spec_step(T, g, cur);
    if (st.ok) z_keep<KEEP>(slot, count, st.x, q0, q1, q2);
    count += st.ok ? 1u : 0u;
    pos += st.used;
  }
  if (KEEP) {
#if RM_ZKEEP == 1
    if (count & 1u) slot[count - 1] = q0;
#elif RM_ZKEEP == 0
    const uint32_t r = count & 3u, c0 = count - r;
    if (r > 0) slot[c0] = q0;
    if (r > 1) slot[c0 + 1] = q1;
    if (r > 2) slot[c0 + 2] = q2;
#endif
  }
  info[(long long)stream * a.nblocks + b] = BlockInfo{att, outs, pos, count};
}

// entries[b] (relative entry of the true path into block b) and true counts.
// Block 0 enters at 0; block b at exit(b-1) - B if b-1 merged.  Failing blocks
// are appended to `bad` for the sequential repair.
__global__ void zig_merge_kernel(ZArgs a, const BlockInfo* __restrict__ info,
                                 uint32_t* __restrict__ entry, uint32_t* __restrict__ tcount,
                                 uint8_t* __restrict__ merged, uint32_t* __restrict__ nbad,
                                 uint64_t* __restrict__ bad) {
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)a.nstreams * a.nblocks) return;
  const int b = (int)(gid % a.nblocks);
  const BlockInfo me = info[gid];
  const uint32_t e = b == 0 ? 0u : info[gid - 1].exit - kZBlock;
  entry[gid] = e;
  if (e < 32 && ((me.att >> e) & 1u)) {
    tcount[gid] = me.count - __popc(me.outs & ((1u << e) - 1u));
    merged[gid] = 1;
  } else {
    tcount[gid] = 0;
    merged[gid] = 0;
    uint32_t slot = atomicAdd(nbad, 1u);
    bad[slot] = (uint64_t)gid;
  }
}

// Parallel repair of isolated failures (predecessor merged, so the stored
// entry is the true one): one thread per bad block re-simulates it, then
// re-checks the successor against the corrected exit.  Failures whose
// predecessor also failed (chains, very rare) go to `left` for the sequential
// pass.
__global__ void __launch_bounds__(128)
    zig_repair_par_kernel(ZArgs a, const ZStream* __restrict__ seeds,
                          const BlockInfo* __restrict__ info, uint32_t* __restrict__ entry,
                          uint32_t* __restrict__ tcount, const uint8_t* __restrict__ merged,
                          uint8_t* __restrict__ valid,
                          const uint32_t* __restrict__ nbad, const uint64_t* __restrict__ bad,
                          uint32_t* __restrict__ nleft, uint64_t* __restrict__ left) {
  __shared__ ZigTables T;
  const uint32_t nb = *nbad;
  if (blockIdx.x * blockDim.x >= nb) return;  // CTA-uniform
  load_tables(&T);
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const long long gid = (long long)bad[i];
  const int stream = (int)(gid / a.nblocks);
  const int b = (int)(gid % a.nblocks);
  if (b > 0 && !merged[gid - 1]) {
    left[atomicAdd(nleft, 1u)] = (uint64_t)gid;  // chain: sequential pass
    return;
  }
  const ZStream zs = seeds[stream];
  const uint32_t e = entry[gid];
  ZGen g{z_jump(zs, (uint64_t)b * kZBlock + e), zs.inc};
  uint32_t pos = e, count = 0;
  while (pos < (uint32_t)kZBlock) {
    double x;
    int extra;
    count += z_attempt(T, g, g.next64(), &x, &extra) ? 1u : 0u;
    pos += 1 + extra;
  }
  tcount[gid] = count;
  if (b + 1 >= a.nblocks) return;
  const uint32_t e2 = pos - kZBlock;
  entry[gid + 1] = e2;
  if (!merged[gid + 1]) return;  // successor is itself bad: the sequential pass owns it
  const BlockInfo nx = info[gid + 1];
  if (e2 < 32 && ((nx.att >> e2) & 1u)) {
    tcount[gid + 1] = nx.count - __popc(nx.outs & ((1u << e2) - 1u));
  } else {
    valid[gid + 1] = 0;
    left[atomicAdd(nleft, 1u)] = (uint64_t)(gid + 1);
  }
}

// Sequential repair of blocks whose speculative path did not merge: one
// thread per stream walks its bad blocks in order and re-simulates from the
// true entry until the path merges again with the next block's speculation.
// Blocks the walk passes through that the merge pass had accepted (so they are on
// neither list) are appended to the merge-failure list `app`, so the fixup regenerates
// them too.
__global__ void zig_repair_kernel(ZArgs a, const ZStream* __restrict__ seeds,
                                  const BlockInfo* __restrict__ info, uint32_t* __restrict__ entry,
                                  uint32_t* __restrict__ tcount, const uint8_t* __restrict__ merged,
                                  uint8_t* __restrict__ valid, const uint32_t* __restrict__ nbad,
                                  const uint64_t* __restrict__ bad, uint32_t* __restrict__ napp,
                                  uint64_t* __restrict__ app) {
  __shared__ ZigTables T;
  const uint32_t nb = *nbad;
  if (nb == 0) return;  // uniform: no leftover blocks (the common case)
  load_tables(&T);
  __syncthreads();
  const int stream = blockIdx.x * blockDim.x + threadIdx.x;
  if (stream >= a.nstreams) return;
  const ZStream zs = seeds[stream];
  long long next_b = -1;
  for (;;) {
    long long best = -1;
    for (uint32_t i = 0; i < nb; i++) {
      const long long gid = (long long)bad[i];
      if (gid / a.nblocks != stream) continue;
      const long long bb = gid % a.nblocks;
      if (bb > next_b && (best < 0 || bb < best)) best = bb;
    }
    if (best < 0) return;
    long long b = best;
    for (;;) {
      const long long gid = (long long)stream * a.nblocks + b;
      const uint32_t e = entry[gid];
      ZGen g{z_jump(zs, (uint64_t)b * kZBlock + e), zs.inc};
      uint32_t pos = e, count = 0;
      while (pos < (uint32_t)kZBlock) {
        double x;
        int extra;
        count += z_attempt(T, g, g.next64(), &x, &extra) ? 1u : 0u;
        pos += 1 + extra;
      }
      tcount[gid] = count;
      valid[gid] = 0;
      next_b = b;
      if (b + 1 >= a.nblocks) return;
      const long long g2 = gid + 1;
      const uint32_t e2 = pos - kZBlock;
      entry[g2] = e2;
      const BlockInfo nx = info[g2];
      // stop only at a block the merge pass accepted (blocks it rejected may
      // carry successor data from a parallel repair with a stale entry)
      if (merged[g2] && e2 < 32 && ((nx.att >> e2) & 1u)) {
        tcount[g2] = nx.count - __popc(nx.outs & ((1u << e2) - 1u));
        valid[g2] = 1;
        break;  // merged again; later blocks keep their speculative entries
      }
      if (merged[g2]) app[atomicAdd(napp, 1u)] = (uint64_t)g2;
      b = b + 1;
    }
  }
}

// per-stream exclusive prefix sum of tcount -> offs
__global__ void zig_scan_kernel(ZArgs a, const uint32_t* __restrict__ tcount,
                                unsigned long long* __restrict__ offs,
                                unsigned long long* __restrict__ total) {
  const int stream = blockIdx.x;
  __shared__ unsigned long long carry;
  __shared__ unsigned long long warp_sums[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const long long base = (long long)stream * a.nblocks;
  for (int c0 = 0; c0 < a.nblocks; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const unsigned long long v = i < a.nblocks ? tcount[base + i] : 0ull;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) warp_sums[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long w = threadIdx.x < (blockDim.x >> 5) ? warp_sums[threadIdx.x] : 0ull;
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      warp_sums[threadIdx.x] = w;
    }
    __syncthreads();
    const unsigned long long before =
        carry + ((threadIdx.x >> 5) ? warp_sums[(threadIdx.x >> 5) - 1] : 0ull);
    if (i < a.nblocks) offs[base + i] = before + x - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[stream] = carry;
}

// Generation + fused quadratic gradient.  A CTA owns kZGenThreads consecutive
// raw blocks of one stream (CTAs ordered stream-fastest so concurrent CTAs
// share lam / w* columns in L2).  Each thread regenerates its block's outputs
// from the true entry in rounds of kZRound; after each round every warp writes
// whole runs of 32 consecutive outputs (coalesced Phi / lam / w* loads and G
// stores).
constexpr int kZRound = 32;

template <typename T>
__global__ void __launch_bounds__(kZGenThreads)
    zig_gen_kernel(ZArgs a, const ZStream* __restrict__ seeds, const uint32_t* __restrict__ entry,
                   const uint32_t* __restrict__ tcount,
                   const unsigned long long* __restrict__ offs, const T* __restrict__ Phi,
                   long long ldp, const double* __restrict__ lam, const double* __restrict__ wopt,
                   double sd, T* __restrict__ G, long long ldg, double* __restrict__ Z,
                   long long ldz) {
  using E = Elem<T>;
  __shared__ ZigTables Tb;
  __shared__ double zbuf[kZGenThreads][kZRound + 1];
  __shared__ int rcount[kZGenThreads];
  __shared__ unsigned long long rbase[kZGenThreads];
  const int groups = (a.nblocks + kZGenThreads - 1) / kZGenThreads;
  const int stream = blockIdx.x % a.nstreams;
  const int b0 = (blockIdx.x / a.nstreams) * kZGenThreads;
  if (b0 >= a.nblocks) return;
  (void)groups;
  const long long base = (long long)stream * a.nblocks;
  if (offs[base + b0] >= (unsigned long long)a.n) return;  // CTA-uniform
  load_tables(&Tb);
  const int b = b0 + threadIdx.x;
  const bool live = b < a.nblocks;
  const ZStream zs = seeds[stream];
  ZGen g{zs.state, zs.inc};
  uint32_t pos = 0, left = 0;
  unsigned long long obase = 0;
  if (live) {
    const long long gid = base + b;
    pos = entry[gid];
    left = tcount[gid];
    obase = offs[gid];
    g.state = z_jump(zs, (uint64_t)b * kZBlock + pos);
    if (obase >= (unsigned long long)a.n) left = 0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (;;) {
    // one round: up to kZRound outputs per thread
    int cnt = 0;
    __syncthreads();  // tables loaded / previous flush done
    while (left > 0 && cnt < kZRound) {
      double x;
      int extra;
      if (z_attempt(Tb, g, g.next64(), &x, &extra)) {
        zbuf[threadIdx.x][cnt++] = x;
        left--;
      }
      pos += 1 + extra;
    }
    rcount[threadIdx.x] = cnt;
    rbase[threadIdx.x] = obase;
    obase += cnt;
    if (!__syncthreads_or(cnt > 0)) break;
    // each warp flushes the runs of threads warp, warp+4, ...; loads of 8 runs
    // are issued before any is consumed (latency hiding)
    constexpr int kBatch = 8;
    for (int t0 = warp; t0 < kZGenThreads; t0 += kBatch * (kZGenThreads / 32)) {
      long long cs[kBatch];
      double w[kBatch], lm[kBatch], wo[kBatch];
      bool on[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; u++) {
        const int t = t0 + u * (kZGenThreads / 32);
        on[u] = false;
        if (t < kZGenThreads && lane < rcount[t]) {
          cs[u] = (long long)rbase[t] + lane;
          on[u] = cs[u] < a.n;
        }
        if (on[u] && G) {
          w[u] = (double)E::ld(Phi + stream * ldp + cs[u], 0);
          lm[u] = lam[cs[u]];
          wo[u] = wopt[cs[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < kBatch; u++) {
        if (!on[u]) continue;
        const int t = t0 + u * (kZGenThreads / 32);
        const double z = zbuf[t][lane];
        if (Z) Z[stream * ldz + cs[u]] = z;
        if (G) {
          // objectives.py:87-90: gradient(w) + noise_sd * z, gradient = lam * (w - w*)
          const double gr = __dmul_rn(lm[u], __dsub_rn(w[u], wo[u]));
          G[stream * ldg + cs[u]] = E::st((typename E::acc)__dadd_rn(gr, __dmul_rn(sd, z)));
        }
      }
    }
  }
}

// ---- fast path: the speculative outputs are kept in a scratch buffer ----
// One warp per raw block copies its (merged) speculative outputs, skipping the
// ones before the true entry, and writes G for them — coalesced reads of the
// scratch and of Phi / lam / w*, coalesced G stores.  Blocks whose speculation
// did not merge are regenerated by zig_fixup_kernel (~2e-4 of the blocks).
template <typename T>
__device__ __forceinline__ void emit_grad(const ZArgs& a, int stream, long long c, double z,
                                          const T* __restrict__ Phi, long long ldp,
                                          const double* __restrict__ lam,
                                          const double* __restrict__ wopt, double sd,
                                          T* __restrict__ G, long long ldg,
                                          double* __restrict__ Z, long long ldz) {
  using E = Elem<T>;
  if (Z) Z[stream * ldz + c] = z;
  if (G) {
    // objectives.py:87-90: gradient(w) + noise_sd * z, gradient = lam * (w - w*)
    const double w = (double)E::ld(Phi + stream * ldp + c, 0);
    const double gr = __dmul_rn(lam[c], __dsub_rn(w, wopt[c]));
    G[stream * ldg + c] = E::st((typename E::acc)__dadd_rn(gr, __dmul_rn(sd, z)));
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
    zig_copy_kernel(ZArgs a, const BlockInfo* __restrict__ info,
                    const uint32_t* __restrict__ entry, const uint32_t* __restrict__ tcount,
                    const unsigned long long* __restrict__ offs, const uint8_t* __restrict__ valid,
                    const double* __restrict__ scratch, const T* __restrict__ Phi, long long ldp,
                    const double* __restrict__ lam, const double* __restrict__ wopt, double sd,
                    T* __restrict__ G, long long ldg, double* __restrict__ Z, long long ldz) {
  // stream-fastest warp order: concurrent warps cover the same columns, so
  // lam / w* (fp64[d], read once per learner) are served from L2
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long long)a.nstreams * a.nblocks) return;
  const int stream = (int)(w % a.nstreams);
  const long long gid = (long long)stream * a.nblocks + w / a.nstreams;
  if (!valid[gid]) return;
  const unsigned long long base = offs[gid];
  if (base >= (unsigned long long)a.n) return;
  const uint32_t e = entry[gid];
  const uint32_t skip = __popc(info[gid].outs & ((1u << e) - 1u));
  const uint32_t cnt = tcount[gid];
  const double* src = scratch + gid * kZBlock + skip;
  // all loads of the block first (cnt <= kZBlock = 8 * 32), then the stores
  const uint32_t lim = min((unsigned long long)cnt, (unsigned long long)a.n - base);
  double z[kZBlock / 32];
#pragma unroll
  for (int j = 0; j < kZBlock / 32; ++j) {
    const uint32_t i = lane + 32 * j;
    z[j] = i < lim ? __ldcs(src + i) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < kZBlock / 32; ++j) {
    const uint32_t i = lane + 32 * j;
    if (i < lim) emit_grad<T>(a, stream, (long long)base + i, z[j], Phi, ldp, lam, wopt, sd, G, ldg, Z, ldz);
  }
}

template <typename T>
__global__ void __launch_bounds__(128)
    zig_fixup_kernel(ZArgs a, const ZStream* __restrict__ seeds, const uint32_t* __restrict__ entry,
                     const unsigned long long* __restrict__ offs, const uint8_t* __restrict__ valid,
                     const uint32_t* __restrict__ nbad, const uint64_t* __restrict__ bad,
                     const uint32_t* __restrict__ nleft, const uint64_t* __restrict__ left,
                     const T* __restrict__ Phi, long long ldp, const double* __restrict__ lam,
                     const double* __restrict__ wopt, double sd, T* __restrict__ G, long long ldg,
                     double* __restrict__ Z, long long ldz) {
  __shared__ ZigTables Tb;
  const uint32_t n1 = *nbad, n2 = *nleft;
  if (blockIdx.x * blockDim.x >= n1 + n2) return;  // CTA-uniform
  load_tables(&Tb);
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n1 + n2) return;
  const long long gid = (long long)(i < n1 ? bad[i] : left[i - n1]);
  if (valid[gid]) return;
  unsigned long long o = offs[gid];
  if (o >= (unsigned long long)a.n) return;
  const int stream = (int)(gid / a.nblocks);
  const int b = (int)(gid % a.nblocks);
  const ZStream zs = seeds[stream];
  uint32_t pos = entry[gid];
  ZGen g{z_jump(zs, (uint64_t)b * kZBlock + pos), zs.inc};
  while (pos < (uint32_t)kZBlock && o < (unsigned long long)a.n) {
    double x;
    int extra;
    if (z_attempt(Tb, g, g.next64(), &x, &extra))
      emit_grad<T>(a, stream, (long long)o++, x, Phi, ldp, lam, wopt, sd, G, ldg, Z, ldz);
    pos += 1 + extra;
  }
}

static bool g_jump_ready[64];

static int ensure_jump_tables() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && g_jump_ready[dev]) return 0;
  // host-side 128-bit arithmetic with unsigned __int128
  typedef unsigned __int128 u128;
  const u128 M = ((u128)2549297995355413924ull << 64) | 4865540595714422341ull;
  U128d A[64], S[64];
  u128 a = M, s = 1;  // 2^0 steps: A = M, S = 1
  for (int i = 0; i < 64; i++) {
    A[i] = {(uint64_t)(a >> 64), (uint64_t)a};
    S[i] = {(uint64_t)(s >> 64), (uint64_t)s};
    // doubling: A_{2r} = A_r^2, S_{2r} = S_r * (A_r + 1)
    s = s * (a + 1);
    a = a * a;
  }
  cudaError_t e = cudaMemcpyToSymbol(c_jumpA, A, sizeof(A));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_jumpS, S, sizeof(S));
  if (e != cudaSuccess) return fail_cuda(e, "cudaMemcpyToSymbol(jump tables)");
  if (dev >= 0 && dev < 64) g_jump_ready[dev] = true;
  return 0;
}

}  // namespace rm

using namespace rm;

// Workspace bytes for nstreams x n normals.
extern "C" int64_t rm_normal_workspace_bytes(int nstreams, int64_t n) {
  if (nstreams < 1 || n < 0) return -1;
  const long long nblocks = (long long)((1.04 * (double)n + 64.0 * sqrt((double)n + 1.0)) /
                                        kZBlock) + 8;
  const long long nb = nblocks * nstreams;
  // per block: info, offs (8), entry (4), tcount (4), bad (8), left (8), merged (1);
  // per stream: total (8), seed; alignment padding and the two counters
  return (int64_t)(nb * (sizeof(BlockInfo) + 8 + 4 + 4 + 8 + 8 + 1 + 1) +
                   nstreams * (8 + sizeof(ZStream)) + 64 + 16 + 16 + 1024);
}

// Workspace for the fast path: the base layout plus the speculative outputs of
// every raw block (kZBlock doubles each, ~8.4 bytes per normal).
extern "C" int64_t rm_normal_workspace_bytes_fast(int nstreams, int64_t n) {
  const int64_t base = rm_normal_workspace_bytes(nstreams, n);
  if (base < 0) return base;
  const long long nblocks = (long long)((1.04 * (double)n + 64.0 * sqrt((double)n + 1.0)) /
                                        kZBlock) + 8;
  return base + 256 + nblocks * nstreams * kZBlock * (int64_t)sizeof(double);
}

namespace rm {

static int z_nblocks(long long n) {
  return (int)((1.04 * (double)n + 64.0 * sqrt((double)n + 1.0)) / kZBlock) + 8;
}

// Workspace carve-up shared by every generator entry (the layout rm_normal_stats_offset
// describes; the scratch and the fused step's tables follow the base layout).
struct ZWs {
  BlockInfo* info;
  unsigned long long* offs;
  uint32_t* entry;
  uint32_t* tcount;
  uint64_t* bad;
  unsigned long long* total;
  ZStream* seeds;
  uint64_t* left;
  uint8_t* merged;
  uint32_t* nbad;
  uint32_t* nleft;
  uint8_t* valid;
  double* scratch;   // null: compact layout
  uint32_t* skip;    // fused step only
  ZDesc* desc;       // fused step only
  double* means;     // fused uniform step (copy side): column means
};

static long long z_groups(long long n) { return (n + kZGroup - 1) / kZGroup; }

static ZWs z_carve(const ZArgs& a, void* workspace, bool fast, bool fused) {
  const long long nb = (long long)a.nblocks * a.nstreams;
  ZWs w{};
  char* ws = static_cast<char*>(workspace);
  w.info = reinterpret_cast<BlockInfo*>(ws);
  ws += nb * sizeof(BlockInfo);
  w.offs = reinterpret_cast<unsigned long long*>(ws);
  ws += nb * 8;
  w.entry = reinterpret_cast<uint32_t*>(ws);
  ws += nb * 4;
  w.tcount = reinterpret_cast<uint32_t*>(ws);
  ws += nb * 4;
  w.bad = reinterpret_cast<uint64_t*>(ws);
  ws += nb * 8;
  w.total = reinterpret_cast<unsigned long long*>(ws);
  ws += a.nstreams * 8;
  ws = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 63) & ~(uintptr_t)63);
  w.seeds = reinterpret_cast<ZStream*>(ws);
  ws += a.nstreams * sizeof(ZStream);
  w.left = reinterpret_cast<uint64_t*>(ws);
  ws += nb * 8;
  w.merged = reinterpret_cast<uint8_t*>(ws);
  ws += nb;
  ws = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 15) & ~(uintptr_t)15);
  w.nbad = reinterpret_cast<uint32_t*>(ws);
  w.nleft = w.nbad + 1;
  ws += 16;
  // validity of the speculative outputs per block (1 = merged at its true entry)
  w.valid = reinterpret_cast<uint8_t*>(ws);
  ws += nb;
  if (fast) {
    ws = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    w.scratch = reinterpret_cast<double*>(ws);
    ws += nb * kZBlock * sizeof(double);
  }
  if (fused) {
    w.skip = reinterpret_cast<uint32_t*>(ws);
    ws += nb * 4;
    ws = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 15) & ~(uintptr_t)15);
    w.desc = reinterpret_cast<ZDesc*>(ws);
    ws += (long long)a.nstreams * z_groups(a.n) * (long long)sizeof(ZDesc);
    ws = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    w.means = reinterpret_cast<double*>(ws);
  }
  return w;
}

// seeding, speculation, merge, repairs and the per-stream scan (steps 1-3)
static int z_front(const ZArgs& a, const ZWs& w, cudaStream_t st) {
  const long long nb = (long long)a.nblocks * a.nstreams;
  cudaError_t e = cudaMemsetAsync(w.nbad, 0, 8, st);
  if (e != cudaSuccess) return fail_cuda(e, "cudaMemsetAsync");
  const int threads = 128;
  const long long grid = (nb + threads - 1) / threads;
  zig_seed_kernel<<<(a.nstreams + 63) / 64, 64, 0, st>>>(a, w.seeds);
  RM_CHECK_LAUNCH("zig_seed_kernel");
  if (w.scratch)
    zig_spec_kernel<true><<<(int)grid, threads, 0, st>>>(a, w.seeds, w.info, w.scratch);
  else
    zig_spec_kernel<false><<<(int)grid, threads, 0, st>>>(a, w.seeds, w.info, w.scratch);
  RM_CHECK_LAUNCH("zig_spec_kernel");
  zig_merge_kernel<<<(int)grid, threads, 0, st>>>(a, w.info, w.entry, w.tcount, w.merged, w.nbad,
                                                  w.bad);
  RM_CHECK_LAUNCH("zig_merge_kernel");
  e = cudaMemcpyAsync(w.valid, w.merged, nb, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return fail_cuda(e, "cudaMemcpyAsync(valid)");
  // isolated failures in parallel (grid sized for the worst case; idle CTAs exit at once)
  zig_repair_par_kernel<<<(int)grid, threads, 0, st>>>(a, w.seeds, w.info, w.entry, w.tcount,
                                                        w.merged, w.valid, w.nbad, w.bad, w.nleft,
                                                        w.left);
  RM_CHECK_LAUNCH("zig_repair_par_kernel");
  zig_repair_kernel<<<(a.nstreams + 31) / 32, 32, 0, st>>>(a, w.seeds, w.info, w.entry, w.tcount,
                                                           w.merged, w.valid, w.nleft, w.left,
                                                           w.nbad, w.bad);
  RM_CHECK_LAUNCH("zig_repair_kernel");
  zig_scan_kernel<<<a.nstreams, 1024, 0, st>>>(a, w.tcount, w.offs, w.total);
  RM_CHECK_LAUNCH("zig_scan_kernel");
  return 0;
}

// rm_set_shard_streams: the calling thread's learner interleave for the next generator calls
static thread_local int g_stream_run = 0;
static thread_local long long g_stream_period = 0;

static int z_args(ZArgs* a, const uint32_t* prefix, int nprefix, int append, uint64_t k,
                  int nstreams, long long n, long long stream0 = 0) {
  *a = ZArgs{};
  a->run = g_stream_run;
  a->period = g_stream_period;
  for (int i = 0; i < nprefix; i++) a->prefix[i] = prefix[i];
  a->nprefix = nprefix;
  a->append = append;
  a->k = k;
  a->nstreams = nstreams;
  a->n = n;
  a->nblocks = z_nblocks(n);
  a->stream0 = stream0;
  return ensure_jump_tables();
}

// Quadratic-oracle gradients for all learners of step k (see header).
template <typename T>
static int quad_grad(const uint32_t* prefix, int nprefix, int append, uint64_t k, int nstreams,
                     int64_t n,
                     const T* Phi, int64_t ldp, const double* lam, const double* wopt, double sd,
                     T* G, int64_t ldg, double* Z, int64_t ldz, void* workspace,
                     int64_t workspace_bytes, void* stream, long long stream0 = 0) {
  if (nprefix < 0 || nprefix > kZMaxPrefix || nstreams < 1 || n < 0 || append < 0 ||
      stream0 < 0 ||
      append > 2 || (append < 2 && nstreams != 1) ||
      workspace == nullptr || (G != nullptr && (Phi == nullptr || lam == nullptr ||
                                                wopt == nullptr || ldg < n || ldp < n)) ||
      (Z != nullptr && ldz < n)) {
    set_error("invalid normal/gradient arguments");
    return RM_EINVAL;
  }
  if (n == 0) return 0;
  const int64_t need = rm_normal_workspace_bytes(nstreams, n);
  if (workspace_bytes < need) {
    set_error("normal workspace too small: need %lld bytes", (long long)need);
    return RM_ERANGE;
  }
  ZArgs a;
  int rc = z_args(&a, prefix, nprefix, append, k, nstreams, n, stream0);
  if (rc) return rc;
  const long long nb = (long long)a.nblocks * nstreams;
  const ZWs w = z_carve(a, workspace,
                        workspace_bytes >= rm_normal_workspace_bytes_fast(nstreams, n), false);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = z_front(a, w, st))) return rc;
  if (w.scratch) {
    zig_copy_kernel<T><<<(int)((nb * 32 + 255) / 256), 256, 0, st>>>(
        a, w.info, w.entry, w.tcount, w.offs, w.valid, w.scratch, Phi, ldp, lam, wopt, sd, G, ldg,
        Z, ldz);
    RM_CHECK_LAUNCH("zig_copy_kernel");
    zig_fixup_kernel<T><<<(int)((2 * nb + 127) / 128), 128, 0, st>>>(
        a, w.seeds, w.entry, w.offs, w.valid, w.nbad, w.bad, w.nleft, w.left, Phi, ldp, lam, wopt,
        sd, G, ldg, Z, ldz);
    RM_CHECK_LAUNCH("zig_fixup_kernel");
  } else {
    const long long groups = (a.nblocks + kZGenThreads - 1) / kZGenThreads;
    zig_gen_kernel<T><<<(int)(groups * nstreams), kZGenThreads, 0, st>>>(
        a, w.seeds, w.entry, w.tcount, w.offs, Phi, ldp, lam, wopt, sd, G, ldg, Z, ldz);
    RM_CHECK_LAUNCH("zig_gen_kernel");
  }
  return 0;
}

// ---- fused gradient + mix step (zsrc.cuh) ----
// Blocks whose speculation did not merge: their true outputs are regenerated into their
// own scratch slot from index 0 (skip 0 in the descriptors).
__global__ void __launch_bounds__(128)
    zig_fixup_scratch_kernel(ZArgs a, const ZStream* __restrict__ seeds,
                             const uint32_t* __restrict__ entry, const uint8_t* __restrict__ valid,
                             const uint32_t* __restrict__ nbad, const uint64_t* __restrict__ bad,
                             const uint32_t* __restrict__ nleft, const uint64_t* __restrict__ left,
                             double* __restrict__ scratch) {
  __shared__ ZigTables Tb;
  const uint32_t n1 = *nbad, n2 = *nleft;
  if (blockIdx.x * blockDim.x >= n1 + n2) return;  // CTA-uniform
  load_tables(&Tb);
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n1 + n2) return;
  const long long gid = (long long)(i < n1 ? bad[i] : left[i - n1]);
  if (valid[gid]) return;
  const int stream = (int)(gid / a.nblocks);
  const int b = (int)(gid % a.nblocks);
  const ZStream zs = seeds[stream];
  uint32_t pos = entry[gid], cnt = 0;
  ZGen g{z_jump(zs, (uint64_t)b * kZBlock + pos), zs.inc};
  double* dst = scratch + gid * kZBlock;
  while (pos < (uint32_t)kZBlock) {
    double x;
    int extra;
    if (z_attempt(Tb, g, g.next64(), &x, &extra)) dst[cnt++] = x;
    pos += 1 + extra;
  }
}

__device__ __forceinline__ uint32_t z_skip_of(const BlockInfo* info, const uint32_t* entry,
                                              const uint8_t* valid, long long gid) {
  if (!valid[gid]) return 0u;
  const uint32_t e = entry[gid];
  return __popc(info[gid].outs & ((1u << e) - 1u));
}

// skip per block and the (stream, 128-column group) descriptors of zsrc.cuh: the block
// that holds a group's first column writes the group's descriptor
__global__ void __launch_bounds__(256)
    zig_zindex_kernel(ZArgs a, const BlockInfo* __restrict__ info,
                      const uint32_t* __restrict__ entry, const uint32_t* __restrict__ tcount,
                      const unsigned long long* __restrict__ offs,
                      const uint8_t* __restrict__ valid, uint32_t* __restrict__ skip,
                      ZDesc* __restrict__ desc, long long ngroups, int force_walk) {
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)a.nstreams * a.nblocks) return;
  const int stream = (int)(gid / a.nblocks);
  const int b = (int)(gid % a.nblocks);
  const uint32_t sk = z_skip_of(info, entry, valid, gid);
  skip[gid] = sk;
  const long long lo = (long long)offs[gid], cnt = tcount[gid], hi = lo + cnt;
  if (cnt == 0 || lo >= a.n) return;
  for (long long s = (lo + kZGroup - 1) & ~(long long)(kZGroup - 1); s < hi && s < a.n;
       s += kZGroup) {
    ZDesc g;
    g.zb = gid * kZBlock + sk - lo;
    g.dz = 0;
    g.brk = kZGroup;
    const long long e = min(s + kZGroup, a.n);
    if (force_walk) {
      g.zb = gid;
      g.brk = -1;
    } else if (hi < e) {
      // the group continues in block b + 1 (which exists: the stream has outputs left)
      const long long g1 = gid + 1;
      const long long cnt1 = b + 1 < a.nblocks ? (long long)tcount[g1] : 0;
      if (cnt1 == 0 || hi + cnt1 < e) {
        g.zb = gid;   // three or more blocks: walk (zsrc.cuh)
        g.brk = -1;
      } else {
        const long long zb1 = g1 * kZBlock + z_skip_of(info, entry, valid, g1) - hi;
        g.dz = (int)(zb1 - g.zb);
        g.brk = (int)(hi - s);
      }
    }
    desc[(long long)stream * ngroups + (s >> kZGroupLog2)] = g;
  }
}

// ---- fused gradient + mix, copy side ----
// One warp per raw block of one stream (stream-fastest order, like zig_copy_kernel): the
// warp's true normals are read coalesced from the scratch and, for each output column c,
//   out[j][c] = fl_T( ring3(W[a][c], W[b][c], W[cc][c]) - fl(lr * g) )    (ring)
//   out[j][c] = fl_T( M[c] - fl(lr * g) )                                 (uniform)
// with g = fl_T(lam[c] (Phi[j][c] - w*[c]) + sd z) — the operations of the two-pass path.
// Concurrent warps cover the same column window of every stream (the streams' output
// offsets differ by a few blocks), so the neighbour rows' W is read from HBM once and
// served from L2 to the other two readers.
template <typename T, bool RING, bool PHI>
__global__ void __launch_bounds__(256)
    zig_mix_kernel(ZArgs a, const BlockInfo* __restrict__ info, const uint32_t* __restrict__ entry,
                   const uint32_t* __restrict__ tcount, const unsigned long long* __restrict__ offs,
                   const uint8_t* __restrict__ valid, const double* __restrict__ scratch,
                   const T* __restrict__ W, long long ldw, const T* __restrict__ Phi,
                   long long ldp, const int32_t* __restrict__ left,
                   const int32_t* __restrict__ right, const double* __restrict__ means,
                   const double* __restrict__ lam, const double* __restrict__ wopt, double sd,
                   double lr, T* __restrict__ out, long long ldo,
                   unsigned long long* __restrict__ absmax) {
  using E = Elem<T>;
  using A = typename E::acc;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  typename E::amax_t amax = 0;
  if (w < (long long)a.nstreams * a.nblocks) {
    const int j = (int)(w % a.nstreams);
    const long long gid = (long long)j * a.nblocks + w / a.nstreams;
    const unsigned long long base = offs[gid];
    if (base < (unsigned long long)a.n) {
      const uint32_t skip = z_skip_of(info, entry, valid, gid);
      const uint32_t lim = min((unsigned long long)tcount[gid], (unsigned long long)a.n - base);
      const double* src = scratch + gid * kZBlock + skip;
      int x0 = j, x1 = j, x2 = j, self = 0;
      if (RING) {
        int t;
        x0 = left[j];
        x2 = right[j];
        if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
        if (x2 < x1) { t = x1; x1 = x2; x2 = t; }
        if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
        self = x0 == j ? 0 : (x1 == j ? 1 : 2);
      }
      const T* wa = W + (long long)x0 * ldw + base;
      const T* wb = W + (long long)x1 * ldw + base;
      const T* wc = W + (long long)x2 * ldw + base;
      const T* ph = PHI ? Phi + (long long)j * ldp + base : W + (long long)j * ldw + base;
      T* dst = out + (long long)j * ldo + base;
      // two halves of four 32-column runs: every load of a half is issued before use
#pragma unroll
      for (int h = 0; h < kZBlock / 32; h += 4) {
        double z[4], lm[4], wo[4], mm[4], pv[4];
        A va[4], vb[4], vc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t i = lane + 32 * (h + q);
          const bool on = i < lim;
          const unsigned long long c = base + i;
          z[q] = on ? __ldcs(src + i) : 0.0;
          lm[q] = on ? __ldg(lam + c) : 0.0;
          wo[q] = on ? __ldg(wopt + c) : 0.0;
          if (RING) {
            va[q] = on ? (A)E::ld(wa + i, 0) : (A)0;
            vb[q] = on ? (A)E::ld(wb + i, 0) : (A)0;
            vc[q] = on ? (A)E::ld(wc + i, 0) : (A)0;
          } else {
            mm[q] = on ? __ldg(means + c) : 0.0;
          }
          if (PHI || !RING) pv[q] = on ? (double)E::ld(ph + i, 0) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t i = lane + 32 * (h + q);
          if (i >= lim) continue;
          A m;
          double phi;
          if (RING) {
            m = ring3<A>(va[q], vb[q], vc[q]);
            phi = PHI ? pv[q] : (double)(self == 0 ? va[q] : (self == 1 ? vb[q] : vc[q]));
          } else {
            m = (A)mm[q];
            phi = pv[q];
          }
          const T g = E::st((A)z_grad(lm[q], wo[q], sd, phi, z[q]));
          const T y = E::st(r_sub(m, r_mul((A)lr, (A)g)));
          amax = E::amax_acc(amax, y);
          __stcs(dst + i, y);
        }
      }
    }
  }
  if (absmax) {
    unsigned long long bits = E::amax_bits(amax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
      bits = other > bits ? other : bits;
    }
    if (lane == 0) absmax_publish(absmax, bits);
  }
}

template <typename T>
int quad_mix_copy(const uint32_t* prefix, int nprefix, uint64_t k, const T* W, const T* Phi,
                  T* out, const int32_t* left, const int32_t* right, int L, long long d,
                  long long ldw, long long ldp, long long ldo, const double* lam,
                  const double* wopt, double sd, double lr, unsigned long long* absmax, void* ws,
                  long long ws_bytes, void* stream, long long stream0, const double* ext_means,
                  void* means_ready) {
  const long long need = quad_z_workspace_bytes(L, d);
  if (ws == nullptr || ws_bytes < need) {
    set_error("fused gradient workspace too small: need %lld bytes", need);
    return RM_ERANGE;
  }
  ZArgs a;
  int rc = z_args(&a, prefix, nprefix, 2, k, L, d, stream0);
  if (rc) return rc;
  const long long nb = (long long)a.nblocks * L;
  ZWs w = z_carve(a, ws, true, true);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool ring = left != nullptr;
  if (ext_means != nullptr) {
    // means computed elsewhere (a learner-sharded run's global average, produced
    // concurrently on other streams / GPUs): only the mix waits for them
    w.means = const_cast<double*>(ext_means);
  } else if (!ring) {
    // the uniform step's column means (numpy pairwise order, the two-pass mean's bits)
    rc = sizeof(T) == 4 ? rm_column_mean_f32(reinterpret_cast<const float*>(W), L, d, ldw,
                                             w.means, stream)
                        : rm_column_mean_f64(reinterpret_cast<const double*>(W), L, d, ldw,
                                             w.means, stream);
    if (rc) return rc;
  }
  if ((rc = z_front(a, w, st))) return rc;
  zig_fixup_scratch_kernel<<<(int)((2 * nb + 127) / 128), 128, 0, st>>>(
      a, w.seeds, w.entry, w.valid, w.nbad, w.bad, w.nleft, w.left, w.scratch);
  RM_CHECK_LAUNCH("zig_fixup_scratch_kernel");
  if (means_ready != nullptr) {
    const cudaError_t e = cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(means_ready), 0);
    if (e != cudaSuccess) return fail_cuda(e, "cudaStreamWaitEvent(means_ready)");
  }
  const long long grid = (nb * 32 + 255) / 256;
  auto launch = [&](auto kern) {
    kern<<<(int)grid, 256, 0, st>>>(a, w.info, w.entry, w.tcount, w.offs, w.valid, w.scratch, W,
                                     ldw, Phi, ldp, left, right, w.means, lam, wopt, sd, lr, out,
                                     ldo, absmax);
  };
  if (ring) {
    if (Phi) launch(zig_mix_kernel<T, true, true>);
    else launch(zig_mix_kernel<T, true, false>);
  } else {
    if (Phi) launch(zig_mix_kernel<T, false, true>);
    else launch(zig_mix_kernel<T, false, false>);
  }
  RM_CHECK_LAUNCH("zig_mix_kernel");
  return 0;
}
template int quad_mix_copy<float>(const uint32_t*, int, uint64_t, const float*, const float*,
                                  float*, const int32_t*, const int32_t*, int, long long,
                                  long long, long long, long long, const double*, const double*,
                                  double, double, unsigned long long*, void*, long long, void*,
                                  long long, const double*, void*);
template int quad_mix_copy<double>(const uint32_t*, int, uint64_t, const double*, const double*,
                                   double*, const int32_t*, const int32_t*, int, long long,
                                   long long, long long, long long, const double*, const double*,
                                   double, double, unsigned long long*, void*, long long, void*,
                                   long long, const double*, void*);

long long quad_z_workspace_bytes(int nstreams, long long n) {
  const int64_t fast = rm_normal_workspace_bytes_fast(nstreams, n);
  if (fast < 0) return fast;
  const long long nb = (long long)z_nblocks(n) * nstreams;
  // + the column means of the uniform step (copy-side fused kernel)
  return fast + nb * 4 + 16 + (long long)nstreams * z_groups(n) * (long long)sizeof(ZDesc) +
         n * 8 + 256;
}

int quad_z_prepare(const uint32_t* prefix, int nprefix, uint64_t k, int nstreams, long long n,
                   void* workspace, long long workspace_bytes, void* stream, ZSrc* z,
                   long long stream0) {
  if (nprefix < 0 || nprefix > kZMaxPrefix || nstreams < 1 || n < 0 || workspace == nullptr ||
      stream0 < 0) {
    set_error("invalid fused gradient arguments");
    return RM_EINVAL;
  }
  if (n == 0) return 0;
  const long long need = quad_z_workspace_bytes(nstreams, n);
  if (workspace_bytes < need) {
    set_error("fused gradient workspace too small: need %lld bytes", need);
    return RM_ERANGE;
  }
  ZArgs a;
  int rc = z_args(&a, prefix, nprefix, 2, k, nstreams, n, stream0);
  if (rc) return rc;
  const long long nb = (long long)a.nblocks * nstreams;
  const ZWs w = z_carve(a, workspace, true, true);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = z_front(a, w, st))) return rc;
  zig_fixup_scratch_kernel<<<(int)((2 * nb + 127) / 128), 128, 0, st>>>(
      a, w.seeds, w.entry, w.valid, w.nbad, w.bad, w.nleft, w.left, w.scratch);
  RM_CHECK_LAUNCH("zig_fixup_scratch_kernel");
  const long long ngroups = z_groups(n);
  // RINGMIX_ZDESC_WALK=1 (tests): every lookup takes the walk fallback of zsrc.cuh
  const char* walk = getenv("RINGMIX_ZDESC_WALK");
  zig_zindex_kernel<<<(int)((nb + 255) / 256), 256, 0, st>>>(
      a, w.info, w.entry, w.tcount, w.offs, w.valid, w.skip, w.desc, ngroups,
      walk != nullptr && walk[0] == '1');
  RM_CHECK_LAUNCH("zig_zindex_kernel");
  z->scratch = w.scratch;
  z->desc = w.desc;
  z->ngroups = ngroups;
  z->offs = w.offs;
  z->tcount = w.tcount;
  z->skip = w.skip;
  return 0;
}

}  // namespace rm

// Learner sets of an interleaved sharding (numpy-order D1D: a rank holds runs of `run`
// consecutive learners every `period`): stream s of the following rm_quadratic_grad_shard_* /
// rm_quadratic_mean_step_shard_* calls from this host thread is learner
// learner0 + (s / run) * period + s % run.  run = 0 restores contiguous learners.
extern "C" int rm_set_shard_streams(int run, int64_t period) {
  if (run < 0 || (run > 0 && period < run)) {
    set_error("invalid learner interleave (run %d, period %lld)", run, (long long)period);
    return RM_EINVAL;
  }
  g_stream_run = run;
  g_stream_period = run > 0 ? period : 0;
  return 0;
}

extern "C" int rm_quadratic_grad_f32(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                     int L, int64_t d, const float* Phi, int64_t ldp,
                                     const double* lam, const double* wopt, double noise_sd,
                                     float* G, int64_t ldg, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  return quad_grad<float>(prefix_words, n_prefix, 2, k, L, d, Phi, ldp, lam, wopt, noise_sd, G, ldg,
                          nullptr, 0, workspace, workspace_bytes, stream);
}

extern "C" int rm_quadratic_grad_f64(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                     int L, int64_t d, const double* Phi, int64_t ldp,
                                     const double* lam, const double* wopt, double noise_sd,
                                     double* G, int64_t ldg, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  return quad_grad<double>(prefix_words, n_prefix, 2, k, L, d, Phi, ldp, lam, wopt, noise_sd, G, ldg,
                           nullptr, 0, workspace, workspace_bytes, stream);
}

// Learners [learner0, learner0 + L) of a learner-sharded run (stream index learner0 + l).
extern "C" int rm_quadratic_grad_shard_f32(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                           int64_t learner0, int L, int64_t d, const float* Phi,
                                           int64_t ldp, const double* lam, const double* wopt,
                                           double noise_sd, float* G, int64_t ldg,
                                           void* workspace, int64_t workspace_bytes,
                                           void* stream) {
  return quad_grad<float>(prefix_words, n_prefix, 2, k, L, d, Phi, ldp, lam, wopt, noise_sd, G, ldg,
                          nullptr, 0, workspace, workspace_bytes, stream, learner0);
}

extern "C" int rm_quadratic_grad_shard_f64(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                           int64_t learner0, int L, int64_t d, const double* Phi,
                                           int64_t ldp, const double* lam, const double* wopt,
                                           double noise_sd, double* G, int64_t ldg,
                                           void* workspace, int64_t workspace_bytes,
                                           void* stream) {
  return quad_grad<double>(prefix_words, n_prefix, 2, k, L, d, Phi, ldp, lam, wopt, noise_sd, G,
                           ldg, nullptr, 0, workspace, workspace_bytes, stream, learner0);
}

// D1D step of a learner-sharded run with the oracle's gradient fused in:
//   Wout[l] = M - lr * G(Phi[l]),  G of learner learner0 + l  (simulation.py:304-312)
// M = the global column means, produced concurrently (other streams / GPUs); the generator
// runs at once and only the final mix waits for `means_ready` (a cudaEvent_t, may be NULL).
#define RM_DEFINE_MEAN_STEP_SHARD(SUFFIX, CT)                                                  \
  extern "C" int rm_quadratic_mean_step_shard_##SUFFIX(                                        \
      const uint32_t* prefix_words, int n_prefix, uint64_t k, int64_t learner0,               \
      const double* M, const CT* Phi, CT* Wout, int L, int64_t d, int64_t ldp, int64_t ldo,   \
      const double* lam, const double* wopt, double noise_sd, double lr,                       \
      unsigned long long* absmax_bits, void* workspace, int64_t workspace_bytes, void* stream, \
      void* means_ready) {                                                                     \
    if (M == nullptr || Phi == nullptr || Wout == nullptr || lam == nullptr || wopt == nullptr || \
        L < 1 || d < 1 || ldp < d || ldo < d || learner0 < 0) {                                \
      set_error("invalid sharded mean-step arguments");                                       \
      return RM_EINVAL;                                                                        \
    }                                                                                          \
    return quad_mix_copy<CT>(prefix_words, n_prefix, k, Phi, Phi, Wout, nullptr, nullptr, L, d, \
                             ldp, ldp, ldo, lam, wopt, noise_sd, lr, absmax_bits, workspace,   \
                             workspace_bytes, stream, learner0, M, means_ready);               \
  }
RM_DEFINE_MEAN_STEP_SHARD(f32, float)
RM_DEFINE_MEAN_STEP_SHARD(f64, double)

extern "C" int rm_standard_normal_f64(const uint32_t* prefix_words, int n_prefix, int append,
                                      uint64_t k, int nstreams, int64_t n, double* Z,
                                      int64_t ldz, void* workspace, int64_t workspace_bytes,
                                      void* stream) {
  return quad_grad<double>(prefix_words, n_prefix, append, k, nstreams, n, nullptr, 0, nullptr, nullptr,
                           0.0, nullptr, 0, Z, ldz, workspace, workspace_bytes, stream);
}

// Element-wise glibc-compatible log1p (pins glibc_log1p against the host libm in tests).
namespace rm {
__global__ void log1p_kernel(const double* __restrict__ x, double* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = glibc_log1p(x[i]);
}
}  // namespace rm

extern "C" int rm_log1p_f64(const double* x, double* y, int64_t n, void* stream) {
  if (x == nullptr || y == nullptr || n < 0) {
    set_error("invalid log1p arguments");
    return RM_EINVAL;
  }
  if (n == 0) return 0;
  long long blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  log1p_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, y, n);
  RM_CHECK_LAUNCH("log1p_kernel");
  return 0;
}

// Byte offset, inside the workspace of the last rm_quadratic_grad_* /
// rm_standard_normal_f64 call with this shape, of two uint32 counters:
// speculation failures and failures left to the sequential repair (diagnostics).
extern "C" int64_t rm_normal_stats_offset(int nstreams, int64_t n) {
  if (nstreams < 1 || n < 0) return -1;
  const long long nblocks = (long long)((1.04 * (double)n + 64.0 * sqrt((double)n + 1.0)) /
                                        kZBlock) + 8;
  const long long nb = nblocks * nstreams;
  uintptr_t off = (uintptr_t)(nb * (sizeof(BlockInfo) + 8 + 4 + 4 + 8) + nstreams * 8);
  off = (off + 63) & ~(uintptr_t)63;
  off += nstreams * sizeof(ZStream) + nb * 8 + nb;
  off = (off + 15) & ~(uintptr_t)15;
  return (int64_t)off;
}
