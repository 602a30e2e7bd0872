// Arithmetic shared by the mix kernels: storage traits, rounding-explicit
// fp ops, the reference's ring FMA chain and numpy's pairwise summation
// (DESIGN.md §4), plus the 2-D TMA helpers.
#pragma once
#include "common.cuh"
#include <cuda.h>

namespace rm {

// ----------------------------------------------------------------------------
// element traits
// ----------------------------------------------------------------------------
template <typename T>
struct Elem;

// max|y| is tracked on the bit pattern of |y| in the storage type (monotone for
// non-negative IEEE values; NaN patterns sort above inf) and widened to the
// double bit pattern once at the end.
template <>
struct Elem<float> {
  using acc = double;
  using amax_t = uint32_t;
  static constexpr int VEC = 4;
  __device__ static __forceinline__ uint32_t amax_acc(uint32_t m, float y) {
    return max(m, __float_as_uint(y) & 0x7fffffffu);
  }
  __device__ static __forceinline__ unsigned long long amax_bits(uint32_t m) {
    return abs_bits((double)__uint_as_float(m));
  }
  __device__ static __forceinline__ double ld(const float* p, int i) { return (double)p[i]; }
  // explicit shared-memory load (generic pointers into smem otherwise compile
  // to generic LD.E)
  __device__ static __forceinline__ double lds(const float* p) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return (double)v;
  }
  __device__ static __forceinline__ float st(double y) { return __double2float_rn(y); }
  __device__ static __forceinline__ double absd(float y) { return fabs((double)y); }
};

template <>
struct Elem<double> {
  using acc = double;
  using amax_t = unsigned long long;
  static constexpr int VEC = 2;
  __device__ static __forceinline__ unsigned long long amax_acc(unsigned long long m, double y) {
    unsigned long long b = abs_bits(y);
    return b > m ? b : m;
  }
  __device__ static __forceinline__ unsigned long long amax_bits(unsigned long long m) {
    return m;
  }
  __device__ static __forceinline__ double ld(const double* p, int i) { return p[i]; }
  __device__ static __forceinline__ double lds(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
    return v;
  }
  __device__ static __forceinline__ double st(double y) { return y; }
  __device__ static __forceinline__ double absd(double y) { return fabs(y); }
};

template <>
struct Elem<__nv_bfloat16> {
  using acc = float;
  using amax_t = uint32_t;
  static constexpr int VEC = 8;
  __device__ static __forceinline__ uint32_t amax_acc(uint32_t m, __nv_bfloat16 y) {
    return max(m, (uint32_t)(__bfloat16_as_ushort(y) & 0x7fffu));
  }
  __device__ static __forceinline__ unsigned long long amax_bits(uint32_t m) {
    return abs_bits((double)__bfloat162float(__ushort_as_bfloat16((unsigned short)m)));
  }
  __device__ static __forceinline__ float ld(const __nv_bfloat16* p, int i) {
    return __bfloat162float(p[i]);
  }
  __device__ static __forceinline__ float lds(const __nv_bfloat16* p) {
    unsigned short v;
    asm volatile("ld.shared.b16 %0, [%1];" : "=h"(v) : "r"(smem_u32(p)));
    return __bfloat162float(__ushort_as_bfloat16(v));
  }
  __device__ static __forceinline__ __nv_bfloat16 st(float y) { return __float2bfloat16_rn(y); }
  __device__ static __forceinline__ double absd(__nv_bfloat16 y) {
    return fabs((double)__bfloat162float(y));
  }
};

// rounding-explicit arithmetic (never contracted)
__device__ __forceinline__ double r_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float r_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double r_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float r_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double r_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float r_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double r_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float r_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double r_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float r_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

template <typename A>
__device__ __forceinline__ A third();
template <>
__device__ __forceinline__ double third<double>() { return 1.0 / 3.0; }
template <>
__device__ __forceinline__ float third<float>() { return 1.0f / 3.0f; }

template <typename A>
__device__ __forceinline__ A ring3(A wa, A wb, A wc) {
  const A t = third<A>();
  A acc = r_mul(wa, t);
  acc = r_fma(wb, t, acc);
  return r_fma(wc, t, acc);
}

// numpy DOUBLE_pairwise_sum over n values at stride `st` (generic, recursive
// in blocks; used by the scalar paths).  `get(i)` loads value i.
template <typename A, typename F>
__device__ A pairwise_sum(F get, int lo, int n) {
  if (n < 8) {
    A res = -0.0;
    for (int i = 0; i < n; i++) res = r_add(res, get(lo + i));
    return res;
  }
  if (n <= 128) {
    A r[8];
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = get(lo + k);
    int i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int k = 0; k < 8; k++) r[k] = r_add(r[k], get(lo + i + k));
    }
    A res = r_add(r_add(r_add(r[0], r[1]), r_add(r[2], r[3])),
                  r_add(r_add(r[4], r[5]), r_add(r[6], r[7])));
    for (; i < n; i++) res = r_add(res, get(lo + i));
    return res;
  }
  // recursion depth is log2(L/128); L <= 2^31 keeps it tiny.  Iterate the
  // left spine explicitly to avoid deep device recursion.
  int n2 = n / 2;
  n2 -= n2 % 8;
  A left = pairwise_sum<A>(get, lo, n2);
  A right = pairwise_sum<A>(get, lo + n2, n - n2);
  return r_add(left, right);
}

template <typename T>
struct Vec {
  uint4 raw;
  __device__ __forceinline__ const T* e() const { return reinterpret_cast<const T*>(&raw); }
  __device__ __forceinline__ T* e() { return reinterpret_cast<T*>(&raw); }
};

__device__ __forceinline__ void tma_load_2d(void* sdst, const CUtensorMap* map, int c, int r,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sdst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(r), "r"(smem_u32(bar))
      : "memory");
}

// TMA tensor store shared -> global (bulk-group completion), and its ordering helpers
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* ssrc, int c,
                                             int r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c), "r"(r), "r"(smem_u32(ssrc))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}


}  // namespace rm
