// The step on the reference's own array layout: W, G, W' as (d, L) C-order
// matrices — row r holds coordinate r of every learner (simulation.py:209, 267;
// mixing.py:125 computes W @ T on exactly this array).  In this layout the mix
// never leaves a row: out[r, j] = ring3(W[r, a], W[r, b], W[r, c]) - lr * G[r, j]
// with {a, b, c} = sorted {left[j], j, right[j]}, and the D1D mean is the
// pairwise sum of row r's L contiguous values.  So no transpose is needed: a
// CTA stages a tile of R whole rows of W in shared memory (coalesced 16-byte
// loads), gathers the three inputs of every output from it, and streams G in
// and W' out row-contiguously.
//
// Arithmetic is the learner-major kernels': fp32 / fp64 storage
// computes the reference's fp64 sequence and rounds once; bf16 computes in fp32.
#include "common.cuh"
#include "arith.cuh"
#include "../../include/ringmix_b200.h"

namespace rm {

constexpr int kDLThreads = 256;
constexpr int kDLTileBytes = 32 * 1024;   // W rows staged per tile

struct DLArgs {
  const void* W;
  const void* G;
  void* out;
  long long ldw, ldg, ldo;   // row strides (elements), >= L
  long long d;               // rows
  int L;
  int R;                     // rows per tile
  const int32_t* left;
  const int32_t* right;
  double lr;
  unsigned long long* absmax;
};

template <typename T, bool MEAN, bool HAS_G>
__global__ void __launch_bounds__(kDLThreads) mix_dL_kernel(DLArgs a) {
  using E = Elem<T>;
  using A = typename E::acc;
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = a.L, R = a.R;
  int4* s_tri = reinterpret_cast<int4*>(smem);
  double* s_mean = reinterpret_cast<double*>(s_tri + L);
  T* s_w = reinterpret_cast<T*>(s_mean + ((R + 1) & ~1));   // 16-byte aligned rows
  const T* W = static_cast<const T*>(a.W);
  const T* G = static_cast<const T*>(a.G);
  T* out = static_cast<T*>(a.out);
  const int tid = threadIdx.x;
  pdl_wait();
  if (!MEAN) {
    for (int j = tid; j < L; j += kDLThreads) {
      int x0 = a.left[j], x1 = j, x2 = a.right[j], t;
      if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
      if (x2 < x1) { t = x1; x1 = x2; x2 = t; }
      if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
      s_tri[j] = make_int4(x0, x1, x2, j);
    }
  }
  const A lr = (A)a.lr;
  typename E::amax_t amax = 0;
  const long long ntiles = (a.d + R - 1) / R;
  // 16-byte staging when every row starts 16-byte aligned
  constexpr int VEC = 16 / sizeof(T);
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(W) | (uintptr_t)(a.ldw * sizeof(T))) & 15) == 0 &&
                      L % VEC == 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long r0 = t * R;
    const int rows = (int)min((long long)R, a.d - r0);
    __syncthreads();   // previous tile's readers are done with s_w / s_mean
    if (vec_ok) {
      const int nv = L / VEC;
      for (int i = tid; i < rows * nv; i += kDLThreads) {
        const int r = i / nv, v = i - r * nv;
        const uint4 x = __ldcs(reinterpret_cast<const uint4*>(W + (r0 + r) * a.ldw) + v);
        *reinterpret_cast<uint4*>(s_w + r * L + v * VEC) = x;
      }
    } else {
      for (int i = tid; i < rows * L; i += kDLThreads) {
        const int r = i / L, j = i - r * L;
        s_w[i] = W[(r0 + r) * a.ldw + j];
      }
    }
    __syncthreads();
    if (MEAN) {
      for (int r = tid; r < rows; r += kDLThreads) {
        const T* row = s_w + r * L;
        auto get = [&](int i) { return (A)E::ld(row, i); };
        s_mean[r] = (double)r_div(pairwise_sum<A>(get, 0, L), (A)L);
      }
      __syncthreads();
    }
    for (int i = tid; i < rows * L; i += kDLThreads) {
      const int r = i / L, j = i - r * L;
      A m;
      if (MEAN) {
        m = (A)s_mean[r];
      } else {
        const int4 tri = s_tri[j];
        const T* row = s_w + r * L;
        m = ring3<A>((A)E::ld(row, tri.x), (A)E::ld(row, tri.y), (A)E::ld(row, tri.z));
      }
      if (HAS_G) m = r_sub(m, r_mul(lr, (A)E::ld(G + (r0 + r) * a.ldg + j, 0)));
      const T y = E::st(m);
      out[(r0 + r) * a.ldo + j] = y;
      amax = E::amax_acc(amax, y);
    }
  }
  if (a.absmax) absmax_publish(a.absmax, E::amax_bits(amax));
}

template <typename T, bool MEAN>
static int launch_dL(DLArgs a, cudaStream_t st) {
  const size_t esz = sizeof(T);
  int R = (int)(kDLTileBytes / (a.L * esz));
  if (R < 1) R = 1;
  if (R > 1024) R = 1024;
  a.R = R;
  const size_t smem = (size_t)a.L * sizeof(int4) + (size_t)((R + 1) & ~1) * sizeof(double) +
                      (size_t)R * a.L * esz;
  auto kern = a.G ? mix_dL_kernel<T, MEAN, true> : mix_dL_kernel<T, MEAN, false>;
  static unsigned long long attr_mask = 0;
  if (attr_needed(&attr_mask)) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(mix_dL_kernel<T, MEAN, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024)) !=
            cudaSuccess ||
        (e = cudaFuncSetAttribute(mix_dL_kernel<T, MEAN, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024)) !=
            cudaSuccess)
      return fail_cuda(e, "cudaFuncSetAttribute(mix_dL_kernel)");
    attr_done(&attr_mask);
  }
  if (smem > 160 * 1024) {
    set_error("(d, L) tile does not fit shared memory (L=%d)", a.L);
    return RM_ERANGE;
  }
  const long long ntiles = (a.d + R - 1) / R;
  long long grid = 4LL * sm_count(-1);
  if (grid > ntiles) grid = ntiles;
  cudaError_t e = launch_pdl(kern, dim3((unsigned)grid), dim3(kDLThreads), smem, st, a);
  if (e != cudaSuccess) return fail_cuda(e, "mix_dL_kernel");
  return RM_OK;
}

template <typename T>
int dispatch_dL(const T* W, const T* G, T* out, const int32_t* left, const int32_t* right, int L,
                long long d, long long ldw, long long ldg, long long ldo, double lr,
                unsigned long long* absmax, void* stream) {
  const bool mean = left == nullptr && right == nullptr;
  if (L < 1 || d < 0 || (d > 0 && (W == nullptr || out == nullptr)) || ldw < L || ldo < L ||
      (G != nullptr && ldg < L)) {
    set_error("invalid (d, L) arguments: L=%d d=%lld", L, d);
    return RM_EINVAL;
  }
  if (!mean) {
    if (left == nullptr || right == nullptr) {
      set_error("ring mix needs left/right neighbour tables");
      return RM_EINVAL;
    }
    if (L < 3) {
      set_error("degenerate ring topology: need at least 3 learners, got %d", L);
      return RM_EINVAL;
    }
  }
  if (d == 0) return RM_OK;
  if (W == out) {
    set_error("in-place mixing is a read-after-write hazard across learners; use distinct buffers");
    return RM_EINVAL;
  }
  DLArgs a{};
  a.W = W;
  a.G = G;
  a.out = out;
  a.ldw = ldw;
  a.ldg = ldg;
  a.ldo = ldo;
  a.d = d;
  a.L = L;
  a.left = left;
  a.right = right;
  a.lr = lr;
  a.absmax = absmax;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // mixing.py:122-124: every entry of the 3-ring is 1/L, so the reference takes the
  // exact column-mean path
  if (mean || L == 3) return launch_dL<T, true>(a, st);
  return launch_dL<T, false>(a, st);
}

template int dispatch_dL<float>(const float*, const float*, float*, const int32_t*,
                                const int32_t*, int, long long, long long, long long, long long,
                                double, unsigned long long*, void*);
template int dispatch_dL<double>(const double*, const double*, double*, const int32_t*,
                                 const int32_t*, int, long long, long long, long long, long long,
                                 double, unsigned long long*, void*);

}  // namespace rm

using namespace rm;

#define RM_DEFINE_DL(SUFFIX, CT, T)                                                               \
  extern "C" int rm_gossip_step_dL_##SUFFIX(const CT* W, const CT* G, CT* out,                   \
                                            const int32_t* left, const int32_t* right, int L,    \
                                            int64_t d, int64_t ldw, int64_t ldg, int64_t ldo,    \
                                            double lr, unsigned long long* absmax_bits,          \
                                            void* stream) {                                      \
    return dispatch_dL<T>(reinterpret_cast<const T*>(W), reinterpret_cast<const T*>(G),         \
                          reinterpret_cast<T*>(out), left, right, L, d, ldw, ldg, ldo, lr,       \
                          absmax_bits, stream);                                                  \
  }

RM_DEFINE_DL(f32, float, float)
RM_DEFINE_DL(f64, double, double)
