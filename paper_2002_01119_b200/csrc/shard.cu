// Learner-sharded multi-GPU path (north-star (d)).
//
// Rank g owns learners [row0, row0 + Lg) of the global ring.  Per RAD step
// every rank derives the same permutation from the shared seed (no
// communication); the only cross-GPU traffic is the
// neighbour rows its learners need from other ranks.
//
// mix_shard_kernel fuses that exchange into the mix itself: for every column
// tile, one elected thread TMA-loads the local W and G rows from HBM while all
// threads pull the remote neighbour rows straight out of the peers' HBM over
// NVLink with cp.async (16 B, peer pointers from CUDA IPC); both land in the
// same shared-memory stage and complete on one mbarrier (expect_tx for the TMA
// bytes + one cp.async.mbarrier.arrive per thread).  So the NVLink transfer of
// tile t+2 overlaps the HBM stream and the math of tile t, tile by tile.
//
// The arithmetic is the single-GPU kernel's (ascending *global* learner id FMA
// chain), so a sharded step is bit-identical to the single-GPU step.  With
// `dest` the same kernel serves the ring-position layout (outputs stored to the
// learner's next-step slot on any rank), and with an rm_step_sync it orders
// consecutive steps itself through a multicast flag (no collective).
//
// D1D: rm_partial_sum (local column sums, fp64) -> cross-rank sum -> apply:
// through NCCL (host side), through our in-NVSwitch kernel rm_nvls_mean_f64,
// or all three phases fused into one launch per rank (rm_d1d_fused_nvls_*).
#include "common.cuh"
#include "tma_host.cuh"
#include "arith.cuh"
#include "../../include/ringmix_b200.h"

#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

namespace rm {

// Per device, once: the cross-rank wait bound of this module's kernels
// (RINGMIX_XGPU_TIMEOUT_S seconds, default 600; see xgpu_wait).
static unsigned long long g_xgpu_config_mask = 0;
static void xgpu_config() {
  if (!attr_needed(&g_xgpu_config_mask)) return;
  unsigned long long ns = 600ull * 1000000000ull;
  if (const char* env = getenv("RINGMIX_XGPU_TIMEOUT_S")) {
    const double s = atof(env);
    if (s > 0) ns = (unsigned long long)(s * 1e9);
  }
  if (cudaMemcpyToSymbol(g_xgpu_timeout_ns, &ns, sizeof(ns)) == cudaSuccess)
    attr_done(&g_xgpu_config_mask);
}

// rm_set_shard_remote_rows: the calling thread's bound on the distinct remote rows of a step
static thread_local int g_shard_rmax_hint = 0;

constexpr int kShThreads = 512;
constexpr int kShMaxStages = 6;
constexpr int kShStagesDefault = 3;
constexpr int kShStageTarget = 64 * 1024;

// plan layout (int32): [0] = R (distinct remote rows), [1 .. 1+2Lg) remote
// global ids, [1+2Lg .. 1+2Lg+4Lg) per local learner: staged indices of its
// three inputs ordered by global learner id, then j.
__host__ __device__ inline int plan_ints(int Lg) { return 1 + 2 * Lg + 4 * Lg; }

__global__ void shard_plan_kernel(const int32_t* __restrict__ left,
                                  const int32_t* __restrict__ right, int L, int row0, int Lg,
                                  int32_t* __restrict__ plan) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int32_t* rem = plan + 1;
  int32_t* tri = plan + 1 + 2 * Lg;
  int R = 0;
  auto staged = [&](int x) -> int {
    if (x >= row0 && x < row0 + Lg) return x - row0;
    for (int i = 0; i < R; i++)
      if (rem[i] == x) return Lg + i;
    rem[R] = x;
    return Lg + R++;
  };
  for (int j = 0; j < Lg; j++) {
    const int g = row0 + j;
    int x0 = left[g], x1 = g, x2 = right[g], t;
    if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
    if (x2 < x1) { t = x1; x1 = x2; x2 = t; }
    if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
    tri[4 * j + 0] = staged(x0);
    tri[4 * j + 1] = staged(x1);
    tri[4 * j + 2] = staged(x2);
    tri[4 * j + 3] = j;
  }
  plan[0] = R;
  (void)L;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

struct ShardArgs {
  const uint64_t* row_ptrs;  // L device pointers: row l of the current W (local or peer)
  void* out;
  long long ldo;
  long long d;
  int L, row0, Lg, Rmax;
  int cw, log2_nv;
  long long ntiles;
  const int32_t* plan;
  double lr;
  unsigned long long* absmax;
  const uint64_t* dest;  // optional: output row j goes to dest[j] (local or peer address)
  // optional in-kernel step ordering (rm_step_sync): wait until every rank finished
  // the previous step, signal this rank's completion to every rank at the end
  const uint32_t* sync_done;
  SymRef sync_flag;  // `done` on every rank (multicast address or peer table)
  uint32_t* sync_cnt;
  uint32_t sync_target;
  int nstages;       // shared-memory stages in flight (RINGMIX_SHARD_STAGES, default 3)
};

template <typename T, bool HAS_G>
__global__ void __launch_bounds__(kShThreads, 1)
    mix_shard_kernel(ShardArgs a, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmG) {
  using E = Elem<T>;
  using A = typename E::acc;
  constexpr int VEC = E::VEC;
  extern __shared__ __align__(128) unsigned char smem[];

  const int Lg = a.Lg;
  const int cw = a.cw;
  const int tid = threadIdx.x;
  const int R = a.plan[0];
  if (R > a.Rmax) __trap();   // the caller's remote-row bound was wrong: the stage would overflow
  const int Srows = Lg + R;
  const int w_bytes_max = (Lg + a.Rmax) * cw * (int)sizeof(T);
  const int g_bytes = HAS_G ? Lg * cw * (int)sizeof(T) : 0;
  const int stage_bytes = w_bytes_max + g_bytes;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  int4* s_tri = reinterpret_cast<int4*>(smem + 128);
  const T** s_rptr = reinterpret_cast<const T**>(smem + 128 + ((Lg * 16 + 127) / 128) * 128);
  unsigned char* stages = reinterpret_cast<unsigned char*>(s_rptr) +
                          (((a.Rmax > 0 ? a.Rmax : 1) * 8 + 127) / 128) * 128;

  if (tid == 0) {
    tma_prefetch_desc(&tmW);
    if (HAS_G) tma_prefetch_desc(&tmG);
    for (int s = 0; s < a.nstages; s++) mbar_init(&full[s], 1 + kShThreads);
    fence_mbar_init();
  }
  for (int j = tid; j < Lg; j += kShThreads) {
    const int32_t* t = a.plan + 1 + 2 * Lg + 4 * j;
    s_tri[j] = make_int4(t[0], t[1], t[2], t[3]);
  }
  for (int i = tid; i < R; i += kShThreads)
    s_rptr[i] = reinterpret_cast<const T*>(a.row_ptrs[a.plan[1 + i]]);
  __syncthreads();
  // peers' rows of this step (and the buffers this step overwrites) belong to the
  // previous step of every rank: wait for all of them before the first load
  if (a.sync_done) xgpu_wait(a.sync_done, a.sync_target);

  const int box_c = cw < 256 ? cw : 256;
  const int lg_bc = __ffs(box_c) - 1;
  const int w_box_stride = Srows << lg_bc;
  const int g_box_stride = Lg << lg_bc;
  auto widx = [&](int r, int c) -> int {
    return (c >> lg_bc) * w_box_stride + (r << lg_bc) + (c & (box_c - 1));
  };
  auto gidx = [&](int r, int c) -> int {
    return (c >> lg_bc) * g_box_stride + (r << lg_bc) + (c & (box_c - 1));
  };
  const int nchunk = cw / VEC;  // 16-byte chunks per row per tile

  // refill stage s with tile t: local rows by TMA (one thread), remote rows by
  // cp.async over NVLink (all threads); every thread arrives once.
  auto issue = [&](int s, long long t) {
    const int c0 = (int)(t * cw);
    unsigned char* st = stages + (size_t)s * stage_bytes;
    T* sW = reinterpret_cast<T*>(st);
    if (tid == 0) {
      mbar_arrive_expect_tx(&full[s], (uint32_t)((Lg * cw + (HAS_G ? Lg * cw : 0)) * sizeof(T)));
      for (int cc = 0; cc < cw; cc += box_c) {
        tma_load_2d(sW + widx(0, cc), &tmW, c0 + cc, 0, &full[s]);
        if (HAS_G)
          tma_load_2d(reinterpret_cast<T*>(st + w_bytes_max) + gidx(0, cc), &tmG, c0 + cc, 0,
                      &full[s]);
      }
    }
    const long long dvec = (a.d - c0 + VEC - 1) / VEC;  // chunks inside the row
    for (int q = tid; q < R * nchunk; q += kShThreads) {
      const int i = q / nchunk, ch = q - i * nchunk;
      if (ch < dvec) cp_async16(sW + widx(Lg + i, ch * VEC), s_rptr[i] + c0 + ch * VEC);
    }
    cp_async_mbar_arrive_noinc(&full[s]);
  };

  const long long first = blockIdx.x, stride = gridDim.x;
  for (int s = 0; s < a.nstages; s++) {
    long long t = first + s * stride;
    if (t < a.ntiles) issue(s, t);
  }

  typename E::amax_t amax = 0;
  const A lr = (A)a.lr;
  const int log2_nv = a.log2_nv;
  const int nv_full = 1 << log2_nv;
  T* out = static_cast<T*>(a.out);

  int it = 0;
  for (long long t = first; t < a.ntiles; t += stride, ++it) {
    const int s = it % a.nstages;
    const uint32_t parity = (it / a.nstages) & 1;
    const long long c0 = t * cw;
    const int width = (int)min((long long)cw, a.d - c0);
    const T* sW = reinterpret_cast<const T*>(stages + (size_t)s * stage_bytes);
    const T* sG = reinterpret_cast<const T*>(stages + (size_t)s * stage_bytes + w_bytes_max);
    mbar_wait(&full[s], parity);

    const int nv = (width + VEC - 1) / VEC;
    const int total = Lg << log2_nv;
#pragma unroll 2
    for (int idx = tid; idx < total; idx += kShThreads) {
      const int j = idx >> log2_nv;
      const int v = idx & (nv_full - 1);
      if (v >= nv) continue;
      const int c = v * VEC;
      const int4 tri = s_tri[j];
      Vec<T> va, vb, vc, vg, y;
      va.raw = *reinterpret_cast<const uint4*>(sW + widx(tri.x, c));
      vb.raw = *reinterpret_cast<const uint4*>(sW + widx(tri.y, c));
      vc.raw = *reinterpret_cast<const uint4*>(sW + widx(tri.z, c));
      if (HAS_G) vg.raw = *reinterpret_cast<const uint4*>(sG + gidx(j, c));
#pragma unroll
      for (int e = 0; e < VEC; e++) {
        A m = ring3<A>((A)E::ld(va.e(), e), (A)E::ld(vb.e(), e), (A)E::ld(vc.e(), e));
        if (HAS_G) m = r_sub(m, r_mul(lr, (A)E::ld(vg.e(), e)));
        y.e()[e] = E::st(m);
      }
      T* dst = (a.dest ? reinterpret_cast<T*>(a.dest[j]) : out + j * a.ldo) + c0 + c;
      if (c + VEC <= width) {
#pragma unroll
        for (int e = 0; e < VEC; e++) amax = E::amax_acc(amax, y.e()[e]);
        st_cs_v4(dst, y.raw);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; e++)
          if (c + e < width) {
            amax = E::amax_acc(amax, y.e()[e]);
            dst[e] = y.e()[e];
          }
      }
    }
    __syncthreads();
    long long tn = t + (long long)a.nstages * stride;
    if (tn < a.ntiles) issue(s, tn);
  }
  if (a.absmax) absmax_publish(a.absmax, E::amax_bits(amax));
  if (a.sync_done) {
    // the last CTA resets the counter (the next launch starts after this one on
    // the stream) and bumps every rank's step flag
    xgpu_arrive(a.sync_cnt, gridDim.x, a.sync_flag, 0, true);
  }
}

// ---- D1D pieces ----
// Column sums of the local rows (ascending learner order, fp64) and the apply
// step.  Both stream HBM with 16-byte accesses and several rows in flight per
// thread; the scalar tail handles d % VEC columns.  The bodies are range
// functions over (worker, nworkers) so the fused D1D kernel (below) can run them
// on a subset of its CTAs.
// numpy order (R = chains per rank > 0; fp32 / fp64): the rank holds the learners of
// numpy's pairwise chains [g R, (g + 1) R) — local row i is in chain i % R — and its partial is
// numpy's tree over those chains: chain q summed from its first element, ((c0 + c1) + ...).
// With the ranks' partials combined in the tree order too (sym_ld_sum_tree_f64) the mean is
// numpy's W.mean(axis=1) bit for bit, as on one GPU (8 <= L <= 128, L % 8 == 0).
template <typename T, int R>
__device__ __forceinline__ void partial_sum_numpy_range(const T* __restrict__ W, int Lg,
                                                        long long d, long long ld,
                                                        double* __restrict__ S, long long worker,
                                                        long long nworkers) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const long long nvec = d / VEC;
  for (long long v = worker; v < nvec; v += nworkers) {
    double s[R][VEC];
    const T* p = W + v * VEC;
#pragma unroll
    for (int q = 0; q < R; q++) {
      Vec<T> x;
      x.raw = __ldcs(reinterpret_cast<const uint4*>(p + (long long)q * ld));
#pragma unroll
      for (int e = 0; e < VEC; e++) s[q][e] = (double)E::ld(x.e(), e);
    }
    for (int l = R; l < Lg; l += R) {
      Vec<T> x[R];
#pragma unroll
      for (int q = 0; q < R; q++)
        x[q].raw = __ldcs(reinterpret_cast<const uint4*>(p + (long long)(l + q) * ld));
#pragma unroll
      for (int q = 0; q < R; q++)
#pragma unroll
        for (int e = 0; e < VEC; e++) s[q][e] = __dadd_rn(s[q][e], (double)E::ld(x[q].e(), e));
    }
#pragma unroll
    for (int w = 1; w < R; w *= 2)
#pragma unroll
      for (int q = 0; q + w < R; q += 2 * w)
#pragma unroll
        for (int e = 0; e < VEC; e++) s[q][e] = __dadd_rn(s[q][e], s[q + w][e]);
#pragma unroll
    for (int e = 0; e < VEC; e++) S[v * VEC + e] = s[0][e];
  }
  for (long long c = nvec * VEC + worker; c < d; c += nworkers) {
    double s[R];
#pragma unroll
    for (int q = 0; q < R; q++) s[q] = (double)E::ld(W + (long long)q * ld + c, 0);
    for (int l = R; l < Lg; l += R)
#pragma unroll
      for (int q = 0; q < R; q++) s[q] = __dadd_rn(s[q], (double)E::ld(W + (long long)(l + q) * ld + c, 0));
#pragma unroll
    for (int w = 1; w < R; w *= 2)
#pragma unroll
      for (int q = 0; q + w < R; q += 2 * w) s[q] = __dadd_rn(s[q], s[q + w]);
    S[c] = s[0];
  }
}

template <typename T>
__device__ __forceinline__ void partial_sum_range(const T* __restrict__ W, int Lg, long long d,
                                                  long long ld, double* __restrict__ S,
                                                  long long worker, long long nworkers,
                                                  int chains = 0) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  if constexpr (sizeof(T) >= 4) {
    switch (chains) {
      case 1: return partial_sum_numpy_range<T, 1>(W, Lg, d, ld, S, worker, nworkers);
      case 2: return partial_sum_numpy_range<T, 2>(W, Lg, d, ld, S, worker, nworkers);
      case 4: return partial_sum_numpy_range<T, 4>(W, Lg, d, ld, S, worker, nworkers);
      case 8: return partial_sum_numpy_range<T, 8>(W, Lg, d, ld, S, worker, nworkers);
      default: break;
    }
  }
  const long long nvec = d / VEC;
  for (long long v = worker; v < nvec; v += nworkers) {
    double s[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e++) s[e] = 0.0;
    const T* p = W + v * VEC;
    int l = 0;
    for (; l + 4 <= Lg; l += 4) {
      Vec<T> x[4];
#pragma unroll
      for (int u = 0; u < 4; u++)
        x[u].raw = __ldcs(reinterpret_cast<const uint4*>(p + (long long)(l + u) * ld));
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int e = 0; e < VEC; e++) s[e] = __dadd_rn(s[e], (double)E::ld(x[u].e(), e));
    }
    for (; l < Lg; l++) {
      Vec<T> x;
      x.raw = __ldcs(reinterpret_cast<const uint4*>(p + (long long)l * ld));
#pragma unroll
      for (int e = 0; e < VEC; e++) s[e] = __dadd_rn(s[e], (double)E::ld(x.e(), e));
    }
#pragma unroll
    for (int e = 0; e < VEC; e++) S[v * VEC + e] = s[e];
  }
  // tail columns
  for (long long c = nvec * VEC + worker; c < d; c += nworkers) {
    double s = 0.0;
    for (int l = 0; l < Lg; l++) s = __dadd_rn(s, (double)E::ld(W + l * ld + c, 0));
    S[c] = s;
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
    partial_sum_kernel(const T* __restrict__ W, int Lg, long long d, long long ld,
                       double* __restrict__ S, int chains) {
  partial_sum_range<T>(W, Lg, d, ld, S, blockIdx.x * (long long)blockDim.x + threadIdx.x,
                       (long long)gridDim.x * blockDim.x, chains);
}

// out[j][c] = S[c]/L - lr*G[j][c] for the Lg local learners.  One thread per
// 16-byte column vector reads S once and walks the rows (S is d fp64 values,
// larger than L2, so per-row re-reads would cost Lg x d x 8 bytes).  L == 1
// means S already holds the mean (the NVLS path divides once per column).
template <typename T, bool HAS_G>
__device__ __forceinline__ void apply_mean_range(const double* S, const T* __restrict__ G,
                                                 T* __restrict__ out, int Lg, int L, long long d,
                                                 long long ldg, long long ldo, double lr,
                                                 typename Elem<T>::amax_t& amax, long long worker,
                                                 long long nworkers) {
  using E = Elem<T>;
  using A = typename E::acc;
  constexpr int VEC = E::VEC;
  const long long nvec = (d + VEC - 1) / VEC;
  const double dL = (double)L;
  for (long long v = worker; v < nvec; v += nworkers) {
    const long long c = v * VEC;
    const bool full = c + VEC <= d;
    A m[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e++) {
      double sv = (full || c + e < d) ? S[c + e] : 0.0;
      m[e] = (A)(L == 1 ? sv : __ddiv_rn(sv, dL));
    }
    // rows in batches of 8: all G loads of a batch are in flight before any use
    constexpr int B = 8;
    for (int j0 = 0; j0 < Lg; j0 += B) {
      Vec<T> gv[B];
      if (HAS_G && full) {
#pragma unroll
        for (int u = 0; u < B; u++)
          if (j0 + u < Lg)
            gv[u].raw = __ldcs(reinterpret_cast<const uint4*>(G + (j0 + u) * ldg + c));
      }
#pragma unroll
      for (int u = 0; u < B; u++) {
        const int j = j0 + u;
        if (j >= Lg) break;
        T* o = out + j * ldo;
        Vec<T> y;
#pragma unroll
        for (int e = 0; e < VEC; e++) {
          A r = m[e];
          if (HAS_G) {
            A gg = full ? (A)E::ld(gv[u].e(), e)
                        : ((c + e < d) ? (A)E::ld(G + j * ldg + c + e, 0) : (A)0);
            r = r_sub(r, r_mul((A)lr, gg));
          }
          y.e()[e] = E::st(r);
        }
        if (full) {
#pragma unroll
          for (int e = 0; e < VEC; e++) amax = E::amax_acc(amax, y.e()[e]);
          st_cs_v4(o + c, y.raw);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; e++)
            if (c + e < d) {
              amax = E::amax_acc(amax, y.e()[e]);
              o[c + e] = y.e()[e];
            }
        }
      }
    }
  }
}

template <typename T, bool HAS_G>
__global__ void __launch_bounds__(256)
    apply_mean_kernel(const double* __restrict__ S, const T* __restrict__ G, T* __restrict__ out,
                      int Lg, int L, long long d, long long ldg, long long ldo, double lr,
                      unsigned long long* absmax) {
  using E = Elem<T>;
  typename E::amax_t amax = 0;
  apply_mean_range<T, HAS_G>(S, G, out, Lg, L, d, ldg, ldo, lr, amax,
                             blockIdx.x * (long long)blockDim.x + threadIdx.x,
                             (long long)gridDim.x * blockDim.x);
  if (absmax) absmax_publish(absmax, E::amax_bits(amax));
}

template <typename T, bool HAS_G>
static int launch_shard(ShardArgs a, const T* W_local, long long ldw, const T* G_local,
                        long long ldg, cudaStream_t st) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const size_t esz = sizeof(T);
  auto fn = tma_encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return RM_ENOSYS;
  }
  static int max_optin = -1;
  if (max_optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  const int rows = a.Lg * 2 + a.Rmax;  // staged rows per column (W local+remote, G)
  // tuning knobs (measured defaults): stages in flight and the stage size target
  static int env_stages = -1, env_kb = -1;
  if (env_stages < 0) {
    const char* e1 = getenv("RINGMIX_SHARD_STAGES");
    const char* e2 = getenv("RINGMIX_SHARD_STAGE_KB");
    env_stages = e1 ? atoi(e1) : 0;
    env_kb = e2 ? atoi(e2) : 0;
  }
  a.nstages = (env_stages >= 2 && env_stages <= kShMaxStages) ? env_stages : kShStagesDefault;
  // position layout with <= 32 local rows: 72 KB stages give 1 KB row segments (256 fp32
  // columns) — measured at C3 on 4 GPUs 863 vs 849 G/s; at 64 local rows the 64 KB target
  // (256-byte segments) stays ahead (746-753 vs 736-743), profiles/r2_n4_sweep/
  // few staged rows (position layout, or the fixed ring's two boundary rows) with <= 32
  // local rows: 72 KB stages give >= 1 KB row segments — at C2 on 2 GPUs the fixed ring's
  // kernel runs 1.49 ms against 1.87 ms with 512-byte segments (profiles/r3_ad_rmax/)
  const size_t dflt = (a.Rmax <= 2 && a.Lg <= 32) ? 72 * 1024 : kShStageTarget;
  const size_t target = (env_kb >= 8 && env_kb <= 128) ? (size_t)env_kb * 1024 : dflt;
  int cw = VEC;
  while ((size_t)(cw * 2) * rows * esz <= target && cw * 2 <= 2048) cw *= 2;
  while (cw > VEC && (a.d + cw - 1) / cw < 4LL * sm_count(-1) && cw * esz > 256) cw /= 2;
  if (const char* env = getenv("RINGMIX_TILE_COLS")) {
    int v = atoi(env);
    if (v >= VEC && (v & (v - 1)) == 0) cw = v;
  }
  const size_t stage = (size_t)rows * cw * esz;
  const size_t smem = 128 + ((size_t)(a.Lg * 16 + 127) / 128) * 128 +
                      ((size_t)((a.Rmax > 0 ? a.Rmax : 1) * 8 + 127) / 128) * 128 +
                      a.nstages * stage;
  if (smem > (size_t)max_optin) {
    set_error("sharded tile does not fit shared memory (Lg=%d)", a.Lg);
    return RM_ERANGE;
  }
  a.cw = cw;
  int nv = cw / VEC, lg = 0;
  while ((1 << lg) < nv) lg++;
  a.log2_nv = lg;
  a.ntiles = (a.d + cw - 1) / cw;
  const int box_c = cw < 256 ? cw : 256;
  CUtensorMap tmW, tmG;
  cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)a.Lg};
  cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)a.Lg};
  cuuint32_t estr[2] = {1, 1};
  cuuint64_t sw[1] = {(cuuint64_t)(ldw * esz)};
  if (fn(&tmW, TmaType<T>::v, 2, const_cast<T*>(W_local), dims, sw, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed for local W");
    return RM_EINVAL;
  }
  tmG = tmW;
  if (HAS_G) {
    cuuint64_t sg[1] = {(cuuint64_t)(ldg * esz)};
    if (fn(&tmG, TmaType<T>::v, 2, const_cast<T*>(G_local), dims, sg, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed for local G");
      return RM_EINVAL;
    }
  }
  static unsigned long long attr_mask = 0;
  if (attr_needed(&attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(mix_shard_kernel<T, HAS_G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(mix_shard_kernel)");
    attr_done(&attr_mask);
  }
  long long grid = sm_count(-1);
  if (grid > a.ntiles) grid = a.ntiles;
  mix_shard_kernel<T, HAS_G><<<(int)grid, kShThreads, smem, st>>>(a, tmW, tmG);
  RM_CHECK_LAUNCH("mix_shard_kernel");
  return RM_OK;
}

template <typename T>
static int shard_dispatch(const uint64_t* row_ptrs, const T* W_local, const T* G_local, T* out,
                          int L, int row0, int Lg, long long d, long long ldw, long long ldg,
                          long long ldo, const int32_t* plan, double lr,
                          unsigned long long* absmax, void* stream,
                          const uint64_t* dest = nullptr, const rm_step_sync* sync = nullptr) {
  using E = Elem<T>;
  const size_t esz = sizeof(T);
  if (row_ptrs == nullptr || W_local == nullptr || (out == nullptr && dest == nullptr) ||
      plan == nullptr || L < 4 ||
      Lg < 1 || row0 < 0 || row0 + Lg > L || d < 1 || Lg > 256) {
    set_error("invalid sharded mix arguments (L=%d row0=%d Lg=%d)", L, row0, Lg);
    return RM_EINVAL;
  }
  const uintptr_t al = reinterpret_cast<uintptr_t>(W_local) | reinterpret_cast<uintptr_t>(out) |
                       (G_local ? reinterpret_cast<uintptr_t>(G_local) : 0) |
                       (uintptr_t)(ldw * esz) | (uintptr_t)(ldo * esz) |
                       (G_local ? (uintptr_t)(ldg * esz) : 0);
  if ((al & 15) != 0 || ldw < (d + E::VEC - 1) / E::VEC * E::VEC) {
    set_error("sharded mix needs 16-byte aligned rows padded to a multiple of 16 bytes");
    return RM_EINVAL;
  }
  ShardArgs a{};
  a.row_ptrs = row_ptrs;
  a.out = out;
  a.ldo = ldo;
  a.d = d;
  a.L = L;
  a.row0 = row0;
  a.Lg = Lg;
  a.Rmax = (2 * Lg < L - Lg) ? 2 * Lg : L - Lg;
  if (dest != nullptr && a.Rmax > 2) a.Rmax = 2;  // position layout: two boundary rows
  // caller's bound (rm_set_shard_remote_rows: the fixed ring pulls at most 2 rows)
  if (g_shard_rmax_hint > 0 && g_shard_rmax_hint < a.Rmax) a.Rmax = g_shard_rmax_hint;
  a.plan = plan;
  a.lr = lr;
  a.absmax = absmax;
  a.dest = dest;
  if (sync != nullptr) {
    if (sync->done == nullptr || (sync->done_mc == nullptr && sync->done_peers == nullptr) ||
        sync->counter == nullptr || sync->world < 1 || sync->epoch == 0) {
      set_error("invalid step-sync arguments");
      return RM_EINVAL;
    }
    xgpu_config();
    a.sync_done = sync->done;
    a.sync_flag = SymRef{reinterpret_cast<unsigned long long>(sync->done_mc),
                         reinterpret_cast<const unsigned long long*>(sync->done_peers),
                         sync->world};
    a.sync_cnt = sync->counter;
    a.sync_target = (uint32_t)sync->world * (sync->epoch - 1u);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (G_local) return launch_shard<T, true>(a, W_local, ldw, G_local, ldg, st);
  return launch_shard<T, false>(a, W_local, ldw, nullptr, ldw, st);
}

}  // namespace rm

using namespace rm;

extern "C" int rm_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// The handle names the whole allocation that contains dptr (allocators such as
// PyTorch's sub-allocate), so the byte offset of dptr inside it is returned too;
// the importer adds it to the mapped base.
extern "C" int rm_ipc_get_handle(const void* dptr, void* handle_out, uint64_t* offset_out) {
  if (dptr == nullptr || handle_out == nullptr || offset_out == nullptr) {
    set_error("null pointer");
    return RM_EINVAL;
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dptr));
  if (e != cudaSuccess) return fail_cuda(e, "cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof(h));
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (range == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      set_error("cuMemGetAddressRange unavailable");
      return RM_ENOSYS;
    }
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed");
    return RM_EINVAL;
  }
  *offset_out = reinterpret_cast<uint64_t>(dptr) - (uint64_t)base;
  return 0;
}

extern "C" int rm_ipc_open_handle(const void* handle, void** dptr_out) {
  if (handle == nullptr || dptr_out == nullptr) {
    set_error("null pointer");
    return RM_EINVAL;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail_cuda(e, "cudaIpcOpenMemHandle");
  return 0;
}

extern "C" int rm_ipc_close_handle(void* dptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dptr);
  if (e != cudaSuccess) return fail_cuda(e, "cudaIpcCloseMemHandle");
  return 0;
}

// Stream-ordered wait until every rank finished step `epoch` of an rm_step_sync
// sequence (*done >= world * epoch): what a consumer of the step's outputs other
// than the next step kernel (host reads, other kernels) needs in the push layout,
// whose outputs land in this rank's buffers from every rank.
__global__ void step_sync_wait_kernel(const uint32_t* done, uint32_t target) {
  xgpu_wait(done, target);
}

extern "C" int rm_step_sync_wait(const rm_step_sync* sync, void* stream) {
  if (sync == nullptr || sync->done == nullptr || sync->world < 1) {
    set_error("invalid step-sync arguments");
    return RM_EINVAL;
  }
  if (sync->epoch == 0) return 0;  // no step issued yet
  xgpu_config();
  step_sync_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      sync->done, (uint32_t)sync->world * sync->epoch);
  RM_CHECK_LAUNCH("step_sync_wait_kernel");
  return 0;
}

// Stream-ordered "publish": adds 1 to `done` on every rank, like the end of a step,
// without a step.  Called collectively (every rank, same epoch) after writes to the
// step buffers from outside the step kernels (initialisation, checkpoint restore,
// host edits): the next step kernel of every rank then waits for them.
__global__ void step_sync_publish_kernel(SymRef flag) {
  __threadfence_system();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.alias;" ::: "memory");
    sym_red_add_u32(flag, 0);
  }
}

extern "C" int rm_step_sync_publish(const rm_step_sync* sync, void* stream) {
  if (sync == nullptr || (sync->done_mc == nullptr && sync->done_peers == nullptr) ||
      sync->world < 1) {
    set_error("invalid step-sync arguments");
    return RM_EINVAL;
  }
  step_sync_publish_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      SymRef{reinterpret_cast<unsigned long long>(sync->done_mc),
             reinterpret_cast<const unsigned long long*>(sync->done_peers), sync->world});
  RM_CHECK_LAUNCH("step_sync_publish_kernel");
  return 0;
}

// Overrides the cross-rank wait bound of the current device (seconds > 0).
extern "C" int rm_set_xgpu_timeout(double seconds) {
  if (!(seconds > 0) || seconds > 1e6) {
    set_error("timeout must be in (0, 1e6] seconds");
    return RM_EINVAL;
  }
  const unsigned long long ns = (unsigned long long)(seconds * 1e9);
  cudaError_t e = cudaMemcpyToSymbol(g_xgpu_timeout_ns, &ns, sizeof(ns));
  if (e != cudaSuccess) return fail_cuda(e, "rm_set_xgpu_timeout");
  attr_done(&g_xgpu_config_mask);
  return 0;
}

// Reads and clears this device's cross-rank wait status: bit 0 = a wait gave up
// after RINGMIX_XGPU_TIMEOUT_S (the steps that saw it have unspecified contents).
extern "C" int rm_xgpu_status(unsigned int* status) {
  if (status == nullptr) {
    set_error("null pointer");
    return RM_EINVAL;
  }
  unsigned int zero = 0;
  cudaError_t e = cudaMemcpyFromSymbol(status, g_xgpu_status, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_xgpu_status, &zero, sizeof(zero));
  if (e != cudaSuccess) return fail_cuda(e, "rm_xgpu_status");
  return 0;
}

extern "C" int rm_shard_plan_ints(int Lg) { return plan_ints(Lg); }

extern "C" int rm_shard_plan(const int32_t* left, const int32_t* right, int L, int row0, int Lg,
                             int32_t* plan, void* stream) {
  if (left == nullptr || right == nullptr || plan == nullptr || L < 1 || Lg < 1 || row0 < 0 ||
      row0 + Lg > L) {
    set_error("invalid shard plan arguments (L=%d row0=%d Lg=%d)", L, row0, Lg);
    return RM_EINVAL;
  }
  shard_plan_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(left, right, L, row0, Lg,
                                                                     plan);
  RM_CHECK_LAUNCH("shard_plan_kernel");
  return 0;
}

// Per-host-thread caps on the CTAs per SM of the D1D kernels (0 = defaults).  A
// pipeline that runs the in-switch reduction concurrently with the local
// partial-sum / apply kernels lowers them so the kernels can be co-resident.
static thread_local int g_d1d_psum_cap = 0;
// numpy-order D1D (rm_set_d1d_numpy_order): chains per rank of the partial sums, 0 = legacy
// ascending-row sums and ascending-rank cross-rank sums
static thread_local int g_d1d_chains = 0;
static thread_local int g_d1d_apply_cap = 0;
static thread_local int g_d1d_nvls_cap = 0;

// the partial-sum cap also bounds rm_column_mean_* (the single-GPU D1D average that runs
// beside the gradient generator)
namespace rm {
int d1d_psum_cap() { return g_d1d_psum_cap; }
}  // namespace rm

extern "C" int rm_set_d1d_numpy_order(int chains) {
  if (chains != 0 && chains != 1 && chains != 2 && chains != 4 && chains != 8) {
    set_error("numpy-order D1D: chains per rank must be 0, 1, 2, 4 or 8");
    return RM_EINVAL;
  }
  g_d1d_chains = chains;
  return 0;
}

extern "C" int rm_set_shard_remote_rows(int max_rows) {
  if (max_rows < 0) {
    set_error("remote-row bound must be >= 0 (0 = the layout's own bound)");
    return RM_EINVAL;
  }
  g_shard_rmax_hint = max_rows;
  return 0;
}

extern "C" int rm_set_d1d_ctas_per_sm(int partial_sum, int apply, int nvls) {
  if (partial_sum < 0 || partial_sum > 16 || apply < 0 || apply > 16 || nvls < 0 || nvls > 16) {
    set_error("CTAs per SM must be in [0, 16] (0 = default)");
    return RM_EINVAL;
  }
  g_d1d_psum_cap = partial_sum;
  g_d1d_apply_cap = apply;
  g_d1d_nvls_cap = nvls;
  return 0;
}

#define RM_DEFINE_SHARD(SUFFIX, CT, T)                                                          \
  extern "C" int rm_ring_mix_sgd_sharded_##SUFFIX(                                              \
      const uint64_t* row_ptrs, const CT* W_local, const CT* G_local, CT* out, int L, int row0, \
      int Lg, int64_t d, int64_t ldw, int64_t ldg, int64_t ldo, const int32_t* plan,           \
      double lr, unsigned long long* absmax_bits, void* stream, const rm_step_sync* sync) {     \
    return shard_dispatch<T>(row_ptrs, reinterpret_cast<const T*>(W_local),                    \
                             reinterpret_cast<const T*>(G_local), reinterpret_cast<T*>(out), L, \
                             row0, Lg, d, ldw, ldg, ldo, plan, lr, absmax_bits, stream, nullptr, \
                             sync);                                                             \
  }                                                                                             \
  extern "C" int rm_partial_sum_##SUFFIX(const CT* W, int Lg, int64_t d, int64_t ld, double* S, \
                                         void* stream) {                                        \
    if (W == nullptr || S == nullptr || Lg < 0 || d < 0 || ld < d ||                            \
        ((reinterpret_cast<uintptr_t>(W) | (uintptr_t)(ld * sizeof(CT))) & 15)) {               \
      set_error("invalid partial sum arguments (rows must be 16-byte aligned)");                \
      return RM_EINVAL;                                                                         \
    }                                                                                           \
    if (d == 0) return 0;                                                                       \
    long long blocks = (d + 255) / 256;                                                         \
    const long long cap = (g_d1d_psum_cap ? g_d1d_psum_cap : 16) * (long long)sm_count(-1);     \
    if (blocks > cap) blocks = cap;                                                             \
    if (g_d1d_chains && (sizeof(CT) < 4 || Lg % g_d1d_chains)) {                               \
      set_error("numpy-order partial sums need fp32/fp64 and Lg a multiple of the chains");    \
      return RM_EINVAL;                                                                         \
    }                                                                                           \
    partial_sum_kernel<T><<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(         \
        reinterpret_cast<const T*>(W), Lg, d, ld, S, g_d1d_chains);                             \
    RM_CHECK_LAUNCH("partial_sum_kernel");                                                      \
    return 0;                                                                                   \
  }                                                                                             \
  extern "C" int rm_apply_mean_sgd_##SUFFIX(const double* S, const CT* G, CT* out, int Lg,      \
                                            int L, int64_t d, int64_t ldg, int64_t ldo,         \
                                            double lr, unsigned long long* absmax_bits,         \
                                            void* stream) {                                     \
    if (S == nullptr || out == nullptr || Lg < 0 || L < 1 || d < 0 || ldo < d ||                \
        ((reinterpret_cast<uintptr_t>(out) | (uintptr_t)(ldo * sizeof(CT)) |                    \
          (G ? (reinterpret_cast<uintptr_t>(G) | (uintptr_t)(ldg * sizeof(CT))) : 0)) & 15)) {  \
      set_error("invalid apply-mean arguments (rows must be 16-byte aligned)");                 \
      return RM_EINVAL;                                                                         \
    }                                                                                           \
    if ((long long)Lg * d == 0) return 0;                                                       \
    long long blocks = (d / 4 + 255) / 256 + 1;                                                 \
    const long long cap = (g_d1d_apply_cap ? g_d1d_apply_cap : 8) * (long long)sm_count(-1);    \
    if (blocks > cap) blocks = cap;                                                             \
    if (G)                                                                                      \
      apply_mean_kernel<T, true><<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(  \
          S, reinterpret_cast<const T*>(G), reinterpret_cast<T*>(out), Lg, L, d, ldg, ldo, lr,  \
          absmax_bits);                                                                         \
    else                                                                                        \
      apply_mean_kernel<T, false><<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>( \
          S, nullptr, reinterpret_cast<T*>(out), Lg, L, d, ldg, ldo, lr, absmax_bits);          \
    RM_CHECK_LAUNCH("apply_mean_kernel");                                                       \
    return 0;                                                                                   \
  }

RM_DEFINE_SHARD(f32, float, float)
RM_DEFINE_SHARD(f64, double, double)
RM_DEFINE_SHARD(bf16, uint16_t, __nv_bfloat16)

// ---- D1D cross-GPU sum through NVSwitch multicast (NVLS) ----
// P_mc / M_mc are multicast addresses of symmetric buffers (every rank maps the
// same object).  For the caller's column shard [c0, c1): the switch sums the
// ranks' partial column sums (multimem.ld_reduce.add.f64, in-network reduction)
// and the result is broadcast into every rank's M (multimem.st).  Ordering
// against the partial-sum writes and the readers of M is the caller's barrier.
namespace rm {
__device__ __forceinline__ void nvls_sum_range(const SymRef& P, const SymRef& M, long long c0,
                                               long long c1, double L, long long worker,
                                               long long nworkers, bool tree = false) {
  constexpr int U = 8;
  for (long long c = c0 + worker; c < c1; c += U * nworkers) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const long long cc = c + u * nworkers;
      if (cc < c1) v[u] = tree ? sym_ld_sum_tree_f64(P, cc) : sym_ld_sum_f64(P, cc);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const long long cc = c + u * nworkers;
      if (cc < c1) sym_st_f64(M, cc, __ddiv_rn(v[u], L));
    }
  }
}

__global__ void __launch_bounds__(256)
    nvls_sum_kernel(SymRef P, SymRef M, long long c0, long long c1, double L, bool tree) {
  nvls_sum_range(P, M, c0, c1, L, blockIdx.x * (long long)blockDim.x + threadIdx.x,
                 (long long)gridDim.x * blockDim.x, tree);
}

static int launch_sym_mean(const SymRef& P, const SymRef& M, int64_t c0, int64_t c1, int L,
                           void* stream) {
  if (c1 == c0) return 0;
  long long blocks = (c1 - c0 + 2047) / 2048;
  const long long cap = (g_d1d_nvls_cap ? g_d1d_nvls_cap : 8) * (long long)sm_count(-1);
  if (blocks > cap) blocks = cap;
  if (g_d1d_chains && P.mc && P.world > 2) {
    set_error("numpy-order D1D over more than 2 ranks needs peer tables (the switch's "
              "summation order is unspecified)");
    return RM_EINVAL;
  }
  nvls_sum_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      P, M, c0, c1, (double)L, g_d1d_chains != 0);
  RM_CHECK_LAUNCH("nvls_sum_kernel");
  return 0;
}
}  // namespace rm

extern "C" int rm_nvls_mean_f64(const double* P_mc, double* M_mc, int64_t c0, int64_t c1,
                                int L, void* stream) {
  if (P_mc == nullptr || M_mc == nullptr || c0 < 0 || c1 < c0 || L < 1) {
    set_error("invalid NVLS reduction arguments");
    return RM_EINVAL;
  }
  return launch_sym_mean(SymRef{reinterpret_cast<unsigned long long>(P_mc), nullptr, 1},
                         SymRef{reinterpret_cast<unsigned long long>(M_mc), nullptr, 1}, c0, c1,
                         L, stream);
}

// Same reduction with peer tables instead of multicast addresses: P_peers /
// M_peers are device uint64[world] tables of every rank's P / M (NVLink P2P
// without NVSwitch multicast, or all ranks' buffers on one GPU).  The sum runs
// in ascending rank order.
extern "C" int rm_p2p_mean_f64(const uint64_t* P_peers, const uint64_t* M_peers, int world,
                               int64_t c0, int64_t c1, int L, void* stream) {
  if (P_peers == nullptr || M_peers == nullptr || world < 1 || c0 < 0 || c1 < c0 || L < 1) {
    set_error("invalid peer-table reduction arguments");
    return RM_EINVAL;
  }
  return launch_sym_mean(
      SymRef{0, reinterpret_cast<const unsigned long long*>(P_peers), world},
      SymRef{0, reinterpret_cast<const unsigned long long*>(M_peers), world}, c0, c1, L, stream);
}

// ---- D1D across GPUs in ONE kernel: partial sums, in-switch reduction, apply ----
// The CTAs of a persistent grid take three roles and walk the column chunks in
// order: partial-sum CTAs write the chunk's fp64 column sums of the local
// learners into the symmetric buffer P and, when the last of them is done,
// bump flagsA[c] on EVERY rank (multimem.red.release); reduce CTAs wait until
// flagsA[c] shows all ranks, sum their 1/N slice of the chunk across ranks in
// the switch (multimem.ld_reduce) and broadcast the means into every rank's M
// (multimem.st), then bump flagsB[c] everywhere; apply CTAs wait on flagsB[c]
// and write mean - lr*G for the local learners.  The in-switch reduction of
// chunk c thus overlaps the partial sums of later chunks and the apply of
// earlier ones inside one launch.  Flags and the per-role counters only grow
// (targets world*epoch and n_role*epoch), so nothing is reset between steps.
// All CTAs must be co-resident (the host sizes the grid by occupancy); waits
// trap after 20 s instead of hanging.
namespace rm {
// One rank's buffers of the fused D1D step (local addresses).  A launch drives
// one rank (the normal multi-process case) or, with peer-table SymRefs, every
// rank of a world whose buffers all live on this GPU (single-device emulation:
// CTA block r * per_rank .. (r+1) * per_rank - 1 plays rank r).
struct D1DRank {
  const void* W;
  const void* G;
  void* out;
  unsigned long long* absmax;
  double* P;                 // partial sums (symmetric buffer)
  const double* M;           // means (symmetric buffer)
  const uint32_t* flags;     // [2 * max_chunks]: A (partials of chunk c ready), B (means ready)
  uint32_t* counters;        // [2 * max_chunks] role counters (local)
  int Lg, rank;
};

constexpr int kD1DMaxLocalRanks = 8;

struct D1DFusedArgs {
  D1DRank r[kD1DMaxLocalRanks];
  int nlocal, per_rank;
  int L;
  long long d, ldw, ldg, ldo;
  double lr;
  SymRef P, M, F;            // every rank's P / M / flags
  int world;
  long long chunk;
  int nchunks, max_chunks;
  uint32_t epoch;
  int nP, nR, nA;
  int chains;                // numpy-order partial sums (0 = ascending rows / ranks)
};

template <typename T, bool HAS_G, int MINB>
__global__ void __launch_bounds__(256, MINB) d1d_fused_kernel(const __grid_constant__ D1DFusedArgs a) {
  using E = Elem<T>;
  const int lr_ = blockIdx.x / a.per_rank;
  const int bid = blockIdx.x - lr_ * a.per_rank;
  const D1DRank& R = a.r[lr_];
  const T* W = static_cast<const T*>(R.W);
  const T* G = static_cast<const T*>(R.G);
  T* out = static_cast<T*>(R.out);
  const uint32_t* flagsA = R.flags;
  const uint32_t* flagsB = R.flags + a.max_chunks;
  uint32_t* cntP = R.counters;
  uint32_t* cntR = R.counters + a.max_chunks;
  const uint32_t all_ranks = (uint32_t)a.world * a.epoch;
  if (bid < a.nP) {
    const long long w = bid * (long long)blockDim.x + threadIdx.x;
    const long long nw = (long long)a.nP * blockDim.x;
    for (int c = 0; c < a.nchunks; c++) {
      const long long b = c * a.chunk, e = min(b + a.chunk, a.d);
      partial_sum_range<T>(W + b, R.Lg, e - b, a.ldw, R.P + b, w, nw, a.chains);
      xgpu_arrive(cntP + c, (uint32_t)a.nP * a.epoch, a.F, c);
    }
  } else if (bid < a.nP + a.nR) {
    const long long w = (bid - a.nP) * (long long)blockDim.x + threadIdx.x;
    const long long nw = (long long)a.nR * blockDim.x;
    for (int c = 0; c < a.nchunks; c++) {
      const long long b = c * a.chunk, e = min(b + a.chunk, a.d);
      long long sl = (e - b + a.world - 1) / a.world;
      sl = (sl + 31) / 32 * 32;
      const long long s0 = min(e, b + R.rank * sl), s1 = min(e, s0 + sl);
      xgpu_wait(flagsA + c, all_ranks);
      nvls_sum_range(a.P, a.M, s0, s1, (double)a.L, w, nw, a.chains != 0);
      xgpu_arrive(cntR + c, (uint32_t)a.nR * a.epoch, a.F, a.max_chunks + c);
    }
  } else {
    const long long w = (bid - a.nP - a.nR) * (long long)blockDim.x + threadIdx.x;
    const long long nw = (long long)a.nA * blockDim.x;
    typename E::amax_t amax = 0;
    for (int c = 0; c < a.nchunks; c++) {
      const long long b = c * a.chunk, e = min(b + a.chunk, a.d);
      xgpu_wait(flagsB + c, all_ranks);
      apply_mean_range<T, HAS_G>(R.M + b, HAS_G ? G + b : nullptr, out + b, R.Lg, 1, e - b,
                                 a.ldg, a.ldo, a.lr, amax, w, nw);
    }
    if (R.absmax) absmax_publish(R.absmax, E::amax_bits(amax));
  }
}

// ranks: nlocal entries (host array); P / M / F: every rank's symmetric buffers
template <typename T>
static int d1d_fused(const D1DRank* ranks, int nlocal, int L, int64_t d, int64_t ldw, int64_t ldg,
                     int64_t ldo, double lr, const SymRef& P, const SymRef& M, const SymRef& F,
                     int world, int64_t chunk_cols, int max_chunks, uint32_t epoch,
                     int pct_partial, int pct_reduce, void* stream) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  if (nlocal < 1 || nlocal > kD1DMaxLocalRanks || nlocal > world || L < 1 || d < 0 ||
      ldw < d || ldo < d || world < 1 || epoch == 0 || max_chunks < 1 || pct_partial < 1 ||
      pct_reduce < 1 || pct_partial + pct_reduce > 98 || (!P.mc && !P.peers) ||
      (!M.mc && !M.peers) || (!F.mc && !F.peers)) {
    set_error("invalid fused D1D arguments");
    return RM_EINVAL;
  }
  const bool has_g = ranks[0].G != nullptr;
  for (int i = 0; i < nlocal; i++) {
    const D1DRank& r = ranks[i];
    if (r.Lg < 1 || r.Lg > L || r.rank < 0 || r.rank >= world || r.W == nullptr ||
        r.out == nullptr || r.P == nullptr || r.M == nullptr || r.flags == nullptr ||
        r.counters == nullptr || (r.G != nullptr) != has_g || (has_g && ldg < d)) {
      set_error("invalid fused D1D arguments (rank entry %d)", i);
      return RM_EINVAL;
    }
    if (((reinterpret_cast<uintptr_t>(r.W) | reinterpret_cast<uintptr_t>(r.out) |
          (uintptr_t)(ldw * sizeof(T)) | (uintptr_t)(ldo * sizeof(T)) |
          (has_g ? (reinterpret_cast<uintptr_t>(r.G) | (uintptr_t)(ldg * sizeof(T))) : 0)) & 15) ||
        VEC * sizeof(T) != 16) {
      set_error("fused D1D needs 16-byte aligned rows");
      return RM_EINVAL;
    }
  }
  if (g_d1d_chains) {
    if (sizeof(T) < 4 || (P.mc && world > 2)) {
      set_error("numpy-order D1D needs fp32/fp64 and, above 2 ranks, peer tables");
      return RM_EINVAL;
    }
    for (int i = 0; i < nlocal; i++)
      if (ranks[i].Lg % g_d1d_chains) {
        set_error("numpy-order D1D: Lg must be a multiple of the chains per rank");
        return RM_EINVAL;
      }
  }
  if (chunk_cols < 32LL * world || chunk_cols % (32LL * world) != 0) {
    set_error("chunk_cols must be a positive multiple of 32 * world");
    return RM_EINVAL;
  }
  if (d == 0) return 0;
  const long long nchunks = (d + chunk_cols - 1) / chunk_cols;
  if (nchunks > max_chunks) {
    set_error("%lld chunks exceed the %d flag slots", nchunks, max_chunks);
    return RM_ERANGE;
  }
  xgpu_config();
  // CTAs per SM the kernel is compiled for (registers): more resident CTAs give the
  // HBM-bound roles more loads in flight (RINGMIX_D1D_FUSED_OCC = 2 / 3 / 4)
  static int occ_env = -1;
  if (occ_env < 0) {
    const char* env = getenv("RINGMIX_D1D_FUSED_OCC");
    occ_env = env ? atoi(env) : 4;
    if (occ_env < 2 || occ_env > 4) occ_env = 4;
  }
  auto kern = occ_env == 2 ? (has_g ? d1d_fused_kernel<T, true, 2> : d1d_fused_kernel<T, false, 2>)
              : occ_env == 4 ? (has_g ? d1d_fused_kernel<T, true, 4> : d1d_fused_kernel<T, false, 4>)
                             : (has_g ? d1d_fused_kernel<T, true, 3> : d1d_fused_kernel<T, false, 3>);
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
  if (e != cudaSuccess) return fail_cuda(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (occ < 1) {
    set_error("fused D1D kernel cannot be resident");
    return RM_EINVAL;
  }
  // every CTA must be resident at once (roles wait on each other — across the
  // local ranks too when several share this GPU)
  const int per_rank = occ * sm_count(-1) / nlocal;
  D1DFusedArgs a{};
  for (int i = 0; i < nlocal; i++) a.r[i] = ranks[i];
  a.nlocal = nlocal;
  a.per_rank = per_rank;
  a.L = L;
  a.d = d;
  a.ldw = ldw;
  a.ldg = ldg;
  a.ldo = ldo;
  a.lr = lr;
  a.P = P;
  a.M = M;
  a.F = F;
  a.world = world;
  a.chunk = chunk_cols;
  a.nchunks = (int)nchunks;
  a.max_chunks = max_chunks;
  a.epoch = epoch;
  a.nP = max(1, per_rank * pct_partial / 100);
  a.nR = max(1, per_rank * pct_reduce / 100);
  a.nA = per_rank - a.nP - a.nR;
  a.chains = g_d1d_chains;
  if (a.nA < 1) {
    set_error("fused D1D: no CTAs left for the apply role");
    return RM_EINVAL;
  }
  kern<<<per_rank * nlocal, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  RM_CHECK_LAUNCH("d1d_fused_kernel");
  return 0;
}
}  // namespace rm

#define RM_DEFINE_D1D_FUSED(SUFFIX, CT, T)                                                      \
  extern "C" int rm_d1d_fused_nvls_##SUFFIX(                                                    \
      const CT* W, const CT* G, CT* out, int Lg, int L, int64_t d, int64_t ldw, int64_t ldg,    \
      int64_t ldo, double lr, unsigned long long* absmax_bits, double* P, const double* P_mc,  \
      const double* M, double* M_mc, uint32_t* flags, uint32_t* flags_mc, uint32_t* counters,  \
      int rank, int world, int64_t chunk_cols, int max_chunks, uint32_t epoch, int pct_partial, \
      int pct_reduce, void* stream) {                                                           \
    if (P_mc == nullptr || M_mc == nullptr || flags_mc == nullptr) {                            \
      set_error("invalid fused D1D arguments (multicast addresses)");                          \
      return RM_EINVAL;                                                                         \
    }                                                                                           \
    D1DRank r{W, G, out, absmax_bits, P, M, flags, counters, Lg, rank};                         \
    return d1d_fused<T>(&r, 1, L, d, ldw, ldg, ldo, lr,                                         \
                        SymRef{reinterpret_cast<unsigned long long>(P_mc), nullptr, world},     \
                        SymRef{reinterpret_cast<unsigned long long>(M_mc), nullptr, world},     \
                        SymRef{reinterpret_cast<unsigned long long>(flags_mc), nullptr, world}, \
                        world, chunk_cols, max_chunks, epoch, pct_partial, pct_reduce, stream); \
  }                                                                                             \
  extern "C" int rm_d1d_fused_p2p_##SUFFIX(                                                     \
      const rm_d1d_rank* ranks, int nlocal, int L, int64_t d, int64_t ldw, int64_t ldg,         \
      int64_t ldo, double lr, const uint64_t* P_peers, const uint64_t* M_peers,                 \
      const uint64_t* flags_peers, int world, int64_t chunk_cols, int max_chunks,               \
      uint32_t epoch, int pct_partial, int pct_reduce, void* stream) {                          \
    if (ranks == nullptr || P_peers == nullptr || M_peers == nullptr || flags_peers == nullptr || \
        nlocal < 1 || nlocal > kD1DMaxLocalRanks) {                                             \
      set_error("invalid fused D1D arguments (peer tables / ranks)");                          \
      return RM_EINVAL;                                                                         \
    }                                                                                           \
    D1DRank r[kD1DMaxLocalRanks];                                                               \
    for (int i = 0; i < nlocal; i++)                                                            \
      r[i] = D1DRank{ranks[i].W, ranks[i].G, ranks[i].out, ranks[i].absmax_bits, ranks[i].P,    \
                     ranks[i].M, ranks[i].flags, ranks[i].counters, ranks[i].Lg, ranks[i].rank}; \
    auto peer = [&](const uint64_t* t) {                                                        \
      return SymRef{0, reinterpret_cast<const unsigned long long*>(t), world};                  \
    };                                                                                          \
    return d1d_fused<T>(r, nlocal, L, d, ldw, ldg, ldo, lr, peer(P_peers), peer(M_peers),       \
                        peer(flags_peers), world, chunk_cols, max_chunks, epoch, pct_partial,   \
                        pct_reduce, stream);                                                    \
  }
RM_DEFINE_D1D_FUSED(f32, float, float)
RM_DEFINE_D1D_FUSED(f64, double, double)
RM_DEFINE_D1D_FUSED(bf16, uint16_t, __nv_bfloat16)

// ---- RAD in ring-position order ("push") ----
// Storage slot x (owned by the rank with positions [g0, g0+Lg)) holds the
// learner at ring position x of the CURRENT step's permutation: inv_k[x].
// The mix of position x reads positions x-1, x, x+1 — all local except the
// two boundary slots g0-1 and g0+Lg — and the output of learner l = inv_k[x]
// is written straight to its slot for the NEXT step, p_{k+1}[l], on whichever
// GPU owns it (P2P store in the epilogue).  The FMA chain still runs in
// ascending learner id, so the step is bit-identical to the single-GPU step.
namespace rm {
// Optional placement tables (NULL = identity, slot x holds position x): with a
// placement, global slot s (rank s / Lg, row s % Lg) holds ring position
// pos_of_slot[s], and position q lives in slot slot_of_pos[q]; every rank's slots
// hold a contiguous arc of positions, so a step still reads exactly two remote
// boundary rows.  slot_of_pos_next is the placement of step k + 1.
__global__ void pos_plan_kernel(const int32_t* __restrict__ inv_k,
                                const int32_t* __restrict__ perm_next, int L, int g0, int Lg,
                                const uint64_t* __restrict__ next_slot_ptrs,
                                int32_t* __restrict__ plan, uint64_t* __restrict__ dest,
                                const int32_t* __restrict__ pos_tab,
                                const int32_t* __restrict__ sop_tab,
                                const int32_t* __restrict__ sop_next) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  auto pos_of_slot = [&](int sl) { return pos_tab ? pos_tab[sl] : sl; };
  auto slot_of_pos = [&](int q) { return sop_tab ? sop_tab[q] : q; };
  // the arc's outer neighbours: left of the first slot's position, right of the last's
  const int xl = slot_of_pos((pos_of_slot(g0) - 1 + L) % L);
  const int xr = slot_of_pos((pos_of_slot(g0 + Lg - 1) + 1) % L);
  const bool local_l = xl >= g0 && xl < g0 + Lg, local_r = xr >= g0 && xr < g0 + Lg;
  if (i == 0) {
    // remote boundary slots (0, 1 or 2 of them) in the plan's remote list
    int R = 0;
    if (!local_l) plan[1 + R++] = xl;
    if (!local_r && xr != xl) plan[1 + R++] = xr;
    plan[0] = R;
  }
  if (i >= Lg) return;
  auto staged = [&](int y) -> int {
    if (y >= g0 && y < g0 + Lg) return y - g0;
    if (y == xl && !local_l) return Lg;
    return Lg + (local_l ? 0 : 1);
  };
  const int x = pos_of_slot(g0 + i);
  int p[3] = {(x - 1 + L) % L, x, (x + 1) % L};
  int id[3] = {inv_k[p[0]], inv_k[p[1]], inv_k[p[2]]};
  // sort by learner id (the reference's FMA order), carrying positions
  for (int u = 0; u < 2; u++)
    for (int v = 0; v < 2 - u; v++)
      if (id[v + 1] < id[v]) {
        int t = id[v]; id[v] = id[v + 1]; id[v + 1] = t;
        t = p[v]; p[v] = p[v + 1]; p[v + 1] = t;
      }
  int32_t* tri = plan + 1 + 2 * Lg + 4 * i;
  tri[0] = staged(slot_of_pos(p[0]));
  tri[1] = staged(slot_of_pos(p[1]));
  tri[2] = staged(slot_of_pos(p[2]));
  tri[3] = i;
  const int qn = perm_next[inv_k[x]];
  dest[i] = next_slot_ptrs[sop_next ? sop_next[qn] : qn];
}

// Placement of step k + 1 for the ring-position layout (L % world == 0, Lg = L / world):
// the ring of step k + 1 is cut into `world` arcs of Lg consecutive positions starting
// at a rotation r, and arc a goes to rank sigma(a).  Any choice gives the same result
// (the mix only sees neighbour relations); the one chosen keeps the most learners on
// the rank that computes their output, which is what the relabelling stores move over
// NVLink.  One CTA, thread r scores rotation r: counts[a][g] = learners whose next
// position falls in arc a and whose current slot is on rank g; the best arc -> rank
// assignment (exhaustive for world <= 5, greedy above) maximises the learners that stay.
// Deterministic (ties: smallest r, first assignment), so every rank computes the same.
constexpr int kPlMaxWorld = 8;

__device__ __forceinline__ int score_assignment(const int* cnt, int n, int* sigma) {
  int best = -1;
  if (n <= 5) {
    int perm[5] = {0, 1, 2, 3, 4};
    // lexicographic enumeration (next_permutation)
    for (;;) {
      int sc = 0;
      for (int a = 0; a < n; a++) sc += cnt[a * kPlMaxWorld + perm[a]];
      if (sc > best) {
        best = sc;
        for (int a = 0; a < n; a++) sigma[a] = perm[a];
      }
      int i = n - 2;
      while (i >= 0 && perm[i] >= perm[i + 1]) i--;
      if (i < 0) break;
      int j = n - 1;
      while (perm[j] <= perm[i]) j--;
      int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
      for (int lo = i + 1, hi = n - 1; lo < hi; lo++, hi--) {
        t = perm[lo]; perm[lo] = perm[hi]; perm[hi] = t;
      }
    }
    return best;
  }
  bool used_a[kPlMaxWorld] = {}, used_g[kPlMaxWorld] = {};
  best = 0;
  for (int step = 0; step < n; step++) {
    int ba = -1, bg = -1, bv = -1;
    for (int a = 0; a < n; a++) {
      if (used_a[a]) continue;
      for (int g = 0; g < n; g++) {
        if (used_g[g]) continue;
        if (cnt[a * kPlMaxWorld + g] > bv) { bv = cnt[a * kPlMaxWorld + g]; ba = a; bg = g; }
      }
    }
    used_a[ba] = used_g[bg] = true;
    sigma[ba] = bg;
    best += bv;
  }
  return best;
}

__global__ void pos_placement_kernel(const int32_t* __restrict__ inv_k,
                                     const int32_t* __restrict__ perm_next,
                                     const int32_t* __restrict__ sop_k, int L, int n,
                                     int32_t* __restrict__ pos_next, int32_t* __restrict__ sop_next,
                                     int32_t* __restrict__ moved) {
  extern __shared__ int sh[];
  int* owner = sh;           // [L] rank holding learner l at step k
  int* qn = owner + L;       // [L] position of learner l at step k + 1
  int* score = qn + L;       // [blockDim] best score of rotation r
  int* sig = score + blockDim.x;   // [blockDim] packed sigma (3 bits per arc)
  __shared__ int s_best_r, s_best_sig;
  const int Lg = L / n;
  const int tid = threadIdx.x;
  for (int q = tid; q < L; q += blockDim.x) {
    const int l = inv_k[q];
    owner[l] = (sop_k ? sop_k[q] : q) / Lg;
    qn[l] = perm_next[l];
  }
  __syncthreads();
  for (int r = tid; r < L; r += blockDim.x) {
    int cnt[kPlMaxWorld * kPlMaxWorld];
    for (int i = 0; i < kPlMaxWorld * kPlMaxWorld; i++) cnt[i] = 0;
    for (int l = 0; l < L; l++) {
      const int a = ((qn[l] - r + L) % L) / Lg;
      cnt[a * kPlMaxWorld + owner[l]]++;
    }
    int sigma[kPlMaxWorld];
    const int sc = score_assignment(cnt, n, sigma);
    int packed = 0;
    for (int a = 0; a < n; a++) packed |= sigma[a] << (3 * a);
    if (r < (int)blockDim.x) { score[r] = sc; sig[r] = packed; }
  }
  __syncthreads();
  if (tid == 0) {
    int br = 0;
    for (int r = 1; r < min(L, (int)blockDim.x); r++)
      if (score[r] > score[br]) br = r;
    s_best_r = br;
    s_best_sig = sig[br];
  }
  __syncthreads();
  const int r = s_best_r, packed = s_best_sig;
  for (int q = tid; q < L; q += blockDim.x) {
    const int u = (q - r + L) % L;
    const int a = u / Lg;
    const int slot = ((packed >> (3 * a)) & 7) * Lg + u % Lg;
    sop_next[q] = slot;
    pos_next[slot] = q;
  }
  if (moved != nullptr) {
    __syncthreads();
    for (int g = tid; g < n; g += blockDim.x) moved[g] = 0;
    __syncthreads();
    for (int l = tid; l < L; l += blockDim.x) {
      const int u = (qn[l] - r + L) % L;
      const int dst = (packed >> (3 * (u / Lg))) & 7;
      if (dst != owner[l]) atomicAdd(&moved[owner[l]], 1);
    }
  }
}
}  // namespace rm

extern "C" int rm_pos_plan(const int32_t* inv_k, const int32_t* perm_next, int L, int g0, int Lg,
                           const uint64_t* next_slot_ptrs, int32_t* plan, uint64_t* dest,
                           void* stream) {
  if (inv_k == nullptr || perm_next == nullptr || next_slot_ptrs == nullptr || plan == nullptr ||
      dest == nullptr || L < 4 || Lg < 1 || g0 < 0 || g0 + Lg > L) {
    set_error("invalid position-plan arguments (L=%d g0=%d Lg=%d)", L, g0, Lg);
    return RM_EINVAL;
  }
  pos_plan_kernel<<<(Lg + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      inv_k, perm_next, L, g0, Lg, next_slot_ptrs, plan, dest, nullptr, nullptr, nullptr);
  RM_CHECK_LAUNCH("pos_plan_kernel");
  return 0;
}

extern "C" int rm_pos_plan_placed(const int32_t* inv_k, const int32_t* perm_next,
                                  const int32_t* pos_of_slot, const int32_t* slot_of_pos,
                                  const int32_t* slot_of_pos_next, int L, int g0, int Lg,
                                  const uint64_t* next_slot_ptrs, int32_t* plan, uint64_t* dest,
                                  void* stream) {
  if (inv_k == nullptr || perm_next == nullptr || next_slot_ptrs == nullptr || plan == nullptr ||
      dest == nullptr || pos_of_slot == nullptr || slot_of_pos == nullptr ||
      slot_of_pos_next == nullptr || L < 4 || Lg < 1 || g0 < 0 || g0 + Lg > L) {
    set_error("invalid position-plan arguments (L=%d g0=%d Lg=%d)", L, g0, Lg);
    return RM_EINVAL;
  }
  pos_plan_kernel<<<(Lg + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      inv_k, perm_next, L, g0, Lg, next_slot_ptrs, plan, dest, pos_of_slot, slot_of_pos,
      slot_of_pos_next);
  RM_CHECK_LAUNCH("pos_plan_kernel");
  return 0;
}

extern "C" int rm_pos_placement(const int32_t* inv_k, const int32_t* perm_next,
                                const int32_t* slot_of_pos, int L, int world,
                                int32_t* pos_of_slot_next, int32_t* slot_of_pos_next,
                                int32_t* moved, void* stream) {
  if (inv_k == nullptr || perm_next == nullptr || pos_of_slot_next == nullptr ||
      slot_of_pos_next == nullptr || world < 1 || world > kPlMaxWorld || L < world ||
      L % world != 0 || L > 1024) {
    set_error("invalid placement arguments (L=%d world=%d; need L %% world == 0, world <= %d, "
              "L <= 1024)", L, world, kPlMaxWorld);
    return RM_EINVAL;
  }
  const int threads = L < 1024 ? ((L + 31) / 32) * 32 : 1024;
  const size_t smem = (2 * (size_t)L + 2 * (size_t)threads) * sizeof(int);
  pos_placement_kernel<<<1, threads, smem, static_cast<cudaStream_t>(stream)>>>(
      inv_k, perm_next, slot_of_pos, L, world, pos_of_slot_next, slot_of_pos_next, moved);
  RM_CHECK_LAUNCH("pos_placement_kernel");
  return 0;
}

#define RM_DEFINE_POS(SUFFIX, CT, T)                                                           \
  extern "C" int rm_ring_mix_sgd_pos_##SUFFIX(                                                 \
      const uint64_t* slot_ptrs, const CT* W_local, const CT* G_local, int L, int g0, int Lg,  \
      int64_t d, int64_t ldw, int64_t ldg, const int32_t* plan, const uint64_t* dest,          \
      double lr, unsigned long long* absmax_bits, void* stream, const rm_step_sync* sync) {     \
    return shard_dispatch<T>(slot_ptrs, reinterpret_cast<const T*>(W_local),                  \
                             reinterpret_cast<const T*>(G_local), nullptr, L, g0, Lg, d, ldw,  \
                             ldg, ldw, plan, lr, absmax_bits, stream, dest, sync);             \
  }
RM_DEFINE_POS(f32, float, float)
RM_DEFINE_POS(f64, double, double)
RM_DEFINE_POS(bf16, uint16_t, __nv_bfloat16)
