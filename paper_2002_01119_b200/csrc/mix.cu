// Fused learner-averaging kernels: gossip mix + SGD (RAD / AD / D-PSGD),
// uniform mean + SGD (D1D), and S-PSGD — the reference's
//   simulation._gossip_step (pkg/src/ringmix/simulation.py:263-268)
//   W_next = apply_mixing(W, T) - lr * G        (mixing.py:106-125)
// and step_spsgd (simulation.py:251-260), one HBM pass per step.
//
// HBM layout: learner-major (L, d) rows with leading dimension ld (elements);
// the reference's (d, L) matrix is the transpose view.
//
// Design: a persistent kernel walks column tiles [c0, c0+cw)
// of all L rows.  Per tile, one thread issues 2-D tensor-map TMA loads
// (cp.async.bulk.tensor.2d, boxes of [L rows x <= 256 columns]) of W[:, tile]
// and G[:, tile] into a shared-memory stage, completion tracked by an mbarrier
// (expect_tx).  Three stages are in flight per CTA, so every W element crosses
// HBM exactly once although it feeds three outputs (itself and its two ring
// neighbours).  Consumers read the stage with 16-byte shared loads and write
// W' with 16-byte streaming stores.  Mean tiles (D1D, S-PSGD) first reduce each
// column in numpy's pairwise order, then apply the update.
//
// Arithmetic: fp32/fp64 storage computes in fp64 with the
// reference's exact rounding sequence, so results are the reference's fp64
// result rounded once to the storage type:
//   ring:    acc = fl(w_a*t); acc = fma(w_b,t,acc); acc = fma(w_c,t,acc)
//            (a<b<c the sorted neighbour triple, t = fl64(1/3): OpenBLAS dgemm
//            accumulates ascending k with FMA; zero terms add exactly)
//   uniform: numpy pairwise sum over the learner axis, then / L
//   update:  y = mix - fl(lr*g)        (numpy evaluates lr*G first)
// bf16 storage computes the same sequence in fp32.
// A fused epilogue publishes max|W'| (NaN sorts above inf) for the
// reference's _check_divergence (simulation.py:390-395): zero extra bytes.
#include "common.cuh"
#include "tma_host.cuh"
#include "arith.cuh"
#include "zsrc.cuh"
#include "../../include/ringmix_b200.h"

#include <stdlib.h>
#include <cuda.h>
#include <cudaTypedefs.h>

namespace rm {

// kRingZ / kMeanZ: the ring / uniform step with the quadratic oracle's gradient
// produced in the epilogue from the generator's normals (zsrc.cuh); HAS_G then means
// "Phi (the weights the gradient is taken at) is staged separately" — without it Phi = W.
enum Mode { kRing = 0, kMean = 1, kSpsgd = 2, kRingZ = 3, kMeanZ = 4 };

__host__ __device__ constexpr bool mode_ring(int m) { return m == kRing || m == kRingZ; }
__host__ __device__ constexpr bool mode_z(int m) { return m == kRingZ || m == kMeanZ; }

// items per thread in flight in the output phase (build-time tuning knob)
#ifndef RM_RING_UNROLL
#define RM_RING_UNROLL 2
#endif

constexpr int kRingUnroll = RM_RING_UNROLL;
// RM_TMA_STORE (build-time experiment): ring steps with G write W' over their G tile in
// shared memory and one thread stores the tile with a 2-D tensor-map TMA store; a stage is
// refilled one tile later, after its store has read it
#ifndef RM_TMA_STORE
#define RM_TMA_STORE 0
#endif
constexpr int kRingThreads = 512;   // ring tiles: one 512-thread CTA per SM
constexpr int kMeanThreads = 256;   // mean tiles: two 256-thread CTAs per SM
constexpr int kStages = 3;
// Z modes: more (smaller) W stages, and the normals of iteration i + kZDist are copied
// (cp.async, 8 bytes per thread and element) into one of kZBufs shared buffers while
// iteration i computes
constexpr int kZStages = 4;
constexpr int kZDist = 2;
constexpr int kZBufs = kZDist + 1;
constexpr int kZTileRing = 4096;   // L * cw per z buffer (fp64 elements): 32 KB
constexpr int kZTileMean = 2048;   // two CTAs per SM: 16 KB
constexpr int kMaxTmaL = 256;   // one TMA row box per tile
constexpr int kStageTarget = 64 * 1024;      // ring
constexpr int kMeanStageTarget = 32 * 1024;  // mean (two CTAs per SM)
constexpr int kSmallRingStageTarget = 24 * 1024;  // ring with L <= 32 (two CTAs per SM)

struct MixArgs {
  const void* W;
  const void* G;
  void* out;
  long long ldw, ldg, ldo;
  long long d;       // columns
  long long d_main;  // columns covered by the tiled TMA path (multiple of VEC)
  int L;
  int cw;        // tile width (elements), power of two, multiple of VEC
  int log2_nv;   // log2(cw / VEC)
  int zdcols;    // Z modes: descriptor columns (uint64) per staged tile
  int zslots;    // Z modes: doubles per z buffer
  long long ntiles;
  const int32_t* left;
  const int32_t* right;
  double lr;
  unsigned long long* absmax;  // may be null
  unsigned int* mismatch;      // kSpsgd: set nonzero if W rows differ
  ZSrc z;                      // kRingZ / kMeanZ
};

// gradient element (row j, column c) of the Z modes in the accumulation type, rounded to
// the storage type first exactly as the generator's G output
template <typename T>
__device__ __forceinline__ typename Elem<T>::acc z_grad_elem(const ZSrc& z, int j, long long c,
                                                             double phi) {
  using E = Elem<T>;
  const double zv = __ldcs(z.scratch + z_index(z, z_desc(z, j, c), c));
  return (typename E::acc)E::st(
      (typename E::acc)z_grad(__ldg(z.lam + c), __ldg(z.wopt + c), z.sd, phi, zv));
}

// ----------------------------------------------------------------------------
// scalar path: any alignment / any L; one thread per (row, column)
// Used for unaligned layouts, very large L, and the < VEC tail columns.
// ----------------------------------------------------------------------------
template <typename T, int MODE, bool HAS_G>
__global__ void __launch_bounds__(256) mix_scalar_kernel(MixArgs a, long long c_begin) {
  using E = Elem<T>;
  using A = typename E::acc;
  const T* W = static_cast<const T*>(a.W);
  const T* G = static_cast<const T*>(a.G);
  T* out = static_cast<T*>(a.out);
  const long long ncols = a.d - c_begin;
  const long long total = ncols * a.L;
  unsigned long long amax = 0;
  const A lr = (A)a.lr;
  if (!mode_ring(MODE)) {
    // one thread per column: the column mean once (numpy pairwise, any L),
    // then every learner's output
    for (long long cc = blockIdx.x * (long long)blockDim.x + threadIdx.x; cc < ncols;
         cc += (long long)gridDim.x * blockDim.x) {
      const long long c = c_begin + cc;
      const T* src = MODE == kSpsgd ? G : W;
      const long long lds = MODE == kSpsgd ? a.ldg : a.ldw;
      auto get = [&](int i) { return (A)E::ld(src + i * lds + c, 0); };
      const A m = r_div(pairwise_sum<A>(get, 0, a.L), (A)a.L);
      for (int j = 0; j < a.L; j++) {
        A y;
        if (MODE == kMeanZ) {
          const double phi = HAS_G ? (double)E::ld(G + j * a.ldg + c, 0)
                                   : (double)E::ld(W + j * a.ldw + c, 0);
          y = r_sub(m, r_mul(lr, z_grad_elem<T>(a.z, j, c, phi)));
        } else if (MODE == kMean) {
          y = HAS_G ? r_sub(m, r_mul(lr, (A)E::ld(G + j * a.ldg + c, 0))) : m;
        } else {  // kSpsgd: W - lr * mean_l(G)
          if (a.mismatch && !(W[j * a.ldw + c] == W[c])) atomicOr(a.mismatch, 1u);
          y = r_sub((A)E::ld(W + j * a.ldw + c, 0), r_mul(lr, m));
        }
        const T ys = E::st(y);
        out[j * a.ldo + c] = ys;
        const unsigned long long b = abs_bits((double)E::absd(ys));
        amax = b > amax ? b : amax;
      }
    }
    if (a.absmax) absmax_publish(a.absmax, amax);
    return;
  }
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(idx / ncols);
    const long long c = c_begin + idx % ncols;
    A y;
    {
      int x0 = a.left[j], x1 = j, x2 = a.right[j], t;
      if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
      if (x2 < x1) { t = x1; x1 = x2; x2 = t; }
      if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
      y = ring3<A>(E::ld(W + x0 * a.ldw + c, 0), E::ld(W + x1 * a.ldw + c, 0),
                   E::ld(W + x2 * a.ldw + c, 0));
      if (MODE == kRingZ) {
        const double phi = HAS_G ? (double)E::ld(G + j * a.ldg + c, 0)
                                 : (double)E::ld(W + j * a.ldw + c, 0);
        y = r_sub(y, r_mul(lr, z_grad_elem<T>(a.z, j, c, phi)));
      } else if (HAS_G) {
        y = r_sub(y, r_mul(lr, E::ld(G + j * a.ldg + c, 0)));
      }
    }
    T ys = E::st(y);
    out[j * a.ldo + c] = ys;
    unsigned long long b = abs_bits((double)E::absd(ys));
    amax = b > amax ? b : amax;
  }
  if (a.absmax) absmax_publish(a.absmax, amax);
}

// ----------------------------------------------------------------------------
// tiled TMA path (2-D tensor maps)
//
// Each tile is [L rows x cw columns] of W (and of G).  One elected thread
// loads it with cp.async.bulk.tensor.2d boxes of at most 256 x 256 elements —
// one TMA instruction per tensor per tile for L <= 256 — into a shared-memory
// stage laid out row-major [L][cw].  (A first version issued one 1-D bulk copy
// per row; ncu showed the per-copy cost of 128 x 512 B copies per tile capped
// DRAM at 35 %: profiles/r1_v1_bulk1d.md.)  Out-of-range columns of the last
// tile are zero-filled by TMA and skipped by the consumers.
// ----------------------------------------------------------------------------
constexpr int kBox = 256;  // TMA box dimension limit (elements)

// NT threads per CTA: ring tiles run one 512-thread CTA per SM; mean tiles
// (D1D / S-PSGD) run two 256-thread CTAs per SM, so one CTA's mean phase
// overlaps the other's output phase.
// element-wise round-to-nearest fp32 add of two pairs (FADD2 on sm_100; each lane of
// the pair is an ordinary IEEE add, nothing is contracted)
__device__ __forceinline__ float2 fadd2_rn(float2 a, float2 b) {
  unsigned long long ra, rb, rc;
  memcpy(&ra, &a, 8);
  memcpy(&rb, &b, 8);
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rc) : "l"(ra), "l"(rb));
  float2 c;
  memcpy(&c, &rc, 8);
  return c;
}

// two adjacent bf16 columns of a staged row as floats (exact conversion)
template <typename T>
__device__ __forceinline__ float2 lds_pair(const T* p) {
  uint32_t w;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(smem_u32(p)));
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// The VEC column means of one output vector: 16-byte shared loads (lanes own
// VEC consecutive columns, so scalar loads would be 2·VEC-way bank conflicts).
template <int VEC>
__device__ __forceinline__ void load_means(const double* s_mean, int c, double (&m)[VEC]) {
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const double2 t = *reinterpret_cast<const double2*>(s_mean + c + e);
    m[e] = t.x;
    m[e + 1] = t.y;
  }
}

// Element e of a staged vector in the accumulation type.  RM_FAST_F2D (build-time
// experiment): fp32 -> fp64 widening of normal numbers by re-biasing the exponent with
// integer ops (exact), F2F only for zero / subnormal / inf / NaN.
template <typename T>
__device__ __forceinline__ typename Elem<T>::acc widen(const T* v, int e) {
#ifdef RM_FAST_F2D
  if constexpr (sizeof(T) == 4) {
    const uint32_t u = __float_as_uint(v[e]);
    if (((u >> 23) & 0xffu) - 1u < 254u) {
      const uint32_t hi = (((u & 0x7fffffffu) >> 3) + (896u << 20)) | (u & 0x80000000u);
      return __hiloint2double((int)hi, (int)(u << 29));
    }
  }
#endif
  return (typename Elem<T>::acc)Elem<T>::ld(v, e);
}

template <typename T, int MODE, bool HAS_G, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
    mix_tma_kernel(MixArgs a, const __grid_constant__ CUtensorMap tmW,
                   const __grid_constant__ CUtensorMap tmG,
                   const __grid_constant__ CUtensorMap tmD,
                   const __grid_constant__ CUtensorMap tmLam,
                   const __grid_constant__ CUtensorMap tmOpt) {
  constexpr int kThreads = NT;
  using E = Elem<T>;
  using A = typename E::acc;
  constexpr int VEC = E::VEC;
  extern __shared__ __align__(128) unsigned char smem[];

  const int L = a.L;
  const int cw = a.cw;
  const int w_bytes = L * cw * (int)sizeof(T);
  constexpr bool ZM = mode_z(MODE);
  constexpr bool TSTORE = RM_TMA_STORE && MODE == kRing && HAS_G;
  // Z modes take a separate Phi through the cp.async buffers, not the stage
  constexpr bool stage_g = (HAS_G && !ZM) || MODE == kSpsgd;
  constexpr int kSt = ZM ? kZStages : kStages;
  // Z modes: the tile's normal descriptors [L][zdcols] (uint64) and its lam / w* columns
  // (fp64 [cw] each) ride in the stage, each piece 128-byte aligned
  const int wg_bytes = w_bytes * (stage_g ? 2 : 1);
  const int zd_off = (wg_bytes + 127) & ~127;
  const int zl_off = zd_off + ((L * a.zdcols * 8 + 127) & ~127);
  const int zo_off = zl_off + ((cw * 8 + 127) & ~127);
  const int stage_bytes = ZM ? zo_off + ((cw * 8 + 127) & ~127) : wg_bytes;
  const uint32_t stage_tx = ZM ? wg_bytes + L * a.zdcols * 8 + 2 * cw * 8 : wg_bytes;

  // layout: [mbarriers | tri table (L x int4) | stages | per-column mean]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  int4* s_tri = reinterpret_cast<int4*>(smem + 128);
  unsigned char* stages = smem + 128 + ((L * 16 + 127) / 128) * 128;
  double* s_mean = nullptr;
  A* s_part = nullptr;  // [8][cw] partial sums in the accumulation type (narrow tiles)
  unsigned char* tail = stages + kSt * stage_bytes;
  if (!mode_ring(MODE)) {
    s_mean = reinterpret_cast<double*>(tail);
    s_part = reinterpret_cast<A*>(s_mean + cw);
    tail += a.zslots ? ((size_t)cw * sizeof(double) + 8 * cw * sizeof(A) + 15) / 16 * 16 : 0;
  }
  double* zbuf = ZM ? reinterpret_cast<double*>(tail) : nullptr;  // [kZBufs][zslots]
  // Z modes with a separate Phi: [kZBufs][L][cw] Phi tiles after the normals
  T* pbuf = ZM && HAS_G ? reinterpret_cast<T*>(zbuf + (size_t)kZBufs * a.zslots) : nullptr;

  T* out = static_cast<T*>(a.out);
  const int tid = threadIdx.x;

  if (tid == 0) {
    tma_prefetch_desc(&tmW);
    if (stage_g) tma_prefetch_desc(&tmG);
    if (ZM) {
      tma_prefetch_desc(&tmD);
      tma_prefetch_desc(&tmLam);
      tma_prefetch_desc(&tmOpt);
    }
    for (int s = 0; s < kSt; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  // Programmatic dependent launch: everything above overlaps the previous kernel's
  // tail; W, G and the neighbour tables may be its outputs, so wait for it here.
  pdl_wait();
  if (mode_ring(MODE)) {
    for (int j = tid; j < L; j += kThreads) {
      int x0 = a.left[j], x1 = j, x2 = a.right[j], t;
      if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
      if (x2 < x1) { t = x1; x1 = x2; x2 = t; }
      if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
      // .w: where learner j itself sits in the sorted triple (Z modes take Phi = W from it)
      s_tri[j] = make_int4(x0, x1, x2, x0 == j ? 0 : (x1 == j ? 1 : 2));
    }
  }
  __syncthreads();

  const long long first = blockIdx.x;
  const long long stride = gridDim.x;
  const int box_c = cw < kBox ? cw : kBox;

  // tile t -> stage s (one thread)
  auto issue = [&](int s, long long t) {
    const int c0 = (int)(t * cw);
    unsigned char* st = stages + (size_t)s * stage_bytes;
    mbar_arrive_expect_tx(&full[s], stage_tx);
    // L <= 256: one row box; column boxes of box_c land one after another,
    // each [L][box_c] (see sidx)
    for (int cc = 0; cc < cw; cc += box_c) {
      const int off = cc * L * (int)sizeof(T);
      tma_load_2d(st + off, &tmW, c0 + cc, 0, &full[s]);
      if (stage_g) tma_load_2d(st + w_bytes + off, &tmG, c0 + cc, 0, &full[s]);
    }
    if (ZM) {
      tma_load_2d(st + zd_off, &tmD, (c0 >> kZGroupLog2) * 2, 0, &full[s]);
      for (int cc = 0; cc < cw; cc += box_c) {
        tma_load_2d(st + zl_off + cc * 8, &tmLam, c0 + cc, 0, &full[s]);
        tma_load_2d(st + zo_off + cc * 8, &tmOpt, c0 + cc, 0, &full[s]);
      }
    }
  };
  // element (r, c) of a stage tile (box_c is a power of two)
  const int lg_bc = __ffs(box_c) - 1;
  const int box_stride = L << lg_bc;
  auto sidx = [&](int r, int c) -> int {
    return (c >> lg_bc) * box_stride + (r << lg_bc) + (c & (box_c - 1));
  };

  if (tid == 0) {
    for (int s = 0; s < kSt; s++) {
      long long t = first + s * stride;
      if (t < a.ntiles) issue(s, t);
    }
  }

  typename E::amax_t amax = 0;
  const A lr = (A)a.lr;
  const int log2_nv = a.log2_nv;
  const int nv_full = 1 << log2_nv;
  const int warp = tid >> 5, lane = tid & 31;

  // Z modes: copy the normals of iteration i's tile into z buffer i % kZBufs, laid out
  // [L][cw] like the W tile.  Copy mapping: the thread that would own column vector v of
  // a row instead copies the lane-contiguous columns cb + ln + grp * e (e < VEC) of it —
  // each warp's 8-byte cp.async then read consecutive scratch doubles, and the run lies
  // in one 128-column descriptor group (one descriptor per row and thread).  The
  // descriptors come from the stage, which the TMA filled kSt - kZDist iterations ahead.
  // Every thread commits one cp.async group per call; a buffer is read only after
  // cp_async_wait and the CTA barrier that ends the previous iteration.
  const int lg_cw = __ffs(cw) - 1;
  // position of normal column c in a buffer row: with VEC = 4 (fp32) the two column pairs
  // of a vector live in separate halves of the row, so the consumer's two 16-byte loads
  // per vector are each lane-contiguous (no shared-memory bank conflicts)
  auto zpos = [&](int c) -> int {
    return VEC == 4 ? (((c >> 1) & 1) << (lg_cw - 1)) + ((c >> 2) << 1) + (c & 1) : c;
  };
  const int zgrp = nv_full < 32 ? nv_full : 32;
  const int zv_ = tid & (nv_full - 1);
  const int zcb = (zv_ & ~(zgrp - 1)) * VEC, zln = zv_ & (zgrp - 1);
  auto zissue = [&](int i) {
    const long long t = first + (long long)i * stride;
    if (t < a.ntiles) {
      const int si = i % kSt;
      mbar_wait(&full[si], (uint32_t)(i / kSt) & 1);
      const uint64_t* sD =
          reinterpret_cast<const uint64_t*>(stages + (size_t)si * stage_bytes + zd_off);
      const long long c0 = t * cw;
      const int width = (int)min((long long)cw, a.d - c0);
      double* zb = zbuf + (size_t)(i % kZBufs) * a.zslots;
      const int gi = (int)(((c0 + zcb) >> kZGroupLog2) - (c0 >> kZGroupLog2));
      const int total = L << log2_nv;
      if constexpr (ZM && HAS_G && sizeof(T) >= 4) {
        // Phi: the thread's own column vector of each row, 16-byte copies
        const T* P = static_cast<const T*>(a.G);
        T* pb = pbuf + (size_t)(i % kZBufs) * a.zslots;
        const int cv = (tid & (nv_full - 1)) * VEC;
        if (cv < width) {
          for (int idx = tid; idx < total; idx += kThreads) {
            const int j = idx >> log2_nv;
            const T* src = P + (long long)j * a.ldg + c0 + cv;
            T* dst = pb + (j << lg_cw) + cv;
            if (cv + VEC <= width) {
              cp_async_16(dst, src);
            } else {
              for (int e = 0; e < width - cv; e++) cp_async_elem(dst + e, src + e);
            }
          }
        }
      }
      if (zcb + zln < width) {
        for (int idx = tid; idx < total; idx += kThreads) {
          const int j = idx >> log2_nv;
          const uint64_t d0 = sD[j * a.zdcols + 2 * gi], d1 = sD[j * a.zdcols + 2 * gi + 1];
          ZDesc gd;
          gd.zb = (long long)d0;
          gd.dz = (int)(uint32_t)d1;
          gd.brk = (int)(uint32_t)(d1 >> 32);
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            const int c = zcb + zln + zgrp * e;
            if (c < width)
              cp_async_8(zb + (j << lg_cw) + zpos(c), a.z.scratch + z_index(a.z, gd, c0 + c));
          }
        }
      }
    }
    cp_async_commit();
  };
  if constexpr (ZM) {
    for (int i = 0; i < kZDist; i++) zissue(i);
    cp_async_wait<kZDist - 1>();
    __syncthreads();
  }

  int it = 0;
  for (long long t = first; t < a.ntiles; t += stride, ++it) {
    const int s = it % kSt;
    const uint32_t parity = (it / kSt) & 1;
    if constexpr (ZM) zissue(it + kZDist);
    const long long c0 = t * cw;
    const int width = (int)min((long long)cw, a.d - c0);
    const T* sW = reinterpret_cast<const T*>(stages + (size_t)s * stage_bytes);
    const T* sG = reinterpret_cast<const T*>(stages + (size_t)s * stage_bytes + w_bytes);

    const int nv = (width + VEC - 1) / VEC;
    const int total = L << log2_nv;
    // this CTA's last tile: let the next kernel on the stream start launching (it
    // waits for this grid's completion before touching memory)
    if (tid == 0 && t + stride >= a.ntiles) pdl_launch_dependents();
    mbar_wait(&full[s], parity);

    if (!mode_ring(MODE)) {
      // numpy pairwise mean per column over the L staged rows: one thread per
      // column keeps numpy's 8 partial sums r[0..7] (8 <= n <= 128) in
      // registers (8 independent add chains) and combines them in numpy's
      // order ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail.  Lanes
      // read consecutive columns of one staged row: no bank conflicts.
      const T* src = (MODE == kSpsgd) ? sG : sW;
      const int groups = cw <= kThreads / 2 ? min(8, kThreads / cw) : 1;
      // 2-byte elements: a thread owns a column pair (one 32-bit shared load
      // feeds two columns' chains, full 128-byte wavefronts per warp)
      const int pgroups = sizeof(T) == 2 ? min(8, kThreads / (cw / 2)) : 0;
      if (sizeof(T) == 2 && pgroups >= 2 && cw >= 2) {
        const int n8 = L - (L % 8);
        const int per = 8 / pgroups;
        const int ncp = cw / 2;
        const int g = tid / ncp, col = 2 * (tid % ncp);
        if (g < pgroups && col < width) {
          for (int q = 0; q < per; q++) {
            const int k = g * per + q;
            float2 r = lds_pair(src + sidx(k, col));
            for (int i = 8 + k; i < n8; i += 8) {
              const float2 v = lds_pair(src + sidx(i, col));
              r = fadd2_rn(r, v);  // two independent IEEE adds in one instruction
            }
            s_part[k * cw + col] = r.x;
            s_part[k * cw + col + 1] = r.y;
          }
        }
        __syncthreads();
        if (tid < width) {
          const A* pp = s_part + tid;
          A res = r_add(r_add(r_add((A)pp[0], (A)pp[cw]), r_add((A)pp[2 * cw], (A)pp[3 * cw])),
                        r_add(r_add((A)pp[4 * cw], (A)pp[5 * cw]),
                              r_add((A)pp[6 * cw], (A)pp[7 * cw])));
          for (int i = n8; i < L; i++) res = r_add(res, (A)E::lds(src + sidx(i, tid)));
          s_mean[tid] = (double)r_div(res, (A)L);
        }
      } else if (groups >= 2) {
        // narrow tiles: split the 8 chains over `groups` threads per column so
        // every warp works; partial sums meet in shared memory
        const int n8 = L - (L % 8);
        const int per = 8 / groups;
        const int g = tid / cw, col = tid % cw;
        if (g < groups && col < width) {
          for (int q = 0; q < per; q++) {
            const int k = g * per + q;
            A r = (A)E::lds(src + sidx(k, col));
            for (int i = 8 + k; i < n8; i += 8) r = r_add(r, (A)E::lds(src + sidx(i, col)));
            s_part[k * cw + col] = r;
          }
        }
        __syncthreads();
        if (tid < width) {
          const A* pp = s_part + tid;
          A res = r_add(r_add(r_add((A)pp[0], (A)pp[cw]), r_add((A)pp[2 * cw], (A)pp[3 * cw])),
                        r_add(r_add((A)pp[4 * cw], (A)pp[5 * cw]),
                              r_add((A)pp[6 * cw], (A)pp[7 * cw])));
          for (int i = n8; i < L; i++) res = r_add(res, (A)E::lds(src + sidx(i, tid)));
          s_mean[tid] = (double)r_div(res, (A)L);
        }
      } else {
        // 8 <= L <= 128 here (launch_mix routes other L to the scalar kernel)
        const int n8 = L - (L % 8);
        for (int col = tid; col < width; col += kThreads) {
          A r[8];
#pragma unroll
          for (int k = 0; k < 8; k++) r[k] = (A)E::lds(src + sidx(k, col));
          for (int i = 8; i < n8; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; k++) r[k] = r_add(r[k], (A)E::lds(src + sidx(i + k, col)));
          }
          A res = r_add(r_add(r_add(r[0], r[1]), r_add(r[2], r[3])),
                        r_add(r_add(r[4], r[5]), r_add(r[6], r[7])));
          for (int i = n8; i < L; i++) res = r_add(res, (A)E::lds(src + sidx(i, col)));
          s_mean[col] = (double)r_div(res, (A)L);
        }
      }
      __syncthreads();
    }

    // mean modes: a thread's column vector is the same for all its items (the
    // host guarantees nv_full divides the CTA size), so its means are read once
    A ma[VEC];
    if (!mode_ring(MODE)) {
      double mv[VEC];
      load_means<VEC>(s_mean, (tid & (nv_full - 1)) * VEC, mv);
#pragma unroll
      for (int e = 0; e < VEC; e++) ma[e] = (A)mv[e];
    }
    // Z modes: lam / w* (and the means) of the thread's columns, the same for all its items
    double zlam[ZM ? VEC : 1], zopt[ZM ? VEC : 1];
    if constexpr (ZM) {
      const double* sLam = reinterpret_cast<const double*>(stages + (size_t)s * stage_bytes + zl_off);
      const double* sOpt = reinterpret_cast<const double*>(stages + (size_t)s * stage_bytes + zo_off);
      const int cv = (tid & (nv_full - 1)) * VEC;
      if (cv < width) {
        load_means<VEC>(sLam, cv, zlam);
        load_means<VEC>(sOpt, cv, zopt);
      }
    }
    if constexpr (ZM) {
      const double* zb = zbuf + (size_t)(it % kZBufs) * a.zslots;
#pragma unroll kRingUnroll
      for (int idx = tid; idx < total; idx += kThreads) {
        const int j = idx >> log2_nv;
        const int v = idx & (nv_full - 1);
        if (v >= nv) continue;
        const int c = v * VEC;
        Vec<T> y;
        double zv[VEC];
        {
          const double* zr = zb + (j << lg_cw);
          if (VEC == 4) {
            const double2 p0 = *reinterpret_cast<const double2*>(zr + (c >> 1));
            const double2 p1 = *reinterpret_cast<const double2*>(zr + (cw >> 1) + (c >> 1));
            zv[0] = p0.x;
            zv[1] = p0.y;
            zv[VEC > 2 ? 2 : 0] = p1.x;
            zv[VEC > 3 ? 3 : 0] = p1.y;
          } else {
            load_means<VEC>(zr, c, zv);
          }
        }
        // Phi: its cp.async tile, or (Phi = W) learner j's own operand of the ring
        double phi[VEC];
        if (HAS_G || MODE == kMeanZ) {
          Vec<T> vp;
          vp.raw = HAS_G ? *reinterpret_cast<const uint4*>(
                               pbuf + (size_t)(it % kZBufs) * a.zslots + (j << lg_cw) + c)
                         : *reinterpret_cast<const uint4*>(sW + sidx(j, c));
#pragma unroll
          for (int e = 0; e < VEC; e++) phi[e] = (double)E::ld(vp.e(), e);
        }
        A m[VEC];
        if (MODE == kRingZ) {
          const int4 tri = s_tri[j];
          Vec<T> va, vb, vc;
          va.raw = *reinterpret_cast<const uint4*>(sW + sidx(tri.x, c));
          vb.raw = *reinterpret_cast<const uint4*>(sW + sidx(tri.y, c));
          vc.raw = *reinterpret_cast<const uint4*>(sW + sidx(tri.z, c));
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            const A xa = widen<T>(va.e(), e), xb = widen<T>(vb.e(), e), xc = widen<T>(vc.e(), e);
            m[e] = ring3<A>(xa, xb, xc);
            if (!HAS_G) phi[e] = (double)(tri.w == 0 ? xa : (tri.w == 1 ? xb : xc));
          }
        } else {
#pragma unroll
          for (int e = 0; e < VEC; e++) m[e] = ma[e];
        }
#pragma unroll
        for (int e = 0; e < VEC; e++) {
          const T g = E::st((A)z_grad(zlam[e], zopt[e], a.z.sd, phi[e], zv[e]));
          y.e()[e] = E::st(r_sub(m[e], r_mul(lr, (A)g)));
        }
        T* dst = out + (long long)j * a.ldo + c0 + c;
        if (c + VEC <= width) {
#pragma unroll
          for (int e = 0; e < VEC; e++) amax = E::amax_acc(amax, y.e()[e]);
          st_cs_v4(dst, y.raw);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            if (c + e < width) {
              amax = E::amax_acc(amax, y.e()[e]);
              dst[e] = y.e()[e];
            }
          }
        }
      }
    } else {
#pragma unroll kRingUnroll
      for (int idx = tid; idx < total; idx += kThreads) {
        const int j = idx >> log2_nv;
        const int v = idx & (nv_full - 1);
        if (v >= nv) continue;
        const int c = v * VEC;
        Vec<T> y;
        if (MODE == kRing) {
          const int4 tri = s_tri[j];
          Vec<T> va, vb, vc, vg;
          va.raw = *reinterpret_cast<const uint4*>(sW + sidx(tri.x, c));
          vb.raw = *reinterpret_cast<const uint4*>(sW + sidx(tri.y, c));
          vc.raw = *reinterpret_cast<const uint4*>(sW + sidx(tri.z, c));
          if (HAS_G) vg.raw = *reinterpret_cast<const uint4*>(sG + sidx(j, c));
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            A m = ring3<A>(widen<T>(va.e(), e), widen<T>(vb.e(), e), widen<T>(vc.e(), e));
            if (HAS_G) m = r_sub(m, r_mul(lr, widen<T>(vg.e(), e)));
            y.e()[e] = E::st(m);
          }
        } else if (MODE == kMean) {
          Vec<T> vg;
          if (HAS_G) vg.raw = *reinterpret_cast<const uint4*>(sG + sidx(j, c));
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            A m = ma[e];
            if (HAS_G) m = r_sub(m, r_mul(lr, (A)E::ld(vg.e(), e)));
            y.e()[e] = E::st(m);
          }
        } else {  // kSpsgd
          Vec<T> vw, w0;
          vw.raw = *reinterpret_cast<const uint4*>(sW + sidx(j, c));
          w0.raw = *reinterpret_cast<const uint4*>(sW + sidx(0, c));
          bool diff = false;
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            if (c + e < width) diff |= !(vw.e()[e] == w0.e()[e]);
            A m = ma[e];
            y.e()[e] = E::st(r_sub((A)E::ld(vw.e(), e), r_mul(lr, m)));
          }
          if (diff && a.mismatch) atomicOr(a.mismatch, 1u);
        }
        T* dst = out + (long long)j * a.ldo + c0 + c;
        if (TSTORE) {
          // over this thread's own G vector (read above); the TMA store clips columns >= d
          *reinterpret_cast<uint4*>(const_cast<T*>(sG) + sidx(j, c)) = y.raw;
#pragma unroll
          for (int e = 0; e < VEC; e++)
            if (c + e < width) amax = E::amax_acc(amax, y.e()[e]);
        } else if (c + VEC <= width) {
#pragma unroll
          for (int e = 0; e < VEC; e++) amax = E::amax_acc(amax, y.e()[e]);
          st_cs_v4(dst, y.raw);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; e++) {
            if (c + e < width) {
              amax = E::amax_acc(amax, y.e()[e]);
              dst[e] = y.e()[e];
            }
          }
        }
      }
    }

    if constexpr (ZM) cp_async_wait<kZDist - 1>();  // own copies for the next tile landed
    if constexpr (TSTORE) fence_proxy_async_smem();  // W' tile visible to the TMA
    __syncthreads();  // stage s fully consumed (and s_mean free); next z buffer visible
    if (tid == 0) {
      if constexpr (TSTORE) {
        const unsigned char* sg = stages + (size_t)s * stage_bytes + w_bytes;
        for (int cc = 0; cc < cw; cc += box_c)
          tma_store_2d(&tmD, sg + cc * L * (int)sizeof(T), (int)(c0 + cc), 0);
        bulk_commit();
        if (it > 0) {
          bulk_wait_read<1>();   // the previous tile's store has read its stage
          const long long tn = t - stride + (long long)kSt * stride;
          if (tn < a.ntiles) issue((it - 1) % kSt, tn);
        }
      } else {
        long long tn = t + (long long)kSt * stride;
        if (tn < a.ntiles) issue(s, tn);
      }
    }
  }
  if constexpr (TSTORE) {
    if (tid == 0) bulk_wait<0>();
  }
  if (a.absmax) absmax_publish(a.absmax, E::amax_bits(amax));
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
template <typename T, int MODE, bool HAS_G>
static int launch_scalar(const MixArgs& a, long long c_begin, cudaStream_t st) {
  long long total = (a.d - c_begin) * a.L;
  if (total <= 0) return RM_OK;
  long long blocks = (total + 255) / 256;
  int cap = sm_count(-1) * 8;
  if (blocks > cap) blocks = cap;
  mix_scalar_kernel<T, MODE, HAS_G><<<(int)blocks, 256, 0, st>>>(a, c_begin);
  RM_CHECK_LAUNCH("mix_scalar_kernel");
  return RM_OK;
}

static size_t tma_smem_bytes(int L, int cw, size_t elem, bool stage_g, int mode,
                             int kThreads, int zdcols = 0, int zslots = 0, bool zphi = false) {
  size_t stage = (size_t)L * cw * elem * (stage_g ? 2 : 1);
  if (mode_z(mode)) {
    // descriptor and lam / w* tiles per stage (128-byte aligned pieces), kZStages stages,
    // the mean region at full size (see the kernel), kZBufs normal buffers
    auto r128 = [](size_t x) { return (x + 127) & ~(size_t)127; };
    stage = r128(stage) + r128((size_t)L * zdcols * 8) + 2 * r128((size_t)cw * 8);
    size_t bytes = 128 + ((size_t)(L * 16 + 127) / 128) * 128 + kZStages * stage;
    const size_t acc = elem == 2 ? sizeof(float) : sizeof(double);
    if (!mode_ring(mode)) bytes += ((size_t)cw * sizeof(double) + 8 * cw * acc + 15) / 16 * 16;
    return bytes + (size_t)kZBufs * zslots * (sizeof(double) + (zphi ? elem : 0));
  }
  size_t bytes = 128 + ((size_t)(L * 16 + 127) / 128) * 128 + kStages * stage;
  // per-column means, plus [8][cw] partial sums when the mean phase splits a
  // column's 8 chains over several threads (see the mean phase)
  const bool split = cw <= kThreads / 2 || (elem == 2 && cw <= kThreads);
  // (the partials are in the accumulation type: float for 2-byte elements)
  const size_t acc = elem == 2 ? sizeof(float) : sizeof(double);
  if (!mode_ring(mode)) bytes += (size_t)cw * sizeof(double) + (split ? 8 * cw * acc : 0);
  return bytes;
}

template <typename T>
static bool make_map(CUtensorMap* m, const void* base, long long d, int L, long long ld, int box_c,
                     int box_r) {
  return tma_map_2d<T>(m, base, d, L, ld, box_c, box_r);
}

template <typename T, int MODE, bool HAS_G, int NT>
static int launch_mix(MixArgs a, cudaStream_t st) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const size_t esz = sizeof(T);
  const bool stage_g = (HAS_G && !mode_z(MODE)) || MODE == kSpsgd;
  const uintptr_t align_bits =
      reinterpret_cast<uintptr_t>(a.W) | reinterpret_cast<uintptr_t>(a.out) |
      (stage_g ? reinterpret_cast<uintptr_t>(a.G) : 0) | (uintptr_t)(a.ldw * esz) |
      (uintptr_t)(a.ldo * esz) | (stage_g ? (uintptr_t)(a.ldg * esz) : 0);
  const uintptr_t z_bits =
      mode_z(MODE) ? reinterpret_cast<uintptr_t>(a.z.lam) | reinterpret_cast<uintptr_t>(a.z.wopt) |
                         (HAS_G ? reinterpret_cast<uintptr_t>(a.G) | (uintptr_t)(a.ldg * esz) : 0)
                   : 0;
  const bool aligned = ((align_bits | z_bits) & 15) == 0;
  static int max_optin = -1;
  if (max_optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  // the tiled mean phase covers numpy's non-recursive pairwise case (8 <= L <= 128)
  const bool mean_ok = mode_ring(MODE) || (a.L >= 8 && a.L <= 128);
  bool use_tma = aligned && mean_ok && a.L <= kMaxTmaL && a.d >= VEC && a.d < (1LL << 31) &&
                 tma_encode_fn() != nullptr;
  int cw = 0;
  if (use_tma) {
    // tile width: power of two, stage ~kStageTarget, enough tiles to spread
    // over every SM several times
    size_t per_col = (size_t)a.L * esz * (stage_g ? 2 : 1);
    cw = VEC;
    size_t target = NT == kRingThreads ? kStageTarget
                                       : (mode_ring(MODE) ? kSmallRingStageTarget : kMeanStageTarget);
    // bf16 ring tiles: 32 KB stages (128 columns at L = 64) measured 0.93 of HBM at C2
    // against 0.84 with 64 KB (256 columns) — tools/gpu_bf16_sweep.sh
    if (NT == kRingThreads && esz == 2) target = kStageTarget / 2;
    if (const char* env = getenv("RINGMIX_STAGE_KB")) {  // tuning override
      int kb = atoi(env);
      if (kb >= 4 && kb <= 96) target = (size_t)kb * 1024;
    }
    while ((size_t)(cw * 2) * per_col <= target && cw * 2 <= 2048) cw *= 2;
    if (mode_z(MODE)) {
      // Z modes: a z buffer holds L * cw normals (kZTileRing / kZTileMean)
      const int zt = NT == kRingThreads ? kZTileRing : kZTileMean;
      cw = VEC;
      while (a.L * cw * 2 <= zt && cw * 2 <= 2048) cw *= 2;
    }
    const long long want_tiles = 4LL * sm_count(-1);
    while (cw > VEC && (a.d + cw - 1) / cw < want_tiles && cw * esz > 256) cw /= 2;
    if (const char* env = getenv("RINGMIX_TILE_COLS")) {  // tuning override
      int v = atoi(env);
      if (v >= VEC && (v & (v - 1)) == 0) cw = v;
    }
  }
  if (use_tma) {
    const size_t cap = NT == kRingThreads ? (size_t)max_optin : (size_t)(max_optin / 2 - 1024);
    for (;;) {
      if (mode_z(MODE)) {
        a.zdcols = 2 * (cw >> kZGroupLog2 > 1 ? cw >> kZGroupLog2 : 1);
        a.zslots = a.L * cw;   // one [L][cw] tile of normals per z buffer
      }
      if (tma_smem_bytes(a.L, cw, esz, stage_g, MODE, NT, a.zdcols, a.zslots, HAS_G) <= cap)
        break;
      // Z modes with Phi staged separately: narrower tiles until the stages fit
      if (!mode_z(MODE) || cw <= VEC) {
        use_tma = false;
        break;
      }
      cw /= 2;
    }
  }
  if (!use_tma) return launch_scalar<T, MODE, HAS_G>(a, 0, st);
  int nv = cw / VEC, lg = 0;
  while ((1 << lg) < nv) lg++;

  // mean and Z modes read a thread's column means / lam / w* once per tile (see the kernel)
  if (MODE != kRing && (1 << lg) > NT) return launch_scalar<T, MODE, HAS_G>(a, 0, st);
  a.cw = cw;
  a.d_main = a.d;
  a.log2_nv = lg;
  a.ntiles = (a.d + cw - 1) / cw;
  const int box_c = cw < kBox ? cw : kBox;
  const int box_r = a.L < kBox ? a.L : kBox;
  CUtensorMap tmW, tmG;
  if (!make_map<T>(&tmW, a.W, a.d, a.L, a.ldw, box_c, box_r)) {
    set_error("cuTensorMapEncodeTiled failed for W");
    return RM_EINVAL;
  }
  if (stage_g) {
    if (!make_map<T>(&tmG, a.G, a.d, a.L, a.ldg, box_c, box_r)) {
      set_error("cuTensorMapEncodeTiled failed for G");
      return RM_EINVAL;
    }
  } else {
    tmG = tmW;
  }
  CUtensorMap tmD = tmW, tmLam = tmW, tmOpt = tmW;
  if (RM_TMA_STORE && MODE == kRing && HAS_G &&
      !make_map<T>(&tmD, a.out, a.d, a.L, a.ldo, box_c, box_r)) {
    set_error("cuTensorMapEncodeTiled failed for W'");
    return RM_EINVAL;
  }
  if (mode_z(MODE)) {
    // normal descriptors as a [L][2 * ngroups] uint64 matrix, box [L][zdcols]; lam and
    // w* as one-row fp64 matrices (zero fill past d), boxes of box_c columns
    const long long ld1 = (a.d + 1) & ~1LL;
    if (!tma_map_2d<uint64_t>(&tmD, a.z.desc, 2 * a.z.ngroups, a.L, 2 * a.z.ngroups, a.zdcols,
                              box_r) ||
        !tma_map_2d<double>(&tmLam, a.z.lam, a.d, 1, ld1, box_c, 1) ||
        !tma_map_2d<double>(&tmOpt, a.z.wopt, a.d, 1, ld1, box_c, 1)) {
      set_error("cuTensorMapEncodeTiled failed for the fused gradient's tables");
      return RM_EINVAL;
    }
  }
  size_t smem = tma_smem_bytes(a.L, cw, esz, stage_g, MODE, NT, a.zdcols, a.zslots, HAS_G);
  static unsigned long long attr_set_mask = 0;
  if (attr_needed(&attr_set_mask)) {
    cudaError_t e = cudaFuncSetAttribute(mix_tma_kernel<T, MODE, HAS_G, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(mix_tma_kernel)");
    attr_done(&attr_set_mask);
  }
  long long grid = (long long)sm_count(-1) * (512 / NT);
  if (grid > a.ntiles) grid = a.ntiles;
  cudaError_t e = launch_pdl(mix_tma_kernel<T, MODE, HAS_G, NT>, dim3((unsigned)grid), dim3(NT),
                             smem, st, a, tmW, tmG, tmD, tmLam, tmOpt);
  if (e != cudaSuccess) return fail_cuda(e, "mix_tma_kernel");
  return RM_OK;
}

template <typename T, int MODE>
static int dispatch(const void* W, const void* G, void* out, int L, long long d, long long ldw,
                    long long ldg, long long ldo, const int32_t* left, const int32_t* right,
                    double lr, unsigned long long* absmax, unsigned int* mismatch, void* stream,
                    const ZSrc* z = nullptr) {
  // d == 0 (empty parameter vectors) is valid and may come with null buffers
  if (L < 1 || d < 0 || (d > 0 && (W == nullptr || out == nullptr))) {
    set_error("invalid arguments: L=%d d=%lld", L, d);
    return RM_EINVAL;
  }
  if (ldw < d || ldo < d || (G != nullptr && ldg < d)) {
    set_error("leading dimension smaller than d");
    return RM_EINVAL;
  }
  if (mode_ring(MODE) && L == 3) {
    // mixing.py:122-124: every entry of the 3-ring equals 1/L, so the
    // reference takes the exact column-mean path.
    return dispatch<T, MODE == kRing ? kMean : kMeanZ>(W, G, out, L, d, ldw, ldg, ldo, nullptr,
                                                       nullptr, lr, absmax, nullptr, stream, z);
  }
  if (mode_ring(MODE)) {
    if (L < 3) {
      set_error("degenerate ring topology: need at least 3 learners, got %d", L);
      return RM_EINVAL;
    }
    if (left == nullptr || right == nullptr) {
      set_error("ring mix needs left/right neighbour tables");
      return RM_EINVAL;
    }
  }
  if (d == 0) return RM_OK;
  if (MODE == kSpsgd && G == nullptr) {
    set_error("spsgd needs gradients");
    return RM_EINVAL;
  }
  if (mode_z(MODE) && z == nullptr) {
    set_error("fused gradient step needs the generator's normals");
    return RM_EINVAL;
  }
  if (W == out) {
    set_error("in-place mixing is a read-after-write hazard across learners; use distinct buffers");
    return RM_EINVAL;
  }
  MixArgs a{};
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
  a.mismatch = mismatch;
  if (z) a.z = *z;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // ring tiles: one 512-thread CTA per SM by default; RINGMIX_RING_NT=256 runs
  // two 256-thread CTAs per SM (tuning experiments)
  // Measured on B200 (tools/sweep_ring.py): few learners (L <= 32) stream
  // better with two 256-thread CTAs per SM and 24 KB stages (16 x 16.8 M fp32:
  // 6.54 vs 5.87 TB/s); L = 64 / 128 prefer one 512-thread CTA with 64 KB stages.
  static int ring_nt_env = -1;
  if (ring_nt_env < 0) {
    const char* env = getenv("RINGMIX_RING_NT");
    ring_nt_env = env ? atoi(env) : 0;
  }
  const int ring_nt = ring_nt_env == 256 || ring_nt_env == 512 ? ring_nt_env
                                                               : (L <= 32 ? 256 : 512);
  const bool hg = MODE == kSpsgd || G != nullptr;
  if (!mode_ring(MODE))
    return hg ? launch_mix<T, MODE, true, kMeanThreads>(a, st)
              : launch_mix<T, MODE, false, kMeanThreads>(a, st);
  if (ring_nt == 256)
    return hg ? launch_mix<T, MODE, true, 256>(a, st) : launch_mix<T, MODE, false, 256>(a, st);
  return hg ? launch_mix<T, MODE, true, kRingThreads>(a, st)
            : launch_mix<T, MODE, false, kRingThreads>(a, st);
}

}  // namespace rm

using namespace rm;

#define RM_DEFINE_MIX(SUFFIX, CT, T)                                                              \
  extern "C" int rm_ring_mix_sgd_##SUFFIX(const CT* W, const CT* G, CT* Wout,                   \
                                          const int32_t* left, const int32_t* right, int L,      \
                                          int64_t d, int64_t ldw, int64_t ldg, int64_t ldo,      \
                                          double lr, unsigned long long* absmax_bits,            \
                                          void* stream) {                                        \
    return dispatch<T, kRing>(W, G, Wout, L, d, ldw, ldg, ldo, left, right, lr, absmax_bits,     \
                              nullptr, stream);                                                  \
  }                                                                                              \
  extern "C" int rm_mean_sgd_##SUFFIX(const CT* W, const CT* G, CT* Wout, int L, int64_t d,     \
                                      int64_t ldw, int64_t ldg, int64_t ldo, double lr,          \
                                      unsigned long long* absmax_bits, void* stream) {           \
    return dispatch<T, kMean>(W, G, Wout, L, d, ldw, ldg, ldo, nullptr, nullptr, lr,             \
                              absmax_bits, nullptr, stream);                                     \
  }                                                                                              \
  extern "C" int rm_spsgd_##SUFFIX(const CT* W, const CT* G, CT* Wout, int L, int64_t d,        \
                                   int64_t ldw, int64_t ldg, int64_t ldo, double lr,             \
                                   unsigned int* mismatch, unsigned long long* absmax_bits,      \
                                   void* stream) {                                               \
    return dispatch<T, kSpsgd>(W, G, Wout, L, d, ldw, ldg, ldo, nullptr, nullptr, lr,            \
                               absmax_bits, mismatch, stream);                                   \
  }

RM_DEFINE_MIX(f32, float, float)
RM_DEFINE_MIX(f64, double, double)
RM_DEFINE_MIX(bf16, uint16_t, __nv_bfloat16)

// ----------------------------------------------------------------------------
// Batched ring products for monte_carlo_consensus (spectral.py:273-279):
// product @ T_k for B independent trials, each with its own neighbour tables.
// Uses `@` semantics (dgemm FMA chain, no uniform shortcut even at L == 3).
// ----------------------------------------------------------------------------
namespace rm {
__global__ void __launch_bounds__(256)
    ring_batched_kernel(const double* __restrict__ X, double* __restrict__ Y,
                        const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                        int B, int L, long long d, long long ld, long long bstride) {
  const long long total = (long long)B * L * d;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long c = idx % d;
    const long long bj = idx / d;
    const int j = (int)(bj % L);
    const int b = (int)(bj / L);
    int x0 = left[(long long)b * L + j], x1 = j, x2 = right[(long long)b * L + j], t;
    if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
    if (x2 < x1) { t = x1; x1 = x2; x2 = t; }
    if (x1 < x0) { t = x0; x0 = x1; x1 = t; }
    const double* xb = X + b * bstride;
    Y[b * bstride + j * ld + c] = ring3<double>(xb[x0 * ld + c], xb[x1 * ld + c], xb[x2 * ld + c]);
  }
}
}  // namespace rm

extern "C" int rm_ring_mix_batched_f64(const double* X, double* Y, const int32_t* left,
                                       const int32_t* right, int B, int L, int64_t d, int64_t ld,
                                       int64_t batch_stride, void* stream) {
  if (B < 0 || L < 3 || d < 0 || ld < d || X == nullptr || Y == nullptr || X == Y ||
      left == nullptr || right == nullptr || batch_stride < (int64_t)L * ld) {
    rm::set_error("invalid batched ring mix arguments (B=%d L=%d d=%lld)", B, L, (long long)d);
    return RM_EINVAL;
  }
  long long total = (long long)B * L * d;
  if (total == 0) return 0;
  long long blocks = (total + 255) / 256;
  if (blocks > 8LL * rm::sm_count(-1)) blocks = 8LL * rm::sm_count(-1);
  rm::ring_batched_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      X, Y, left, right, B, L, d, ld, batch_stride);
  RM_CHECK_LAUNCH("ring_batched_kernel");
  return 0;
}

// ----------------------------------------------------------------------------
// Training step with the quadratic oracle's gradient fused into the mix (zsrc.cuh):
// the generator runs up to its normals, then one mix pass produces G in its epilogue.
// ----------------------------------------------------------------------------
namespace rm {
template <typename T>
static int quad_mix_step(const uint32_t* prefix, int nprefix, uint64_t k, const T* W,
                         const T* Phi, T* out, const int32_t* left, const int32_t* right, int L,
                         long long d, long long ldw, long long ldp, long long ldo,
                         const double* lam, const double* wopt, double sd, double lr,
                         unsigned long long* absmax, void* ws, long long ws_bytes, void* stream) {
  if (L < 1 || d < 0 || (d > 0 && (W == nullptr || out == nullptr || lam == nullptr ||
                                   wopt == nullptr))) {
    set_error("invalid fused step arguments: L=%d d=%lld", L, d);
    return RM_EINVAL;
  }
  const bool uniform = left == nullptr && right == nullptr;
  if (!uniform && (left == nullptr || right == nullptr)) {
    set_error("ring mix needs left/right neighbour tables");
    return RM_EINVAL;
  }
  if (!uniform && L < 3) {
    set_error("degenerate ring topology: need at least 3 learners, got %d", L);
    return RM_EINVAL;
  }
  if (Phi == W && ldp == ldw) Phi = nullptr;
  if (Phi != nullptr && ldp < d) {
    set_error("leading dimension smaller than d");
    return RM_EINVAL;
  }
  if (d == 0) return RM_OK;
  if (W == out || Phi == out) {
    set_error("in-place mixing is a read-after-write hazard across learners; use distinct buffers");
    return RM_EINVAL;
  }
  // Two fused kernels compute the same bits: "tile" produces the gradient in
  // mix_tma_kernel's epilogue (kRingZ / kMeanZ); "copy" folds the mix into the generator's
  // output pass (zig_mix_kernel, one warp per raw block, neighbour rows from L2).
  // Measured at C2: tile for ring steps (15.7 vs 16.7 ms), copy for the
  // uniform matrix (17.2 vs 18.2 ms); RINGMIX_FUSED_KERNEL=tile|copy overrides.
  const char* kind = getenv("RINGMIX_FUSED_KERNEL");
  const bool copy_side = kind && kind[0] ? kind[0] == 'c' : (uniform || L == 3);
  if (copy_side) {
    // mixing.py:122-124: the 3-ring is the uniform matrix
    const bool uni = uniform || L == 3;
    return quad_mix_copy<T>(prefix, nprefix, k, W, Phi, out, uni ? nullptr : left,
                            uni ? nullptr : right, L, d, ldw, ldp, ldo, lam, wopt, sd, lr,
                            absmax, ws, ws_bytes, stream);
  }
  ZSrc z{};
  int rc = quad_z_prepare(prefix, nprefix, k, L, d, ws, ws_bytes, stream, &z);
  if (rc) return rc;
  z.lam = lam;
  z.wopt = wopt;
  z.sd = sd;
  if (uniform)
    return dispatch<T, kMeanZ>(W, Phi, out, L, d, ldw, ldp, ldo, nullptr, nullptr, lr, absmax,
                               nullptr, stream, &z);
  return dispatch<T, kRingZ>(W, Phi, out, L, d, ldw, ldp, ldo, left, right, lr, absmax, nullptr,
                             stream, &z);
}
}  // namespace rm

extern "C" int64_t rm_quadratic_mix_workspace_bytes(int L, int64_t d) {
  if (L < 1 || d < 0) return -1;
  return (int64_t)rm::quad_z_workspace_bytes(L, d);
}

#define RM_DEFINE_QMIX(SUFFIX, CT, T)                                                             \
  extern "C" int rm_quadratic_mix_step_##SUFFIX(                                                 \
      const uint32_t* prefix_words, int n_prefix, uint64_t k, const CT* W, const CT* Phi,       \
      CT* Wout, const int32_t* left, const int32_t* right, int L, int64_t d, int64_t ldw,        \
      int64_t ldp, int64_t ldo, const double* lam, const double* wopt, double noise_sd,         \
      double lr, unsigned long long* absmax_bits, void* workspace, int64_t workspace_bytes,     \
      void* stream) {                                                                            \
    return rm::quad_mix_step<T>(prefix_words, n_prefix, k, W, Phi, Wout, left, right, L, d, ldw, \
                                ldp, ldo, lam, wopt, noise_sd, lr, absmax_bits, workspace,       \
                                workspace_bytes, stream);                                        \
  }
RM_DEFINE_QMIX(f32, float, float)
RM_DEFINE_QMIX(f64, double, double)
