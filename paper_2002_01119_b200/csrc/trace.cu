// Fused trace reductions for run_training's _record:
//   cons_sq[l]  = sum_c (W[l,c] - mean_c)^2        consensus_distance (simulation.py:359-362)
//   loss_col[l] = 0.5 * sum_c lam_c (W[l,c] - w*_c)^2   QuadraticObjective.loss_columns
//                                                     (objectives.py:77-79)
//   avg_loss    = 0.5 * sum_c lam_c (mean_c - w*_c)^2   loss(W.mean(axis=1)) (simulation.py:401)
// in ONE pass over W (the reference makes three full passes plus temporaries).
// mean_c uses numpy's pairwise order over the learners; the sums over columns
// are parallel fp64 reductions (the reference sums sequentially), so they agree
// to fp64 rounding, not bitwise.
#include "common.cuh"
#include "tma_host.cuh"
#include "arith.cuh"
#include "../../include/ringmix_b200.h"

namespace rm {

constexpr int kTrThreads = 256;  // = columns per tile
constexpr int kTrMaxL = 128;     // the one-barrier TMA kernel
constexpr int kTrMaxLAny = 4096; // the API (generic kernel: per-warp learner sums in smem)
constexpr int kTrWarps = kTrThreads / 32;

// numpy's pairwise sum of column c over the L learners (n < 8: in order; 8..128:
// eight interleaved partial sums, combined in numpy's order, then the tail).
template <typename T>
__device__ __forceinline__ double column_pairwise(const T* p, int L, long long ld) {
  using E = Elem<T>;
  if (L < 8) {
    double res = -0.0;
    for (int i = 0; i < L; i++) res = __dadd_rn(res, (double)E::ld(p + (long long)i * ld, 0));
    return res;
  }
  if (L > 128) {   // numpy's recursion
    auto get = [&](int i) { return (double)E::ld(p + (long long)i * ld, 0); };
    return pairwise_sum<double>(get, 0, L);
  }
  const int n8 = L - (L % 8);
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; k++) r[k] = (double)E::ld(p + (long long)k * ld, 0);
  for (int i = 8; i < n8; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], (double)E::ld(p + (long long)(i + k) * ld, 0));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int i = n8; i < L; i++) res = __dadd_rn(res, (double)E::ld(p + (long long)i * ld, 0));
  return res;
}

// Per tile of 256 columns: (A) one thread per column computes the column mean
// (coalesced row reads) and the average-model loss term; (B) warp w walks
// learners w, w+8, ... over the tile (rows are L2-resident from phase A) and
// accumulates that learner's consensus and loss sums in registers.  One pass
// over W from HBM; per-learner totals leave with one atomicAdd per CTA.
template <typename T>
__global__ void __launch_bounds__(kTrThreads, 4)
    trace_stats_kernel(const T* __restrict__ W, int L, long long d, long long ld,
                       const double* __restrict__ lam, const double* __restrict__ wopt,
                       double* __restrict__ part) {
  using E = Elem<T>;
  __shared__ double s_mean[kTrThreads];
  __shared__ double s_lm[kTrThreads];
  __shared__ double s_wo[kTrThreads];
  __shared__ double s_red[kTrWarps];
  // warp-private per-learner sums [kTrWarps][per][2] (dynamic: per = ceil(L / 8))
  extern __shared__ double s_dyn[];
  const int per = (L + kTrWarps - 1) / kTrWarps;
  double* s_acc = s_dyn;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool has_obj = lam != nullptr;
  for (int i = lane; i < per; i += 32)
    s_acc[(warp * per + i) * 2] = s_acc[(warp * per + i) * 2 + 1] = 0.0;
  __syncwarp();
  double a_sum = 0.0;
  for (long long c0 = blockIdx.x * (long long)kTrThreads; c0 < d;
       c0 += (long long)gridDim.x * kTrThreads) {
    const long long c = c0 + tid;
    if (c < d) {
      const double mean = __ddiv_rn(column_pairwise<T>(W + c, L, ld), (double)L);
      s_mean[tid] = mean;
      if (has_obj) {
        const double lm = lam[c], wo = wopt[c];
        s_lm[tid] = lm;
        s_wo[tid] = wo;
        const double dm = __dsub_rn(mean, wo);
        a_sum += 0.5 * lm * dm * dm;
      }
    }
    __syncthreads();
    const int width = (int)min((long long)kTrThreads, d - c0);
    for (int j = 0; j < per; j++) {
      const int l = warp + kTrWarps * j;
      if (l >= L) break;
      const T* row = W + (long long)l * ld + c0;
      double v = 0.0, q = 0.0;
      for (int i = lane; i < width; i += 32) {
        const double w = (double)E::ld(row + i, 0);
        const double dv = w - s_mean[i];
        v += dv * dv;
        if (has_obj) {
          const double dw = w - s_wo[i];
          q += s_lm[i] * dw * dw;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
      }
      if (lane == 0) {
        s_acc[(warp * per + j) * 2] += v;
        s_acc[(warp * per + j) * 2 + 1] += q;
      }
    }
    __syncthreads();
  }
  // this CTA's partials, in a fixed order (trace_finalize_kernel sums the CTAs
  // in index order: the result does not depend on scheduling)
  __syncwarp();
  double* out = part + (long long)blockIdx.x * (2 * L + 1);
  for (int i = lane; i < per; i += 32) {
    const int l = warp + kTrWarps * i;
    if (l < L) {
      out[l] = s_acc[(warp * per + i) * 2];
      out[L + l] = has_obj ? 0.5 * s_acc[(warp * per + i) * 2 + 1] : 0.0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) a_sum += __shfl_xor_sync(0xffffffffu, a_sum, o);
  if (lane == 0) s_red[warp] = a_sum;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kTrWarps; w++) t += s_red[w];
    out[2 * L] = has_obj ? t : 0.0;
  }
}

// out[o] += sum over CTAs b (in index order) of part[b][o]
__global__ void trace_finalize_kernel(const double* __restrict__ part, int nparts, int L,
                                      double* __restrict__ cons_sq, double* __restrict__ loss_col,
                                      double* __restrict__ avg_loss) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 2 * L + 1;
  if (o >= n) return;
  double t = 0.0;
  for (int b = 0; b < nparts; b++) t += part[(long long)b * n + o];
  if (o < L) cons_sq[o] += t;
  else if (o < 2 * L) { if (loss_col) loss_col[o - L] += t; }
  else if (avg_loss) *avg_loss += t;
}

// TMA-staged variant (16-byte aligned rows, L <= 128): tiles [L x cw] of W
// arrive in a 3-stage shared-memory ring (one 2-D tensor-map load per tile);
// phase A computes the tile's column means from shared memory, phase B has every
// thread fold its fixed set of (row, 16-byte vector) items into per-row
// register accumulators.  W crosses HBM exactly once, with no L2 re-reads.
constexpr int kTrStages = 3;
constexpr int kTrStageTarget = 32 * 1024;  // two 256-thread CTAs per SM
constexpr int kTrItems = 8;                // (row, vector) items per thread per tile

template <typename T>
__global__ void __launch_bounds__(kTrThreads, 2)
    trace_stats_tma_kernel(const __grid_constant__ CUtensorMap tmW, int L, long long d, int cw,
                           int lg_nv, long long ntiles, const double* __restrict__ lam,
                           const double* __restrict__ wopt, double* __restrict__ part) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  // column means / lam / w* of a tile, double-buffered: phase A of tile t+1 runs in
  // the same barrier interval as phase B of tile t (one __syncthreads per tile)
  double* s_cols = reinterpret_cast<double*>(smem + 128);  // [2][3][cw]
  double* s_rows = s_cols + 6 * cw;                           // [2][L] block totals
  unsigned char* stages =
      reinterpret_cast<unsigned char*>(s_rows + 2 * kTrMaxL) +
      ((128 - (((uintptr_t)(s_rows + 2 * kTrMaxL)) & 127)) & 127);
  const int tid = threadIdx.x;
  const int stage_bytes = L * cw * (int)sizeof(T);
  const bool has_obj = lam != nullptr;
  const int box_c = cw < 256 ? cw : 256;
  const int lg_bc = __ffs(box_c) - 1;
  const int box_stride = L << lg_bc;
  auto sidx = [&](int r, int c) -> int {
    return (c >> lg_bc) * box_stride + (r << lg_bc) + (c & (box_c - 1));
  };
  if (tid == 0) {
    tma_prefetch_desc(&tmW);
    for (int st = 0; st < kTrStages; st++) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 2 * kTrMaxL; i += kTrThreads) s_rows[i] = 0.0;
  __syncthreads();
  auto issue = [&](int st, long long t) {
    mbar_arrive_expect_tx(&full[st], (uint32_t)stage_bytes);
    T* dst = reinterpret_cast<T*>(stages + (size_t)st * stage_bytes);
    for (int cc = 0; cc < cw; cc += box_c)
      tma_load_2d(dst + sidx(0, cc), &tmW, (int)(t * cw + cc), 0, &full[st]);
  };
  const long long first = blockIdx.x, stride = gridDim.x;
  if (tid == 0)
    for (int st = 0; st < kTrStages; st++)
      if (first + st * stride < ntiles) issue(st, first + st * stride);

  // this thread's items: rows (tid >> lg_nv) + k * (kTrThreads >> lg_nv), vector v
  const int nv_full = 1 << lg_nv;
  const int v = tid & (nv_full - 1);
  const int row0 = tid >> lg_nv, row_step = kTrThreads >> lg_nv;
  double acc_c[kTrItems], acc_l[kTrItems];
#pragma unroll
  for (int k = 0; k < kTrItems; k++) acc_c[k] = acc_l[k] = 0.0;
  double a_sum = 0.0;

  // phase A of the tile in local slot `it`: wait for its stage, column means
  // (numpy pairwise order) and the average-model loss into buffer it & 1
  // Phase A split over every warp: lane l < 16 of a warp sums numpy's chains 0-3 of
  // column col, lane l + 16 chains 4-7 of the same column; the halves meet with one
  // shuffle in numpy's order ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)).  (One thread per
  // column left half the warps idle in this phase while the others did both phases:
  // ncu showed barrier stalls first, profiles/r2_trace_c2_onebarrier_ncu.json.)
  const int a_lane = tid & 15, a_half = (tid >> 4) & 1, a_warp = tid >> 5;
  auto phase_a = [&](long long t, int it) {
    const int st = it % kTrStages;
    const long long c0 = t * cw;
    const int width = (int)min((long long)cw, d - c0);
    const T* sW = reinterpret_cast<const T*>(stages + (size_t)st * stage_bytes);
    double* cm = s_cols + (it & 1) * 3 * cw;
    mbar_wait(&full[st], (it / kTrStages) & 1);
    for (int cb = a_warp * 16; cb < width; cb += kTrThreads / 2) {
      const int col = cb + a_lane;
      const bool live = col < width;
      double lm = 0.0, wo = 0.0;
      if (has_obj && live && a_half == 0) {   // issued first: latency under the sums
        lm = lam[c0 + col];
        wo = wopt[c0 + col];
      }
      double res;
      if (L < 8) {
        res = -0.0;
        if (a_half == 0 && live)
          for (int i = 0; i < L; i++) res = __dadd_rn(res, (double)E::lds(sW + sidx(i, col)));
      } else {
        const int n8 = L - (L % 8);
        const int k0 = a_half * 4;
        const int cc = live ? col : 0;
        double r0 = (double)E::lds(sW + sidx(k0, cc)), r1 = (double)E::lds(sW + sidx(k0 + 1, cc));
        double r2 = (double)E::lds(sW + sidx(k0 + 2, cc)), r3 = (double)E::lds(sW + sidx(k0 + 3, cc));
        for (int i = 8; i < n8; i += 8) {
          r0 = __dadd_rn(r0, (double)E::lds(sW + sidx(i + k0, cc)));
          r1 = __dadd_rn(r1, (double)E::lds(sW + sidx(i + k0 + 1, cc)));
          r2 = __dadd_rn(r2, (double)E::lds(sW + sidx(i + k0 + 2, cc)));
          r3 = __dadd_rn(r3, (double)E::lds(sW + sidx(i + k0 + 3, cc)));
        }
        const double h = __dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3));
        const double other = __shfl_xor_sync(0xffffffffu, h, 16);
        res = __dadd_rn(h, other);                 // lane < 16: X + Y in numpy's order
        if (a_half == 0 && live)
          for (int i = n8; i < L; i++) res = __dadd_rn(res, (double)E::lds(sW + sidx(i, col)));
      }
      if (a_half == 0 && live) {
        const double mean = __ddiv_rn(res, (double)L);
        cm[col] = mean;
        if (has_obj) {
          cm[cw + col] = lm;
          cm[2 * cw + col] = wo;
          const double dm = __dsub_rn(mean, wo);
          a_sum += 0.5 * lm * dm * dm;
        }
      }
    }
  };
  // phase B of the tile in slot `it`: this thread's rows over its vector of columns
  auto phase_b = [&](long long t, int it) {
    const int st = it % kTrStages;
    const int width = (int)min((long long)cw, d - t * cw);
    const T* sW = reinterpret_cast<const T*>(stages + (size_t)st * stage_bytes);
    const double* cm = s_cols + (it & 1) * 3 * cw;
    const int c = v * VEC;
    if (c >= width) return;
    // 16-byte shared loads: a thread owns VEC consecutive columns (scalar loads
    // would be 2*VEC-way bank conflicts); entries past `width` are never used
    double m[VEC], lm[VEC], wo[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      const double2 a2 = *reinterpret_cast<const double2*>(cm + c + e);
      m[e] = a2.x;
      m[e + 1] = a2.y;
      if (has_obj) {
        const double2 l2 = *reinterpret_cast<const double2*>(cm + cw + c + e);
        const double2 w2 = *reinterpret_cast<const double2*>(cm + 2 * cw + c + e);
        lm[e] = l2.x;
        lm[e + 1] = l2.y;
        wo[e] = w2.x;
        wo[e + 1] = w2.y;
      } else {
        lm[e] = lm[e + 1] = wo[e] = wo[e + 1] = 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kTrItems; k++) {
      const int j = row0 + k * row_step;
      if (j < L) {
        Vec<T> x;
        x.raw = *reinterpret_cast<const uint4*>(sW + sidx(j, c));
        double vv = 0.0, qq = 0.0;
#pragma unroll
        for (int e = 0; e < VEC; e++) {
          if (c + e < width) {
            const double w = (double)E::ld(x.e(), e);
            const double dv = w - m[e];
            vv += dv * dv;
            const double dw = w - wo[e];
            qq += lm[e] * dw * dw;
          }
        }
        acc_c[k] += vv;
        acc_l[k] += qq;
      }
    }
  };

  if (first < ntiles) phase_a(first, 0);
  __syncthreads();
  int it = 0;
  for (long long t = first; t < ntiles; t += stride, ++it) {
    if (t + stride < ntiles) phase_a(t + stride, it + 1);
    phase_b(t, it);
    __syncthreads();  // tile t's stage and mean buffer are free, tile t+1's means ready
    if (tid == 0) {
      const long long tn = t + (long long)kTrStages * stride;
      if (tn < ntiles) issue(it % kTrStages, tn);
    }
  }
  // deterministic in-CTA reduction: the (drained) stage buffers hold every
  // thread's accumulators; thread j sums the owners of learner j in thread order
  __syncthreads();
  double* s_acc = reinterpret_cast<double*>(stages);  // [kTrThreads][kTrItems][2]
#pragma unroll
  for (int k = 0; k < kTrItems; k++) {
    s_acc[(tid * kTrItems + k) * 2] = acc_c[k];
    s_acc[(tid * kTrItems + k) * 2 + 1] = acc_l[k];
  }
  for (int o = 16; o > 0; o >>= 1) a_sum += __shfl_xor_sync(0xffffffffu, a_sum, o);
  if ((tid & 31) == 0) s_rows[tid >> 5] = a_sum;
  __syncthreads();
  double* out = part + (long long)blockIdx.x * (2 * L + 1);
  for (int j = tid; j < L; j += kTrThreads) {
    const int k = j / row_step, r = j % row_step;
    double c = 0.0, q = 0.0;
    for (int vv = 0; vv < nv_full; vv++) {
      const int owner = (r << lg_nv) | vv;
      c += s_acc[(owner * kTrItems + k) * 2];
      q += s_acc[(owner * kTrItems + k) * 2 + 1];
    }
    out[j] = c;
    out[L + j] = has_obj ? 0.5 * q : 0.0;
  }
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kTrThreads / 32; w++) t += s_rows[w];
    out[2 * L] = has_obj ? t : 0.0;
  }
}

// Compile-time-shaped variant for L in {8, 16, 32, 64, 128} (the configs' learner
// counts): the tile [L x CW] is one TMA box, every shared-memory offset is an immediate,
// full tiles run without column checks, and phase B's items are independent
// accumulator chains the compiler can interleave (the runtime-L kernel above keeps a
// branch per item, which serialised them: ncu showed fixed-latency `wait` stalls first).
// Phase A: TPC = 256 / CW threads per column, each summing CPT = 8 / TPC of numpy's eight
// interleaved chains; the chains' tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) is finished
// inside the thread and then across the column's threads with xor shuffles (IEEE addition
// commutes, so only the tree matters).  L is a power of two: sum / L == sum * (1 / L).
template <typename T, int L>
struct TrShape {
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int CW0 = kTrStageTarget / (L * (int)sizeof(T));
  static constexpr int CW = CW0 > 256 ? 256 : CW0;
  static constexpr int NV = CW / VEC;
  static constexpr int ITEMS = L * NV / kTrThreads;
  static constexpr int ROW_STEP = kTrThreads / NV;
  static constexpr int TPC = kTrThreads / CW;
  static constexpr int CPT = 8 / TPC;
  static constexpr int NCW = 32 / TPC;
  static constexpr int STAGE = L * CW * (int)sizeof(T);
  static_assert(L % 8 == 0 && L <= 128, "numpy's 8-chain form");
  static_assert(TPC >= 1 && TPC <= 8 && ITEMS >= 1 && L * NV == ITEMS * kTrThreads, "shape");
};

template <typename T, int L>
__global__ void __launch_bounds__(kTrThreads, 2)
    trace_tile_kernel(const __grid_constant__ CUtensorMap tmW, long long d, long long ntiles,
                      const double* __restrict__ lam, const double* __restrict__ wopt,
                      double* __restrict__ part) {
  using E = Elem<T>;
  using S = TrShape<T, L>;
  constexpr int VEC = S::VEC, CW = S::CW, NV = S::NV, ITEMS = S::ITEMS;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  double* s_cols = reinterpret_cast<double*>(smem + 128);  // [2][3][CW]
  double* s_red = s_cols + 6 * CW;                            // [kTrWarps]
  unsigned char* stages = smem + 128 + ((6 * CW + kTrWarps) * 8 + 127) / 128 * 128;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool has_obj = lam != nullptr;
  if (tid == 0) {
    tma_prefetch_desc(&tmW);
    for (int st = 0; st < kTrStages; st++) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int st, long long t) {
    mbar_arrive_expect_tx(&full[st], (uint32_t)S::STAGE);
    tma_load_2d(stages + (size_t)st * S::STAGE, &tmW, (int)(t * CW), 0, &full[st]);
  };
  const long long first = blockIdx.x, stride = gridDim.x;
  if (tid == 0)
    for (int st = 0; st < kTrStages; st++)
      if (first + st * stride < ntiles) issue(st, first + st * stride);

  // phase A lanes: column a_col of the tile, chains [a_part * CPT, (a_part + 1) * CPT)
  const int a_col = warp * S::NCW + (lane % S::NCW);
  const int a_part = lane / S::NCW;
  // phase B items: vector b_v of rows b_row0 + k * ROW_STEP
  const int b_v = tid % NV, b_row0 = tid / NV;
  double acc_c[ITEMS], acc_l[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; k++) acc_c[k] = acc_l[k] = 0.0;
  double a_sum = 0.0;

  auto phase_a = [&](long long t, int it) {
    const int st = it % kTrStages;
    const long long c0 = t * CW;
    const T* sW = reinterpret_cast<const T*>(stages + (size_t)st * S::STAGE);
    double* cm = s_cols + (it & 1) * 3 * CW;
    const bool live = c0 + a_col < d;
    double lm = 0.0, wo = 0.0;
    if (has_obj && live && a_part == 0) {   // issued first: latency under the sums
      lm = lam[c0 + a_col];
      wo = wopt[c0 + a_col];
    }
    mbar_wait(&full[st], (it / kTrStages) & 1);
    // columns past d hold TMA's zero fill: summed harmlessly, never stored
    const T* col = sW + a_col;
    double r[S::CPT];
#pragma unroll
    for (int q = 0; q < S::CPT; q++) r[q] = (double)E::lds(col + (a_part * S::CPT + q) * CW);
#pragma unroll
    for (int i = 8; i < L; i += 8) {
#pragma unroll
      for (int q = 0; q < S::CPT; q++)
        r[q] = __dadd_rn(r[q], (double)E::lds(col + (i + a_part * S::CPT + q) * CW));
    }
#pragma unroll
    for (int w = 1; w < S::CPT; w *= 2) {   // this thread's subtree of the chains
#pragma unroll
      for (int q = 0; q < S::CPT; q += 2 * w) r[q] = __dadd_rn(r[q], r[q + w]);
    }
    double res = r[0];
#pragma unroll
    for (int off = S::NCW; off < 32; off *= 2) res = __dadd_rn(res, __shfl_xor_sync(0xffffffffu, res, off));
    if (a_part == 0 && live) {
      const double mean = __dmul_rn(res, 1.0 / L);
      cm[a_col] = mean;
      if (has_obj) {
        cm[CW + a_col] = lm;
        cm[2 * CW + a_col] = wo;
        const double dm = __dsub_rn(mean, wo);
        a_sum += 0.5 * lm * dm * dm;
      }
    }
  };
  auto phase_b = [&](long long t, int it) {
    const int st = it % kTrStages;
    const long long c0 = t * CW;
    const int width = (int)min((long long)CW, d - c0);
    const T* sW = reinterpret_cast<const T*>(stages + (size_t)st * S::STAGE);
    const double* cm = s_cols + (it & 1) * 3 * CW;
    const int c = b_v * VEC;
    double m[VEC], lm[VEC], wo[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      const double2 a2 = *reinterpret_cast<const double2*>(cm + c + e);
      m[e] = a2.x;
      m[e + 1] = a2.y;
      if (has_obj) {
        const double2 l2 = *reinterpret_cast<const double2*>(cm + CW + c + e);
        const double2 w2 = *reinterpret_cast<const double2*>(cm + 2 * CW + c + e);
        lm[e] = l2.x;
        lm[e + 1] = l2.y;
        wo[e] = w2.x;
        wo[e + 1] = w2.y;
      } else {
        lm[e] = lm[e + 1] = wo[e] = wo[e + 1] = 0.0;
      }
    }
    if (width == CW) {
#pragma unroll
      for (int k = 0; k < ITEMS; k++) {
        Vec<T> x;
        x.raw = *reinterpret_cast<const uint4*>(sW + (b_row0 + k * S::ROW_STEP) * CW + c);
#pragma unroll
        for (int e = 0; e < VEC; e++) {
          const double w = (double)E::ld(x.e(), e);
          const double dv = w - m[e];
          acc_c[k] += dv * dv;
          const double dw = w - wo[e];
          acc_l[k] += lm[e] * dw * dw;
        }
      }
    } else if (c < width) {
#pragma unroll
      for (int k = 0; k < ITEMS; k++) {
        Vec<T> x;
        x.raw = *reinterpret_cast<const uint4*>(sW + (b_row0 + k * S::ROW_STEP) * CW + c);
#pragma unroll
        for (int e = 0; e < VEC; e++) {
          if (c + e < width) {
            const double w = (double)E::ld(x.e(), e);
            const double dv = w - m[e];
            acc_c[k] += dv * dv;
            const double dw = w - wo[e];
            acc_l[k] += lm[e] * dw * dw;
          }
        }
      }
    }
  };

  if (first < ntiles) phase_a(first, 0);
  __syncthreads();
  int it = 0;
  for (long long t = first; t < ntiles; t += stride, ++it) {
    if (t + stride < ntiles) phase_a(t + stride, it + 1);
    phase_b(t, it);
    __syncthreads();  // tile t's stage and mean buffer are free, tile t+1's means ready
    if (tid == 0) {
      const long long tn = t + (long long)kTrStages * stride;
      if (tn < ntiles) issue(it % kTrStages, tn);
    }
  }
  // deterministic in-CTA reduction (as trace_stats_tma_kernel): thread j sums the owners
  // of learner j in thread order
  __syncthreads();
  double* s_acc = reinterpret_cast<double*>(stages);  // [kTrThreads][ITEMS][2]
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    s_acc[(tid * ITEMS + k) * 2] = acc_c[k];
    s_acc[(tid * ITEMS + k) * 2 + 1] = acc_l[k];
  }
  for (int o = 16; o > 0; o >>= 1) a_sum += __shfl_xor_sync(0xffffffffu, a_sum, o);
  if (lane == 0) s_red[warp] = a_sum;
  __syncthreads();
  double* out = part + (long long)blockIdx.x * (2 * L + 1);
  for (int j = tid; j < L; j += kTrThreads) {
    const int k = j / S::ROW_STEP, r0 = j % S::ROW_STEP;
    double cs = 0.0, q = 0.0;
    for (int vv = 0; vv < NV; vv++) {
      const int owner = r0 * NV + vv;
      cs += s_acc[(owner * ITEMS + k) * 2];
      q += s_acc[(owner * ITEMS + k) * 2 + 1];
    }
    out[j] = cs;
    out[L + j] = has_obj ? 0.5 * q : 0.0;
  }
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kTrWarps; w++) t += s_red[w];
    out[2 * L] = has_obj ? t : 0.0;
  }
}

template <typename T, int L>
static int trace_tile_launch(const T* W, int64_t d, int64_t ld, const double* lam,
                             const double* wopt, double* part, int* nparts, cudaStream_t st,
                             bool* covered) {
  using S = TrShape<T, L>;
  CUtensorMap tm;
  if (!tma_map_2d<T>(&tm, W, d, L, ld, S::CW, L)) return 0;
  const size_t smem = 128 + ((6 * S::CW + kTrWarps) * 8 + 127) / 128 * 128 +
                      (size_t)kTrStages * S::STAGE;
  static_assert((size_t)kTrThreads * S::ITEMS * 16 <= (size_t)kTrStages * S::STAGE,
                "accumulators fit in the drained stages");
  static unsigned long long attr_mask = 0;
  if (attr_needed(&attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(trace_tile_kernel<T, L>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(trace_tile_kernel)");
    attr_done(&attr_mask);
  }
  *covered = true;
  const long long ntiles = (d + S::CW - 1) / S::CW;
  long long grid = 2LL * sm_count(-1);
  if (grid > ntiles) grid = ntiles;
  *nparts = (int)grid;
  trace_tile_kernel<T, L><<<(int)grid, kTrThreads, smem, st>>>(tm, d, ntiles, lam, wopt, part);
  RM_CHECK_LAUNCH("trace_tile_kernel");
  return 0;
}

template <typename T>
static int trace_stats_tma(const T* W, int L, int64_t d, int64_t ld, const double* lam,
                           const double* wopt, double* part, int* nparts, cudaStream_t st,
                           bool* covered) {
  using E = Elem<T>;
  if (getenv("RINGMIX_TRACE_RUNTIME_L") == nullptr) {
    switch (L) {
      case 8: return trace_tile_launch<T, 8>(W, d, ld, lam, wopt, part, nparts, st, covered);
      case 16: return trace_tile_launch<T, 16>(W, d, ld, lam, wopt, part, nparts, st, covered);
      case 32: return trace_tile_launch<T, 32>(W, d, ld, lam, wopt, part, nparts, st, covered);
      case 64: return trace_tile_launch<T, 64>(W, d, ld, lam, wopt, part, nparts, st, covered);
      case 128: return trace_tile_launch<T, 128>(W, d, ld, lam, wopt, part, nparts, st, covered);
      default: break;
    }
  }
  constexpr int VEC = E::VEC;
  const size_t esz = sizeof(T);
  // tile width: power of two, stage ~32 KB, exactly kTrItems items per thread
  int cw = VEC;
  while ((size_t)(cw * 2) * L * esz <= (size_t)kTrStageTarget && cw * 2 <= 2048) cw *= 2;
  int nv = cw / VEC, lg = 0;
  while ((1 << lg) < nv) lg++;
  *covered = false;
  if ((long long)L * nv > (long long)kTrItems * kTrThreads || nv > kTrThreads) return 0;
  const int box_c = cw < 256 ? cw : 256;
  CUtensorMap tm;
  if (!tma_map_2d<T>(&tm, W, d, L, ld, box_c, L)) return 0;
  const size_t smem = 128 + 6 * (size_t)cw * 8 + 2 * kTrMaxL * 8 + 128 +
                      (size_t)kTrStages * L * cw * esz;
  static unsigned long long attr_mask = 0;
  if (attr_needed(&attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(trace_stats_tma_kernel<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(trace_stats_tma_kernel)");
    attr_done(&attr_mask);
  }
  if (smem > 110 * 1024) return 0;
  *covered = true;
  const long long ntiles = (d + cw - 1) / cw;
  long long grid = 2LL * sm_count(-1);
  if (grid > ntiles) grid = ntiles;
  *nparts = (int)grid;
  trace_stats_tma_kernel<T><<<(int)grid, kTrThreads, smem, st>>>(tm, L, d, cw, lg, ntiles, lam,
                                                                 wopt, part);
  RM_CHECK_LAUNCH("trace_stats_tma_kernel");
  return 0;
}

// per-CTA partial sums: at most max(8, 2) CTAs per SM x (2L + 1) doubles
static int64_t trace_workspace_bytes(int L) {
  return (int64_t)8 * sm_count(-1) * (2 * (int64_t)L + 1) * (int64_t)sizeof(double);
}

template <typename T>
static int trace_stats(const T* W, int L, int64_t d, int64_t ld, const double* lam,
                       const double* wopt, double* cons_sq, double* loss_col, double* avg_loss,
                       void* workspace, int64_t workspace_bytes, void* stream) {
  if (W == nullptr || cons_sq == nullptr || L < 1 || L > kTrMaxLAny || d < 0 || ld < d ||
      (lam != nullptr && (wopt == nullptr || loss_col == nullptr || avg_loss == nullptr))) {
    set_error("invalid trace-stat arguments (L=%d, at most %d)", L, kTrMaxLAny);
    return RM_EINVAL;
  }
  if (workspace == nullptr || workspace_bytes < trace_workspace_bytes(L)) {
    set_error("trace-stat workspace too small (need %lld bytes)",
              (long long)trace_workspace_bytes(L));
    return RM_EINVAL;
  }
  if (d == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(workspace);
  int nparts = 0;
  constexpr int VEC = Elem<T>::VEC;
  const bool aligned = ((reinterpret_cast<uintptr_t>(W) | (uintptr_t)(ld * sizeof(T))) & 15) == 0;
  bool covered = false;
  if (aligned && d >= VEC && d < (1LL << 31) && L <= kTrMaxL && tma_encode_fn() != nullptr &&
      getenv("RINGMIX_TRACE_NO_TMA") == nullptr) {
    const int rc = trace_stats_tma<T>(W, L, d, ld, lam, wopt, part, &nparts, st, &covered);
    if (rc != 0) return rc;
  }
  if (!covered) {
    long long blocks = (d + kTrThreads - 1) / kTrThreads;
    if (blocks > 8LL * sm_count(-1)) blocks = 8LL * sm_count(-1);
    nparts = (int)blocks;
    const size_t dyn = (size_t)kTrWarps * ((L + kTrWarps - 1) / kTrWarps) * 2 * sizeof(double);
    if (dyn > 48 * 1024) {
      static unsigned long long attr_mask = 0;
      if (attr_needed(&attr_mask)) {
        cudaError_t e = cudaFuncSetAttribute(trace_stats_kernel<T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             100 * 1024);
        if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(trace_stats_kernel)");
        attr_done(&attr_mask);
      }
    }
    trace_stats_kernel<T><<<(int)blocks, kTrThreads, dyn, st>>>(W, L, d, ld, lam, wopt, part);
    RM_CHECK_LAUNCH("trace_stats_kernel");
  }
  trace_finalize_kernel<<<(2 * L + 1 + 127) / 128, 128, 0, st>>>(
      part, nparts, L, cons_sq, lam ? loss_col : nullptr, lam ? avg_loss : nullptr);
  RM_CHECK_LAUNCH("trace_finalize_kernel");
  return 0;
}

}  // namespace rm

using namespace rm;

extern "C" int64_t rm_trace_stats_workspace_bytes(int L) {
  if (L < 1 || L > kTrMaxLAny) return -1;
  return trace_workspace_bytes(L);
}

#define RM_DEFINE_TRACE(SUFFIX, CT, T)                                                         \
  extern "C" int rm_trace_stats_##SUFFIX(const CT* W, int L, int64_t d, int64_t ld,           \
                                         const double* lam, const double* wopt,               \
                                         double* cons_sq, double* loss_col, double* avg_loss,  \
                                         void* workspace, int64_t workspace_bytes,             \
                                         void* stream) {                                       \
    return trace_stats<T>(reinterpret_cast<const T*>(W), L, d, ld, lam, wopt, cons_sq,        \
                          loss_col, avg_loss, workspace, workspace_bytes, stream);             \
  }
RM_DEFINE_TRACE(f32, float, float)
RM_DEFINE_TRACE(f64, double, double)
RM_DEFINE_TRACE(bf16, uint16_t, __nv_bfloat16)

// ---- column mean (numpy pairwise order), the D1D average on its own ----
// M[c] = pairwise_sum_l W[l, c] / L, bit-identical to the mean the fused
// D1D tile computes.  Lets the average of W_k run on a side stream while the
// gradient of W_{k-1} is produced (simulation.step_d1d; north-star (c)), after
// which rm_apply_mean_sgd_*(M, G, L = 1) finishes the step.
namespace rm {
int d1d_psum_cap();   // shard.cu: rm_set_d1d_ctas_per_sm's partial-sum cap (0 = default)

template <typename T>
__global__ void __launch_bounds__(256)
    column_mean_kernel(const T* __restrict__ W, int L, long long d, long long ld,
                       double* __restrict__ M) {
  using E = Elem<T>;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d;
       c += (long long)gridDim.x * blockDim.x) {
    const T* p = W + c;
    double res;
    if (L <= kTrMaxL) {
      res = column_pairwise<T>(p, L, ld);
    } else {
      auto get = [&](int i) { return (double)E::ld(p + (long long)i * ld, 0); };
      res = pairwise_sum<double>(get, 0, L);
    }
    M[c] = __ddiv_rn(res, (double)L);
  }
}
}  // namespace rm

#define RM_DEFINE_COLMEAN(SUFFIX, CT, T)                                                      \
  extern "C" int rm_column_mean_##SUFFIX(const CT* W, int L, int64_t d, int64_t ld,          \
                                         double* M, void* stream) {                           \
    if (W == nullptr || M == nullptr || L < 1 || d < 0 || ld < d) {                           \
      set_error("invalid column-mean arguments");                                             \
      return RM_EINVAL;                                                                       \
    }                                                                                         \
    if (d == 0) return 0;                                                                     \
    long long blocks = (d + 255) / 256;                                                       \
    const long long cap = (d1d_psum_cap() ? d1d_psum_cap() : 16) * (long long)sm_count(-1);   \
    if (blocks > cap) blocks = cap;                                                           \
    column_mean_kernel<T><<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(       \
        reinterpret_cast<const T*>(W), L, d, ld, M);                                          \
    RM_CHECK_LAUNCH("column_mean_kernel");                                                    \
    return 0;                                                                                 \
  }
RM_DEFINE_COLMEAN(f32, float, float)
RM_DEFINE_COLMEAN(f64, double, double)
RM_DEFINE_COLMEAN(bf16, uint16_t, __nv_bfloat16)

// ---- exact-order trace reductions: numpy's own summation order, bit for bit ----
// The reference's reductions over the parameters are sequential in c:
//   (dev * dev).sum(axis=0)             -> axis-0 reduce of a C-order (d, L) array: one
//                                          running sum per learner, c = 0, 1, ... (simulation.py:361)
//   einsum("i,il,il->l", lam, dev, dev)  -> the same, of fl(fl(lam_c dev) dev)  (objectives.py:79)
// and the average-model loss np.sum(lam * dev * dev) over a contiguous vector is numpy's
// pairwise sum (objectives.py:72).  A running sum cannot be re-associated without changing
// its rounding, so each learner's chain is one thread walking its row; the pairwise sum is
// parallel over the subtrees of numpy's recursion at a fixed depth (every node above that
// depth has more than 128 values, so it splits exactly as numpy's does) and its top levels
// are combined in tree order.  Cost: d dependent fp64 adds per learner (latency-bound), so
// the host uses it for small d (run_training's records, the sweep) and the one-pass kernel above otherwise.
namespace rm {
constexpr int kExactMaxDepth = 12;   // at most 4096 pairwise subtrees

__host__ __device__ inline int exact_pairwise_depth(long long d) {
  int D = 0;
  while (D < kExactMaxDepth && (d >> (D + 1)) >= 256) D++;
  return D;
}

// One warp per 32 learners; lane l's running sums walk row l.  The row tiles [32 x kExCT]
// (and M, lam, w* of those columns) are staged into shared memory by coalesced cp.async
// copies kExBuf - 1 tiles ahead, so the chains wait on shared-memory latency only (direct
// row loads left every 8-column batch waiting for a global round trip: 7.5 ms at
// 64 x 2^16).  Rows are padded by one element: lane l reading column c of its own row
// hits a different bank than its neighbours.
constexpr int kExCT = 128;
constexpr int kExBuf = 4;

template <typename T>
struct ExTile {
  static constexpr int ROW = kExCT + 1;
  static constexpr size_t W_BYTES = ((size_t)32 * ROW * sizeof(T) + 15) / 16 * 16;
  static constexpr size_t BYTES = W_BYTES + 3 * kExCT * sizeof(double);
};

template <typename T>
__global__ void __launch_bounds__(32)
    trace_exact_rows_kernel(const T* __restrict__ W, int L, long long d, long long ld,
                            const double* __restrict__ M, const double* __restrict__ lam,
                            const double* __restrict__ wopt, double* __restrict__ cons_sq,
                            double* __restrict__ loss_col) {
  using E = Elem<T>;
  using X = ExTile<T>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x;
  const int l0 = blockIdx.x * 32;
  const int nrows = min(32, L - l0);
  const long long ntiles = (d + kExCT - 1) / kExCT;
  const bool has_obj = lam != nullptr;
  auto tile_w = [&](int b) { return reinterpret_cast<T*>(smem + (size_t)b * X::BYTES); };
  auto tile_c = [&](int b) {
    return reinterpret_cast<double*>(smem + (size_t)b * X::BYTES + X::W_BYTES);
  };
  auto issue = [&](long long t) {
    const int b = (int)(t % kExBuf);
    const long long c0 = t * kExCT;
    const int width = (int)min((long long)kExCT, d - c0);
    T* sw = tile_w(b);
    double* sc = tile_c(b);
    for (int r = 0; r < nrows; r++) {
      const T* src = W + (long long)(l0 + r) * ld + c0;
      for (int c = lane; c < width; c += 32) cp_async_elem(sw + r * X::ROW + c, src + c);
    }
    for (int c = lane; c < width; c += 32) {
      cp_async_elem(sc + c, M + c0 + c);
      if (has_obj) {
        cp_async_elem(sc + kExCT + c, lam + c0 + c);
        cp_async_elem(sc + 2 * kExCT + c, wopt + c0 + c);
      }
    }
  };
  // one commit group per tile slot (empty groups past the end keep the count uniform)
#pragma unroll
  for (int t = 0; t < kExBuf - 1; t++) {
    if (t < ntiles) issue(t);
    cp_async_commit();
  }
  double cons = 0.0, loss = 0.0;
  for (long long t = 0; t < ntiles; t++) {
    if (t + kExBuf - 1 < ntiles) issue(t + kExBuf - 1);
    cp_async_commit();
    cp_async_wait<kExBuf - 1>();
    __syncwarp();
    const int b = (int)(t % kExBuf);
    const int width = (int)min((long long)kExCT, d - t * kExCT);
    const T* row = tile_w(b) + lane * X::ROW;
    const double* sc = tile_c(b);
    if (lane < nrows) {
      if (has_obj) {
#pragma unroll 8
        for (int c = 0; c < width; c++) {
          const double w = (double)row[c];
          const double dv = __dsub_rn(w, sc[c]);
          cons = __dadd_rn(cons, __dmul_rn(dv, dv));
          const double dw = __dsub_rn(w, sc[2 * kExCT + c]);
          loss = __dadd_rn(loss, __dmul_rn(__dmul_rn(sc[kExCT + c], dw), dw));
        }
      } else {
#pragma unroll 8
        for (int c = 0; c < width; c++) {
          const double dv = __dsub_rn((double)row[c], sc[c]);
          cons = __dadd_rn(cons, __dmul_rn(dv, dv));
        }
      }
    }
    __syncwarp();   // buffer b is refilled by the next iteration's issue
  }
  cp_async_wait<0>();
  if (lane < nrows) {
    cons_sq[l0 + lane] = cons;
    if (loss_col != nullptr) loss_col[l0 + lane] = __dmul_rn(0.5, loss);
  }
}

// bf16 (2-byte elements, no cp.async of that size): direct row walk
__global__ void __launch_bounds__(128)
    trace_exact_rows_bf16_kernel(const __nv_bfloat16* __restrict__ W, int L, long long d,
                                 long long ld, const double* __restrict__ M,
                                 const double* __restrict__ lam, const double* __restrict__ wopt,
                                 double* __restrict__ cons_sq, double* __restrict__ loss_col) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const __nv_bfloat16* row = W + (long long)l * ld;
  double cons = 0.0, loss = 0.0;
  for (long long c = 0; c < d; c++) {
    const double w = (double)__bfloat162float(row[c]);
    const double dv = __dsub_rn(w, M[c]);
    cons = __dadd_rn(cons, __dmul_rn(dv, dv));
    if (lam != nullptr) {
      const double dw = __dsub_rn(w, wopt[c]);
      loss = __dadd_rn(loss, __dmul_rn(__dmul_rn(lam[c], dw), dw));
    }
  }
  cons_sq[l] = cons;
  if (loss_col != nullptr) loss_col[l] = __dmul_rn(0.5, loss);
}

// subtree t of numpy's pairwise recursion over the terms fl(fl(lam_c dm) dm), dm = M_c - w*_c
__global__ void __launch_bounds__(128)
    trace_exact_avg_leaves_kernel(const double* __restrict__ M, const double* __restrict__ lam,
                                  const double* __restrict__ wopt, long long d, int depth,
                                  double* __restrict__ part) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (1 << depth)) return;
  long long lo = 0, n = d;
  for (int j = depth - 1; j >= 0; j--) {   // descend: bit j of t picks the half
    long long n2 = n / 2;
    n2 -= n2 % 8;
    if ((t >> j) & 1) {
      lo += n2;
      n -= n2;
    } else {
      n = n2;
    }
  }
  auto term = [&](int i) {
    const long long c = lo + i;
    const double dm = __dsub_rn(M[c], wopt[c]);
    return __dmul_rn(__dmul_rn(lam[c], dm), dm);
  };
  part[t] = pairwise_sum<double>(term, 0, (int)n);
}

// the top `depth` levels of the recursion: left + right, level by level
__global__ void __launch_bounds__(1024)
    trace_exact_avg_top_kernel(const double* __restrict__ part, int depth,
                               double* __restrict__ avg_loss) {
  __shared__ double s[1 << kExactMaxDepth];
  const int n = 1 << depth;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = part[i];
  __syncthreads();
  for (int w = n; w > 1; w >>= 1) {
    double v[4];
    const int h = w >> 1;
    int q = 0;
    for (int i = threadIdx.x; i < h; i += blockDim.x) v[q++] = __dadd_rn(s[2 * i], s[2 * i + 1]);
    __syncthreads();
    q = 0;
    for (int i = threadIdx.x; i < h; i += blockDim.x) s[i] = v[q++];
    __syncthreads();
  }
  if (threadIdx.x == 0) *avg_loss = __dmul_rn(0.5, s[0]);
}

static int64_t trace_exact_workspace_bytes(int64_t d) {
  return (d + (1LL << kExactMaxDepth)) * (int64_t)sizeof(double);
}

template <typename T>
static int trace_stats_exact(const T* W, int L, int64_t d, int64_t ld, const double* lam,
                             const double* wopt, double* cons_sq, double* loss_col,
                             double* avg_loss, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  if (W == nullptr || cons_sq == nullptr || L < 1 || L > kTrMaxLAny || d < 1 || ld < d ||
      (lam != nullptr && (wopt == nullptr || loss_col == nullptr || avg_loss == nullptr))) {
    set_error("invalid exact trace-stat arguments (L=%d, at most %d; d >= 1)", L, kTrMaxLAny);
    return RM_EINVAL;
  }
  if (workspace == nullptr || workspace_bytes < trace_exact_workspace_bytes(d)) {
    set_error("exact trace-stat workspace too small (need %lld bytes)",
              (long long)trace_exact_workspace_bytes(d));
    return RM_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* M = static_cast<double*>(workspace);
  double* part = M + d;
  long long blocks = (d + 255) / 256;
  if (blocks > 16LL * sm_count(-1)) blocks = 16LL * sm_count(-1);
  column_mean_kernel<T><<<(int)blocks, 256, 0, st>>>(W, L, d, ld, M);
  RM_CHECK_LAUNCH("column_mean_kernel");
  if constexpr (sizeof(T) == 2) {
    trace_exact_rows_bf16_kernel<<<(L + 127) / 128, 128, 0, st>>>(
        W, L, d, ld, M, lam, wopt, cons_sq, lam ? loss_col : nullptr);
    RM_CHECK_LAUNCH("trace_exact_rows_bf16_kernel");
  } else {
    const size_t smem = (size_t)kExBuf * ExTile<T>::BYTES;
    static unsigned long long attr_mask = 0;
    if (attr_needed(&attr_mask)) {
      cudaError_t e = cudaFuncSetAttribute(trace_exact_rows_kernel<T>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(trace_exact_rows_kernel)");
      attr_done(&attr_mask);
    }
    trace_exact_rows_kernel<T><<<(L + 31) / 32, 32, smem, st>>>(W, L, d, ld, M, lam, wopt,
                                                                cons_sq, lam ? loss_col : nullptr);
    RM_CHECK_LAUNCH("trace_exact_rows_kernel");
  }
  if (lam != nullptr) {
    const int depth = exact_pairwise_depth(d);
    trace_exact_avg_leaves_kernel<<<((1 << depth) + 127) / 128, 128, 0, st>>>(M, lam, wopt, d,
                                                                             depth, part);
    RM_CHECK_LAUNCH("trace_exact_avg_leaves_kernel");
    trace_exact_avg_top_kernel<<<1, 1024, 0, st>>>(part, depth, avg_loss);
    RM_CHECK_LAUNCH("trace_exact_avg_top_kernel");
  }
  return 0;
}
}  // namespace rm

extern "C" int64_t rm_trace_stats_exact_workspace_bytes(int64_t d) {
  if (d < 1) return -1;
  return trace_exact_workspace_bytes(d);
}

#define RM_DEFINE_TRACE_EXACT(SUFFIX, CT, T)                                                   \
  extern "C" int rm_trace_stats_exact_##SUFFIX(                                                \
      const CT* W, int L, int64_t d, int64_t ld, const double* lam, const double* wopt,         \
      double* cons_sq, double* loss_col, double* avg_loss, void* workspace,                     \
      int64_t workspace_bytes, void* stream) {                                                  \
    return trace_stats_exact<T>(reinterpret_cast<const T*>(W), L, d, ld, lam, wopt, cons_sq,   \
                                loss_col, avg_loss, workspace, workspace_bytes, stream);       \
  }
RM_DEFINE_TRACE_EXACT(f32, float, float)
RM_DEFINE_TRACE_EXACT(f64, double, double)
RM_DEFINE_TRACE_EXACT(bf16, uint16_t, __nv_bfloat16)
