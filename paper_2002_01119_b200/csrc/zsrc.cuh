// The quadratic oracle's gradient produced inside the mix kernel (
// reference objectives.py:84-90 called from simulation.py:226-238): G never touches HBM.
//
// The normal generator (csrc/normal.cu) leaves every learner stream's normals in its
// speculative scratch: raw block b of stream j holds its true outputs at
//   scratch[gid * 256 + skip[gid] + (c - offs[gid])],  gid = j * nblocks + b,
// for output indices c in [offs[gid], offs[gid] + tcount[gid]).  zig_zindex_kernel
// condenses that into one 16-byte descriptor per (stream, 128-column group):
//   z(c) = scratch[zb + c]          for c - group_start <  brk
//   z(c) = scratch[zb + dz + c]     for c - group_start >= brk
// (brk = 128 when one block covers the whole group).  A group that spans three or more
// blocks (a middle block with fewer than 128 outputs; never seen in practice) gets
// brk = -1 and zb = the gid of its first block, and the lookup walks offs / tcount.
//
// The gradient element is the generator's own expression (zig_copy_kernel / emit_grad):
//   g = fl_T( lam[c] * (Phi[j][c] - w*[c]) + sd * z )
// so the fused step is bit-identical to gradient pass + ring / mean step.
#pragma once
#include <stdint.h>

namespace rm {

constexpr int kZGroupLog2 = 7;   // 128-column groups
constexpr int kZGroup = 1 << kZGroupLog2;

struct ZDesc {
  long long zb;
  int dz;
  int brk;
};

struct ZSrc {
  const double* scratch;
  const ZDesc* desc;                 // [nstreams][ngroups]
  long long ngroups;
  const unsigned long long* offs;    // walk fallback
  const uint32_t* tcount;
  const uint32_t* skip;
  const double* lam;
  const double* wopt;
  double sd;
};

// scratch index of normal `col` of stream j, given the group descriptor
__device__ __forceinline__ long long z_index(const ZSrc& z, const ZDesc& g, long long col) {
  const int rel = (int)(col & (kZGroup - 1));
  if (g.brk >= 0) return g.zb + col + (rel >= g.brk ? g.dz : 0);
  long long gid = g.zb;
  for (;;) {
    const long long lo = (long long)z.offs[gid];
    if (col < lo + (long long)z.tcount[gid]) return gid * 256 + z.skip[gid] + (col - lo);
    ++gid;
  }
}

__device__ __forceinline__ ZDesc z_desc(const ZSrc& z, int j, long long col) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(z.desc + (long long)j * z.ngroups +
                                                     (col >> kZGroupLog2)));
  ZDesc g;
  g.zb = (long long)(((unsigned long long)(uint32_t)v.y << 32) | (uint32_t)v.x);
  g.dz = v.z;
  g.brk = v.w;
  return g;
}

// the gradient element in fp64 before the storage rounding (objectives.py:87-90)
__device__ __forceinline__ double z_grad(double lam, double wopt, double sd, double phi,
                                         double zv) {
  return __dadd_rn(__dmul_rn(lam, __dsub_rn(phi, wopt)), __dmul_rn(sd, zv));
}

// Generator side: run the generator for step k up to the normals (scratch + descriptors)
// and fill `z` (device pointers into `workspace`).  Defined in normal.cu.
int quad_z_prepare(const uint32_t* prefix, int nprefix, uint64_t k, int nstreams, long long n,
                   void* workspace, long long workspace_bytes, void* stream, ZSrc* z,
                   long long stream0 = 0);
long long quad_z_workspace_bytes(int nstreams, long long n);
// The fused step on the generator's copy side (zig_mix_kernel): left == nullptr = uniform.
template <typename T>
int quad_mix_copy(const uint32_t* prefix, int nprefix, uint64_t k, const T* W, const T* Phi,
                  T* out, const int32_t* left, const int32_t* right, int L, long long d,
                  long long ldw, long long ldp, long long ldo, const double* lam,
                  const double* wopt, double sd, double lr, unsigned long long* absmax, void* ws,
                  long long ws_bytes, void* stream, long long stream0 = 0,
                  const double* ext_means = nullptr, void* means_ready = nullptr);

}  // namespace rm
