// Internal types shared by traverse.cu / execute.cu / engine.cu.
#pragma once

#include "engine.cuh"
#include "series_dev.cuh"

namespace dfgtb {
namespace detail {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr int kMaxGridBlocks = 148 * 16;
constexpr int kSPow = 128;  // s^k, k < kSPow, per slot (scaling of unscaled moments)

enum Kind { kE = 0, kF = 1, kD = 2, kT = 3, kB = 4, kX = 5, kFD = 6 };

struct TreeView {
  const double *lo, *hi, *cen, *side;
  const int *left, *right, *count, *begin, *parent;
  const double* xs;
  const int *depth, *anc;  // node depth; root-first ancestor chains (depth < kMaxAnc)
};

inline TreeView view_of(const DevTree& t)
{
  return TreeView{ t.lo.p, t.hi.p, t.centroid.p, t.max_side.p, t.left.p, t.right.p,
                   t.count.p, t.begin.p, t.parent.p, t.xs.p, t.depth.p, t.anc.p };
}

inline int grid_warps(long long work)
{
  return (int)std::max<long long>(
    1, std::min<long long>(kMaxGridBlocks, (work + kWarpsPerBlock - 1) / kWarpsPerBlock));
}

// Per-slot constants of a batch, in device memory: s = 1/(h sqrt 2), s2 = 1/(2h^2),
// spow[k] = s^k.
struct SlotView {
  const double* s;
  const double* s2;
  const double* spow;  // slot * kSPow + k
};

template <int DT>
__device__ __forceinline__ void box_bounds(const double* alo, const double* ahi, const double* blo,
                                           const double* bhi, int Drt, double& lo2, double& hi2)
{  // kdtree.cpp:122-141
  const int D = DT ? DT : Drt;
  double lo = 0.0, hi = 0.0;
#pragma unroll
  for (int k = 0; k < (DT ? DT : kMaxDim); ++k) {
    if (!DT && k >= D) break;
    const double g1 = blo[k] - ahi[k];
    const double g2 = alo[k] - bhi[k];
    const double l = 0.5 * (g1 + fabs(g1) + g2 + fabs(g2));
    lo = __dadd_rn(lo, __dmul_rn(l, l));  // no FMA: bit-identical to the reference's sums
    const double u1 = bhi[k] - alo[k], u2 = ahi[k] - blo[k];
    const double u = u1 < u2 ? u2 : u1;
    hi = __dadd_rn(hi, __dmul_rn(u, u));
  }
  lo2 = lo;
  hi2 = hi;
}

}  // namespace detail
}  // namespace dfgtb
