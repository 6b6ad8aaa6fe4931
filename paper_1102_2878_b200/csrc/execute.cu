// Execution of the traversal's work lists on sm_100a, batched over bandwidth slots.
//
// Reference path (/root/reference/proj/src):
//   moments_for (leaf moments + F2F)  engine.cpp:368-403  -> k_moment_chunks/reduce (once per tree)
//   summarize D (direct local)        engine.cpp:212-221  -> k_local_chunks + k_local_reduce
//   summarize T (far-to-local)        engine.cpp:223-232  -> k_local_chunks + k_local_reduce
//   post_process L2L                  engine.cpp:294-304  -> k_l2l (local_pushdown = 1) or the
//                                                            direct ancestor evaluation in k_finalize
//   base_case                         engine.cpp:239-269  -> k_base_case (K10, the hot kernel)
//   summarize F (far-field eval)      engine.cpp:200-211  -> k_farfield(_t)
//   post_process leaf + run           engine.cpp:273-291, 85-89 -> k_finalize
//   lkcv / lscv_from_sums             cv.cpp:61-97        -> k_cv_partial
#include "internal.cuh"

#include <cstring>

#include <cub/device/device_scan.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <string>

namespace dfgtb {
using namespace detail;

namespace {

// ------------------------------------------------------------------- moments
__global__ void k_mark_moments(const Item* it, const int* n, int cap, int* flag)
{
  const int m = min(*n, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int kind = it[i].code >> 8;
    if (kind == kF || kind == kT) flag[it[i].r] = 1;
  }
}

// K2/K3 (large tables, lazy): UNSCALED moments (position layout) of the reference
// nodes an F/T item uses and that are not cached yet, one block per node.
__global__ void k_moments(DevSeries g, TreeView R, int nodes, const int* flag, int* done, double* M)
{
  extern __shared__ double sm[];
  for (int n = blockIdx.x; n < nodes; n += gridDim.x) {
    if (!flag[n] || done[n]) continue;
    dev_moments_block(g, R.xs + (size_t)R.begin[n] * g.D, R.count[n], R.cen + (size_t)n * g.D, 1.0,
                      M + (size_t)n * g.T, sm, g.pos);
    __syncthreads();
    if (threadIdx.x == 0) done[n] = 1;
  }
}

// K2/K3 (eager, tables <= 4096 terms): unscaled moments of EVERY reference node, once
// per tree: M~_a(node) = (1/a!) sum_r prod_d (r - c)_d^{a_d}.  The reference's per-h
// moment is s^|a| M~_a with s = 1/(h sqrt 2) -- one pass serves a whole sweep.
// Pass 1: partial sums over 64-point chunks of each node; pass 2: chunks summed in
// order per node; tables stored in the reference's position layout.
constexpr int kMomChunk = 64;
__global__ void k_moment_chunks(DevSeries g, TreeView R, const int* cnode, const int* cstart,
                                int nchunks, double* part)
{
  extern __shared__ double sm[];
  const int D = g.D, pm = g.pmax, per = D * pm;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int n = cnode[c], st = cstart[c];
    const int m = min(kMomChunk, R.begin[n] + R.count[n] - st);
    const double* cen = R.cen + (size_t)n * D;
    __syncthreads();
    for (int w = threadIdx.x; w < m * D; w += blockDim.x) {
      const int pt = w / D, d = w % D;
      const double u = R.xs[(size_t)(st + pt) * D + d] - cen[d];
      double* P = sm + pt * per + d * pm;
      P[0] = 1.0;
      for (int k = 1; k < pm; ++k) P[k] = P[k - 1] * u;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < g.T; i += blockDim.x) {
      const uint64_t a = g.dig[i];
      double sum = 0.0;
      for (int pt = 0; pt < m; ++pt) sum += mono(sm + pt * per, pm, D, a);
      part[(size_t)c * g.T + i] = sum;
    }
  }
}

// Warp reduce-scatter of 32 per-lane values: afterwards lane l holds the sum over the
// warp of value l (five halving exchange steps, fixed order).
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane)
{
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int off = 16 >> st;
    const bool up = lane & off;
    const int h = 16 >> st;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < h) {
        const double send = up ? v[i] : v[i + h];
        const double keep = up ? v[i + h] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
  }
  return v[0];
}

// Specialised pass 1 for the default tables (p_max == PM, <= 64 terms): ONE WARP per
// 64-point chunk, each lane's points' monomials prod_d (r - c)_d^{a_d} for every
// multi-index accumulated in registers (compile-time digits), warp reduce-scatter,
// partials in term order like k_moment_chunks.
template <int D, int PM>
__global__ void __launch_bounds__(128) k_moment_chunks_w(DevSeries g, TreeView R, const int* cnode,
                                                         const int* cstart, int nchunks, double* part)
{
  constexpr int NP = ipow_c(PM, D), NB = (NP + 31) / 32;
  __shared__ int tp[NP];
  for (int p = threadIdx.x; p < NP; p += blockDim.x) tp[p] = g.term_of_pos[p];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks;
       c += (gridDim.x * blockDim.x) >> 5) {
    const int n = cnode[c], st = cstart[c];
    const int m = min(kMomChunk, R.begin[n] + R.count[n] - st);
    double cen[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cen[d] = R.cen[(size_t)n * D + d];
    double acc[NB * 32];
#pragma unroll
    for (int p = 0; p < NB * 32; ++p) acc[p] = 0.0;
    for (int j = lane; j < m; j += 32) {
      double P[D][PM];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double u = R.xs[(size_t)(st + j) * D + d] - cen[d];
        P[d][0] = 1.0;
#pragma unroll
        for (int k = 1; k < PM; ++k) P[d][k] = P[d][k - 1] * u;
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double f = 1.0;
        int rest = p;
#pragma unroll
        for (int d = D - 1; d >= 0; --d) {
          f *= P[d][rest % PM];
          rest /= PM;
        }
        acc[p] += f;
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      double v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = acc[b * 32 + i];
      const double tot = warp_reduce_scatter32(v, lane);
      const int p = b * 32 + lane;
      if (p < NP) part[(size_t)c * NP + tp[p]] = tot;
    }
  }
}

// One CTA per node: thread (term i, stripe k) sums chunks c = c0 + k, c0 + k + S, ...
// (8 loads in flight), then the S stripe sums are added in stripe order: a fixed
// summation order, latency ~count/(8 S) round trips instead of count.
constexpr int kMomRedThreads = 256;
__global__ void __launch_bounds__(kMomRedThreads) k_moment_reduce(DevSeries g, int nodes,
                                                                  const int* coff,
                                                                  const double* part, double* M)
{
  __shared__ double red[kMomRedThreads];
  const int T = g.T;
  const int S = T <= kMomRedThreads ? kMomRedThreads / T : 1;
  for (int n = blockIdx.x; n < nodes; n += gridDim.x) {
    const int c0 = coff[n], c1 = coff[n + 1];
    for (int i0 = 0; i0 < T; i0 += kMomRedThreads / S) {
      const int i = i0 + threadIdx.x % (kMomRedThreads / S), k = threadIdx.x / (kMomRedThreads / S);
      double acc = 0.0;
      if (i < T && k < S) {
        int c = c0 + k;
        for (; c + 7 * S < c1; c += 8 * S) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(c + u * S) * T + i];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += v[u];
        }
        for (; c < c1; c += S) acc += part[(size_t)c * T + i];
      }
      red[threadIdx.x] = acc;
      __syncthreads();
      if (k == 0 && i < T) {
        double sum = 0.0;
        for (int kk = 0; kk < S; ++kk) sum += red[kk * (kMomRedThreads / S) + threadIdx.x];
        M[(size_t)n * T + g.pos[i]] = sum * g.invf[i];
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------- D / T items (local expansions)
// Work split into chunks: a D item over <= kLocChunk reference points, or one T
// item.  Each chunk writes an unsigned partial table; k_local_reduce sums a query
// node's chunks in item order and applies (-1)^|b|/b! (summarize, engine.cpp:212-232).
constexpr int kLocChunk = 1024;  // points per D chunk (staged kLocSub at a time)
constexpr int kLocSub = 64;
struct LChunk {
  int item, start, n;
};

// chunk counts of the D/T items (0 past the item count, so one scan over the
// capacity gives the offsets); counts come from the device
__global__ void k_local_count(const Item* items, const int* n, int cap, TreeView R, int* nch)
{
  const int m = min(*n, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= cap; i += gridDim.x * blockDim.x) {
    int c = 0;
    if (i < m) {
      const int kind = items[i].code >> 8;
      c = kind == kD ? (R.count[items[i].r] + kLocChunk - 1) / kLocChunk : 1;
    }
    nch[i] = c;
  }
}

__global__ void k_local_fill(const Item* items, const int* n, int cap, TreeView R, const int* choff,
                             LChunk* ch, int chcap, int* nch_out)
{
  const int m = min(*n, cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) *nch_out = choff[m];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int kind = items[i].code >> 8;
    const int r = items[i].r;
    if (kind == kD) {
      const int b = R.begin[r], c = R.count[r];
      for (int k = 0, st = 0; st < c; ++k, st += kLocChunk)
        if (choff[i] + k < chcap) ch[choff[i] + k] = LChunk{ i, b + st, min(kLocChunk, c - st) };
    } else if (choff[i] < chcap) {
      ch[choff[i]] = LChunk{ i, -1, 0 };
    }
  }
}

__global__ void k_local_chunks(DevSeries g, TreeView Q, TreeView R, int K, const Item* items,
                               const LChunk* ch, const int* nchp, int chcap, const double* Mt,
                               SlotView sv, double* part)
{
  extern __shared__ double sm[];
  const int nch = min(*nchp, chcap);
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const LChunk lc = ch[c];
    const Item it = items[lc.item];
    const int slot = it.key / K, node = it.key - slot * K;
    const int kind = it.code >> 8, order = it.code & 0xff;
    const double s = sv.s[slot];
    double* P = part + (size_t)c * g.T;
    const double* qc = Q.cen + (size_t)node * g.D;
    if (kind == kD) {
      for (int b = 0; b < lc.n; b += kLocSub)
        dev_direct_local_partial(g, R.xs + (size_t)(lc.start + b) * g.D, min(kLocSub, lc.n - b), qc,
                                 s, order, P, sm, b > 0);
    } else {
      dev_f2l_block(g, Mt + (size_t)it.r * g.T, R.cen + (size_t)it.r * g.D, qc, s, order, P, sm,
                    sv.spow + (size_t)slot * kSPow, 1, g.pos);
    }
  }
}

// Specialised D chunks for the default tables (p_max == PM, <= 64 terms): each thread
// accumulates its points' Hermite products for every multi-index in registers
// (compile-time digits), then the block reduces over threads in a fixed order.  T
// chunks use the generic F2L.  Same partial table as dev_direct_local_partial.
constexpr int kLocThreads = 64;
template <int D, int PM>
__global__ void __launch_bounds__(kLocThreads) k_local_chunks_t(DevSeries g, TreeView Q, TreeView R,
                                                               int K, const Item* items,
                                                               const LChunk* ch, const int* nchp,
                                                               int chcap, const double* Mt,
                                                               SlotView sv, double* part)
{
  constexpr int NP = ipow_c(PM, D);
  __shared__ double red[NP][kLocThreads + 1];
  extern __shared__ double sm[];
  const int nch = min(*nchp, chcap);
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const LChunk lc = ch[c];
    const Item it = items[lc.item];
    const int slot = it.key / K, node = it.key - slot * K;
    const int kind = it.code >> 8, order = it.code & 0xff;
    const double s = sv.s[slot];
    double* P = part + (size_t)c * g.T;
    const double* qc = Q.cen + (size_t)node * D;
    if (kind != kD) {
      dev_f2l_block(g, Mt + (size_t)it.r * g.T, R.cen + (size_t)it.r * D, qc, s, order, P, sm,
                    sv.spow + (size_t)slot * kSPow, 1, g.pos);
      __syncthreads();
      continue;
    }
    double acc[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) acc[p] = 0.0;
    double cq[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cq[d] = qc[d];
    for (int j = threadIdx.x; j < lc.n; j += kLocThreads) {
      const double* rp = R.xs + (size_t)(lc.start + j) * D;
      // Hermite functions H_k(t_d) = exp(-t_d^2) h_k(t_d): the Gaussians of all
      // dimensions are one exp(-|t|^2), folded into dimension 0
      double H[D][PM];
      double tt = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double t = (cq[d] - rp[d]) * s;
        tt = fma(t, t, tt);
        H[d][0] = 1.0;
        if (PM > 1) H[d][1] = 2.0 * t;
#pragma unroll
        for (int k = 1; k + 1 < PM; ++k) H[d][k + 1] = fma(2.0 * t, H[d][k], -2.0 * k * H[d][k - 1]);
      }
      const double e = exp(-tt);
#pragma unroll
      for (int k = 0; k < PM; ++k) H[0][k] *= e;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double f = 1.0;
        int rest = p;
#pragma unroll
        for (int d = D - 1; d >= 0; --d) {
          f *= H[d][rest % PM];
          rest /= PM;
        }
        acc[p] += f;
      }
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) red[p][threadIdx.x] = acc[p];
    __syncthreads();
    for (int p = threadIdx.x; p < NP; p += kLocThreads) {
      int rest = p, mx = 0;
      for (int d = 0; d < D; ++d) {
        mx = max(mx, rest % PM);
        rest /= PM;
      }
      double sum = 0.0;
      for (int k = 0; k < kLocThreads; ++k) sum += red[p][k];
      if (mx < order) P[g.term_of_pos[p]] = sum;
    }
    __syncthreads();
  }
}

// One warp per query-node key that has D/T items (launched over the sorted items; the
// warp of a key's first item does the work), lanes over terms.  Every term sums its
// chunks in item order (8 loads in flight), so the result does not depend on the
// launch shape.
// Specialised D/T chunks for the default tables (p_max == PM): ONE WARP per chunk.
//  D: lanes over the chunk's points, Hermite products of every multi-index in
//     registers (one exp(-|t|^2) per point), warp reduce-scatter per 32 terms.
//  T: far-to-local of the reference node's moments contracted one dimension at a time
//     in the warp's shared scratch: V <- sum_{a_d} V[.., a_d, ..] H_d[a_d + b_d]
//     (D stages of PM^D outputs x PM FMAs instead of PM^{2D} products).
// Both write the same unsigned partial table (term layout, terms < order^D) as
// dev_direct_local_partial / dev_f2l_block.
constexpr int kLocWarps = 4;
#ifndef DFGTB_LOC_MINB
#define DFGTB_LOC_MINB 4  // <= 128 registers (119 at D = 2; D = 3 spills 184 B): measured best of 2 / 4 / 6 / 8
#endif
template <int D, int PM>
__global__ void __launch_bounds__(kLocWarps * 32, DFGTB_LOC_MINB) k_local_chunks_w(
  DevSeries g, TreeView Q, TreeView R, int K, const Item* items, const LChunk* ch, const int* nchp,
  int chcap, const double* Mt, SlotView sv, double* part)
{
  constexpr int NP = ipow_c(PM, D), HL = 2 * PM - 1, NB = (NP + 31) / 32;
  __shared__ int tp[NP];
  __shared__ double wsc[kLocWarps][2 * NP + D * HL];
  for (int p = threadIdx.x; p < NP; p += blockDim.x) tp[p] = g.term_of_pos[p];
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* V0 = wsc[wib];
  double* V1 = V0 + NP;
  double* H = V1 + NP;
  const int nch = min(*nchp, chcap);
  for (int c = blockIdx.x * kLocWarps + wib; c < nch; c += gridDim.x * kLocWarps) {
    const LChunk lc = ch[c];
    const Item it = items[lc.item];
    const int slot = it.key / K, node = it.key - slot * K;
    const int kind = it.code >> 8, order = it.code & 0xff;
    const double s = sv.s[slot];
    double* P = part + (size_t)c * g.T;
    const double* qc = Q.cen + (size_t)node * D;
    if (kind == kD) {
      double acc[NB * 32];
#pragma unroll
      for (int p = 0; p < NB * 32; ++p) acc[p] = 0.0;
      double cq[D];
#pragma unroll
      for (int d = 0; d < D; ++d) cq[d] = qc[d];
      for (int j = lane; j < lc.n; j += 32) {
        const double* rp = R.xs + (size_t)(lc.start + j) * D;
        double Hh[D][PM];
        double tt = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double t = (cq[d] - rp[d]) * s;
          tt = fma(t, t, tt);
          Hh[d][0] = 1.0;
          if (PM > 1) Hh[d][1] = 2.0 * t;
#pragma unroll
          for (int k = 1; k + 1 < PM; ++k) Hh[d][k + 1] = fma(2.0 * t, Hh[d][k], -2.0 * k * Hh[d][k - 1]);
        }
        const double e = exp(-tt);
#pragma unroll
        for (int k = 0; k < PM; ++k) Hh[0][k] *= e;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          double f = 1.0;
          int rest = p;
#pragma unroll
          for (int d = D - 1; d >= 0; --d) {
            f *= Hh[d][rest % PM];
            rest /= PM;
          }
          acc[p] += f;
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = acc[b * 32 + i];
        const double tot = warp_reduce_scatter32(v, lane);
        const int p = b * 32 + lane;
        if (p < NP) {
          int rest = p, mx = 0;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            mx = max(mx, rest % PM);
            rest /= PM;
          }
          if (mx < order) P[tp[p]] = tot;
        }
      }
    } else {
      // Hermite function rows at t = (c_Q - c_R) s, one lane per dimension
      const int r = it.r;
      if (lane < D) {
        const double t = (qc[lane] - R.cen[(size_t)r * D + lane]) * s;
        double* h = H + lane * HL;
        h[0] = exp(-t * t);
        h[1] = 2.0 * t * h[0];
#pragma unroll
        for (int k = 1; k + 1 < HL; ++k) h[k + 1] = 2.0 * t * h[k] - 2.0 * k * h[k - 1];
      }
      // scaled, truncated moments M'_a = s^|a| M~_a (a_d < order), position layout
      const double* sp = sv.spow + (size_t)slot * kSPow;
      for (int p = lane; p < NP; p += 32) {
        int rest = p, mx = 0, deg = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int dg = rest % PM;
          mx = max(mx, dg);
          deg += dg;
          rest /= PM;
        }
        V0[p] = mx < order ? Mt[(size_t)r * NP + p] * sp[deg] : 0.0;
      }
      __syncwarp();
      double* src = V0;
      double* dst = V1;
#pragma unroll
      for (int d = D - 1; d >= 0; --d) {
        const int stride = ipow_c(PM, D - 1 - d);
        const double* hd = H + d * HL;
        for (int p = lane; p < NP; p += 32) {
          const int bd = (p / stride) % PM;
          const int base = p - bd * stride;
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < PM; ++k) acc = fma(src[base + k * stride], hd[k + bd], acc);
          dst[p] = acc;
        }
        __syncwarp();
        double* tmp = src;
        src = dst;
        dst = tmp;
      }
      for (int p = lane; p < NP; p += 32) {
        int rest = p, mx = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          mx = max(mx, rest % PM);
          rest /= PM;
        }
        if (mx < order) P[tp[p]] = src[p];
      }
      __syncwarp();
    }
  }
}

// One warp per (slot, query node) key that has D/T items.  The keys are found from the
// per-key counts, kLrKeys keys per CTA round (coalesced loads, compacted in shared
// memory, dealt to the CTA's warps) -- not by scanning the item list for first-of-key
// items, which cost every warp a chain of dependent loads per item.
#ifndef DFGTB_LR_KEYS
#define DFGTB_LR_KEYS 64
#endif
constexpr int kLrKeys = DFGTB_LR_KEYS;
__global__ void k_local_reduce(DevSeries g, const int* nitems_p, int cap, int nkeys, const int* cnt,
                               const int* off, const Item* items, const int* choff, int capch,
                               const double* part, double* L, int* Lord)
{
  const int nitems = min(*nitems_p, cap);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  __shared__ int s_n, s_key[kLrKeys], s_i0[kLrKeys], s_c[kLrKeys];
  for (int kb = blockIdx.x * kLrKeys; kb < nkeys; kb += gridDim.x * kLrKeys) {
  __syncthreads();
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  if (threadIdx.x < kLrKeys && kb + threadIdx.x < nkeys) {
    const int c = cnt[kb + threadIdx.x];
    if (c > 0) {
      const int o = off[kb + threadIdx.x];
      if (o + c <= nitems) {
        const int pos = atomicAdd(&s_n, 1);  // any order: every key's table is its own
        s_key[pos] = kb + threadIdx.x;
        s_i0[pos] = o;
        s_c[pos] = c;
      }
    }
  }
  __syncthreads();
  for (int j = wib; j < s_n; j += nwb) {
  const int n = s_key[j];
  const int i0 = s_i0[j];
  const int i1 = i0 + s_c[j];
  int ord = 0, omin = 1 << 20;
  for (int k = i0 + lane; k < i1; k += 32) {
    ord = max(ord, items[k].code & 0xff);
    omin = min(omin, items[k].code & 0xff);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ord = max(ord, __shfl_xor_sync(0xffffffffu, ord, o));
    omin = min(omin, __shfl_xor_sync(0xffffffffu, omin, o));
  }
  const int q0 = choff[i0], q1 = choff[i1];
  if (q1 > capch) continue;  // chunks past the chunk buffer were dropped: the batch is rerun
  const int nt = ipow_i(ord, g.D);
  for (int t = lane; t < nt; t += 32) {
    const uint64_t a = g.dig[t];
    int mx = 0;
    for (int d = 0; d < g.D; ++d) mx = max(mx, digit_of(a, d));
    double acc = 0.0;
    if (mx >= omin) {  // a term some item does not carry: walk the items
      for (int k = i0; k < i1; ++k) {
        if (mx >= (items[k].code & 0xff)) continue;  // term beyond this item's order
        for (int q = choff[k]; q < choff[k + 1]; ++q) acc += part[(size_t)q * g.T + t];
      }
    } else {  // every item carries the term: its chunks are one contiguous run
      int q = q0;
      for (; q + 8 <= q1; q += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(q + u) * g.T + t];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; q < q1; ++q) acc += part[(size_t)q * g.T + t];
    }
    const double sg = (g.degree[t] & 1) ? -1.0 : 1.0;
    L[(size_t)n * g.T + t] += sg * g.invf[t] * acc;
  }
  if (lane == 0 && Lord[n] < ord) Lord[n] = ord;
  }
  }
}

// Top-down L2L of one depth level for every slot (post_process, engine.cpp:294-304).
__global__ void k_l2l(DevSeries g, TreeView Q, int K, int nb, const int* nodes_at, int m,
                      SlotView sv, double* L, int* Lord)
{
  extern __shared__ double sm[];
  for (int k = blockIdx.x; k < m * nb; k += gridDim.x) {
    const int slot = k / m;
    const int n = nodes_at[k - slot * m];
    const int key = slot * K + n;
    const int order = Lord[key];
    if (Q.left[n] < 0 || order <= 0) continue;
    const int ch[2] = { slot * K + Q.left[n], slot * K + Q.right[n] };
    const int chn[2] = { Q.left[n], Q.right[n] };
    for (int c = 0; c < 2; ++c) {
      dev_l2l_block(g, L + (size_t)key * g.T, Q.cen + (size_t)n * g.D, Q.cen + (size_t)chn[c] * g.D,
                    sv.s[slot], order, L + (size_t)ch[c] * g.T, sm);
      __syncthreads();
      if (threadIdx.x == 0 && Lord[ch[c]] < order) Lord[ch[c]] = order;
    }
  }
}

// ---------------------------------------------------------------- base case
// Base-case tasks: a (slot, query leaf)'s sorted base items cut into runs of <=
// kTaskItems reference leaves, times 32-query chunks of the leaf.  One warp per task
// writes per-query partial sums; k_finalize adds a query's partials in task order.
constexpr int kTaskItems = 32;  // at most one reference leaf per lane
struct BTask {
  int key, item0, item1, q0;
};

// A (slot, query leaf)'s sorted base items are cut into RUNS of consecutive items
// whose points fit the warp's stream tile (<= rmax points, <= kTaskItems items; a
// single larger leaf is a run of its own and is streamed in tiles).  One warp per
// (slot, leaf): a window of 32 items, inclusive scan of their counts, the run is the
// prefix that fits.  Returns the next run's first item (all lanes).
__device__ __forceinline__ int warp_run_end(const Item* it, int k, int e, const int* rcount, int rmax,
                                            int lane, int* code = nullptr)
{
  const int j = k + lane;
  int pre = 1 << 28;
  if (j < e) {
    const int4 v = *reinterpret_cast<const int4*>(it + j);  // {key, r, code, rank}
    pre = rcount[v.y];
    if (code) *code = v.z;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre = min(pre + v, 1 << 28);
  }
  const unsigned fit = __ballot_sync(0xffffffffu, j < e && (pre <= rmax || lane == 0));
  return k + __popc(fit);
}

// Base-case tasks in one pass: the (slot, leaf)'s warp cuts its items into runs (lane r
// keeps run r's end, a bit mask whether the FP32 kernel may take the run: every item
// carries order bit 2), claims its task range with one atomic (bc[5] = tasks so far; a
// key's tasks stay contiguous, query chunk major, run minor, which is all k_finalize
// relies on), then writes the tasks from the recorded ends (keys with more than 32 runs
// recompute the later ones).  Tasks past tcap are dropped; the host sees bc[5] > tcap and
// reruns.
__global__ void k_task_build(const int* leaves, int nleaves, int nb, int K, const int* cntB,
                             const int* offB, const Item* sB, const int* rcount, int rmax, TreeView Q,
                             BTask* tasks, int tcap, int* ntasks, int* leaf_task, int* leaf_runs,
                             int* tflag)
{
  static_assert(sizeof(Item) == 16, "Item is read as one int4");
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= nleaves * nb) return;
  const int slot = i / nleaves;
  const int leaf = leaves[i - slot * nleaves];
  const int key = slot * K + leaf;
  const int o = offB[key], e = o + cntB[key];
  const int nq = (Q.count[leaf] + 31) / 32;
  int nruns = 0, myend = 0;
  unsigned f32m = 0;
  for (int k = o; k < e;) {
    int code = 0;
    const int j = warp_run_end(sB, k, e, rcount, rmax, lane, &code);
    const bool f32 = __all_sync(0xffffffffu, k + lane >= j || (code & 4));
    if (nruns < 32) {
      if (lane == nruns) myend = j;
      f32m |= (f32 ? 1u : 0u) << nruns;
    }
    k = j;
    ++nruns;
  }
  int t0 = 0;
  if (lane == 0 && nruns) t0 = atomicAdd(ntasks, nruns * nq);
  t0 = __shfl_sync(0xffffffffu, t0, 0);
  int runs = 0;
  for (int k = o; k < e;) {
    int j;
    bool f32;
    if (runs < 32) {
      j = __shfl_sync(0xffffffffu, myend, runs);
      f32 = (f32m >> runs) & 1u;
    } else {
      int code = 0;
      j = warp_run_end(sB, k, e, rcount, rmax, lane, &code);
      f32 = __all_sync(0xffffffffu, k + lane >= j || (code & 4));
    }
    for (int qi = lane; qi < nq; qi += 32)
      if (t0 + qi * nruns + runs < tcap) {
        tasks[t0 + qi * nruns + runs] = BTask{ key, k, j, 32 * qi };
        tflag[t0 + qi * nruns + runs] = f32 ? 1 : 0;
      }
    k = j;
    ++runs;
  }
  if (lane == 0) {
    leaf_task[key] = t0;
    leaf_runs[key] = runs;
  }
}

// Table-driven exp(-y), 0 <= y <= 708: -y = (64 m + j) ln2/64 + r, |r| <= ln2/128,
// exp(-y) = 2^m * 2^(j/64) * e^r with 2^(j/64) from a 64-entry shared-memory table and
// e^r by a degree-5 Taylor polynomial (truncation r^6/6! < 3.5e-17 relative).  The
// reduction uses ONE rounded constant C = RN(ln2/64) in a single FMA: its error,
// |n| |C - ln2/64| <= y * 1.1e-16 absolute in r, is of the same size as the rounding
// already present in y = |q'-r'|^2 itself (y * 2-3 ulp), so the pair's relative error
// stays y * O(1e-16) as with libdevice exp of the same y: nothing is charged to eps.
// 10 FP64 instructions (libdevice exp: ~16 plus integer work).
// c_exp64 = {64 log2 e, RN(ln2/64), 1/5!, 1/4!, 1/3!, 1/2!}.
__constant__ double c_exp64[6];
__constant__ double c_exp2tab[64];  // 2^(j/64)

// The table is addressed by its shared-window address `tabs` (512-byte aligned): the
// entry address is one shift and one AND-OR, the exponent increment (m << 20, taken
// from the low word k of t as (k & ~63) << 14) one AND and one multiply-add.
__device__ __forceinline__ double exp_negy_s(double y, unsigned tabs)
{
  const double magic = 6755399441055744.0;
  const double t = fma(-y, c_exp64[0], magic);
  const double n = t - magic;
  const double r = fma(n, -c_exp64[1], -y);
  double p = fma(c_exp64[2], r, c_exp64[3]);
  p = fma(p, r, c_exp64[4]);
  p = fma(p, r, c_exp64[5]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = __double2loint(t);
  double c;
  asm volatile("{\n\t.reg .b32 a;\n\tshl.b32 a, %1, 3;\n\tlop3.b32 a, a, 504, %2, 0xea;\n\t"
               "ld.shared.f64 %0, [a];\n\t}"
               : "=d"(c) : "r"(k), "r"(tabs));
  const double v = p * c;
  int hi;
  asm("{\n\t.reg .b32 m;\n\tand.b32 m, %1, -64;\n\tmad.lo.s32 %0, m, 16384, %2;\n\t}"
      : "=r"(hi) : "r"(k), "r"(__double2hiint(v)));
  return __hiloint2double(hi, __double2loint(v));
}

// exp(-y) for any y >= 0, branch-free, with the underflow range: beyond y = 708 the
// argument is shifted by 64 ln2 into the fast range and the result scaled by 2^-64
// (one rounding into the subnormals, as libm's exp rounds there); y > 752 gives
// exp(-708) 2^-64, which rounds to 0 like exp(-y) itself.
__device__ __forceinline__ double exp_negy_c(double y, unsigned tabs)
{
  const bool big = y > 708.0;
  const double yy = big ? y - 44.3614195558365 : y;  // 64 ln 2
  const double e = exp_negy_s(fmin(yy, 708.0), tabs);
  return big ? e * 0x1p-64 : e;
}

// MUFU exp for the fast base case (eps >= kMufuMinEps; the traversal runs with
// eps - kMufuCharge so the per-term error below is paid for).
// Coordinates are scaled by sqrt(log2 e) / (h sqrt 2) and centred on the chunk's first
// query, so z = y log2 e = |q|^2 + |r|^2 - 2 q.r is formed in FP64 directly on top of
// the fixed-point magic: t = M + b - 896 + z with M = 1.5 2^32 (ulp 2^-20), so the low
// word of t is (z + b - 896) in signed 12.20 fixed point (b = kMufuBias units keeps
// z + b >= 0 under the D + 2 roundings; 0 <= z <= 1021.4 on the fast path).  Then
//   2^-z = 2^-n 2^-(f - b 2^-20),  (n - 896) << 20 = lo & 0xFFF00000,  f = lo & (2^20 - 1),
// 2^-(f - b) by ex2.approx.ftz.f32 of an exact FP32 argument, and 2^-n spliced into the
// exponent while widening to FP64 (hi = (G >> 3) - ((n - 896) << 20); n <= 1021 keeps
// the result normal).  Per-term relative error <= (D + 2) ln2 2^-21 (fixed-point
// rounding) + ex2.approx's error (exhaustively measured by the tests over every
// reachable argument).
constexpr int kMufuBias = 4;
// t above this (high word 0x41F80000, low word (125 << 20) | 0xFFFFF) is z > 1021 - b
constexpr double kMufuClampT = 0x1.8000007dfffffp+32;
template <bool CLAMP = false>
__device__ __forceinline__ double exp2_neg_fixed(double t, unsigned fbits)
{
  // z > 1021 -> 0 (terms < 2^-1021; only where the traversal pays for it): one FP64
  // compare on t (positive doubles order like their bit patterns), the term is computed
  // from whatever t is and discarded
  const bool under = CLAMP && t > kMufuClampT;
  const int lo = __double2loint(t);
  // fbits = 0x4B000000 held in a register (one LOP3: (lo & mask) | fbits)
  const float x = __uint_as_float(((unsigned)lo & 0xFFFFFu) | fbits);  // 2^23 + f
  const float a = fmaf(x, -0x1p-20f, 8.0f + kMufuBias * 0x1p-20f);     // (b - f) 2^-20, exact
  float g;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(a));
  const unsigned G = __float_as_uint(g);
  const unsigned hi = (G >> 3) - ((unsigned)lo & 0xFFF00000u);
  const double v = __hiloint2double((int)hi, (int)(G << 29));
  return under ? 0.0 : v;
}
constexpr double kMufuMagic = 6442450944.0 - 896.0 + kMufuBias * 0x1p-20;  // M - 896 + b 2^-20
constexpr double kSqrtLog2e = 1.2011224087864498;                           // sqrt(log2 e)
constexpr double kLn2 = 0.6931471805599453;

// Scaled, centred, padded coordinates for the base case, per slot:
// x' = (x - c0) f / (h sqrt 2) so that |q' - r'|^2 = f^2 |q - r|^2 / (2 h^2) (stride DP);
// f = sqrt(log2 e) when the base case uses the MUFU exp (2^-z), else 1 (e^-y).
__global__ void k_scale_points(const double* xs, int n, int D, int DP, int nb, const double* c0,
                               SlotView sv, double f, double* out)
{
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t per = (size_t)n * DP;
  if (i >= per * nb) return;
  const int slot = (int)(i / per);
  const size_t j = i - (size_t)slot * per;
  const size_t p = j / DP;
  const int d = (int)(j % DP);
  out[i] = d < D ? (xs[p * D + d] - c0[d]) * (sv.s[slot] * f) : 0.0;
}

template <int DT>
struct PtLoad {
  static constexpr int DP = DT == 1 ? 1 : (DT + 1) / 2 * 2;
  __device__ __forceinline__ static void load(const double* base, int j, double (&v)[DP])
  {
    if constexpr (DT == 1) {
      v[0] = base[j];
    } else {
      const double2* b2 = reinterpret_cast<const double2*>(base + (size_t)j * DP);
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) {
        const double2 t = b2[k];
        v[2 * k] = t.x;
        v[2 * k + 1] = t.y;
      }
    }
  }
  // point j of src -> point j2 of dst (16-byte vectors)
  __device__ __forceinline__ static void copy2(const double* src, int j, double* dst, int j2)
  {
    if constexpr (DT == 1) {
      dst[j2] = src[j];
    } else {
      const double2* s2 = reinterpret_cast<const double2*>(src + (size_t)j * DP);
      double2* d2 = reinterpret_cast<double2*>(dst + (size_t)j2 * DP);
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) d2[k] = s2[k];
    }
  }
  // point j of src -> point j of dst (16-byte vectors)
  __device__ __forceinline__ static void copy(const double* src, int j, double* dst)
  {
    if constexpr (DT == 1) {
      dst[j] = src[j];
    } else {
      const double2* s2 = reinterpret_cast<const double2*>(src + (size_t)j * DP);
      double2* d2 = reinterpret_cast<double2*>(dst + (size_t)j * DP);
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) d2[k] = s2[k];
    }
  }
};

// Compact reference-leaf records for the base case, in sorted item order:
// {first sorted position, count | flags << 28}; flags bit 0: the traversal proved
// y <= 708 for every pair; bit 1: terms may be clamped at 2^-1021; bit 2: the FP32 base
// case applies (see traverse.cu).
__global__ void k_base_records(const Item* items, const int* n, int cap, TreeView R, int2* rec)
{
  const int m = min(*n, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const Item it = items[i];
    const int c = R.count[it.r];
    rec[i] = make_int2(R.begin[it.r], c | ((it.code & 7) << 28));
  }
}

// K10: exhaustive base case (Traversal::base_case, engine.cpp:239-269).  One warp per
// task = (slot, query leaf, 32-query chunk, run of <= kTaskItems reference leaves),
// tasks handed out by an atomic counter (results are written per task, so the order
// of execution does not change a bit).  The task's reference points are staged, as
// one contiguous stream, into the warp's shared-memory tile; LANES RUN OVER REFERENCE
// POINTS and each lane holds a group of G queries in registers, so all 32 lanes are
// busy whatever the leaf sizes (only the stream's last 32-block is partial) and each
// reference point is read once per G pairs.  The G partial sums are combined across
// the warp by a transpose-reduction (G values in log2(32) exchange steps) in a fixed
// order: bit-reproducible.  Chunks whose leaves the traversal proved to have y <= 708
// for every pair run the branch-free table exp; others the careful path (libdevice
// exp beyond the fast range: exact underflow behaviour).
template <int DT>
struct BaseGeo {
  static constexpr int DP = PtLoad<DT>::DP;
#ifndef DFGTB_BASE_G
#define DFGTB_BASE_G 8
#endif
  static constexpr int G = DT <= 2 ? DFGTB_BASE_G : 4;            // queries per lane
#ifndef DFGTB_BASE_GM
#define DFGTB_BASE_GM 8
#endif
#ifndef DFGTB_BASE_GM3
#define DFGTB_BASE_GM3 8  // measured 2-4% faster than 4 on cfg3 / cfg5
#endif
  static constexpr int GM = DT <= 2 ? DFGTB_BASE_GM : DT == 3 ? DFGTB_BASE_GM3 : 4;  // MUFU path
  static constexpr int RMAX = DT == 1 ? 512 : 256;              // stream tile (points)
  static constexpr int WARPS = 4;                                 // per CTA
  static constexpr int DM = (DT + 2) / 2 * 2;                     // MUFU stream stride
  static constexpr int DS = DM > DP ? DM : DP;
  static constexpr int WORDS = RMAX * DS + 32 * DS + 32;          // refs | queries | sums
};

template <int DT, int GG, bool FAST>
__device__ __forceinline__ void base_group(const double* rs, int n, const double* qs, double* qsum,
                                           const double* tab, double ysc, int lane)
{
  constexpr int D = DT, DP = BaseGeo<DT>::DP;
  constexpr int LG = GG == 8 ? 3 : GG == 4 ? 2 : GG == 2 ? 1 : 0;
  double qv[GG][D];
#pragma unroll
  for (int i = 0; i < GG; ++i)
#pragma unroll
    for (int d = 0; d < D; ++d) qv[i][d] = qs[i * DP + d];
  double acc[GG];
#pragma unroll
  for (int i = 0; i < GG; ++i) acc[i] = 0.0;
  const unsigned tabs = (unsigned)__cvta_generic_to_shared(tab);
  auto body = [&](int j) {
    double r[DP];
    PtLoad<DT>::load(rs, j, r);
#pragma unroll
    for (int i = 0; i < GG; ++i) {
      double y = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double t = qv[i][d] - r[d];
        y = fma(t, t, y);
      }
      if constexpr (FAST) acc[i] += exp_negy_s(y, tabs);
      else acc[i] += exp_negy_c(y * ysc, tabs);  // ysc = ln 2 on log2e-scaled points
    }
  };
  // one copy of the body (instruction-cache footprint): lanes past the end of the
  // stream idle in the last 32-block only
  const int nceil = (n + 31) & ~31;
  for (int j = lane; j < nceil; j += 32)
    if (j < n) body(j);
  // transpose-reduction: split steps on lane bits 4, 3, .. (each lane keeps half of its
  // values, adds the partner's copy of that half), then butterflies on the rest
#pragma unroll
  for (int s = 0; s < LG; ++s) {
    const int off = 16 >> s;
    const bool up = lane & off;
    const int h = GG >> (s + 1);
#pragma unroll
    for (int i = 0; i < GG / 2; ++i) {
      if (i < h) {
        const double send = up ? acc[i] : acc[i + h];
        const double keep = up ? acc[i + h] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
  }
#pragma unroll
  for (int off = 16 >> LG; off >= 1; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
  if ((lane & ((32 >> LG) - 1)) == 0) qsum[lane >> (5 - LG)] += acc[0];
}

// A point's DP scaled coordinates in registers (vector loads; staging loads all of a
// tile's points before storing them).
template <int DT>
struct RawPt {
  static constexpr int DP = PtLoad<DT>::DP;
  double x[DP];
  __device__ __forceinline__ static RawPt load(const double* src, int j)
  {
    RawPt r;
    PtLoad<DT>::load(src, j, r.x);
    return r;
  }
  // point j2 of dst (stride DP, 16-byte vectors)
  __device__ __forceinline__ void store(double* dst, int j2) const
  {
    if constexpr (DT == 1) {
      dst[j2] = x[0];
    } else {
      double2* d2 = reinterpret_cast<double2*>(dst + (size_t)j2 * DP);
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) d2[k] = make_double2(x[2 * k], x[2 * k + 1]);
    }
  }
};

// MUFU variant: the stream holds centred (log2e-scaled) points r and |r|^2 (stride DM),
// the query tile the same (q, |q|^2); per pair t = fma(-2q_d, r_d, .. (M + |q|^2) + |r|^2).
template <int DT>
struct MPt {
  static constexpr int DM = (DT + 2) / 2 * 2;  // D coordinates + |r|^2, padded to 16 bytes
  static constexpr int PL = BaseGeo<DT>::RMAX * 2;  // stream: DM / 2 planes of double2
  // stream point j: plane k holds its elements (2k, 2k+1) -- 16-byte lane stride, so a
  // warp's LDS.128 of 32 consecutive points is conflict-free
  __device__ __forceinline__ static void load(const double* base, int j, double (&v)[DM])
  {
#pragma unroll
    for (int k = 0; k < DM / 2; ++k) {
      const double2 t = reinterpret_cast<const double2*>(base + k * PL)[j];
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
  }
  // point j of src (stride DP, log2e-scaled coordinates) -> centred on c, |r|^2
  __device__ __forceinline__ static void centred(const double* src, int j, const double* c,
                                                 double (&v)[DM])
  {
    constexpr int DP = PtLoad<DT>::DP;
    double rr = 0.0;
#pragma unroll
    for (int d = 0; d < DT; ++d) {
      v[d] = src[(size_t)j * DP + d] - c[d];
      rr = fma(v[d], v[d], rr);
    }
    v[DT] = rr;
#pragma unroll
    for (int d = DT + 1; d < DM; ++d) v[d] = 0.0;
  }
  __device__ __forceinline__ static void stage(const RawPt<DT>& p, const double* c, double* dst, int j2)
  {
    double v[DM];
    centred(p.x, 0, c, v);
#pragma unroll
    for (int k = 0; k < DM / 2; ++k)
      reinterpret_cast<double2*>(dst + k * PL)[j2] = make_double2(v[2 * k], v[2 * k + 1]);
  }
  // query tile (broadcast reads): point-major, stride DM
  __device__ __forceinline__ static void stage_q(const double* src, int j, const double* c,
                                                 double* dst)
  {
    double v[DM];
    centred(src, j, c, v);
#pragma unroll
    for (int k = 0; k < DM / 2; ++k)
      reinterpret_cast<double2*>(dst + (size_t)j * DM)[k] = make_double2(v[2 * k], v[2 * k + 1]);
  }
};

template <int DT, int GG, bool CLAMP>
__device__ __forceinline__ void base_group_mufu(const double* rs, int n, const double* qs, double* qsum,
                                                int lane)
{
  constexpr int D = DT, DM = MPt<DT>::DM;
  constexpr int LG = GG == 16 ? 4 : GG == 8 ? 3 : GG == 4 ? 2 : GG == 2 ? 1 : 0;
  double m[GG][D], A[GG], acc[GG];
#pragma unroll
  for (int i = 0; i < GG; ++i) {
#pragma unroll
    for (int d = 0; d < D; ++d) m[i][d] = -2.0 * qs[i * DM + d];
    A[i] = kMufuMagic + qs[i * DM + D];
    acc[i] = 0.0;
  }
  // the G chains of a reference point are written stage by stage (independent
  // instructions back to back) so the warp always has work while one chain waits
  unsigned fbits;
  asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(fbits));  // opaque: stays in a register
  auto body = [&](int j) {
    double r[DM];
    MPt<DT>::load(rs, j, r);
    double t[GG];
#pragma unroll
    for (int i = 0; i < GG; ++i) t[i] = A[i] + r[D];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int i = 0; i < GG; ++i) t[i] = fma(m[i][d], r[d], t[i]);
#pragma unroll
    for (int i = 0; i < GG; ++i) acc[i] += exp2_neg_fixed<CLAMP>(t[i], fbits);
  };
  // full 32-blocks without a predicate, then the partial last block
  const int nfull = n & ~31;
  int j = lane;
  for (; j < nfull; j += 32) body(j);
  if (j < n) body(j);
#pragma unroll
  for (int s = 0; s < LG; ++s) {
    const int off = 16 >> s;
    const bool up = lane & off;
    const int h = GG >> (s + 1);
#pragma unroll
    for (int i = 0; i < GG / 2; ++i) {
      if (i < h) {
        const double send = up ? acc[i] : acc[i + h];
        const double keep = up ? acc[i + h] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
  }
#pragma unroll
  for (int off = 16 >> LG; off >= 1; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
  if ((lane & ((32 >> LG) - 1)) == 0) qsum[lane >> (5 - LG)] += acc[0];
}

template <int DT, int GG, bool CLAMP>
__device__ __noinline__ void base_group_mufu_call(const double* rs, int n, const double* qs,
                                                  double* qsum, int lane)
{
  base_group_mufu<DT, GG, CLAMP>(rs, n, qs, qsum, lane);
}

template <int DT, bool CLAMP>
__device__ __forceinline__ void base_groups_mufu(const double* rs, int n, const double* qs, double* qsum,
                                                 int qc, int lane)
{
  constexpr int DM = MPt<DT>::DM, G = BaseGeo<DT>::GM;
  int g0 = 0;
  for (; g0 + G <= qc; g0 += G) base_group_mufu_call<DT, G, CLAMP>(rs, n, qs + g0 * DM, qsum + g0, lane);
  if constexpr (G >= 16) {
    if (qc - g0 >= 8) {
      base_group_mufu_call<DT, 8, CLAMP>(rs, n, qs + g0 * DM, qsum + g0, lane);
      g0 += 8;
    }
  }
  if constexpr (G >= 8) {
    if (qc - g0 >= 4) {
      base_group_mufu_call<DT, 4, CLAMP>(rs, n, qs + g0 * DM, qsum + g0, lane);
      g0 += 4;
    }
  }
  if (qc - g0 >= 2) {
    base_group_mufu_call<DT, 2, CLAMP>(rs, n, qs + g0 * DM, qsum + g0, lane);
    g0 += 2;
  }
  if (qc - g0 >= 1) base_group_mufu_call<DT, 1, CLAMP>(rs, n, qs + g0 * DM, qsum + g0, lane);
}

// FP32 base case (leaf pairs the traversal flagged with order bit 2: the query leaf's box
// diagonal is <= kF32Diam = 150 in units where |q - r|^2 = z, and the query sums are
// provably >= 1e-20 (Q != R) or >= 1 (Q = R: the self term)).  Points are
// centred on the query leaf's box centre in FP64 (every query within 75 of it) and rounded
// to FP32 (q~, r~), and per pair
//   z' = sum_d (q~_d - r~_d)^2 - S,   term = ex2.approx.ftz(-z') = 2^S 2^-z,   S = kF32Shift = 64,
// D FP32 subtractions, D multiply-adds (the first one adds -S), one MUFU and one FP32 add:
// no FP64 instruction in the pair loop; each tile's FP32 sum is scaled back by 2^-S
// exactly in FP64.  The shift keeps terms down to 2^-190 (z <= 190) out of the flush
// range at no cost (sums of <= 256 terms <= 2^S per tile stay below 2^72).  Terms below
// 2^-190 flush to 0: absolute error <= |R| 2^-190, against sums >= 1e-20 (Q != R) or
// >= 1 (Q = R: below the 2^-53 resolution of the FP64 sum G that is returned, from which
// the CV scores form G - 1, cv.cpp:17-25).  Q = R: the self pairs
// are masked out of the FP32 sums (their tiles run the SELF variant) and K(0) = 1 is
// added exactly in FP64 at the end, so the partial sums hold only G - 1, to 21 u relative.
// Per-term relative error for z <= 127 (|q| <= 75, |r| <= 75 + sqrt z, unit roundoff
// u = 2^-24; z = sum_d a_d^2 with a_d = q~_d - r~_d):
//   coordinate rounding   |d(q - r)| <= u (|q| + |r|) <= u (150 + sqrt z)
//                         -> |dz| <= 2 sqrt(z) u (150 + sqrt z)
//   differences           a~_d = a_d (1 + d), |d| <= u        -> |dz| <= 2 z u
//   squares and sums      D roundings of partial sums, each <= max(z, S) <= 127
//                                                              -> |dz| <= D 127 u
//   total at z = 127, D = 5:
//     2 sqrt(127) (150 + sqrt(127)) u + 2 127 u + 5 127 u
//       = 3635 u + 254 u + 635 u = 4524 u = 2.70e-4 = 2 sqrt(127) (150 + 2 sqrt(127)) u + 5 127 u,
//   |dz| ln 2 <= 1.87e-4 relative, + ex2.approx (< 2^-22 = 2.4e-7 over every argument in
//   [-126, S], measured exhaustively by dfgtb_f32_exp_error) + FP32 partial sums (<= 16
//   roundings per lane + 5 reduction levels: 21 u = 1.3e-6): 1.89e-4 < kF32Charge = 2e-4,
//   which the traversal pays for.  Terms with 127 < z <= 190 (below 2^-127 each) carry up
//   to 2.5e-4 relative error but weigh at most |R| 2^-127 against G >= 1e-20 (Q != R) or
//   G >= 1 (Q = R): below 1e-15 of G, inside the charge's margin.
template <int DT>
struct FPt {
  static constexpr int DF = DT <= 4 ? 4 : 8;  // floats per point (coordinates, pad)
  static constexpr int DP = PtLoad<DT>::DP;
  struct Raw {
    double x[DT];
  };
  __device__ __forceinline__ static Raw load_raw(const double* src, int j)
  {
    Raw r;
#pragma unroll
    for (int d = 0; d < DT; ++d) r.x[d] = __ldg(src + (size_t)j * DP + d);
    return r;
  }
  // coordinates centred on c (FP64), rounded to FP32
  __device__ __forceinline__ static void centred(const Raw& p, const double* c, float (&v)[DF])
  {
#pragma unroll
    for (int d = 0; d < DT; ++d) v[d] = (float)(p.x[d] - c[d]);
#pragma unroll
    for (int d = DT; d < DF; ++d) v[d] = 0.f;
  }
};

__device__ __forceinline__ float ex2_ftz(float t)
{
  float g;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(t));
  return g;
}

// z - kF32Shift = |q~ - r~|^2 - 64 in FP32, in the loop's order
template <int DT>
__device__ __forceinline__ float f32_z(const float* q, const float* r)
{
  const float a0 = q[0] - r[0];
  float z = fmaf(a0, a0, -kF32Shift);
#pragma unroll
  for (int d = 1; d < DT; ++d) {
    const float a = q[d] - r[d];
    z = fmaf(a, a, z);
  }
  return z;
}

// One FP32 pair term exactly as the loop forms it, still scaled by 2^kF32Shift (tests).
template <int DT>
__device__ __forceinline__ float f32_term(const float* q, const float* r)
{
  return ex2_ftz(-f32_z<DT>(q, r));
}

// P2 partial sums per lane (lanes over points) combined across the warp by a
// transpose-reduction in a fixed order: lane l ends with the sum of value l >> (5 - LG).
template <int P2, int LG>
__device__ __forceinline__ float transpose_reduce(float (&acc)[P2], int lane)
{
#pragma unroll
  for (int s = 0; s < LG; ++s) {
    const int off = 16 >> s;
    const bool up = lane & off;
    const int h = P2 >> (s + 1);
#pragma unroll
    for (int i = 0; i < P2 / 2; ++i) {
      if (i < h) {
        const float send = up ? acc[i] : acc[i + h];
        const float keep = up ? acc[i + h] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
  }
#pragma unroll
  for (int off = 16 >> LG; off >= 1; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
  return acc[0];
}

// Queries in groups of G, the remainder in groups of 4, 2, 1.  Each group size is one
// out-of-line copy, to keep the kernel's hot code small.
template <int DT, int GG, bool FAST>
__device__ __noinline__ void base_group_call(const double* rs, int n, const double* qs, double* qsum,
                                             const double* tab, double ysc, int lane)
{
  base_group<DT, GG, FAST>(rs, n, qs, qsum, tab, ysc, lane);
}

template <int DT, bool FAST>
__device__ __forceinline__ void base_groups(const double* rs, int n, const double* qs, double* qsum,
                                            int qc, const double* tab, double ysc, int lane)
{
  constexpr int DP = BaseGeo<DT>::DP, G = BaseGeo<DT>::G;
  int g0 = 0;
  for (; g0 + G <= qc; g0 += G)
    base_group_call<DT, G, FAST>(rs, n, qs + g0 * DP, qsum + g0, tab, ysc, lane);
  if constexpr (G >= 8) {
    if (qc - g0 >= 4) {
      base_group_call<DT, 4, FAST>(rs, n, qs + g0 * DP, qsum + g0, tab, ysc, lane);
      g0 += 4;
    }
  }
  if (qc - g0 >= 2) {
    base_group_call<DT, 2, FAST>(rs, n, qs + g0 * DP, qsum + g0, tab, ysc, lane);
    g0 += 2;
  }
  if (qc - g0 >= 1) base_group_call<DT, 1, FAST>(rs, n, qs + g0 * DP, qsum + g0, tab, ysc, lane);
}

#ifndef DFGTB_BASE_MINB
#define DFGTB_BASE_MINB 4  // CTAs per SM: 125 registers, chains interleaved by ptxas
#endif
// A base-case task as one warp sees it: lane k < nit holds item k's record; the
// items' points form one stream (item k at stream positions [sk, sk + count)).
struct TaskView {
  int slot, leaf, nit, qc, qb, total, sk, okk;
  int2 rc;
};

__device__ __forceinline__ TaskView task_view(const BTask& t, TreeView Q, int K, const int2* rec, int lane)
{
  TaskView v;
  v.slot = t.key / K;
  v.leaf = t.key - v.slot * K;
  v.nit = t.item1 - t.item0;  // all records at once (kTaskItems <= 32)
  v.rc = lane < v.nit ? rec[t.item0 + lane] : make_int2(0, 0);
  v.qc = min(32, Q.count[v.leaf] - t.q0);
  v.qb = Q.begin[v.leaf];
  const int cnt = v.rc.y & 0x0FFFFFFF;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < kTaskItems; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  v.total = __shfl_sync(0xffffffffu, incl, kTaskItems - 1);
  v.sk = incl - cnt;       // lane k < nit: stream start of item k
  v.okk = v.rc.x - v.sk;   // its source position = okk + stream position
  return v;
}

// Stage the stream of an item set (lane k < ni: item k starts at stream position skk,
// source position = ok + stream position) in tiles of RMAX positions and run `groups` on
// each tile.  Owner item of position c0 + 32 i + lane: (items started at
// or before c0) + (starts in word i at or below this lane's bit) + (starts in earlier
// words) - 1, from a bit mask of the item starts.  Global loads of B positions per lane
// are issued back to back before their shared-memory stores (one L2 round trip per B,
// not per point).
#ifndef DFGTB_STAGE_B
#define DFGTB_STAGE_B 4  // measured: 8 spills and is 2% slower on cfg2
#endif
#ifndef DFGTB_STAGE_B3
#define DFGTB_STAGE_B3 0  // D = 3 override (0: the rule below)
#endif
constexpr int stage_batch(int D)
{
  return D == 3 && DFGTB_STAGE_B3 > 0 ? DFGTB_STAGE_B3
         : (DFGTB_STAGE_B >> (D <= 2 ? 0 : D <= 4 ? 1 : 2)) > 0 ? (DFGTB_STAGE_B >> (D <= 2 ? 0 : D <= 4 ? 1 : 2))
                                                                 : 1;
}
template <int RMAX, int B, class Load, class Store, class Groups>
__device__ __forceinline__ void stream_passes(unsigned* smask, int ni, int skk, int ok, int tot, int lane,
                                              Load load, Store store, Groups groups)
{
  for (int c0 = 0; c0 < tot; c0 += RMAX) {
    const int n = min(RMAX, tot - c0);
    if (lane < RMAX / 32) smask[lane] = 0u;
    __syncwarp();
    if (lane < ni && skk > c0 && skk < c0 + n) atomicOr(&smask[(skk - c0) >> 5], 1u << ((skk - c0) & 31));
    int kb = __popc(__ballot_sync(0xffffffffu, lane < ni && skk <= c0)) - 1;
    __syncwarp();
    const unsigned le = 0xffffffffu >> (31 - lane);
    for (int i0 = 0; 32 * i0 < n; i0 += B) {
      decltype(load(0)) buf[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int e = lane + 32 * (i0 + b);
        const unsigned wm = smask[i0 + b];
        const int off = __shfl_sync(0xffffffffu, ok, kb + __popc(wm & le));
        kb += __popc(wm);
        if (e < n) buf[b] = load(off + c0 + e);
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int e = lane + 32 * (i0 + b);
        if (e < n) store(buf[b], e);
      }
    }
    __syncwarp();
    groups(n, c0);
    __syncwarp();
  }
}

// Tasks of one base-case kernel: indices into the task array, split by the path their
// leaf pairs qualify for (k_task_split); results go to part[task * 32 + query].
__device__ __forceinline__ int next_task(int* next, int lane)
{
  int w = 0;
  if (lane == 0) w = atomicAdd(next, 1);
  return __shfl_sync(0xffffffffu, w, 0);
}

template <int DT>
__global__ void __launch_bounds__(BaseGeo<DT>::WARPS * 32, DFGTB_BASE_MINB)
  k_base_case(TreeView Q, int K, const BTask* tasks, const int* tlist, const int* ntl, const int2* rec,
              const double* xq, const double* xr, int nq, int nr, double* part, int* next, int mufu,
              const double* c0, SlotView sv, double f)
{
  const int nl = *ntl;
  using Geo = BaseGeo<DT>;
  constexpr int DP = Geo::DP, RMAX = Geo::RMAX;
  __shared__ __align__(512) double tab[64];
  extern __shared__ __align__(16) double dsm[];  // WARPS x WORDS (dynamic: > 48 KB for D >= 3)
  __shared__ unsigned smask_all[Geo::WARPS][RMAX / 32];
  if (threadIdx.x < 64) tab[threadIdx.x] = c_exp2tab[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double* rs = dsm + (size_t)(threadIdx.x >> 5) * Geo::WORDS;
  double* qs = rs + RMAX * Geo::DS;
  double* qsum = qs + 32 * Geo::DS;
  unsigned* smask = smask_all[threadIdx.x >> 5];
  for (int i = next_task(next, lane); i < nl;) {
    const int w = tlist[i];
    const BTask t = tasks[w];
    const int inext = next_task(next, lane);  // the next task, fetched early
    const TaskView v = task_view(t, Q, K, rec, lane);
    const bool fast = __all_sync(0xffffffffu, lane >= v.nit || (v.rc.y & (1 << 28)));
    const bool clampok = __all_sync(0xffffffffu, lane >= v.nit || (v.rc.y & (3 << 28)));
    const bool mf = (fast || clampok) && (mufu & 1);
    const double* qsrc = xq + ((size_t)v.slot * nq + v.qb + t.q0) * DP;
    double cq[DT];  // MUFU path: centre = the chunk's first query
#pragma unroll
    for (int d = 0; d < DT; ++d) cq[d] = qsrc[d];
    if (lane < v.qc) {
      if (mf) MPt<DT>::stage_q(qsrc, lane, cq, qs);
      else PtLoad<DT>::copy(qsrc, lane, qs);
    }
    qsum[lane] = 0.0;
    const double* xrs = xr + (size_t)v.slot * nr * DP;
    stream_passes<RMAX, stage_batch(DT)>(
      smask, v.nit, v.sk, v.okk, v.total, lane, [&](int src) { return RawPt<DT>::load(xrs, src); },
      [&](const RawPt<DT>& p, int pos) {
        if (mf) MPt<DT>::stage(p, cq, rs, pos);
        else p.store(rs, pos);
      },
      [&](int n, int) {
        if (mf && fast) base_groups_mufu<DT, false>(rs, n, qs, qsum, v.qc, lane);
        else if (mf) base_groups_mufu<DT, true>(rs, n, qs, qsum, v.qc, lane);
        else if (fast) base_groups<DT, true>(rs, n, qs, qsum, v.qc, tab, 1.0, lane);
        else base_groups<DT, false>(rs, n, qs, qsum, v.qc, tab, (mufu & 1) ? kLn2 : 1.0, lane);
      });
    // Q = R: the run holding the query leaf itself contains every query's self pair,
    // whose MUFU value is 1 +- O(2^-20).  Replace it by exactly K(0) = 1 (the LOO CV
    // scores subtract exactly 1): recompute it with the loop's own operations and order.
    if (mf && xq == xr && __any_sync(0xffffffffu, lane < v.nit && v.rc.x == v.qb) && lane < v.qc) {
      constexpr int DM = MPt<DT>::DM;
      unsigned fbits;
      asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(fbits));
      const double qq = qs[lane * DM + DT];
      double tq = (kMufuMagic + qq) + qq;
#pragma unroll
      for (int d = 0; d < DT; ++d) tq = fma(-2.0 * qs[lane * DM + d], qs[lane * DM + d], tq);
      qsum[lane] += 1.0 - exp2_neg_fixed<false>(tq, fbits);
    }
    __syncwarp();
    if (lane < v.qc) part[(size_t)w * 32 + lane] = qsum[lane];
    __syncwarp();
    i = inext;
  }
}

// ---- packed FP32x2 base case (Blackwell FADD2 / FFMA2) ------------------------------
// Lanes own reference points (P per pass, registers); the warp walks the task's queries
// in PAIRS: one packed instruction forms a coordinate difference for two queries against
// one point (the point's coordinate is the instruction's scalar broadcast operand, so
// points are stored once, not duplicated), so per two (q, r) pairs the loop issues
// D FADD2 + D FFMA2 (the first one adds -S) + 2 MUFU.EX2 + 1 FADD2 (accumulate): 3.5
// issue slots per pair at D = 2 against the MUFU rate's budget of 8.  The arithmetic per
// term is exactly FPt's (q~ + (-r~) = q~ - r~; FFMA onto -S, FFMAs, all round-to-nearest),
// so kF32Charge's derivation holds; each lane's accumulator of a query sums
// <= RMAX / 32 = 16 terms per tile.
//   points: negated centred FP32 coordinates, zero padded to PF floats per point, in
//           planes of V-float vectors (conflict-free LDS.64 / LDS.128 per lane);
//   queries: pair k, dimension d at float2 index k * DT + d = (q_2k[d], q_2k+1[d]);
//            padding queries (>= qc) sit at 1e18 (their terms are 0, their sums unused).
#ifndef DFGTB_F32_KB
#define DFGTB_F32_KB 2
#endif
template <int DT>
struct F2Pt {
  static constexpr int PF = DT <= 2 ? 2 : DT <= 4 ? 4 : 8;  // floats per point
  static constexpr int V = PF >= 4 ? 4 : 2;                 // floats per vector
  static constexpr int NPL = PF / V;                        // planes
#ifndef DFGTB_F32_RMAX
#define DFGTB_F32_RMAX 512  // measured: 11% faster than 256 on cfg3 / cfg5 with 512-point runs
#endif
  static constexpr int RMAX = DFGTB_F32_RMAX;
  static constexpr int PL = RMAX * V;                       // floats per plane
  static constexpr int P = DT <= 3 ? 4 : 2;                 // points per lane per pass
  static constexpr int QF = 32 * DT;                        // floats of the query tile
  static constexpr int FLOATS = RMAX * PF + QF;
  __device__ __forceinline__ static void store(const typename FPt<DT>::Raw& p, const double* c, float* dst, int j)
  {
    float v[PF];
#pragma unroll
    for (int d = 0; d < DT; ++d) v[d] = -(float)(p.x[d] - c[d]);
#pragma unroll
    for (int k = DT; k < PF; ++k) v[k] = 0.f;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      if constexpr (V == 4)
        reinterpret_cast<float4*>(dst + k * PL)[j] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      else
        reinterpret_cast<float2*>(dst + k * PL)[j] = make_float2(v[2 * k], v[2 * k + 1]);
    }
  }
  __device__ __forceinline__ static void load(const float* base, int j, float (&r)[DT])
  {
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      float t[V];
      if constexpr (V == 4) {
        const float4 u = reinterpret_cast<const float4*>(base + k * PL)[j];
        t[0] = u.x; t[1] = u.y; t[2] = u.z; t[3] = u.w;
      } else {
        const float2 u = reinterpret_cast<const float2*>(base + k * PL)[j];
        t[0] = u.x; t[1] = u.y;
      }
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (V * k + i < DT) r[V * k + i] = t[i];
    }
  }
  // query `lane` of the chunk (lane >= qc: padding) into the pair layout
  __device__ __forceinline__ static void stage_q(const double* src, int lane, int qc, const double* c, float* qs)
  {
    float v[DT];
    if (lane < qc) {
      const typename FPt<DT>::Raw p = FPt<DT>::load_raw(src, lane);
#pragma unroll
      for (int d = 0; d < DT; ++d) v[d] = (float)(p.x[d] - c[d]);
    } else {
#pragma unroll
      for (int d = 0; d < DT; ++d) v[d] = 1e18f;
    }
#pragma unroll
    for (int d = 0; d < DT; ++d) qs[((lane >> 1) * DT + d) * 2 + (lane & 1)] = v[d];
  }
};

// One tile of n <= RMAX points against the chunk's qc queries; adds each query's tile sum
// (scaled back by 2^-S) to qsum (FP64).  SELF: query k's own point sits at tile position
// sb + k (Q = R); those pairs are masked to 0 (the caller adds K(0) = 1 exactly).
template <int DT, bool SELF>
__device__ __forceinline__ void base_tile_f32x2(const float* rs, int n, const float* qs, double* qsum, int qc,
                                                int lane, int sb)
{
  constexpr int P = F2Pt<DT>::P;
  constexpr int KB = DFGTB_F32_KB;  // query pairs per branch-free block
  const float2* q2 = reinterpret_cast<const float2*>(qs);
  const int np = (qc + 1) >> 1;
  const float2 mS = make_float2(-kF32Shift, -kF32Shift);
  float2 acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = make_float2(0.f, 0.f);
  for (int c = 0; c < n; c += 32 * P) {
    float r[P][DT];
    int dl[P];  // SELF: the chunk query whose own point point p is
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int j = c + 32 * p + lane;
      if constexpr (SELF) dl[p] = j - sb;
      if (j < n) F2Pt<DT>::load(rs, j, r[p]);
      else
#pragma unroll
        for (int d = 0; d < DT; ++d) r[p][d] = -1e18f;
    }
#pragma unroll
    for (int k = 0; k < 16; k += KB) {
      if (k < np) {  // KB query pairs per block, branch-free inside (padding queries add 0)
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          float2 q[DT];
#pragma unroll
          for (int d = 0; d < DT; ++d) q[d] = q2[(k + kk) * DT + d];
          float2 e[P];
#pragma unroll
          for (int p = 0; p < P; ++p) {
            float2 a = __fadd2_rn(q[0], make_float2(r[p][0], r[p][0]));  // scalar broadcast operand
            float2 z = __ffma2_rn(a, a, mS);
#pragma unroll
            for (int d = 1; d < DT; ++d) {
              a = __fadd2_rn(q[d], make_float2(r[p][d], r[p][d]));
              z = __ffma2_rn(a, a, z);
            }
            e[p] = make_float2(ex2_ftz(-z.x), ex2_ftz(-z.y));
            if constexpr (SELF) {
              if (dl[p] == 2 * (k + kk)) e[p].x = 0.f;
              if (dl[p] == 2 * (k + kk) + 1) e[p].y = 0.f;
            }
          }
          // the P terms by a fixed tree, then into the accumulator
#pragma unroll
          for (int w = P / 2; w >= 1; w >>= 1)
#pragma unroll
            for (int p = 0; p < w; ++p) e[p] = __fadd2_rn(e[p], e[p + w]);
          acc[k + kk] = __fadd2_rn(acc[k + kk], e[0]);
        }
      }
    }
  }
  float a32[32];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    a32[2 * k] = acc[k].x;
    a32[2 * k + 1] = acc[k].y;
  }
  const float v = transpose_reduce<32, 5>(a32, lane);  // lane l: query l's tile sum
  if (lane < qc) qsum[lane] += (double)v * kF32Unshift;  // 2^-S, exact
}

// FP32 base case kernel (tasks whose every leaf pair carries order bit 2).
// A base-case task's metadata (from its packed list record).
template <int DT>
struct TaskMeta {
  int w, key, item0, nit, q0;
  int2 rc;         // lane < nit: item lane's record
  int qcount, qb;  // query leaf count and first position
  double cen[DT];  // query leaf's box centre
  double s;        // slot scale
};

template <int DT>
__device__ __forceinline__ TaskMeta<DT> fetch_meta(const int4& r, bool ok, TreeView Q, int K, const int2* rec,
                                                   SlotView sv, int lane)
{
  TaskMeta<DT> m;
  m.w = r.w;
  m.key = r.x;
  m.item0 = r.y;
  m.nit = r.z & 63;
  m.q0 = (r.z >> 6) << 5;
  const int slot = ok ? r.x / K : 0, leaf = ok ? r.x - slot * K : 0;
  m.rc = ok && lane < m.nit ? rec[m.item0 + lane] : make_int2(0, 0);
  m.qcount = ok ? Q.count[leaf] : 0;
  m.qb = ok ? Q.begin[leaf] : 0;
#pragma unroll
  for (int d = 0; d < DT; ++d) m.cen[d] = ok ? Q.cen[(size_t)leaf * DT + d] : 0.0;
  m.s = ok ? sv.s[slot] : 0.0;
  return m;
}

// TaskView from prefetched metadata (same fields as task_view, no memory access).
__device__ __forceinline__ TaskView task_view_m(int key, int K, int nit, int q0, int2 rc, int qcount, int qb, int lane)
{
  TaskView v;
  v.slot = key / K;
  v.leaf = key - v.slot * K;
  v.nit = nit;
  v.rc = rc;
  v.qc = min(32, qcount - q0);
  v.qb = qb;
  const int cnt = v.rc.y & 0x0FFFFFFF;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < kTaskItems; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  v.total = __shfl_sync(0xffffffffu, incl, kTaskItems - 1);
  v.sk = incl - cnt;
  v.okk = v.rc.x - v.sk;
  return v;
}

template <int DT>
struct F32Geo {
  static constexpr int RMAX = F2Pt<DT>::RMAX;  // stream tile (points)
  static constexpr int WARPS = 4;
  static constexpr int FLOATS = F2Pt<DT>::FLOATS;  // stream | query tile
};
#ifndef DFGTB_BF32_MINB
#define DFGTB_BF32_MINB 5
#endif
// Tasks come from the packed list (one 16-byte record per task; measured: prefetching
// the next task's metadata a task ahead gains nothing -- the MUFU pipe, not the fetch
// chain, bounds this kernel).
template <int DT>
__global__ void __launch_bounds__(F32Geo<DT>::WARPS * 32, DFGTB_BF32_MINB)
  k_base_f32(TreeView Q, int K, const int4* tl, const int* ntl, const int2* rec, const double* xq,
             const double* xr, int nq, int nr, double* part, int* next, const double* c0, SlotView sv,
             double f)
{
  using Geo = F32Geo<DT>;
  constexpr int DP = PtLoad<DT>::DP, RMAX = Geo::RMAX;
  const int nl = *ntl;
  extern __shared__ __align__(16) float fsm[];  // WARPS x FLOATS
  __shared__ double qsum_all[Geo::WARPS][32];
  __shared__ unsigned smask_all[Geo::WARPS][RMAX / 32];
  const int lane = threadIdx.x & 31;
  float* rs = fsm + (size_t)(threadIdx.x >> 5) * Geo::FLOATS;
  float* qs = rs + RMAX * F2Pt<DT>::PF;
  double* qsum = qsum_all[threadIdx.x >> 5];
  unsigned* smask = smask_all[threadIdx.x >> 5];
  for (int i = next_task(next, lane); i < nl;) {
    const int4 r4 = tl[i];
    const int inext = next_task(next, lane);
    const TaskMeta<DT> mc = fetch_meta<DT>(r4, true, Q, K, rec, sv, lane);
    const TaskView v = task_view_m(mc.key, K, mc.nit, mc.q0, mc.rc, mc.qcount, mc.qb, lane);
    const double* qsrc = xq + ((size_t)v.slot * nq + v.qb + mc.q0) * DP;
    double cq[DT];  // centre = the query leaf's box centre, scaled like the points
    const double sc = mc.s * f;
#pragma unroll
    for (int d = 0; d < DT; ++d) cq[d] = (mc.cen[d] - c0[d]) * sc;
    F2Pt<DT>::stage_q(qsrc, lane, v.qc, cq, qs);
    qsum[lane] = 0.0;
    const double* xrs = xr + (size_t)v.slot * nr * DP;
    // Q = R: the item that is the query leaf itself holds every query's self pair, at
    // stream position sself + k for chunk query k
    int sself = -1;
    if (xq == xr) {
      const unsigned bm = __ballot_sync(0xffffffffu, lane < v.nit && v.rc.x == v.qb);
      if (bm) sself = __shfl_sync(0xffffffffu, v.sk, __ffs(bm) - 1) + mc.q0;
    }
#if defined(DFGTB_EXP_NOSTAGE)  // timing experiments only (results wrong)
    for (int c0t = 0; c0t < v.total; c0t += RMAX)
      base_tile_f32x2<DT, false>(rs, min(RMAX, v.total - c0t), qs, qsum, v.qc, lane, 0);
#else
    stream_passes<RMAX, stage_batch(DT)>(
      smask, v.nit, v.sk, v.okk, v.total, lane, [&](int src) { return FPt<DT>::load_raw(xrs, src); },
      [&](const typename FPt<DT>::Raw& p, int pos) { F2Pt<DT>::store(p, cq, rs, pos); },
      [&](int n, int c0t) {
#if !defined(DFGTB_EXP_NOCOMPUTE)
        const int sb = sself - c0t;  // tile position of chunk query 0's own point
        if (sself >= 0 && sb < n && sb + v.qc > 0) base_tile_f32x2<DT, true>(rs, n, qs, qsum, v.qc, lane, sb);
        else base_tile_f32x2<DT, false>(rs, n, qs, qsum, v.qc, lane, 0);
#endif
      });
#endif
    __syncwarp();
    if (lane < v.qc) part[(size_t)mc.w * 32 + lane] = qsum[lane] + (sself >= 0 ? 1.0 : 0.0);  // + K(0) exactly
    __syncwarp();
    i = inext;
  }
}

// Split the task array by path: tasks whose every item carries order bit 2 (and the
// engine runs the FP32 base case) -> list A, the rest -> list B.  cnt[0], cnt[1] count
// them (zeroed by the caller).  The order inside a list is irrelevant: every task
// writes its own partial sums.
__global__ void k_task_split(const int* leaves, int nleaves, int nb, int K, const int* cntB,
                             const int* leaf_task, const int* leaf_runs, TreeView Q, int tcap,
                             const int* tflag, int f32, int* listA, int* listB, int* cnt,
                             const BTask* tasks, int4* l4A, int4* l4B)
{
  // one warp per (slot, leaf) key in key order, lanes over its tasks: the lists keep a
  // key's tasks together (the query tile and reference leaves stay hot in L1 / L2)
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nleaves * nb;
       i += (gridDim.x * blockDim.x) >> 5) {
    const int slot = i / nleaves;
    const int leaf = leaves[i - slot * nleaves];
    const int key = slot * K + leaf;
    if (!cntB[key]) continue;
    const int t0 = leaf_task[key];
    const int nt = leaf_runs[key] * ((Q.count[leaf] + 31) / 32);
    for (int j0 = 0; j0 < nt; j0 += 32) {
      const int w = t0 + j0 + lane;
      const bool in = j0 + lane < nt && w < tcap;
      const bool a = in && f32 && tflag[w];
      const unsigned ma = __ballot_sync(0xffffffffu, a), mb = __ballot_sync(0xffffffffu, in && !a);
      int baseA = 0, baseB = 0;
      if (lane == 0) {
        if (ma) baseA = atomicAdd(cnt, __popc(ma));
        if (mb) baseB = atomicAdd(cnt + 1, __popc(mb));
      }
      baseA = __shfl_sync(0xffffffffu, baseA, 0);
      baseB = __shfl_sync(0xffffffffu, baseB, 0);
      // packed copies {key, item0, nit | (q0 / 32) << 6, w}: the base kernels' task fetch
      // is ONE 16-byte load (no index -> record chain)
      int4 rec4 = make_int4(0, 0, 0, 0);
      if (in) {
        const BTask t = tasks[w];
        rec4 = make_int4(t.key, t.item0, (t.item1 - t.item0) | ((t.q0 >> 5) << 6), w);
      }
      if (a) {
        listA[baseA + __popc(ma & below)] = w;
        l4A[baseA + __popc(ma & below)] = rec4;
      } else if (in) {
        listB[baseB + __popc(mb & below)] = w;
        l4B[baseB + __popc(mb & below)] = rec4;
      }
    }
  }
}

// (q, r) pairs of the tasks in a list (diagnostics: Engine::base_split)
__global__ void k_task_pairs(const BTask* tasks, const int* list, const int* nl, const int2* rec, TreeView Q,
                             int K, unsigned long long* out)
{
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  unsigned long long acc = 0;
  for (int i = w0; i < *nl; i += nw) {
    const BTask t = tasks[list[i]];
    const int k = t.item0 + lane;
    const unsigned c = k < t.item1 ? (unsigned)(rec[k].y & 0x0FFFFFFF) : 0u;
    const unsigned tot = __reduce_add_sync(0xffffffffu, c);
    acc += (unsigned long long)tot * (unsigned long long)min(32, Q.count[t.key % K] - t.q0);
  }
  if (lane == 0 && acc) atomicAdd(out, acc);
}

// Generic dimension (D > 5): scalar loads of the scaled coordinates, libdevice exp.
__global__ void __launch_bounds__(kBlock) k_base_case_any(TreeView Q, TreeView R, int K, int D,
                                                          const BTask* tasks, const int* ntasks_p,
                                                          int tcap,
                                                          const Item* items, const double* xq,
                                                          const double* xr, int nq, int nr,
                                                          double* part)
{
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ntasks = min(*ntasks_p, tcap);
  for (int w = w0; w < ntasks; w += nw) {
    const BTask t = tasks[w];
    const int slot = t.key / K, leaf = t.key - slot * K;
    const double* xqs = xq + (size_t)slot * nq * D;
    const double* xrs = xr + (size_t)slot * nr * D;
    const int qb = Q.begin[leaf] + t.q0;
    const bool act = lane < Q.count[leaf] - t.q0;
    double q[kMaxDim];
    for (int d = 0; d < D; ++d) q[d] = xqs[(size_t)(act ? qb + lane : qb) * D + d];
    double acc = 0.0;
    for (int k = t.item0; k < t.item1; ++k) {
      const int r = items[k].r;
      const double* rp = xrs + (size_t)R.begin[r] * D;
      for (int j = 0; j < R.count[r]; ++j) {
        double y = 0.0;
        for (int d = 0; d < D; ++d) {
          const double ta = q[d] - rp[(size_t)j * D + d];
          y = fma(ta, ta, y);
        }
        acc += exp(-y);
      }
    }
    part[(size_t)w * 32 + lane] = acc;
  }
}

// ---------------------------------------------------------------- far field
// ancestor of `leaf` (depth dep) at depth k <= dep: the precomputed chain, or a parent
// walk for leaves at least kMaxAnc deep
__device__ __forceinline__ int ancestor_at(const TreeView& Q, int leaf, int dep, int k)
{
  if (dep < kMaxAnc) return Q.anc[(size_t)leaf * kMaxAnc + k];
  int node = leaf;
  for (int j = dep; j > k; --j) node = Q.parent[node];
  return node;
}

// Every query evaluates the far-field expansions attached to its leaf or any ancestor,
// root first (eval_farfield per query, engine.cpp:200-211).  One warp per (slot, leaf).
__global__ void __launch_bounds__(kBlock) k_farfield(DevSeries g, TreeView Q, TreeView R, int K,
                                                     int nb, const int* leaves, int nleaves,
                                                     const int* cnt, const int* off,
                                                     const Item* items, const double* Mt,
                                                     SlotView sv, int nq, double* s_ff)
{
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int D = g.D;
  for (int li = w0; li < nleaves * nb; li += nw) {
    const int slot = li / nleaves;
    const int leaf = leaves[li - slot * nleaves];
    const double s = sv.s[slot];
    const double* spw = sv.spow + (size_t)slot * kSPow;
    const int qb = Q.begin[leaf], qc = Q.count[leaf];
    const int dep = Q.depth[leaf];
    for (int q0 = 0; q0 < qc; q0 += 32) {
      const int qi = q0 + lane;
      const bool act = qi < qc;
      const double* qp = Q.xs + (size_t)(qb + (act ? qi : 0)) * D;
      double acc = 0.0;
      for (int k = 0; k <= dep; ++k) {
        const int key = slot * K + ancestor_at(Q, leaf, dep, k);
        const int c = cnt[key];
        const Item* it = items + off[key];
        for (int t = 0; t < c; ++t) {
          const int r = it[t].r, order = it[t].code & 0xff;
          acc += dev_eval_farfield(g, Mt + (size_t)r * g.T, R.cen + (size_t)r * D, qp, s, order,
                                   spw, g.pos);
        }
      }
      if (act) s_ff[(size_t)slot * nq + qb + qi] = acc;
    }
  }
}

// Specialised far-field evaluation for the default tables (p_max == PM).  With
// t = (q - c) s, h_k the Hermite polynomials and the Gaussian factored out of the
// Hermite functions (prod_d exp(-t_d^2) = exp(-|t|^2), ONE exp per (query, item)):
//   sum_a M_a s^|a| prod_d H_{a_d}(t_d) = exp(-|t|^2) sum_a M_a prod_d (s^{a_d} h_{a_d}(t_d)),
// contracted one dimension at a time (last dimension first; position layout p =
// sum_d a_d PM^(D-1-d)) over the truncation cube a_d < order: PM^D + PM^(D-1) + ..
// FMAs instead of (D + 1) PM^D multiplies.  The moments are warp-uniform 16-byte loads.
template <int D, int PM, int O>
__device__ __forceinline__ double ff_eval_o(const double* Mt, const double (&h)[D][PM])
{  // contraction over the truncation cube a_d < O (moments in position layout, stride PM)
  constexpr int NO = ipow_c(O, D);
  double v[NO];
#pragma unroll
  for (int p = 0; p < NO; ++p) {
    int rest = p, pos = 0, mul = 1;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      pos += (rest % O) * mul;
      rest /= O;
      mul *= PM;
    }
    v[p] = Mt[pos];
  }
  int len = NO;
#pragma unroll
  for (int d = D - 1; d >= 0; --d) {
    len /= O;
#pragma unroll
    for (int r = 0; r < ipow_c(O, D - 1); ++r) {
      if (r < len) {
        double acc = 0.0;
#pragma unroll
        for (int k = O - 1; k >= 0; --k) acc = fma(v[r * O + k], h[d][k], acc);
        v[r] = acc;
      }
    }
  }
  return v[0];
}

template <int D, int PM>
__device__ __forceinline__ double ff_eval_t(const double* Mt, const double* c, const double* q,
                                            double s, int order,
                                            const double (&spw)[D * (PM - 1) + 1])
{
  double h[D][PM];
  double tt = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double t = (q[d] - c[d]) * s;
    tt = fma(t, t, tt);
    h[d][0] = 1.0;
    if (PM > 1) h[d][1] = 2.0 * t;
#pragma unroll
    for (int k = 1; k + 1 < PM; ++k) h[d][k + 1] = fma(2.0 * t, h[d][k], -2.0 * k * h[d][k - 1]);
#pragma unroll
    for (int k = 1; k < PM; ++k) h[d][k] *= spw[k];
  }
  double v;
  switch (order) {  // warp-uniform: one item per iteration for the whole warp
  case 1: v = ff_eval_o<D, PM, 1>(Mt, h); break;
  case 2: v = ff_eval_o<D, PM, (PM >= 2 ? 2 : 1)>(Mt, h); break;
  case 3: v = ff_eval_o<D, PM, (PM >= 3 ? 3 : 1)>(Mt, h); break;
  case 4: v = ff_eval_o<D, PM, (PM >= 4 ? 4 : 1)>(Mt, h); break;
  case 5: v = ff_eval_o<D, PM, (PM >= 5 ? 5 : 1)>(Mt, h); break;
  case 6: v = ff_eval_o<D, PM, (PM >= 6 ? 6 : 1)>(Mt, h); break;
  case 7: v = ff_eval_o<D, PM, (PM >= 7 ? 7 : 1)>(Mt, h); break;
  default: v = ff_eval_o<D, PM, PM>(Mt, h); break;
  }
  return exp(-tt) * v;
}

#ifndef DFGTB_FF_MINB
#define DFGTB_FF_MINB 3  // 80 registers, 3 CTAs per SM: measured 1-7% faster than the unbounded 96-register build
#endif
template <int D, int PM>
__global__ void __launch_bounds__(kBlock, DFGTB_FF_MINB) k_farfield_t(TreeView Q, TreeView R, int K, int nb,
                                                       const int* leaves, int nleaves,
                                                       const int* cnt, const int* off,
                                                       const Item* items, const double* Mt,
                                                       SlotView sv, int nq, double* s_ff)
{
  constexpr int T = ipow_c(PM, D);
  constexpr int ND = D * (PM - 1) + 1;
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = w0; li < nleaves * nb; li += nw) {
    const int slot = li / nleaves;
    const int leaf = leaves[li - slot * nleaves];
    const double s = sv.s[slot];
    double spw[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) spw[k] = sv.spow[(size_t)slot * kSPow + k];
    const int qb = Q.begin[leaf], qc = Q.count[leaf];
    const int dep = Q.depth[leaf];
    // the ancestors carrying far-field items, root first: one coalesced load of the
    // leaf's chain per 32 levels and a ballot (deeper leaves walk parent pointers)
    int anode[2] = { -1, -1 };
    unsigned amask[2] = { 0u, 0u };
    if (dep < kMaxAnc) {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int k = w * 32 + lane;
        if (k <= dep) anode[w] = Q.anc[(size_t)leaf * kMaxAnc + k];
        amask[w] = __ballot_sync(0xffffffffu, anode[w] >= 0 && cnt[slot * K + anode[w]] > 0);
      }
    }
    for (int q0 = 0; q0 < qc; q0 += 32) {
      const int qi = q0 + lane;
      const bool act = qi < qc;
      double qv[D];
#pragma unroll
      for (int d = 0; d < D; ++d) qv[d] = Q.xs[(size_t)(qb + (act ? qi : 0)) * D + d];
      double acc = 0.0;
      auto visit = [&](int node) {
        const int key = slot * K + node;
        const int c = cnt[key];
        const Item* it = items + off[key];
        for (int t = 0; t < c; ++t) {
          const int r = it[t].r, order = it[t].code & 0xff;
          acc += ff_eval_t<D, PM>(Mt + (size_t)r * T, R.cen + (size_t)r * D, qv, s, order, spw);
        }
      };
      if (dep < kMaxAnc) {
#pragma unroll
        for (int w = 0; w < 2; ++w)
          for (unsigned m = amask[w]; m; m &= m - 1)
            visit(__shfl_sync(0xffffffffu, anode[w], __ffs(m) - 1));
      } else {
        for (int k = 0; k <= dep; ++k) visit(ancestor_at(Q, leaf, dep, k));
      }
      if (act) s_ff[(size_t)slot * nq + qb + qi] = acc;
    }
  }
}

// ---------------------------------------------------------------- finalize
// Local evaluation, the base-case partials in task order, and the final sum
// (post_process leaf branch and Traversal::run, engine.cpp:273-291, 85-89); results
// scattered to input order.  direct != 0: the local expansions of ALL ancestors are
// evaluated at the query (root first) instead of being pushed down by L2L first --
// the same polynomial, re-centred exactly, without the per-level launch chain.
__global__ void k_finalize(DevSeries g, TreeView Q, int K, int nb, const int* leaf_of_pos,
                           const int* perm, int n, const double* L, const int* Lord,
                           const int* cntB, const int* leaf_task, const int* leaf_runs,
                           const double* part, int tcap,
                           const double* s_ff, SlotView sv, int direct, double* out)
{
  const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= (long long)n * nb) return;
  const int slot = (int)(gi / n);
  const int i = (int)(gi - (long long)slot * n);
  const int leaf = leaf_of_pos[i];
  const int lkey = slot * K + leaf;
  const double s = sv.s[slot];
  const double* qp = Q.xs + (size_t)i * g.D;
  double loc = 0.0;
  if (direct) {
    const int dep = Q.depth[leaf];
    for (int k = 0; k <= dep; ++k) {
      const int a = ancestor_at(Q, leaf, dep, k);
      const int key = slot * K + a;
      const int order = Lord[key];
      if (order > 0)
        loc += dev_eval_local(g, L + (size_t)key * g.T, Q.cen + (size_t)a * g.D, qp, s, order);
    }
  } else {
    const int order = Lord[lkey];
    if (order > 0)
      loc = dev_eval_local(g, L + (size_t)lkey * g.T, Q.cen + (size_t)leaf * g.D, qp, s, order);
  }
  const int li = i - Q.begin[leaf];
  const int nic = cntB[lkey] ? leaf_runs[lkey] : 0;
  double ex = 0.0;
  if (nic) {
    const int t0 = leaf_task[lkey] + (li >> 5) * nic;
    // (tasks past the task buffer were dropped: the batch is rerun, nothing is read there)
    if (t0 + nic <= tcap)
      for (int k = 0; k < nic; ++k) ex += part[(size_t)(t0 + k) * 32 + (li & 31)];
  }
  out[(size_t)slot * n + perm[i]] = loc + s_ff[(size_t)slot * n + i] + ex;
}

// sum over the cube b_d < O of L_b prod_d u_d^{b_d}, Horner one dimension at a time
// (tp: position -> term index of the table; entries beyond the table's order are 0)
template <int D, int PM, int O>
__device__ __forceinline__ double local_horner(const double* Lk, const int* tp, const double (&u)[D])
{
  constexpr int NO = ipow_c(O, D);
  double v[NO];
#pragma unroll
  for (int p = 0; p < NO; ++p) {
    int rest = p, pos = 0, mul = 1;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      pos += (rest % O) * mul;
      rest /= O;
      mul *= PM;
    }
    v[p] = Lk[tp[pos]];
  }
  int len = NO;
#pragma unroll
  for (int d = D - 1; d >= 0; --d) {
    len /= O;
#pragma unroll
    for (int r = 0; r < ipow_c(O, D - 1); ++r) {
      if (r < len) {
        double acc = v[r * O + O - 1];
#pragma unroll
        for (int k = O - 2; k >= 0; --k) acc = fma(acc, u[d], v[r * O + k]);
        v[r] = acc;
      }
    }
  }
  return v[0];
}

// Specialised finalize for the default tables (p_max == PM): every ancestor's local
// table is evaluated as a polynomial in u = (q - c) s, contracted one dimension at a
// time (Horner per dimension, position layout via term_of_pos staged in shared
// memory; entries beyond a table's order are zero).  Ancestors are walked from the
// leaf up (no per-thread chain array).
#ifndef DFGTB_FIN_MINB
#define DFGTB_FIN_MINB 8  // 64 registers (the full-order Horner spills, it is rare): latency-bound, occupancy pays --
                          // k_finalize_t 69 -> 57 us (cfg2), 0.54 -> 0.39 ms (cfg3) against 128 registers
#endif
template <int D, int PM>
__global__ void __launch_bounds__(128, DFGTB_FIN_MINB) k_finalize_t(DevSeries g, TreeView Q, int K, int nb,
                                                    const int* leaf_of_pos, const int* perm, int n,
                                                    const double* L, const int* Lord,
                                                    const int* cntB, const int* leaf_task,
                                                    const int* leaf_runs, const double* part, int tcap,
                                                    const double* s_ff, SlotView sv, double* out)
{
  constexpr int NP = ipow_c(PM, D);
  __shared__ int tp[NP];
  for (int p = threadIdx.x; p < NP; p += blockDim.x) tp[p] = g.term_of_pos[p];
  __syncthreads();
  const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= (long long)n * nb) return;
  const int slot = (int)(gi / n);
  const int i = (int)(gi - (long long)slot * n);
  const int leaf = leaf_of_pos[i];
  const int lkey = slot * K + leaf;
  const double s = sv.s[slot];
  double q[D];
#pragma unroll
  for (int d = 0; d < D; ++d) q[d] = Q.xs[(size_t)i * D + d];
  double loc = 0.0;
  const int dep = Q.depth[leaf];
  const int* anc = Q.anc + (size_t)leaf * kMaxAnc;
  auto eval = [&](int a) {
    const int key = slot * K + a;
    const int ord = Lord[key];
    if (ord <= 0) return;
    const double* Lk = L + (size_t)key * g.T;
    double u[D];
#pragma unroll
    for (int d = 0; d < D; ++d) u[d] = (q[d] - Q.cen[(size_t)a * D + d]) * s;
    if (ord == 1) {
      loc += Lk[0];  // the finite-difference constant term only
    } else if (ord == 2) {
      loc += local_horner<D, PM, (PM >= 2 ? 2 : 1)>(Lk, tp, u);
    } else if (ord == 3) {
      loc += local_horner<D, PM, (PM >= 3 ? 3 : 1)>(Lk, tp, u);
    } else {
      loc += local_horner<D, PM, PM>(Lk, tp, u);
    }
  };
  if (dep < kMaxAnc) {
    // which ancestors (anc[k], depth k <= dep; anc[dep] = the leaf) hold a table: the
    // order loads of 8 ancestors are issued together (independent chains anc -> Lord),
    // then only the holders are visited, leaf first (the same order of additions as the
    // plain walk below)
    static_assert(kMaxAnc <= 64, "ancestor mask");
    unsigned long long act = 0;
#pragma unroll 1
    for (int k0 = 0; k0 <= dep; k0 += 8) {
      int o[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) o[u] = k0 + u <= dep ? Lord[slot * K + anc[k0 + u]] : 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (o[u] > 0) act |= 1ull << (k0 + u);
    }
    while (act) {
      const int k = 63 - __clzll((long long)act);
      act &= ~(1ull << k);
      eval(anc[k]);
    }
  } else {
    for (int k = dep, a = leaf; k >= 0; --k, a = Q.parent[a]) eval(a);
  }
  const int li = i - Q.begin[leaf];
  const int nic = cntB[lkey] ? leaf_runs[lkey] : 0;
  double ex = 0.0;
  if (nic) {
    const int t0 = leaf_task[lkey] + (li >> 5) * nic;
    // (tasks past the task buffer were dropped: the batch is rerun, nothing is read there)
    if (t0 + nic <= tcap)
      for (int k = 0; k < nic; ++k) ex += part[(size_t)(t0 + k) * 32 + (li & 31)];
  }
  out[(size_t)slot * n + perm[i]] = loc + s_ff[(size_t)slot * n + i] + ex;
}

__global__ void k_leaf_of_pos(const int* leaves, int nleaves, const int* begin, const int* count,
                              int* leaf_of_pos)
{
  const int i = blockIdx.x;
  if (i >= nleaves) return;
  const int leaf = leaves[i];
  for (int k = threadIdx.x; k < count[leaf]; k += blockDim.x) leaf_of_pos[begin[leaf] + k] = leaf;
}

// ---------------------------------------------------------------------- CV
// K11 (cv.cpp:17-25, 61-97): per scale k (blockIdx.y), deterministic two-stage sums of
// log LOO density, clamp count and the least-squares term.
constexpr int kRedBlocks = 148;
struct CvNorm {
  double nh[kMaxSlots], nc[kMaxSlots];
};
__global__ void k_cv_partial(const double* sums, const double* conv, int n, CvNorm cn, double* part)
{
  __shared__ double sl[kBlock / 32], ss[kBlock / 32], sc[kBlock / 32];
  const int k = blockIdx.y;
  const double* S = sums + (size_t)k * n;
  const double* C = conv ? conv + (size_t)k * n : nullptr;
  const double nh = cn.nh[k], nc = cn.nc[k];
  double lk = 0.0, ls = 0.0, cl = 0.0;
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int b = blockIdx.x * per, e = min(n, b + per);
  for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
    double loo = S[i] - 1.0;
    if (loo <= 0.0) {
      loo = DBL_MIN;
      cl += 1.0;
    }
    lk += log(loo / nh);
    if (C) ls += (C[i] - 1.0) / nc - 2.0 * ((S[i] - 1.0) / nh);
  }
  lk = warp_sum(lk);
  ls = warp_sum(ls);
  cl = warp_sum(cl);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sl[w] = lk;
    ss[w] = ls;
    sc[w] = cl;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b2 = 0, c = 0;
    for (int q = 0; q < kBlock / 32; ++q) {
      a += sl[q];
      b2 += ss[q];
      c += sc[q];
    }
    double* P = part + ((size_t)k * gridDim.x + blockIdx.x) * 3;
    P[0] = a;
    P[1] = b2;
    P[2] = c;
  }
}

// K12: exhaustive FP64 sums, 128 queries per block, reference tiles through smem.
__global__ void k_naive(const double* q, int nq, const double* r, int nr, int D, double scale,
                        double* out)
{
  extern __shared__ double tile[];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double qq[kMaxDim];
  for (int d = 0; d < D; ++d) qq[d] = i < nq ? q[(size_t)i * D + d] : 0.0;
  double acc = 0.0;
  const int TR = 256;
  for (int b = 0; b < nr; b += TR) {
    const int m = min(TR, nr - b);
    __syncthreads();
    for (int k = threadIdx.x; k < m * D; k += blockDim.x) tile[k] = r[(size_t)b * D + k];
    __syncthreads();
    for (int j = 0; j < m; ++j) {
      double d2 = 0.0;
      for (int d = 0; d < D; ++d) {
        const double t = qq[d] - tile[j * D + d];
        d2 += t * t;
      }
      acc += exp(scale * d2);
    }
  }
  if (i < nq) out[i] = acc;
}

__global__ void k_dfma_peak(double* out, int iters)
{
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 42.0) out[0] = 1.0;
}

// Points per task run: the base case's stream tile (k_base_case_any streams directly),
// or DFGTB_RUN_POINTS.
#ifndef DFGTB_RUN_POINTS
#define DFGTB_RUN_POINTS 512  // measured: 512-point runs 5-11% faster than 256 (FP32 tile 512); 1024 slower
#endif
int base_rmax(int D)
{
  return D <= 5 ? DFGTB_RUN_POINTS : 256;  // k_base_case_any (D > 5) streams its own tiles
}

int padded_dim(int D) { return D == 1 ? 1 : (D <= 5 ? (D + 1) / 2 * 2 : D); }

// Persistent grids: as many CTAs as fit on the GPU (or fewer for small task lists).
// ws = [nextA, nextB, cntA, cntB, pairsA (u64), pairsB (u64), listA (tcap), listB (tcap),
// task flags (tcap, written by k_task_build)]; the lists come from k_task_split.  Then the
// FP32 kernel over list A, then the FP64 kernel over list B.
#ifndef DFGTB_PREP_STREAM_DEFAULT
#define DFGTB_PREP_STREAM_DEFAULT 1
#endif
#ifndef DFGTB_FF_STREAM_DEFAULT
#define DFGTB_FF_STREAM_DEFAULT 1  // measured: cfg2 -1.4%, cfg3 / cfg5 -0.4% against the far field queued behind the local chain
#endif
#ifndef DFGTB_BASE_CONC
#define DFGTB_BASE_CONC 0  // measured: side by side is no faster than one after the other (c32) or slower
#endif
#ifndef DFGTB_CONC_F32
#define DFGTB_CONC_F32 4
#endif
#ifndef DFGTB_CONC_FP64
#define DFGTB_CONC_FP64 1
#endif
constexpr int kConcF32 = DFGTB_CONC_F32, kConcFP64 = DFGTB_CONC_FP64;  // CTAs per SM side by side
struct BaseConc {
  cudaStream_t s3 = nullptr;  // nullptr: the two kernels run one after the other on `s`
  cudaEvent_t fork3 = nullptr, join3 = nullptr, b0 = nullptr, b1 = nullptr;
};
template <class KF>
int persistent_grid(KF kern, int threads, int smem, int slack, int tcap, int warps)
{
  int dev = 0, nsm = 0, per_sm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  per_sm = std::max(per_sm, 1);
  // leave `slack` CTA slots per SM to the kernels of the second stream
  return (int)std::min<long long>((long long)nsm * std::max(1, per_sm - slack), (tcap + warps - 1) / warps);
}

template <int DT>
void launch_base_t(const int* ntasks, int tcap, cudaStream_t s, TreeView Q, int K, const BTask* tasks,
                   const int2* rec, const double* xq, const double* xr, int nq, int nr, double* part,
                   int* ws, int mufu, int slack, const double* c0, SlotView sv, double f, cudaEvent_t mid,
                   const BaseConc& cc)
{
  static int gridB = 0, gridA = 0;
  constexpr int threads = BaseGeo<DT>::WARPS * 32;
  constexpr int smem = BaseGeo<DT>::WARPS * BaseGeo<DT>::WORDS * (int)sizeof(double);
  constexpr int threadsA = F32Geo<DT>::WARPS * 32;
  constexpr int smemA = F32Geo<DT>::WARPS * F32Geo<DT>::FLOATS * (int)sizeof(float);
  if (!gridB) {
    gridB = persistent_grid(k_base_case<DT>, threads, smem, slack, INT32_MAX / 2, BaseGeo<DT>::WARPS);
    gridA = persistent_grid(k_base_f32<DT>, threadsA, smemA, slack, INT32_MAX / 2, F32Geo<DT>::WARPS);
  }
  const int cap_grid = (tcap + 3) / 4;
  int* listB = ws + 8 + tcap;
  (void)ntasks;  // the lists were built by k_task_split (launch_phases)
  if ((mufu & 2) && cc.s3) {
    // both kernels at once: the FP32 one (XU / FP32 pipes) on `s` with kConcF32 CTAs per
    // SM, the FP64 one (FP64 pipe) on `s3` with the register file's remainder
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    CK(cudaEventRecord(cc.fork3, s));
    CK(cudaStreamWaitEvent(cc.s3, cc.fork3, 0));
    CK(cudaEventRecord(cc.b0, cc.s3));
    k_base_case<DT><<<std::min(nsm * kConcFP64, cap_grid), threads, smem, cc.s3>>>(
      Q, K, tasks, listB, ws + 3, rec, xq, xr, nq, nr, part, ws + 1, mufu, c0, sv, f);
    CK_LAUNCH();
    CK(cudaEventRecord(cc.b1, cc.s3));
    CK(cudaEventRecord(cc.join3, cc.s3));
    k_base_f32<DT><<<std::min(nsm * kConcF32, cap_grid), threadsA, smemA, s>>>(
      Q, K, reinterpret_cast<const int4*>(tasks + tcap), ws + 2, rec, xq, xr, nq, nr, part, ws, c0, sv, f);
    CK_LAUNCH();
    if (mid) CK(cudaEventRecord(mid, s));
    CK(cudaStreamWaitEvent(s, cc.join3, 0));
    return;
  }
  if (mufu & 2) {
    k_base_f32<DT><<<std::min(gridA, cap_grid), threadsA, smemA, s>>>(
      Q, K, reinterpret_cast<const int4*>(tasks + tcap), ws + 2, rec, xq, xr, nq, nr, part, ws, c0, sv, f);
    CK_LAUNCH();
  }
  if (mid) CK(cudaEventRecord(mid, s));
  k_base_case<DT><<<std::min(gridB, cap_grid), threads, smem, s>>>(Q, K, tasks, listB, ws + 3, rec, xq, xr,
                                                                  nq, nr, part, ws + 1, mufu, c0, sv, f);
}

void launch_base(int D, cudaStream_t s, TreeView Q, TreeView R, int K, const BTask* tasks,
                 const int* ntasks, int tcap, const Item* items, const int2* rec, const double* xq,
                 const double* xr, int nq, int nr, double* part, int* next, int mufu, int slack,
                 const double* c0, SlotView sv, double f, cudaEvent_t mid, const BaseConc& cc)
{
#define BASE(DD)                                                                                 \
  launch_base_t<DD>(ntasks, tcap, s, Q, K, tasks, rec, xq, xr, nq, nr, part, next, mufu, slack, c0, sv, f, mid, cc)
  switch (D) {
  case 1: BASE(1); break;
  case 2: BASE(2); break;
  case 3: BASE(3); break;
  case 4: BASE(4); break;
  case 5: BASE(5); break;
  default:
    if (mid) CK(cudaEventRecord(mid, s));
    k_base_case_any<<<148 * 16, kBlock, 0, s>>>(Q, R, K, D, tasks, ntasks, tcap, items, xq, xr, nq, nr,
                                                part);
    break;
  }
#undef BASE
  CK_LAUNCH();
}

}  // namespace

void init_exp_constants(cudaStream_t s)
{  // base-case exp(-y): 64 log2(e), ln2/64, 1/5! .. 1/2!, table 2^(j/64)
  double k64[6] = { 64.0 * 1.4426950408889634, 0.6931471805599453 / 64.0,  // RN(ln 2) / 2^6
                    1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5 };
  double tab[64];
  for (int j = 0; j < 64; ++j) tab[j] = std::exp2((double)j / 64.0);  // correctly rounded in glibc
  CK(cudaMemcpyToSymbolAsync(c_exp64, k64, sizeof(k64), 0, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyToSymbolAsync(c_exp2tab, tab, sizeof(tab), 0, cudaMemcpyHostToDevice, s));
}

// Unscaled moments of every reference node, once per tree (tables <= 4096 terms).
// Queued on s2_ without a host wait: every consumer of Mt_ runs on s2_ after it, so
// the moments overlap whatever the caller does next (the first batch's traversal).
void Engine::eager_moments()
{
  const DevTree& t = rt_;
  const int K = t.nodes, T = ser_.T;
  std::vector<int> cnode, cstart, coff(K + 1, 0);
  for (int n = 0; n < K; ++n) {
    coff[n] = (int)cnode.size();
    for (int st = 0; st < t.h_count[n]; st += kMomChunk) {
      cnode.push_back(n);
      cstart.push_back(t.h_begin[n] + st);
    }
  }
  coff[K] = (int)cnode.size();
  const int nch = (int)cnode.size();
  DevBuf<int>& dn = mom_node_;
  DevBuf<int>& ds = mom_start_;
  DevBuf<int>& dof = mom_off_;
  DevBuf<double>& part = mom_part_;  // members: alive until the queued kernels are done
  cudaStream_t s2 = s2_;
  CK(cudaEventRecord(fork_, s_));
  CK(cudaStreamWaitEvent(s2, fork_, 0));
  dn.reserve(nch);
  ds.reserve(nch);
  dof.reserve(K + 1);
  part.reserve((size_t)nch * T);
  CK(cudaMemcpyAsync(dn.p, cnode.data(), sizeof(int) * nch, cudaMemcpyHostToDevice, s2));
  CK(cudaMemcpyAsync(ds.p, cstart.data(), sizeof(int) * nch, cudaMemcpyHostToDevice, s2));
  CK(cudaMemcpyAsync(dof.p, coff.data(), sizeof(int) * (K + 1), cudaMemcpyHostToDevice, s2));
  Mt_.reserve((size_t)K * T);
  CK(cudaEventRecord(mom_ev_[0], s2));
  const DevSeries g = dev_series();
  const int smem = kMomChunk * D_ * ser_.pmax * (int)sizeof(double);
  const int pm = ser_.pmax;
  const int gw = std::min(ceil_div(nch, 4), 148 * 16);
#define MOM_T(DD, PP) k_moment_chunks_w<DD, PP><<<gw, 128, 0, s2>>>(g, view_of(t), dn.p, ds.p, nch, part.p)
  if (D_ == 1 && pm == 8) MOM_T(1, 8);
  else if (D_ == 2 && pm == 6) MOM_T(2, 6);
  else if (D_ == 3 && pm == 4) MOM_T(3, 4);
  else if (D_ == 4 && pm == 2) MOM_T(4, 2);
  else if (D_ == 5 && pm == 2) MOM_T(5, 2);
  else
    k_moment_chunks<<<std::min(nch, 148 * 16), 128, smem, s2>>>(g, view_of(t), dn.p, ds.p, nch,
                                                                 part.p);
#undef MOM_T
  CK_LAUNCH();
  k_moment_reduce<<<std::min(K, 148 * 8), kMomRedThreads, 0, s2>>>(g, K, dof.p, part.p, Mt_.p);
  CK_LAUNCH();
  CK(cudaEventRecord(mom_ev_[1], s2));
}

void Engine::setup_leaves(const DevTree& t)
{
  qleaves_host_.clear();
  for (int i = 0; i < t.nodes; ++i)
    if (t.h_left[i] < 0) qleaves_host_.push_back(i);
  const int nl = (int)qleaves_host_.size();
  leaves_.reserve(nl);
  CK(cudaMemcpyAsync(leaves_.p, qleaves_host_.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, s_));
  leaf_of_pos_.reserve(t.n);
  k_leaf_of_pos<<<nl, 64, 0, s_>>>(leaves_.p, nl, t.begin.p, t.count.p, leaf_of_pos_.p);
  CK_LAUNCH();  // ordered on s_ before the batch that follows (qleaves_host_ is a member: the
                // upload's source outlives the call)
}

// One batch: every launch is queued without a host round trip (counts live in bc_);
// the host synchronises once at the end, reads the traversal verdict and the chunk /
// task totals, and reruns the batch with larger buffers if anything overflowed.
void Engine::run_phases(const DevTree& qt, const double* h, int nb, double* d_out)
{
  for (int attempt = 0;; ++attempt) {
    launch_phases(qt, h, nb, d_out);
    if (post_batch_) post_batch_();
    // the traversal verdict and the chunk / task totals come back with the one wait
    if (!hpin_) hpin_ = pinned_alloc(kHostPinBytes);
    int* hb = static_cast<int*>(hpin_);
    traverse_fetch_async();
    CK(cudaMemcpyAsync(hb, bc_.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    const bool trav_ok = traverse_finish(true);
    bool ok = trav_ok;
    if (trav_ok) {
      auto grow = [&](long long need) {
        if (need > (1 << 28))
          throw OutOfMemory("batch needs more than 2^28 chunks / tasks (" + std::to_string(hb[4]) +
                            ", " + std::to_string(hb[5]) + ")");
        return (int)(need + need / 4 + 1024);
      };
      if (hb[4] > capCh_) {
        capCh_ = grow(hb[4]);
        ok = false;
      }
      if (hb[5] > capTask_) {
        capTask_ = grow(hb[5]);
        ok = false;
      }
    }
    if (ok) break;
    if (attempt > 10) throw OutOfMemory("batch buffers keep overflowing");
  }
  CK(cudaEventElapsedTime(&tim_.traverse_ms, ev_[2], ev_[3]));
  CK(cudaEventElapsedTime(&tim_.moments_ms, ev_[3], ev_[4]));
  CK(cudaEventElapsedTime(&tim_.local_ms, ev_[4], ev_[5]));
  CK(cudaEventElapsedTime(&tim_.base_ms, ev_[9], ev_[10]));
  CK(cudaEventElapsedTime(&tim_.base_f32_ms, ev_[9], ev_[11]));
  if (base_conc_) CK(cudaEventElapsedTime(&tim_.base_fp64_ms, ev_[12], ev_[13]));
  else CK(cudaEventElapsedTime(&tim_.base_fp64_ms, ev_[11], ev_[10]));
  CK(cudaEventElapsedTime(&tim_.farfield_ms, ev_[6], ev_[7]));
  CK(cudaEventElapsedTime(&tim_.final_ms, ev_[14], ev_[8]));
  CK(cudaEventElapsedTime(&tim_.total_ms, ev_[2], ev_[8]));
  if (std::getenv("DFGTB_TIMELINE")) {  // event times of the batch, ms after its start
    const int ids[] = { 3, 4, 5, 6, 7, 9, 11, 10, 14, 8 };
    const char* names[] = { "traversal_end", "local_start", "local_end", "ff_start", "ff_end", "base_start",
                            "base_f32_end", "base_end", "joined", "end" };
    std::fprintf(stderr, "DFGTB_TIMELINE");
    for (int k = 0; k < 10; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev_[2], ev_[ids[k]]) != cudaSuccess) cudaGetLastError();
      std::fprintf(stderr, " %s %.3f", names[k], ms);
    }
    std::fprintf(stderr, "\n");
  }
}

void Engine::launch_phases(const DevTree& qt, const double* h, int nb, double* d_out)
{
  last_q_ = &qt;
  last_K_ = qt.nodes;
  cudaStream_t s = s_;
  const DevSeries g = dev_series();
  const TreeView Q = view_of(qt), R = view_of(rt_);
  const int K = qt.nodes, T = ser_.T;
  const int KB = K * nb;
  nb_ = nb;
  // per-slot constants: s, s2, s^k
  {
    std::vector<double> hp((size_t)nb * (2 + kSPow));
    for (int b = 0; b < nb; ++b) {
      const double sc = inv_scale(h[b]);
      hp[b] = sc;
      hp[nb + b] = 1.0 / (2.0 * h[b] * h[b]);
      double* sp = hp.data() + 2 * nb + (size_t)b * kSPow;
      sp[0] = 1.0;
      for (int k = 1; k < kSPow; ++k) sp[k] = sp[k - 1] * sc;
    }
    slotp_.reserve(hp.size());
    CK(cudaMemcpyAsync(slotp_.p, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice, s));
  }
  const SlotView sv{ slotp_.p, slotp_.p + nb, slotp_.p + 2 * nb };
  CK(cudaEventRecord(ev_[2], s));
  traverse(qt, h, nb);
  const int* dnF = bc_.p + 0;
  const int* dnDT = bc_.p + 1;
  const int* dnB = bc_.p + 2;
  CK(cudaEventRecord(ev_[3], s));
  // Fork: the local expansions (D/T items) and the far field run on s2_ beside the
  // base-case chain on s_ (they only read the traversal's sorted items and write their
  // own buffers); the base case leaves a CTA slot per SM for them.  Join before
  // finalize.
  cudaStream_t s2 = one_stream_ ? s : s2_;  // DFGTB_ONE_STREAM: isolated kernel timings
  CK(cudaEventRecord(fork_, s));
  CK(cudaStreamWaitEvent(s2, fork_, 0));
  const int nleaves = (int)qleaves_host_.size();
  const int nlb = nleaves * nb;
  // base-case tasks and records: queued first (host order) on the preparation stream
  leaf_task_.reserve(KB);
  leaf_runs_.reserve(KB);
  const int rmax = base_rmax(D_);
  capTask_ = std::max(capTask_, std::max(4096, capB_ / 8));
  tasks_.reserve((size_t)capTask_ * 12);  // BTask array | packed list A | packed list B
  bnext_.reserve(8 + 3 * (size_t)capTask_);  // base-case lists and task flags (launch_base_t)
  // the preparation kernels run on their own top-priority stream (DFGTB_PREP_STREAM=0: on
  // s): on s they were queued behind the expansion kernels and delayed the base case by
  // ~0.15 ms on cfg2
  static const int prep_env = std::getenv("DFGTB_PREP_STREAM") ? std::atoi(std::getenv("DFGTB_PREP_STREAM")) : DFGTB_PREP_STREAM_DEFAULT;
  cudaStream_t sp = (prep_env && !one_stream_ && s4_) ? s4_ : s;
  if (sp != s) CK(cudaStreamWaitEvent(sp, fork_, 0));
  CK(cudaMemsetAsync(bc_.p + 5, 0, sizeof(int), sp));
  k_task_build<<<ceil_div(nlb, 8), 256, 0, sp>>>(leaves_.p, nleaves, nb, K, cntB_.p, offB_.p, sB_.p,
                                                  R.count, rmax, Q, reinterpret_cast<BTask*>(tasks_.p),
                                                  capTask_, bc_.p + 5, leaf_task_.p, leaf_runs_.p,
                                                  bnext_.p + 8 + 2 * (size_t)capTask_);
  CK_LAUNCH();
  CK(cudaMemsetAsync(bnext_.p, 0, 8 * sizeof(int), sp));
  k_task_split<<<ceil_div(nlb, 8), 256, 0, sp>>>(leaves_.p, nleaves, nb, K, cntB_.p, leaf_task_.p, leaf_runs_.p, Q,
                                                  capTask_, bnext_.p + 8 + 2 * (size_t)capTask_, f32_ ? 1 : 0,
                                                  bnext_.p + 8, bnext_.p + 8 + capTask_, bnext_.p + 2,
                                                  reinterpret_cast<const BTask*>(tasks_.p),
                                                  reinterpret_cast<int4*>(tasks_.p + (size_t)capTask_ * 4),
                                                  reinterpret_cast<int4*>(tasks_.p + (size_t)capTask_ * 8));
  CK_LAUNCH();
  bpart_.reserve((size_t)capTask_ * 32);
  brec_.reserve((size_t)capB_ * 2 + 2);
  k_base_records<<<148 * 4, 256, 0, sp>>>(sB_.p, dnB, capB_, R, reinterpret_cast<int2*>(brec_.p));
  CK_LAUNCH();
  // scaled, centred, padded coordinates per slot (Q and, if different, R)
  const int DP = padded_dim(D_);
  xq_.reserve((size_t)qt.n * DP * nb);
  k_scale_points<<<ceil_div((long long)qt.n * DP * nb, 256), 256, 0, sp>>>(
    qt.xs.p, qt.n, D_, DP, nb, rt_.centroid.p, sv, mufu_ ? kSqrtLog2e : 1.0, xq_.p);
  CK_LAUNCH();
  const double* xq = xq_.p;
  const double* xr = xq_.p;
  if (&qt != &rt_) {
    xr_.reserve((size_t)rt_.n * DP * nb);
    k_scale_points<<<ceil_div((long long)rt_.n * DP * nb, 256), 256, 0, sp>>>(
      rt_.xs.p, rt_.n, D_, DP, nb, rt_.centroid.p, sv, mufu_ ? kSqrtLog2e : 1.0, xr_.p);
    CK_LAUNCH();
    xr = xr_.p;
  }
  if (sp != s) {
    CK(cudaEventRecord(prep_ev_, sp));
    CK(cudaStreamWaitEvent(s, prep_ev_, 0));
    if (prep_env == 2) {  // the expansion chains start with the base case, after the preparation
      CK(cudaStreamWaitEvent(s2, prep_ev_, 0));
      if (s3_) CK(cudaStreamWaitEvent(s3_, prep_ev_, 0));
    }
  }
  // moments of the reference nodes used by F/T items (large tables only; small
  // tables were computed for every node when the engine was built)
  if (!eager_ && cfg_.mode == 1) {
    mflag_.reserve(rt_.nodes);
    CK(cudaMemsetAsync(mflag_.p, 0, sizeof(int) * rt_.nodes, s2));
    k_mark_moments<<<148 * 4, 256, 0, s2>>>(sF_.p, dnF, capF_, mflag_.p);
    CK_LAUNCH();
    k_mark_moments<<<148 * 4, 256, 0, s2>>>(sDT_.p, dnDT, capDT_, mflag_.p);
    CK_LAUNCH();
    const int smem = 32 * D_ * ser_.pmax * (int)sizeof(double);
    k_moments<<<std::min(rt_.nodes, 148 * 8), 128, smem, s2>>>(g, R, rt_.nodes, mflag_.p, mdone_.p,
                                                              Mt_.p);
    CK_LAUNCH();
  }
  // far field: on s2_ after the local chain, or (DFGTB_FF_STREAM = 1 / 2, tables built
  // with the engine) on a third stream beside it, queued after / before the local chain
  static const int ff_env = std::getenv("DFGTB_FF_STREAM") ? std::atoi(std::getenv("DFGTB_FF_STREAM")) : DFGTB_FF_STREAM_DEFAULT;
  const int ff_mode = (one_stream_ || !s3_ || (cfg_.mode == 1 && !eager_)) ? 0 : ff_env;
  cudaStream_t sff = ff_mode ? s3_ : s2;
  if (ff_mode) CK(cudaStreamWaitEvent(sff, fork_, 0));
  auto launch_ff = [&]() {
    s_ff_.reserve((size_t)qt.n * nb);
    CK(cudaEventRecord(ev_[6], sff));
    if (cfg_.mode == 1) {
      const int gw = grid_warps(nlb);
      const int pm = ser_.pmax;
  #define FF_T(DD, PP)                                                                              \
    k_farfield_t<DD, PP><<<gw, kBlock, 0, sff>>>(Q, R, K, nb, leaves_.p, nleaves, cntF_.p, offF_.p,  \
                                                sF_.p, Mt_.p, sv, qt.n, s_ff_.p)
      if (D_ == 1 && pm == 8) FF_T(1, 8);
      else if (D_ == 2 && pm == 6) FF_T(2, 6);
      else if (D_ == 3 && pm == 4) FF_T(3, 4);
      else if (D_ == 4 && pm == 2) FF_T(4, 2);
      else if (D_ == 5 && pm == 2) FF_T(5, 2);
      else
        k_farfield<<<gw, kBlock, 0, sff>>>(g, Q, R, K, nb, leaves_.p, nleaves, cntF_.p, offF_.p, sF_.p,
                                         Mt_.p, sv, qt.n, s_ff_.p);
  #undef FF_T
      CK_LAUNCH();
    } else {
      CK(cudaMemsetAsync(s_ff_.p, 0, sizeof(double) * qt.n * nb, sff));
    }
    CK(cudaEventRecord(ev_[7], sff));
    if (ff_mode) CK(cudaEventRecord(join3_, sff));
  };
  if (ff_mode == 2) launch_ff();
  CK(cudaEventRecord(ev_[4], s2));
  // D/T items -> chunked partial tables -> per-(slot, query node) reduction
  if (cfg_.mode == 1) {
    lnch_.reserve((size_t)capDT_ + 1);
    lchoff_.reserve((size_t)capDT_ + 1);
    k_local_count<<<148 * 4, 256, 0, s2>>>(sDT_.p, dnDT, capDT_, R, lnch_.p);
    CK_LAUNCH();
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, lnch_.p, lchoff_.p, capDT_ + 1, s2);
    scan_tmp2_.reserve(need + 256);
    size_t have = scan_tmp2_.cap;
    cub::DeviceScan::ExclusiveSum(scan_tmp2_.p, have, lnch_.p, lchoff_.p, capDT_ + 1, s2);
    capCh_ = std::max(capCh_, std::max(4096, capDT_));
    lchunk_.reserve((size_t)capCh_ * 3);
    LChunk* ch = reinterpret_cast<LChunk*>(lchunk_.p);
    k_local_fill<<<148 * 4, 256, 0, s2>>>(sDT_.p, dnDT, capDT_, R, lchoff_.p, ch, capCh_, bc_.p + 4);
    CK_LAUNCH();
    lpart_.reserve((size_t)capCh_ * T);
    const int smem = std::max(kLocSub * D_ * ser_.pmax, D_ * (2 * ser_.pmax)) * (int)sizeof(double);
    const int gl = 148 * 16;
    const int pm = ser_.pmax;
    const int* dnch = bc_.p + 4;
#define LOC_T(DD, PP)                                                                            \
  k_local_chunks_w<DD, PP><<<gl, kLocWarps * 32, 0, s2>>>(g, Q, R, K, sDT_.p, ch, dnch, capCh_,  \
                                                          Mt_.p, sv, lpart_.p)
    if (D_ == 1 && pm == 8) LOC_T(1, 8);
    else if (D_ == 2 && pm == 6) LOC_T(2, 6);
    else if (D_ == 3 && pm == 4) LOC_T(3, 4);
    else if (D_ == 4 && pm == 2) LOC_T(4, 2);
    else if (D_ == 5 && pm == 2) LOC_T(5, 2);
    else
      k_local_chunks<<<gl, 64, smem, s2>>>(g, Q, R, K, sDT_.p, ch, dnch, capCh_, Mt_.p, sv, lpart_.p);
#undef LOC_T
    CK_LAUNCH();
    k_local_reduce<<<148 * 8, 256, 0, s2>>>(g, dnDT, capDT_, (int)KB, cntDT_.p, offDT_.p, sDT_.p, lchoff_.p,
                                            capCh_, lpart_.p, L_.p, Lord_.p);
    CK_LAUNCH();
  }
  if (cfg_.local_pushdown == 1) {
    const int smem = D_ * ser_.pmax * (int)sizeof(double);
    for (int d = 0; d + 1 < qt.height; ++d) {
      const int b = qt.depth_off[d], e = qt.depth_off[d + 1];
      k_l2l<<<std::min((e - b) * nb, 148 * 8), 64, smem, s2>>>(g, Q, K, nb, qt.by_depth.p + b, e - b,
                                                              sv, L_.p, Lord_.p);
      CK_LAUNCH();
    }
  }
  CK(cudaEventRecord(ev_[5], s2));
  if (ff_mode != 2) launch_ff();
  CK(cudaEventRecord(join_, s2));
  CK(cudaEventRecord(ev_[9], s));
  BaseConc conc;
  if (DFGTB_BASE_CONC && f32_ && !std::getenv("DFGTB_BASE_SERIAL")) {
    conc.s3 = s3_;
    conc.fork3 = fork3_;
    conc.join3 = join3_;
    conc.b0 = ev_[12];
    conc.b1 = ev_[13];
  }
  base_conc_ = conc.s3 != nullptr;
  launch_base(D_, s, Q, R, K, reinterpret_cast<const BTask*>(tasks_.p), bc_.p + 5, capTask_, sB_.p,
              reinterpret_cast<const int2*>(brec_.p), xq, xr, qt.n, rt_.n, bpart_.p, bnext_.p,
              (mufu_ ? 1 : 0) | (f32_ ? 2 : 0), base_cta_slack_, rt_.centroid.p, sv,
              mufu_ ? kSqrtLog2e : 1.0, ev_[11], conc);
  CK(cudaEventRecord(ev_[10], s));
  // join, finalize
  CK(cudaStreamWaitEvent(s, join_, 0));
  if (ff_mode) CK(cudaStreamWaitEvent(s, join3_, 0));
  CK(cudaEventRecord(ev_[14], s));  // both chains joined: finalize starts
  {
    const int fgrid = ceil_div((long long)qt.n * nb, 128);
    const int pm = ser_.pmax;
    const bool direct = cfg_.local_pushdown == 0;
#define FIN_T(DD, PP)                                                                             \
  k_finalize_t<DD, PP><<<fgrid, 128, 0, s>>>(g, Q, K, nb, leaf_of_pos_.p, qt.perm.p, qt.n, L_.p,  \
                                             Lord_.p, cntB_.p, leaf_task_.p, leaf_runs_.p,        \
                                             bpart_.p, capTask_, s_ff_.p, sv, d_out)
    if (direct && cfg_.mode == 1 && D_ == 1 && pm == 8) FIN_T(1, 8);
    else if (direct && cfg_.mode == 1 && D_ == 2 && pm == 6) FIN_T(2, 6);
    else if (direct && cfg_.mode == 1 && D_ == 3 && pm == 4) FIN_T(3, 4);
    else if (direct && cfg_.mode == 1 && D_ == 4 && pm == 2) FIN_T(4, 2);
    else if (direct && cfg_.mode == 1 && D_ == 5 && pm == 2) FIN_T(5, 2);
    else
      k_finalize<<<fgrid, 128, 0, s>>>(g, Q, K, nb, leaf_of_pos_.p, qt.perm.p, qt.n, L_.p, Lord_.p,
                                       cntB_.p, leaf_task_.p, leaf_runs_.p, bpart_.p, capTask_, s_ff_.p,
                                       sv, direct, d_out);
#undef FIN_T
  }
  CK_LAUNCH();
  CK(cudaEventRecord(ev_[8], s));
}

void Engine::cv_enqueue(const double* d_sums, const double* h, const double* d_conv,
                        const double* conv_h, int ns)
{
  const size_t n = n_;
  if (n < 2) throw InvalidArgument("CV requires at least 2 points");
  if (ns < 1 || ns > kMaxSlots) throw InvalidArgument("CV batch size outside [1, 64]");
  const double two_pi = 6.283185307179586476925286766559;
  CvNorm cn{};
  for (int k = 0; k < ns; ++k) {
    cn.nh[k] = (double)(n - 1) * std::pow(two_pi * h[k] * h[k], 0.5 * D_);
    cn.nc[k] = d_conv ? (double)(n - 1) * std::pow(two_pi * conv_h[k] * conv_h[k], 0.5 * D_) : 1.0;
  }
  red_.reserve((size_t)kRedBlocks * 3 * ns);
  k_cv_partial<<<dim3(kRedBlocks, ns), kBlock, 0, s_>>>(d_sums, d_conv, (int)n, cn, red_.p);
  CK_LAUNCH();
  static_assert(kRedBlocks == 148, "kHostPinBytes holds 148 x 3 x kMaxSlots partial sums");
  if (!hpin_) hpin_ = pinned_alloc(kHostPinBytes);
  CK(cudaMemcpyAsync(static_cast<char*>(hpin_) + 64, red_.p, sizeof(double) * kRedBlocks * 3 * ns,
                     cudaMemcpyDeviceToHost, s_));
}

// the block partials in fixed order (after the stream wait that follows cv_enqueue)
void Engine::cv_collect(int ns, double* lk, int* clamped, double* ls) const
{
  const double* part = reinterpret_cast<const double*>(static_cast<const char*>(hpin_) + 64);
  const size_t n = n_;
  for (int k = 0; k < ns; ++k) {
    double a = 0, b = 0, c = 0;
    for (int q = 0; q < kRedBlocks; ++q) {
      const double* P = part + ((size_t)k * kRedBlocks + q) * 3;
      a += P[0];
      b += P[1];
      c += P[2];
    }
    if (lk) lk[k] = a / (double)n;
    if (clamped) clamped[k] = (int)c;
    if (ls) ls[k] = b / (double)n;
  }
}

void Engine::cv_reduce(const double* d_sums, const double* h, const double* d_conv,
                       const double* conv_h, int ns, double* lk, int* clamped, double* ls)
{
  DeviceGuard dg(dev_);
  cv_enqueue(d_sums, h, d_conv, conv_h, ns);
  CK(cudaStreamSynchronize(s_));
  cv_collect(ns, lk, clamped, ls);
}

void Engine::compute_batch_cv(const double* h, int nb, double* d_out, const double* bw,
                              const double* conv_h, int ns, double* lk, int* clamped, double* ls)
{
  DeviceGuard dg(dev_);
  struct Clear {
    std::function<void()>& f;
    ~Clear() { f = nullptr; }
  } clear{ post_batch_ };
  post_batch_ = [&] { cv_enqueue(d_out, bw, conv_h ? d_out + n_ * (size_t)ns : nullptr, conv_h, ns); };
  compute_batch(nullptr, n_, h, nb, d_out);
  cv_collect(ns, lk, clamped, ls);
}

void naive_device(const double* d_q, size_t nq, const double* d_r, size_t nr, int D, double h,
                  double* d_out, cudaStream_t s)
{
  const int TR = 256;
  k_naive<<<ceil_div(nq, 128), 128, TR * D * sizeof(double), s>>>(d_q, (int)nq, d_r, (int)nr, D,
                                                                 -1.0 / (2.0 * h * h), d_out);
  CK_LAUNCH();
}

// Exhaustive error of exp2_neg_fixed over every fixed-point argument the fast base
// case can form: t = M - 896 + u 2^-20 for every u in [0, 1022 2^20), value
// 2^-(u - b) 2^-20, against libdevice exp2 in FP64; and of the clamped variant beyond
// z = 1021 (value exactly 0).  Max relative error as ordered bits in *out.
__global__ void k_mufu_check(unsigned long long* out)
{
  unsigned long long worst = 0;
  const unsigned long long nz = 1022ull << 20;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       i < nz + (4ull << 20); i += (unsigned long long)gridDim.x * blockDim.x) {
    const double t = (kMufuMagic - kMufuBias * 0x1p-20) + (double)i * 0x1p-20;
    double got, want;
    if (i < nz) {
      got = exp2_neg_fixed<false>(t, 0x4B000000u);
      want = exp2(-((double)i - kMufuBias) * 0x1p-20);
    } else {  // clamp: any z >= 1022 - b -> 2^-(1021 + frac of the clamp point)
      got = exp2_neg_fixed<true>(t + 8192.0 * (double)(i & 7), 0x4B000000u);
      if (got != 0.0) worst = 0x7FF0000000000000ull;  // clamped terms must be exactly 0
      continue;
    }
    const double rel = fabs(got - want) / want;
    const unsigned long long b = (unsigned long long)__double_as_longlong(rel);
    worst = b > worst ? b : worst;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, worst, o);
    worst = v > worst ? v : worst;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, worst);
}

double mufu_exp_max_error()
{
  DevBuf<unsigned long long> o;
  o.reserve(1);
  CK(cudaMemset(o.p, 0, sizeof(unsigned long long)));
  k_mufu_check<<<148 * 8, 256>>>(o.p);
  CK_LAUNCH();
  unsigned long long b = 0;
  CK(cudaMemcpy(&b, o.p, sizeof(b), cudaMemcpyDeviceToHost));
  double v;
  std::memcpy(&v, &b, sizeof(v));
  return v;
}

// Exhaustive relative error of ex2.approx.ftz.f32 over every FP32 argument in
// [-126, S] (the FP32 base case's argument S - z; S = kF32Shift) against libdevice exp2
// in FP64.  Max as ordered bits in *out.
__global__ void k_f32_exp_check(unsigned long long* out)
{
  if (blockIdx.x == 0 && threadIdx.x == 0 && (ex2_ftz(kF32Shift) != 0x1p64f || ex2_ftz(0.0f) != 1.0f))
    atomicMax(out, 0x7FF0000000000000ull);  // coincident points (z = 0): exactly 2^S -> 1
  const unsigned lo_pos = 0u, hi_pos = __float_as_uint(kF32Shift);  // [+0, S]
  const unsigned lo_neg = 0x80000001u, hi_neg = __float_as_uint(-126.0f);  // (-0, -126]
  const unsigned long long npos = hi_pos - lo_pos + 1ull, nneg = hi_neg - lo_neg + 1ull;
  unsigned long long worst = 0;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < npos + nneg;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned bits = i < npos ? lo_pos + (unsigned)i : lo_neg + (unsigned)(i - npos);
    const float t = __uint_as_float(bits);
    const double want = exp2((double)t);
    const double rel = fabs((double)ex2_ftz(t) - want) / want;
    const unsigned long long b = (unsigned long long)__double_as_longlong(rel);
    worst = b > worst ? b : worst;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, worst, o);
    worst = v > worst ? v : worst;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, worst);
}

template <int DT>
__global__ void k_f32_terms(const double* q, const double* r, const double* c, int n, double* out)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  constexpr int DF = FPt<DT>::DF;
  double cc[DT];
#pragma unroll
  for (int d = 0; d < DT; ++d) cc[d] = c[d];
  float vq[DF], vr[DF];
  FPt<DT>::centred(FPt<DT>::load_raw(q, i), cc, vq);
  FPt<DT>::centred(FPt<DT>::load_raw(r, i), cc, vr);
  // exactly as base_tile_f32x2 forms it: q~ + (-r~) packed, FFMA2 onto -S, FFMA2s, 2^-S
  float2 a = __fadd2_rn(make_float2(vq[0], vq[0]), make_float2(-vr[0], -vr[0]));
  float2 z = __ffma2_rn(a, a, make_float2(-kF32Shift, -kF32Shift));
#pragma unroll
  for (int d = 1; d < DT; ++d) {
    a = __fadd2_rn(make_float2(vq[d], vq[d]), make_float2(-vr[d], -vr[d]));
    z = __ffma2_rn(a, a, z);
  }
  out[i] = (double)ex2_ftz(-z.x) * kF32Unshift;
  if (ex2_ftz(-z.y) != ex2_ftz(-z.x) || ex2_ftz(-z.x) != f32_term<DT>(vq, vr)) out[i] = -1.0;  // lanes agree
}

__global__ void k_ex2_peak(float* out, int iters)
{
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = -0.001f * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 42.0f) out[0] = s;
}

void Engine::base_split(int& f32_tasks, int& fp64_tasks, unsigned long long& f32_pairs,
                        unsigned long long& fp64_pairs)
{
  DeviceGuard dg(dev_);
  int v[6] = { 0, 0, 0, 0, 0, 0 };
  if (bnext_.p && tasks_.p && brec_.p) {
    CK(cudaMemsetAsync(bnext_.p + 4, 0, 4 * sizeof(int), s_));
    const TreeView Q = view_of(last_q_ ? *last_q_ : rt_);
    auto* pr = reinterpret_cast<unsigned long long*>(bnext_.p + 4);
    const BTask* tk = reinterpret_cast<const BTask*>(tasks_.p);
    const int2* rc = reinterpret_cast<const int2*>(brec_.p);
    k_task_pairs<<<148 * 4, 256, 0, s_>>>(tk, bnext_.p + 8, bnext_.p + 2, rc, Q, last_K_, pr);
    k_task_pairs<<<148 * 4, 256, 0, s_>>>(tk, bnext_.p + 8 + capTask_, bnext_.p + 3, rc, Q, last_K_, pr + 1);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s_));
    CK(cudaMemcpy(v, bnext_.p + 2, sizeof(v), cudaMemcpyDeviceToHost));
  }
  f32_tasks = v[0];
  fp64_tasks = v[1];
  std::memcpy(&f32_pairs, v + 2, 8);
  std::memcpy(&fp64_pairs, v + 4, 8);
}

double f32_exp_max_error()
{
  DevBuf<unsigned long long> o;
  o.reserve(1);
  CK(cudaMemset(o.p, 0, sizeof(unsigned long long)));
  k_f32_exp_check<<<148 * 8, 256>>>(o.p);
  CK_LAUNCH();
  unsigned long long b = 0;
  CK(cudaMemcpy(&b, o.p, sizeof(b), cudaMemcpyDeviceToHost));
  double v;
  std::memcpy(&v, &b, sizeof(v));
  return v;
}

void f32_terms_host(int d, const double* q, const double* r, const double* c, size_t n, double* out)
{
  const int DP = padded_dim(d);
  std::vector<double> hq(n * DP, 0.0), hr(n * DP, 0.0);
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) {
      hq[i * DP + k] = q[i * d + k];
      hr[i * DP + k] = r[i * d + k];
    }
  DevBuf<double> dq, dr, dc, dout;
  dq.reserve(n * DP);
  dr.reserve(n * DP);
  dc.reserve(d);
  dout.reserve(n);
  CK(cudaMemcpy(dq.p, hq.data(), sizeof(double) * n * DP, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dr.p, hr.data(), sizeof(double) * n * DP, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dc.p, c, sizeof(double) * d, cudaMemcpyHostToDevice));
  const int g = (int)((n + 255) / 256);
  switch (d) {
  case 1: k_f32_terms<1><<<g, 256>>>(dq.p, dr.p, dc.p, (int)n, dout.p); break;
  case 2: k_f32_terms<2><<<g, 256>>>(dq.p, dr.p, dc.p, (int)n, dout.p); break;
  case 3: k_f32_terms<3><<<g, 256>>>(dq.p, dr.p, dc.p, (int)n, dout.p); break;
  case 4: k_f32_terms<4><<<g, 256>>>(dq.p, dr.p, dc.p, (int)n, dout.p); break;
  default: k_f32_terms<5><<<g, 256>>>(dq.p, dr.p, dc.p, (int)n, dout.p); break;
  }
  CK_LAUNCH();
  CK(cudaMemcpy(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
}

// Measured MUFU.EX2 throughput (ex2/s): the MUFU base case's roofline denominator.
double measure_ex2_peak(int device)
{
  cudaDeviceProp p{};
  CK(cudaGetDeviceProperties(&p, device));
  DevBuf<float> o;
  o.reserve(1);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  k_ex2_peak<<<blocks, threads>>>(o.p, 64);
  CK(cudaEventRecord(a));
  k_ex2_peak<<<blocks, threads>>>(o.p, iters);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
}

double measure_dfma_peak(int device)
{
  cudaDeviceProp p{};
  CK(cudaGetDeviceProperties(&p, device));
  DevBuf<double> o;
  o.reserve(1);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  k_dfma_peak<<<blocks, threads>>>(o.p, 64);
  CK(cudaEventRecord(a));
  k_dfma_peak<<<blocks, threads>>>(o.p, iters);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
}

}  // namespace dfgtb
