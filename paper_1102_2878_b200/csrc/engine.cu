// DFGT engine on sm_100a: level-synchronous dual-tree traversal and the kernels
// that execute its work lists.
//
// Reference path (all under /root/reference/proj/src):
//   DualTreeEngine::compute       engine.cpp:405-424
//   Traversal::recurse            engine.cpp:113-195   -> k_classify + k_emit (per level)
//   choose_best_method            truncation.cpp:130-166 -> dev_choose
//   Traversal::summarize F/D/T    engine.cpp:197-237   -> k_farfield / k_local_items
//   Traversal::base_case          engine.cpp:239-269   -> k_base_case
//   Traversal::post_process       engine.cpp:271-318   -> k_l2l (top-down) + k_finalize
//   moments_for                   engine.cpp:368-403   -> k_moments (direct, per used node)
//
// Schedule (the reference's recursion replaced; results differ only within eps):
// the frontier of live (Q, R) node pairs is kept grouped by query node (an antichain:
// every query node appears at most once per level), one warp per query node.  The
// error budget of a pair is tau = eps |R| G^l(Q) / |R_total| where G^l(Q) is a valid
// lower bound on every G(q), q in Q:  sum of |R'| K(d_max) over all pairs retired at
// Q or its ancestors (pruned, summarised or sent to the base case) plus over all
// frontier pairs of Q.  Those pairs partition the reference set, so the per-query
// error stays <= eps G(q) exactly as in the reference's proof.
// Work items (F/D/T/base) are appended per level with a per-node rank and counting-
// sorted by query node afterwards, so every kernel accumulates in a fixed order:
// results are bit-reproducible run to run.
#include "engine.cuh"
#include "series_dev.cuh"

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <math_constants.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstring>

namespace dfgtb {

uint64_t& launch_counter()
{
  static uint64_t n = 0;
  return n;
}

int default_p_max(int D)
{  // truncation.cpp:168-186
  switch (D) {
  case 1: return 8;
  case 2: return 6;
  case 3: return 4;
  case 4:
  case 5: return 2;
  default: return 1;
  }
}

namespace cg = cooperative_groups;

namespace {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr int kMaxGridBlocks = 148 * 16;
enum Kind { kE = 0, kF = 1, kD = 2, kT = 3, kB = 4, kX = 5, kFD = 6 };

// ------------------------------------------------------------------ truncation
__device__ double d_binomial(int n, int k)
{
  double b = 1.0;
  for (int i = 1; i <= k; ++i) b *= (double)(n - k + i) / (double)i;
  return b;
}
__device__ double d_sqrt_factorial(int p)
{
  double f = 1.0;
  for (int k = 2; k <= p; ++k) f *= k;
  return sqrt(f);
}
__device__ double d_ipow(double x, int n)
{
  double r = 1.0;
  for (int i = 0; i < n; ++i) r *= x;
  return r;
}
// truncation.cpp:40-54
__device__ double d_bound_sum(double count, double s, int dpow, double a, double b, int dim)
{
  double sum = 0.0;
  for (int k = 0; k < dim; ++k) sum += d_binomial(dim, k) * d_ipow(a, k) * d_ipow(b, dim - k);
  const double pre = count / d_ipow(1.0 - s, dim * dpow);
  double bound = pre * sum;
  if (!isfinite(bound) && count > 0.0 && sum > 0.0)
    bound = exp(log(count) - (double)(dim * dpow) * log1p(-s) + log(sum));
  return bound;
}
__device__ double d_ff_bound(double count, double r, int p, int dim)
{  // truncation.cpp:58-65
  if (count <= 0.0) return 0.0;
  const double rp = d_ipow(r, p);
  return d_bound_sum(count, r, 1, 1.0 - rp, rp / d_sqrt_factorial(p), dim);
}
__device__ double d_f2l_bound(double count, double r, int p, int dim)
{  // truncation.cpp:72-81
  if (count <= 0.0) return 0.0;
  const double s = 2.0 * r, sp = d_ipow(s, p);
  return d_bound_sum(count, s, 2, (1.0 - sp) * (1.0 - sp), sp * (2.0 - sp) / d_sqrt_factorial(p),
                     dim);
}
__device__ int d_order_ff(double ratio, double count, double tau, int pmax, int dim)
{  // truncation.cpp:85-112
  if (ratio >= 1.0) return 0;
  for (int p = 1; p <= pmax; ++p)
    if (d_ff_bound(count, ratio, p, dim) <= tau) return p;
  return 0;
}
__device__ int d_order_f2l(double ratio, double count, double tau, int pmax, int dim)
{  // truncation.cpp:114-128
  if (ratio >= 0.5) return 0;
  for (int p = 1; p <= pmax; ++p)
    if (d_f2l_bound(count, ratio, p, dim) <= tau) return p;
  return 0;
}
// choose_best_method, truncation.cpp:130-166 (ties F > D > T > E)
__device__ void dev_choose(double nq, double nr, double sq, double sr, double h, double tau,
                           int pmax, int dim, int cost, int& kind, int& order)
{
  const int pf = d_order_ff(sr / (2.0 * h), nr, tau, pmax, dim);
  const int pd = d_order_ff(sq / (2.0 * h), nr, tau, pmax, dim);
  const int pt = d_order_f2l((sq < sr ? sr : sq) / (4.0 * h), nr, tau, pmax, dim);
  const double D = (double)dim;
  double cf = CUDART_INF, cd = CUDART_INF, ct = CUDART_INF;
  if (cost == 0) {  // exponential model; integer powers are exact
    if (pf) cf = nq * d_ipow(D, pf + 1);
    if (pd) cd = nr * d_ipow(D, pd + 1);
    if (pt) ct = d_ipow(D, 2 * pt + 1);
  } else {
    if (pf) cf = nq * d_ipow((double)pf, dim);
    if (pd) cd = nr * d_ipow((double)pd, dim);
    if (pt) ct = D * d_ipow((double)pt, 2 * dim);
  }
  const double ce = D * nq * nr;
  const double m1 = cd < cf ? cd : cf, m2 = ce < ct ? ce : ct;
  const double best = m2 < m1 ? m2 : m1;
  if (cf == best) { kind = kF; order = pf; }
  else if (cd == best) { kind = kD; order = pd; }
  else if (ct == best) { kind = kT; order = pt; }
  else { kind = kE; order = 0; }
}

// ------------------------------------------------------------------ traversal
struct TreeView {
  const double *lo, *hi, *cen, *side;
  const int *left, *right, *count, *begin, *parent;
  const double* xs;
};

// Device-resident traversal state.  The level loop runs without host round trips:
// every kernel reads the frontier size and the bandwidth from here, and k_advance
// decides (cudaGraphSetConditional) whether the graph's WHILE node runs another
// level.  Capacities are checked before anything is written; on overflow the loop
// stops and the host regrows the buffers and reruns (engine.cu: Engine::traverse).
struct TravState {
  double h, scale, eps, ntot;          // per compute (host)
  int capE, capP, capF, capDT, capB;   // buffer capacities (host)
  int cur;                             // frontier buffer of the current level
  int m[2], p[2];                      // entries / pairs in each frontier buffer
  int nF, nDT, nB;                     // items emitted so far
  int overflow, levels;
  int done;                            // CTAs finished with their tile sum (k_traverse)
  Cnt lvl;                             // totals of the current level
  unsigned long long pairs, fd, f, dt, t, b, kev;
};

__device__ __forceinline__ Cnt ldcg_cnt(const Cnt* p)
{
  const int* q = reinterpret_cast<const int*>(p);
  return Cnt{ __ldcg(q), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3), __ldcg(q + 4), __ldcg(q + 5),
              __ldcg(q + 6) };
}

struct TravArgs {
  TreeView Q, R;
  int D, pmax, cost, series, T;
  TravState* st;
  int *fq[2], *foff[2], *flen[2], *fr[2];
  double* fbase[2];
  double *pkmax, *pkmin;
  int* dec;
  Cnt *cnt, *cntoff, *tsum, *toff;
  int* childlen;
  double* newbase;
  double* L;
  int* Lord;
  Item *itF, *itDT, *itB;
  int *cntF, *cntDT, *cntB;
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
    lo += l * l;
    const double u1 = bhi[k] - alo[k], u2 = ahi[k] - blo[k];
    const double u = u1 < u2 ? u2 : u1;
    hi += u * u;
  }
  lo2 = lo;
  hi2 = hi;
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total)
{
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

struct CntSum {
  __host__ __device__ Cnt operator()(const Cnt& x, const Cnt& y) const
  {
    return Cnt{ x.e + y.e, x.p + y.p, x.f + y.f, x.dt + y.dt, x.t + y.t, x.b + y.b, x.fd + y.fd };
  }
};

// Root pair (Q root, R root) and a fresh state (host-owned fields untouched).
__global__ void k_trav_init(TravArgs a)
{
  TravState& st = *a.st;
  st.cur = 0;
  st.m[0] = 1;
  st.p[0] = 1;
  st.m[1] = st.p[1] = 0;
  st.nF = st.nDT = st.nB = 0;
  st.overflow = 0;
  st.levels = 0;
  st.done = 0;
  st.lvl = Cnt{};
  st.pairs = st.fd = st.f = st.dt = st.t = st.b = st.kev = 0;
  a.fq[0][0] = 0;
  a.foff[0][0] = 0;
  a.flen[0][0] = 1;
  a.fbase[0][0] = 0.0;
  a.fr[0][0] = 0;
}

// Per-level inputs every warp needs (read once from the state).
struct LevelView {
  int cur, m;
  double h, scale, eps, ntot;
};

__device__ __forceinline__ LevelView level_view(const TravState& st)
{
  return LevelView{ st.cur, st.m[st.cur], st.h, st.scale, st.eps, st.ntot };
}

// One warp, one frontier query node: kernel bounds of every live pair, the lower
// bound G^l, and the prune / summarise / base / expand decision per pair
// (Traversal::recurse, engine.cpp:113-195).
template <int DT>
__device__ __forceinline__ void classify_entry(const TravArgs& a, const LevelView& v, int e, int lane)
{
  const int cur = v.cur;
  const int* fr = a.fr[cur];
  const int D = DT ? DT : a.D;
  const int Q = a.fq[cur][e];
  const int off = a.foff[cur][e], len = a.flen[cur][e];
  const double fb = a.fbase[cur][e];
  const double* qlo = a.Q.lo + (size_t)Q * D;
  const double* qhi = a.Q.hi + (size_t)Q * D;
  const bool qleaf = a.Q.left[Q] < 0;
  const double nq = (double)a.Q.count[Q];
  const double sq = a.Q.side[Q];
  // pass 1: kernel bounds and the lower-bound mass of every live pair
  double part = 0.0;
  for (int j = lane; j < len; j += 32) {
    const int R = fr[off + j];
    double dl, du;
    box_bounds<DT>(qlo, qhi, a.R.lo + (size_t)R * D, a.R.hi + (size_t)R * D, D, dl, du);
    const double kmax = exp(v.scale * dl);  // kernel at closest approach
    const double kmin = exp(v.scale * du);
    a.pkmax[off + j] = kmax;
    a.pkmin[off + j] = kmin;
    part += (double)a.R.count[R] * kmin;
  }
  const double glo = fb + warp_sum(part);
  // pass 2: decisions
  double fd_dlo = 0.0, fd_const = 0.0, ret = 0.0;
  int nF = 0, nDT = 0, nT = 0, nB = 0, nFD = 0, slots = 0;
  unsigned long long kev = 0;
  for (int j = lane; j < len; j += 32) {
    const int R = fr[off + j];
    const double kmax = a.pkmax[off + j], kmin = a.pkmin[off + j];
    const double nr = (double)a.R.count[R];
    const double dlo = nr * kmin;
    const double tau = v.eps * nr * glo / v.ntot;
    int kind = kX, order = 0;
    if (0.5 * nr * (kmax - kmin) <= tau) {  // kernel-difference prune, engine.cpp:137-148
      kind = kFD;
      fd_dlo += dlo;
      fd_const += 0.5 * nr * (kmax + kmin);
      ++nFD;
    } else {
      if (a.series) {
        dev_choose(nq, nr, sq, a.R.side[R], v.h, tau, a.pmax, D, a.cost, kind, order);
        if (kind == kE) kind = kX;
      }
      if (kind == kX && qleaf && a.R.left[R] < 0) kind = kB;
      if (kind == kX) {
        slots += a.R.left[R] < 0 ? 1 : 2;
      } else if (kind == kB) {
        ++nB;
        kev += (unsigned long long)a.Q.count[Q] * (unsigned long long)a.R.count[R];
        ret += dlo;
      } else {
        ret += dlo;
        if (kind == kF) ++nF;
        else {
          ++nDT;
          if (kind == kT) ++nT;
        }
      }
    }
    a.dec[off + j] = kind | (order << 8);
  }
  fd_dlo = warp_sum(fd_dlo);
  fd_const = warp_sum(fd_const);
  ret = warp_sum(ret);
  nF = warp_sum_i(nF);
  nDT = warp_sum_i(nDT);
  nT = warp_sum_i(nT);
  nB = warp_sum_i(nB);
  nFD = warp_sum_i(nFD);
  slots = warp_sum_i(slots);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kev += __shfl_xor_sync(0xffffffffu, kev, o);
  if (lane == 0) {
    const int ne = slots > 0 ? (qleaf ? 1 : 2) : 0;
    a.cnt[e] = Cnt{ ne, ne * slots, nF, nDT, nT, nB, nFD };
    a.childlen[e] = slots;
    a.newbase[e] = fb + (fd_dlo + ret);
    if (nFD) {
      a.L[(size_t)Q * a.T] += fd_const;  // constant local term (order 1)
      if (a.Lord[Q] < 1) a.Lord[Q] = 1;
    }
    if (kev) atomicAdd(&a.st->kev, kev);
  }
}

template <int DT>
__global__ void __launch_bounds__(kBlock) k_classify(TravArgs a)
{
  const LevelView v = level_view(*a.st);
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w0; e < v.m; e += nw) classify_entry<DT>(a, v, e, lane);
}


// Device-side exclusive scan of the per-entry counts (frontier size read from the
// state): tile sums -> one-block scan of the tiles (+ capacity check) -> tile rescan.
constexpr int kScanTiles = 256;
__global__ void __launch_bounds__(256) k_scan_tiles(TravArgs a)
{
  const TravState& st = *a.st;
  const int m = st.m[st.cur];
  const int per = (m + kScanTiles - 1) / kScanTiles;
  const int b0 = blockIdx.x * per, b1 = min(m, b0 + per);
  Cnt acc{};
  for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) acc = CntSum()(acc, a.cnt[i]);
  using BR = cub::BlockReduce<Cnt, 256>;
  __shared__ typename BR::TempStorage tmp;
  const Cnt tot = BR(tmp).Reduce(acc, CntSum());
  if (threadIdx.x == 0) a.tsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanTiles) k_scan_top(TravArgs a)
{
  TravState& st = *a.st;
  using BS = cub::BlockScan<Cnt, kScanTiles>;
  __shared__ typename BS::TempStorage tmp;
  Cnt agg;
  Cnt out;
  BS(tmp).ExclusiveScan(a.tsum[threadIdx.x], out, Cnt{}, CntSum(), agg);
  a.toff[threadIdx.x] = out;
  if (threadIdx.x == 0) {
    st.lvl = agg;
    if (agg.e > st.capE || agg.p > st.capP || (long long)st.nF + agg.f > st.capF ||
        (long long)st.nDT + agg.dt > st.capDT || (long long)st.nB + agg.b > st.capB)
      st.overflow = 1;
  }
}

__global__ void __launch_bounds__(256) k_scan_local(TravArgs a)
{
  const TravState& st = *a.st;
  const int m = st.m[st.cur];
  const int per = (m + kScanTiles - 1) / kScanTiles;
  const int b0 = blockIdx.x * per, b1 = min(m, b0 + per);
  using BS = cub::BlockScan<Cnt, 256>;
  __shared__ typename BS::TempStorage tmp;
  Cnt carry = a.toff[blockIdx.x];
  for (int base = b0; base < b1; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const Cnt v = i < b1 ? a.cnt[i] : Cnt{};
    Cnt ex, agg;
    BS(tmp).ExclusiveScan(v, ex, Cnt{}, CntSum(), agg);
    if (i < b1) a.cntoff[i] = CntSum()(carry, ex);
    carry = CntSum()(carry, agg);
    __syncthreads();
  }
}

// One warp, one frontier query node: write its part of the next frontier and its
// work items at the offsets `o` (exclusive scan of the level's counts).
__device__ __forceinline__ void emit_entry(const TravArgs& a, int cur, int gF, int gDT, int gB,
                                           int e, const Cnt& o, int lane)
{
  const int nxt = cur ^ 1;
  const int* fr = a.fr[cur];
  int* nr = a.fr[nxt];
  const Cnt c = a.cnt[e];
  const int Q = a.fq[cur][e];
  const int off = a.foff[cur][e], len = a.flen[cur][e];
  const bool qleaf = a.Q.left[Q] < 0;
  const int cl = a.childlen[e];
  if (lane == 0 && c.e) {
    const double nb = a.newbase[e];
    if (qleaf) {
      a.fq[nxt][o.e] = Q;
      a.fbase[nxt][o.e] = nb;
      a.foff[nxt][o.e] = o.p;
      a.flen[nxt][o.e] = cl;
    } else {
      a.fq[nxt][o.e] = a.Q.left[Q];
      a.fq[nxt][o.e + 1] = a.Q.right[Q];
      a.fbase[nxt][o.e] = nb;
      a.fbase[nxt][o.e + 1] = nb;
      a.foff[nxt][o.e] = o.p;
      a.foff[nxt][o.e + 1] = o.p + cl;
      a.flen[nxt][o.e] = cl;
      a.flen[nxt][o.e + 1] = cl;
    }
  }
  const int rF = a.cntF[Q], rDT = a.cntDT[Q], rB = a.cntB[Q];
  int runX = 0, runF = 0, runDT = 0, runB = 0;
  for (int j0 = 0; j0 < len; j0 += 32) {
    const int j = j0 + lane;
    int kind = kE, order = 0, R = 0;
    if (j < len) {
      const int dcode = a.dec[off + j];
      kind = dcode & 0xff;
      order = dcode >> 8;
      R = fr[off + j];
    }
    const bool rleaf = (j < len) ? a.R.left[R] < 0 : true;
    int tot;
    const int px = warp_excl_scan(kind == kX ? (rleaf ? 1 : 2) : 0, lane, tot);
    if (kind == kX) {
      const int dst = o.p + runX + px;
      if (rleaf) {
        nr[dst] = R;
        if (!qleaf) nr[dst + cl] = R;
      } else {
        nr[dst] = a.R.left[R];
        nr[dst + 1] = a.R.right[R];
        if (!qleaf) {
          nr[dst + cl] = a.R.left[R];
          nr[dst + cl + 1] = a.R.right[R];
        }
      }
    }
    runX += tot;
    int t2;
    const int pf = warp_excl_scan(kind == kF, lane, t2);
    if (kind == kF) a.itF[gF + o.f + runF + pf] = Item{ Q, R, order | (kF << 8), rF + runF + pf };
    runF += t2;
    const int pd = warp_excl_scan(kind == kD || kind == kT, lane, t2);
    if (kind == kD || kind == kT)
      a.itDT[gDT + o.dt + runDT + pd] = Item{ Q, R, order | (kind << 8), rDT + runDT + pd };
    runDT += t2;
    const int pb = warp_excl_scan(kind == kB, lane, t2);
    if (kind == kB) a.itB[gB + o.b + runB + pb] = Item{ Q, R, kB << 8, rB + runB + pb };
    runB += t2;
  }
  if (lane == 0) {
    a.cntF[Q] = rF + runF;
    a.cntDT[Q] = rDT + runDT;
    a.cntB[Q] = rB + runB;
  }
}

__global__ void __launch_bounds__(kBlock) k_emit(TravArgs a)
{
  const TravState& st = *a.st;
  if (st.overflow) return;
  const int cur = st.cur, m = st.m[cur];
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w0; e < m; e += nw) emit_entry(a, cur, st.nF, st.nDT, st.nB, e, a.cntoff[e], lane);
}

// The whole level loop in ONE cooperative launch (one CTA per SM): per level
//   classify (warp per entry, grid-stride) | grid sync |
//   tile sums over contiguous entry ranges; the last CTA to finish scans the tiles,
//   checks capacities and publishes the level totals | grid sync |
//   each CTA rescans its range and emits it (offsets are local) | grid sync.
// Every CTA advances an identical private copy of (cur, m, item offsets), so no
// extra barrier is needed to publish them; CTA 0 writes the state back at the end.
constexpr int kPBlock = 512;
template <int DT>
__global__ void __launch_bounds__(kPBlock) k_traverse(TravArgs a)
{
  cg::grid_group grid = cg::this_grid();
  TravState& st = *a.st;
  __shared__ int s_last;
  using BR = cub::BlockReduce<Cnt, kPBlock>;
  using BS = cub::BlockScan<Cnt, kPBlock>;
  __shared__ union {
    typename BR::TempStorage r;
    typename BS::TempStorage s;
  } tmp;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int G = gridDim.x;
  int cur = 0, m = 1, p = 1, gF = 0, gDT = 0, gB = 0, levels = 0;
  unsigned long long pairs = 0, fd = 0, f = 0, dt = 0, t = 0, b = 0;
  bool overflow = false;
  LevelView v{ 0, 1, st.h, st.scale, st.eps, st.ntot };
  for (;;) {
    v.cur = cur;
    v.m = m;
    for (int e = gw; e < m; e += nw) classify_entry<DT>(a, v, e, lane);
    grid.sync();
    // tile sums (contiguous ranges of entries per CTA)
    const int per = (m + G - 1) / G;
    const int b0 = min(m, blockIdx.x * per), b1 = min(m, b0 + per);
    Cnt acc{};
    for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) acc = CntSum()(acc, a.cnt[i]);
    const Cnt tot = BR(tmp.r).Reduce(acc, CntSum());
    if (threadIdx.x == 0) {
      a.tsum[blockIdx.x] = tot;
      __threadfence();
      s_last = atomicAdd(&st.done, 1) == G - 1;
    }
    __syncthreads();
    if (s_last) {  // last CTA: scan the tile sums, publish totals and the overflow verdict
      __threadfence();
      Cnt run{};
      for (int base = 0; base < G; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const Cnt x = i < G ? ldcg_cnt(a.tsum + i) : Cnt{};  // other CTAs' tiles: bypass L1
        Cnt ex, agg;
        __syncthreads();
        BS(tmp.s).ExclusiveScan(x, ex, Cnt{}, CntSum(), agg);
        if (i < G) a.toff[i] = CntSum()(run, ex);
        run = CntSum()(run, agg);
      }
      if (threadIdx.x == 0) {
        st.lvl = run;
        st.overflow = run.e > st.capE || run.p > st.capP || (long long)gF + run.f > st.capF ||
                      (long long)gDT + run.dt > st.capDT || (long long)gB + run.b > st.capB;
        st.done = 0;
        __threadfence();
      }
    }
    grid.sync();
    const Cnt lv2 = ldcg_cnt(&st.lvl);
    overflow = __ldcg(&st.overflow) != 0;
    if (overflow) break;
    // local rescan of this CTA's range, then emit it (warp per entry)
    Cnt carry = a.toff[blockIdx.x];
    for (int base = b0; base < b1; base += blockDim.x) {
      const int i = base + threadIdx.x;
      const Cnt x = i < b1 ? a.cnt[i] : Cnt{};
      Cnt ex, agg;
      __syncthreads();
      BS(tmp.s).ExclusiveScan(x, ex, Cnt{}, CntSum(), agg);
      if (i < b1) a.cntoff[i] = CntSum()(carry, ex);
      carry = CntSum()(carry, agg);
    }
    __syncthreads();
    for (int e = b0 + wib; e < b1; e += blockDim.x / 32)
      emit_entry(a, cur, gF, gDT, gB, e, a.cntoff[e], lane);
    // advance (identical in every CTA)
    pairs += p;
    fd += lv2.fd;
    f += lv2.f;
    dt += lv2.dt;
    t += lv2.t;
    b += lv2.b;
    gF += lv2.f;
    gDT += lv2.dt;
    gB += lv2.b;
    cur ^= 1;
    m = lv2.e;
    p = lv2.p;
    ++levels;
    grid.sync();
    if (m == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st.cur = cur;
    st.m[cur] = m;
    st.p[cur] = p;
    st.nF = gF;
    st.nDT = gDT;
    st.nB = gB;
    st.levels = levels;
    st.pairs = pairs;
    st.fd = fd;
    st.f = f;
    st.dt = dt;
    st.t = t;
    st.b = b;
  }
}


// Close the level: fold its totals into the state, flip the frontier buffers and
// tell the WHILE node whether another level follows.
__global__ void k_advance(TravArgs a, cudaGraphConditionalHandle hc, int use_cond)
{
  TravState& st = *a.st;
  if (!st.overflow) {
    const Cnt l = st.lvl;
    st.pairs += st.p[st.cur];
    st.fd += l.fd;
    st.f += l.f;
    st.dt += l.dt;
    st.t += l.t;
    st.b += l.b;
    st.nF += l.f;
    st.nDT += l.dt;
    st.nB += l.b;
    st.m[st.cur ^ 1] = l.e;
    st.p[st.cur ^ 1] = l.p;
    st.cur ^= 1;
    st.levels += 1;
  }
  const bool more = !st.overflow && st.m[st.cur] > 0;
  if (use_cond) cudaGraphSetConditional(hc, more ? 1u : 0u);
}


__global__ void k_scatter_items(const Item* in, int n, const int* noff, Item* out)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const Item it = in[i];
    out[noff[it.q] + it.rank] = it;
  }
}

__global__ void k_mark_moments(const Item* it, int n, int* flag)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int kind = it[i].code >> 8;
    if (kind == kF || kind == kT) flag[it[i].r] = 1;
  }
}

// K2/K3 (large tables, lazy): UNSCALED moments of the reference nodes an F/T item
// uses and that are not cached yet, one block per node over its contiguous points.
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

// K2/K3 (eager, tables <= 4096 terms): unscaled moments of EVERY reference node,
// computed once per tree.  M~_a(node) = (1/a!) sum_r prod_d (r - c)_d^{a_d}; the
// reference's per-h moment is s^|a| M~_a with s = 1/(h sqrt 2) (engine.cpp:368-403
// recomputes per h; one pass serves the whole sweep).  Pass 1: partial sums over
// 64-point chunks of each node; pass 2: per node, chunks summed in order.
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

__global__ void k_moment_reduce(DevSeries g, int nodes, const int* coff, const double* part,
                                double* M)
{
  for (int n = blockIdx.x; n < nodes; n += gridDim.x)
    for (int i = threadIdx.x; i < g.T; i += blockDim.x) {
      double acc = 0.0;
      for (int c = coff[n]; c < coff[n + 1]; ++c) acc += part[(size_t)c * g.T + i];
      M[(size_t)n * g.T + g.pos[i]] = acc * g.invf[i];
    }
}

// s^k, k <= D(p_max-1), for scaling unscaled moments inside F / T kernels.
struct SPow {
  double v[128];
};

// D/T work split into chunks: a D item over <= kLocChunk reference points or one
// T item.  Each chunk writes an unsigned partial table; k_local_reduce sums a query
// node's chunks in item order and applies (-1)^|b|/b! (summarize, engine.cpp:212-232).
constexpr int kLocChunk = 1024;  // points per D chunk (staged 64 at a time)
constexpr int kLocSub = 64;
struct LChunk {
  int item, start, n;
};

__global__ void k_local_count(const Item* items, int n, TreeView R, int* nch)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int kind = items[i].code >> 8;
  nch[i] = kind == kD ? (R.count[items[i].r] + kLocChunk - 1) / kLocChunk : 1;
}

__global__ void k_local_fill(const Item* items, int n, TreeView R, const int* choff, LChunk* ch)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int kind = items[i].code >> 8;
  const int r = items[i].r;
  if (kind == kD) {
    const int b = R.begin[r], c = R.count[r];
    for (int k = 0, st = 0; st < c; ++k, st += kLocChunk)
      ch[choff[i] + k] = LChunk{ i, b + st, min(kLocChunk, c - st) };
  } else {
    ch[choff[i]] = LChunk{ i, -1, 0 };
  }
}

__global__ void k_local_chunks(DevSeries g, TreeView Q, TreeView R, const Item* items,
                               const LChunk* ch, int nch, const double* Mt, SPow sp, double s,
                               double* part)
{
  extern __shared__ double sm[];
  __shared__ double spw[128];
  for (int k = threadIdx.x; k < 128; k += blockDim.x) spw[k] = sp.v[k];
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const LChunk lc = ch[c];
    const Item it = items[lc.item];
    const int kind = it.code >> 8, order = it.code & 0xff;
    double* P = part + (size_t)c * g.T;
    const double* qc = Q.cen + (size_t)it.q * g.D;
    if (kind == kD)
      for (int b = 0; b < lc.n; b += kLocSub)
        dev_direct_local_partial(g, R.xs + (size_t)(lc.start + b) * g.D, min(kLocSub, lc.n - b), qc,
                                 s, order, P, sm, b > 0);
    else
      dev_f2l_block(g, Mt + (size_t)it.r * g.T, R.cen + (size_t)it.r * g.D, qc, s, order, P, sm,
                    spw, 1, g.pos);
  }
}

__global__ void k_local_reduce(DevSeries g, int nodes, const int* cnt, const int* off,
                               const Item* items, const int* choff, const double* part, double* L,
                               int* Lord)
{
  for (int n = blockIdx.x; n < nodes; n += gridDim.x) {
    const int c = cnt[n];
    if (!c) continue;
    const int i0 = off[n], i1 = i0 + c;
    int ord = 0;
    for (int k = i0; k < i1; ++k) ord = max(ord, items[k].code & 0xff);
    const int nt = ipow_i(ord, g.D);
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
      const uint64_t a = g.dig[t];
      int mx = 0;
      for (int d = 0; d < g.D; ++d) mx = max(mx, digit_of(a, d));
      double acc = 0.0;
      for (int k = i0; k < i1; ++k) {
        if (mx >= (items[k].code & 0xff)) continue;  // term beyond this item's order
        for (int q = choff[k]; q < choff[k + 1]; ++q) acc += part[(size_t)q * g.T + t];
      }
      const double sg = (g.degree[t] & 1) ? -1.0 : 1.0;
      L[(size_t)n * g.T + t] += sg * g.invf[t] * acc;
    }
    if (threadIdx.x == 0 && Lord[n] < ord) Lord[n] = ord;
  }
}

// Base-case tasks: a query leaf's (sorted) base items cut into runs of <= kTaskItems
// reference leaves, times 32-query chunks of the leaf.  One warp per task writes
// per-query partial sums; k_finalize adds a query's partials in task order.
constexpr int kTaskItems = 8;
struct BTask {
  int leaf, item0, item1, q0;
};

__global__ void k_task_count(const int* leaves, int nleaves, const int* cntB, TreeView Q, int* nt)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  const int leaf = leaves[i];
  const int ic = (cntB[leaf] + kTaskItems - 1) / kTaskItems;
  nt[i] = ic * ((Q.count[leaf] + 31) / 32);
}

__global__ void k_task_fill(const int* leaves, int nleaves, const int* cntB, const int* offB,
                            TreeView Q, const int* toff, BTask* tasks, int* leaf_task)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  const int leaf = leaves[i];
  const int c = cntB[leaf], o = offB[leaf];
  const int ic = (c + kTaskItems - 1) / kTaskItems;
  int t = toff[i];
  leaf_task[leaf] = t;
  for (int q0 = 0; q0 < Q.count[leaf]; q0 += 32)
    for (int k = 0; k < ic; ++k)
      tasks[t++] = BTask{ leaf, o + k * kTaskItems, o + min(c, (k + 1) * kTaskItems), q0 };
}

// Top-down L2L of one depth level (post_process, engine.cpp:294-304).
__global__ void k_l2l(DevSeries g, TreeView Q, const int* nodes_at, int m, double s, double* L,
                      int* Lord)
{
  extern __shared__ double sm[];
  for (int k = blockIdx.x; k < m; k += gridDim.x) {
    const int n = nodes_at[k];
    const int order = Lord[n];
    if (Q.left[n] < 0 || order <= 0) continue;
    const int ch[2] = { Q.left[n], Q.right[n] };
    for (int c = 0; c < 2; ++c) {
      dev_l2l_block(g, L + (size_t)n * g.T, Q.cen + (size_t)n * g.D, Q.cen + (size_t)ch[c] * g.D, s,
                    order, L + (size_t)ch[c] * g.T, sm);
      __syncthreads();
      if (threadIdx.x == 0 && Lord[ch[c]] < order) Lord[ch[c]] = order;
    }
  }
}

// exp(-y), 0 <= y <= 708.39, to ~1 ulp: Cody-Waite reduction y*log2(e) = n + f,
// r = -y - n ln2 (|r| <= ln2/2), degree-12 Taylor polynomial (truncation
// <= 1.7e-16 relative), 2^n spliced into the exponent field.  Coefficients sit in
// the constant bank so every DFMA takes its constant operand from c[] (libdevice
// exp re-materialises its 64-bit constants with integer moves inside hot loops).
// Same accuracy class as libdevice exp; no reduced precision is charged to eps.
__constant__ double c_expk[15];

__device__ __forceinline__ double exp_negy(double y)
{
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: round to nearest integer
  const double t = fma(-y, c_expk[0], magic);
  const double n = t - magic;
  double r = fma(n, -c_expk[1], -y);
  r = fma(n, -c_expk[2], r);
  double p = c_expk[3];
#pragma unroll
  for (int k = 4; k < 15; ++k) p = fma(p, r, c_expk[k]);
  p = fma(p, r, 1.0);
  const int ni = __double2loint(t);  // n in the low word of t
  return __hiloint2double(__double2hiint(p) + (ni << 20), __double2loint(p));
}

// Scaled, centred, padded coordinates for the base case: x' = (x - c0) / (h sqrt 2)
// so that |q' - r'|^2 = |q - r|^2 / (2 h^2) directly (stride DP, zero padding).
__global__ void k_scale_points(const double* xs, int n, int D, int DP, const double* c0, double s,
                               double* out)
{
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * DP) return;
  const size_t p = i / DP;
  const int d = (int)(i % DP);
  out[i] = d < D ? (xs[p * D + d] - c0[d]) * s : 0.0;
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
};

// K10: exhaustive base case (Traversal::base_case, engine.cpp:239-269).  One warp
// per task = (query leaf, 32-query chunk, run of <= kTaskItems reference leaves):
// lanes own queries, each reference point arrives as one warp-uniform vector load
// (broadcast), two pairs in flight per iteration.  A reference leaf whose box bound
// guarantees y <= 708 for every pair takes the branch-free path; otherwise pairs
// beyond the fast range fall back to libdevice exp (exact underflow behaviour).
template <int DT>
__global__ void __launch_bounds__(kBlock) k_base_case(TreeView Q, TreeView R, const BTask* tasks,
                                                      int ntasks, const Item* items,
                                                      const double* xq, const double* xr,
                                                      double s2, double* part)
{
  constexpr int D = DT;
  constexpr int DP = PtLoad<DT>::DP;
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int w = w0; w < ntasks; w += nw) {
    const BTask t = tasks[w];
    const int qb = Q.begin[t.leaf] + t.q0;
    const bool act = lane < Q.count[t.leaf] - t.q0;
    double q[DP];
    PtLoad<DT>::load(xq, act ? qb + lane : qb, q);
    const double* qlo = Q.lo + (size_t)t.leaf * D;
    const double* qhi = Q.hi + (size_t)t.leaf * D;
    double acc0 = 0.0, acc1 = 0.0;
    for (int k = t.item0; k < t.item1; ++k) {
      const int r = items[k].r;
      const double* rp = xr + (size_t)R.begin[r] * DP;
      const int rc = R.count[r];
      double dl, du;
      box_bounds<DT>(qlo, qhi, R.lo + (size_t)r * D, R.hi + (size_t)r * D, D, dl, du);
      if (s2 * du <= 708.0) {
        int j = 0;
        for (; j + 1 < rc; j += 2) {
          double a[DP], b[DP];
          PtLoad<DT>::load(rp, j, a);
          PtLoad<DT>::load(rp, j + 1, b);
          double ya = 0.0, yb = 0.0;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double ta = q[d] - a[d], tb = q[d] - b[d];
            ya = fma(ta, ta, ya);
            yb = fma(tb, tb, yb);
          }
          acc0 += exp_negy(ya);
          acc1 += exp_negy(yb);
        }
        if (j < rc) {
          double a[DP];
          PtLoad<DT>::load(rp, j, a);
          double ya = 0.0;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double ta = q[d] - a[d];
            ya = fma(ta, ta, ya);
          }
          acc0 += exp_negy(ya);
        }
      } else {
        for (int j = 0; j < rc; ++j) {
          double a[DP];
          PtLoad<DT>::load(rp, j, a);
          double ya = 0.0;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double ta = q[d] - a[d];
            ya = fma(ta, ta, ya);
          }
          acc0 += ya <= 708.0 ? exp_negy(ya) : exp(-ya);
        }
      }
    }
    part[(size_t)w * 32 + lane] = acc0 + acc1;
  }
}

// Generic dimension (D > 5): scalar loads of the scaled coordinates, libdevice exp.
__global__ void __launch_bounds__(kBlock) k_base_case_any(TreeView Q, TreeView R, int D,
                                                          const BTask* tasks, int ntasks,
                                                          const Item* items, const double* xq,
                                                          const double* xr, double* part)
{
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int w = w0; w < ntasks; w += nw) {
    const BTask t = tasks[w];
    const int qb = Q.begin[t.leaf] + t.q0;
    const bool act = lane < Q.count[t.leaf] - t.q0;
    double q[kMaxDim];
    for (int d = 0; d < D; ++d) q[d] = xq[(size_t)(act ? qb + lane : qb) * D + d];
    double acc = 0.0;
    for (int k = t.item0; k < t.item1; ++k) {
      const int r = items[k].r;
      const double* rp = xr + (size_t)R.begin[r] * D;
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

// F items: every query of a leaf evaluates the far-field expansions attached to the
// leaf or any ancestor, root first (eval_farfield per query, engine.cpp:200-211).
__global__ void __launch_bounds__(kBlock) k_farfield(DevSeries g, TreeView Q, TreeView R,
                                                     const int* leaves, int nleaves,
                                                     const int* cnt, const int* off,
                                                     const Item* items, const double* Mt, SPow sp,
                                                     double s, double* s_ff)
{
  __shared__ double spw[128];
  for (int k = threadIdx.x; k < 128; k += blockDim.x) spw[k] = sp.v[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int D = g.D;
  for (int li = w0; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const int qb = Q.begin[leaf], qc = Q.count[leaf];
    int chain[64];
    int depth = 0;
    for (int n = leaf; n >= 0 && depth < 64; n = Q.parent[n]) chain[depth++] = n;
    for (int q0 = 0; q0 < qc; q0 += 32) {
      const int qi = q0 + lane;
      const bool act = qi < qc;
      const double* qp = Q.xs + (size_t)(qb + (act ? qi : 0)) * D;
      double acc = 0.0;
      for (int k = depth - 1; k >= 0; --k) {
        const int n = chain[k];
        const int c = cnt[n];
        const Item* it = items + off[n];
        for (int t = 0; t < c; ++t) {
          const int r = it[t].r, order = it[t].code & 0xff;
          acc += dev_eval_farfield(g, Mt + (size_t)r * g.T, R.cen + (size_t)r * D, qp, s, order,
                                   spw, g.pos);
        }
      }
      if (act) s_ff[qb + qi] = acc;
    }
  }
}

// Specialised far-field evaluation for the default tables (p_max == PM): every
// multi-index is a compile-time constant, so the Hermite rows, s^|a| and the digit
// products live in registers and the (position-layout) moments are read as
// warp-uniform broadcast loads.  Same sum as dev_eval_farfield, same term order.
template <int D, int PM>
__device__ __forceinline__ double ff_eval_t(const double* Mt, const double* c, const double* q,
                                            double s, int order, const double (&spw)[D * (PM - 1) + 1])
{
  double H[D][PM];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double t = (q[d] - c[d]) * s;
    H[d][0] = exp(-t * t);
    if (PM > 1) H[d][1] = 2.0 * t * H[d][0];
#pragma unroll
    for (int k = 1; k + 1 < PM; ++k) H[d][k + 1] = 2.0 * t * H[d][k] - 2.0 * k * H[d][k - 1];
  }
  double sum = 0.0;
  constexpr int NP = ipow_c(PM, D);
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    int dig[D], mx = 0, deg = 0, rest = p;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      dig[d] = rest % PM;
      rest /= PM;
      mx = dig[d] > mx ? dig[d] : mx;
      deg += dig[d];
    }
    if (mx < order) {
      double f = Mt[p] * spw[deg];
#pragma unroll
      for (int d = 0; d < D; ++d) f *= H[d][dig[d]];
      sum += f;
    }
  }
  return sum;
}

template <int D, int PM>
__global__ void __launch_bounds__(kBlock) k_farfield_t(TreeView Q, TreeView R, const int* leaves,
                                                       int nleaves, const int* cnt, const int* off,
                                                       const Item* items, const double* Mt, SPow sp,
                                                       double s, double* s_ff)
{
  constexpr int T = ipow_c(PM, D);
  constexpr int ND = D * (PM - 1) + 1;
  double spw[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) spw[k] = sp.v[k];
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = w0; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const int qb = Q.begin[leaf], qc = Q.count[leaf];
    int chain[64];
    int depth = 0;
    for (int n = leaf; n >= 0 && depth < 64; n = Q.parent[n]) chain[depth++] = n;
    for (int q0 = 0; q0 < qc; q0 += 32) {
      const int qi = q0 + lane;
      const bool act = qi < qc;
      double qv[D];
#pragma unroll
      for (int d = 0; d < D; ++d) qv[d] = Q.xs[(size_t)(qb + (act ? qi : 0)) * D + d];
      double acc = 0.0;
      for (int k = depth - 1; k >= 0; --k) {
        const int n = chain[k];
        const int c = cnt[n];
        const Item* it = items + off[n];
        for (int t = 0; t < c; ++t) {
          const int r = it[t].r, order = it[t].code & 0xff;
          acc += ff_eval_t<D, PM>(Mt + (size_t)r * T, R.cen + (size_t)r * D, qv, s, order, spw);
        }
      }
      if (act) s_ff[qb + qi] = acc;
    }
  }
}

// Local evaluation at the leaves, the base-case partials in task order, and the final
// sum (post_process leaf branch and Traversal::run, engine.cpp:273-291, 85-89);
// results scattered to input order.
// direct != 0: the local expansions of ALL ancestors are evaluated at the query
// (root first) instead of being pushed down by L2L first -- the same polynomial,
// re-centred exactly, without the per-level launch chain.
__global__ void k_finalize(DevSeries g, TreeView Q, const int* leaf_of_pos, const int* perm, int n,
                           const double* L, const int* Lord, const int* cntB,
                           const int* leaf_task, const double* part, const double* s_ff,
                           double s, int direct, double* out)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int leaf = leaf_of_pos[i];
  const double* qp = Q.xs + (size_t)i * g.D;
  double loc = 0.0;
  if (direct) {
    int chain[64];
    int depth = 0;
    for (int a = leaf; a >= 0 && depth < 64; a = Q.parent[a]) chain[depth++] = a;
    for (int k = depth - 1; k >= 0; --k) {
      const int a = chain[k];
      const int order = Lord[a];
      if (order > 0)
        loc += dev_eval_local(g, L + (size_t)a * g.T, Q.cen + (size_t)a * g.D, qp, s, order);
    }
  } else {
    const int order = Lord[leaf];
    if (order > 0)
      loc = dev_eval_local(g, L + (size_t)leaf * g.T, Q.cen + (size_t)leaf * g.D, qp, s, order);
  }
  const int li = i - Q.begin[leaf];
  const int nic = (cntB[leaf] + kTaskItems - 1) / kTaskItems;
  double ex = 0.0;
  if (nic) {
    const int t0 = leaf_task[leaf] + (li >> 5) * nic;
    for (int k = 0; k < nic; ++k) ex += part[(size_t)(t0 + k) * 32 + (li & 31)];
  }
  out[perm[i]] = loc + s_ff[i] + ex;
}

__global__ void k_leaf_of_pos(const int* leaves, int nleaves, const int* begin, const int* count,
                              int* leaf_of_pos)
{
  const int i = blockIdx.x;
  if (i >= nleaves) return;
  const int leaf = leaves[i];
  for (int k = threadIdx.x; k < count[leaf]; k += blockDim.x) leaf_of_pos[begin[leaf] + k] = leaf;
}

// K11: CV reductions (cv.cpp:17-25, 61-97), deterministic two-stage.
constexpr int kRedBlocks = 148;
__global__ void k_cv_partial(const double* sums, const double* conv, int n, double nh, double nc,
                             double* part)
{
  __shared__ double sl[kBlock / 32], ss[kBlock / 32], sc[kBlock / 32];
  double lk = 0.0, ls = 0.0, cl = 0.0;
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int b = blockIdx.x * per, e = min(n, b + per);
  for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
    double loo = sums[i] - 1.0;
    if (loo <= 0.0) {
      loo = DBL_MIN;
      cl += 1.0;
    }
    lk += log(loo / nh);
    if (conv) ls += (conv[i] - 1.0) / nc - 2.0 * ((sums[i] - 1.0) / nh);
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
    for (int k = 0; k < kBlock / 32; ++k) {
      a += sl[k];
      b2 += ss[k];
      c += sc[k];
    }
    part[blockIdx.x * 3 + 0] = a;
    part[blockIdx.x * 3 + 1] = b2;
    part[blockIdx.x * 3 + 2] = c;
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

TreeView view_of(const DevTree& t)
{
  return TreeView{ t.lo.p, t.hi.p, t.centroid.p, t.max_side.p, t.left.p, t.right.p,
                   t.count.p, t.begin.p, t.parent.p, t.xs.p };
}

int grid_warps(long long work)
{
  return (int)std::max<long long>(1, std::min<long long>(kMaxGridBlocks, (work + kWarpsPerBlock - 1) / kWarpsPerBlock));
}

void launch_classify(int D, int grid, cudaStream_t s, const TravArgs& a)
{
  switch (D) {
  case 1: k_classify<1><<<grid, kBlock, 0, s>>>(a); break;
  case 2: k_classify<2><<<grid, kBlock, 0, s>>>(a); break;
  case 3: k_classify<3><<<grid, kBlock, 0, s>>>(a); break;
  case 4: k_classify<4><<<grid, kBlock, 0, s>>>(a); break;
  case 5: k_classify<5><<<grid, kBlock, 0, s>>>(a); break;
  default: k_classify<0><<<grid, kBlock, 0, s>>>(a); break;
  }
  CK_LAUNCH();
}

void launch_base(int D, int grid, cudaStream_t s, TreeView Q, TreeView R, const BTask* tasks,
                 int ntasks, const Item* items, const double* xq, const double* xr, double s2,
                 double* part)
{
  switch (D) {
  case 1: k_base_case<1><<<grid, kBlock, 0, s>>>(Q, R, tasks, ntasks, items, xq, xr, s2, part); break;
  case 2: k_base_case<2><<<grid, kBlock, 0, s>>>(Q, R, tasks, ntasks, items, xq, xr, s2, part); break;
  case 3: k_base_case<3><<<grid, kBlock, 0, s>>>(Q, R, tasks, ntasks, items, xq, xr, s2, part); break;
  case 4: k_base_case<4><<<grid, kBlock, 0, s>>>(Q, R, tasks, ntasks, items, xq, xr, s2, part); break;
  case 5: k_base_case<5><<<grid, kBlock, 0, s>>>(Q, R, tasks, ntasks, items, xq, xr, s2, part); break;
  default: k_base_case_any<<<grid, kBlock, 0, s>>>(Q, R, D, tasks, ntasks, items, xq, xr, part); break;
  }
  CK_LAUNCH();
}

int padded_dim(int D) { return D == 1 ? 1 : (D <= 5 ? (D + 1) / 2 * 2 : D); }

}  // namespace

// ======================================================================= Engine

Engine::Engine(const double* refs, size_t n, size_t d, const Config& cfg, bool on_device)
  : cfg_(cfg)
{
  if (n == 0 || d == 0) throw InvalidArgument("PointSet requires N >= 1 and D >= 1");
  if (n > (size_t)INT32_MAX / 2) throw InvalidArgument("N too large for 32-bit node ids");
  if (cfg.epsilon < 0.0) throw InvalidArgument("epsilon must be >= 0");
  if (cfg.leaf_threshold < 1) throw InvalidArgument("leaf_threshold must be >= 1");
  D_ = (int)d;
  n_ = n;
  const int pm = cfg.mode == 0 ? 1 : (cfg.p_max > 0 ? cfg.p_max : default_p_max(D_));
  if (cfg.p_max < 0 || (cfg.mode == 1 && cfg.p_max > 15)) throw InvalidArgument("SeriesGeometry requires dim >= 1 and 1 <= p_max <= 15");
  ser_ = SeriesTables(D_, pm);
  if (D_ * (pm - 1) >= 128) throw InvalidArgument("D * (p_max - 1) must be < 128");
  if (D_ > kMaxDim) throw InvalidArgument("dimension > 16 is not supported by the device engine");
  CK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
  for (auto& e : ev_) CK(cudaEventCreate(&e));
  x_.reserve(n * d);
  CK(cudaMemcpyAsync(x_.p, refs, sizeof(double) * n * d,
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s_));
  upload_series(ser_, ser_dev_, s_);
  {  // exp_negy constants: log2(e), Cody-Waite ln2 split, 1/12! ... 1/1!
    double k[15];
    k[0] = 1.4426950408889634;
    k[1] = 6.93147180369123816490e-01;
    k[2] = 1.90821492927058770002e-10;
    double f = 1.0;
    for (int i = 1; i <= 12; ++i) {
      f *= i;
      k[3 + (12 - i)] = 1.0 / f;
    }
    CK(cudaMemcpyToSymbolAsync(c_expk, k, sizeof(k), 0, cudaMemcpyHostToDevice, s_));
  }
  CK(cudaEventRecord(ev_[0], s_));
  build_tree(rt_, x_.p, (int)n, D_, cfg.leaf_threshold, s_);
  if (cfg.mode == 1) {
    if (ser_.T <= 4096) {
      eager_ = true;
      eager_moments();
    } else {
      Mt_.reserve((size_t)rt_.nodes * ser_.T);
      mdone_.reserve(rt_.nodes);
      CK(cudaMemsetAsync(mdone_.p, 0, sizeof(int) * rt_.nodes, s_));
    }
  }
  CK(cudaEventRecord(ev_[1], s_));
  CK(cudaStreamSynchronize(s_));
  CK(cudaEventElapsedTime(&tim_.tree_ms, ev_[0], ev_[1]));
  dstat_.reserve(4);
}

Engine::~Engine()
{
  if (s_) cudaStreamSynchronize(s_);
  destroy_graph();
  if (hst_) cudaFreeHost(hst_);
  for (auto& e : ev_) cudaEventDestroy(e);
  if (s_) cudaStreamDestroy(s_);
}

DevSeries Engine::dev_series() const { return series_view(ser_, ser_dev_); }

void upload_series(const SeriesTables& t, DevBuf<unsigned char>& dev, cudaStream_t s)
{
  const int T = t.T;
  const size_t bytes = sizeof(uint64_t) * T + sizeof(double) * 2 * T + sizeof(int) * 3 * T;
  dev.reserve(bytes);
  std::vector<unsigned char> blob(bytes);
  unsigned char* p = blob.data();
  std::memcpy(p, t.dig.data(), sizeof(uint64_t) * T);
  p += sizeof(uint64_t) * T;
  std::memcpy(p, t.invf.data(), sizeof(double) * T);
  p += sizeof(double) * T;
  std::memcpy(p, t.fact.data(), sizeof(double) * T);
  p += sizeof(double) * T;
  std::memcpy(p, t.degree.data(), sizeof(int) * T);
  p += sizeof(int) * T;
  std::memcpy(p, t.term_of_pos.data(), sizeof(int) * T);
  p += sizeof(int) * T;
  std::memcpy(p, t.pos.data(), sizeof(int) * T);
  CK(cudaMemcpyAsync(dev.p, blob.data(), bytes, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

DevSeries series_view(const SeriesTables& t, const DevBuf<unsigned char>& dev)
{
  const int T = t.T;
  const unsigned char* p = dev.p;
  DevSeries g;
  g.D = t.D;
  g.pmax = t.pmax;
  g.T = T;
  g.dig = (const uint64_t*)p;
  p += sizeof(uint64_t) * T;
  g.invf = (const double*)p;
  p += sizeof(double) * T;
  g.fact = (const double*)p;
  p += sizeof(double) * T;
  g.degree = (const int*)p;
  p += sizeof(int) * T;
  g.term_of_pos = (const int*)p;
  p += sizeof(int) * T;
  g.pos = (const int*)p;
  return g;
}

// The kernels of one traversal level (all sizes read from the device state).
constexpr int kLevelKernels = 6;
static void launch_level(const TravArgs& a, int D, cudaStream_t s, cudaGraphConditionalHandle hc,
                         int use_cond)
{
  const int grid = 148 * 4;
  launch_classify(D, grid, s, a);
  k_scan_tiles<<<kScanTiles, 256, 0, s>>>(a);
  CK_LAUNCH();
  k_scan_top<<<1, kScanTiles, 0, s>>>(a);
  CK_LAUNCH();
  k_scan_local<<<kScanTiles, 256, 0, s>>>(a);
  CK_LAUNCH();
  k_emit<<<grid, kBlock, 0, s>>>(a);
  CK_LAUNCH();
  k_advance<<<1, 1, 0, s>>>(a, hc, use_cond);
  CK_LAUNCH();
}

void Engine::destroy_graph()
{
  if (gexec_) cudaGraphExecDestroy(gexec_);
  if (graph_) cudaGraphDestroy(graph_);
  gexec_ = nullptr;
  graph_ = nullptr;
  gsig_.clear();
}

// Runs the whole level loop.  Preferred: one CUDA graph whose WHILE node repeats the
// level kernels until k_advance clears the condition -- no host round trip per
// level.  Fallback (graph build failed): the host launches levels and polls.
void Engine::run_levels(const void* args, const std::vector<const void*>& sig)
{
  const TravArgs& a = *static_cast<const TravArgs*>(args);
  if (use_persistent_) {
    void* fn = nullptr;
    switch (D_) {
    case 1: fn = (void*)k_traverse<1>; break;
    case 2: fn = (void*)k_traverse<2>; break;
    case 3: fn = (void*)k_traverse<3>; break;
    case 4: fn = (void*)k_traverse<4>; break;
    case 5: fn = (void*)k_traverse<5>; break;
    default: fn = (void*)k_traverse<0>; break;
    }
    int dev = 0, nsm = 0, per_sm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPBlock, 0));
    if (per_sm >= 1) {
      TravArgs copy = a;
      void* kargs[] = { &copy };
      CK(cudaLaunchCooperativeKernel(fn, nsm, kPBlock, kargs, 0, s_));
      ++launch_counter();
      return;
    }
    use_persistent_ = false;  // cannot co-schedule one CTA per SM: use the graph loop
  }
  if (use_graph_ && sig != gsig_) {
    destroy_graph();
    const uint64_t before = launch_counter();
    try {
      CK(cudaGraphCreate(&graph_, 0));
      CK(cudaGraphConditionalHandleCreate(&hc_, graph_, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams p = {};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = hc_;
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, graph_, nullptr, 0, &p));
      cudaGraph_t body = p.conditional.phGraph_out[0];
      CK(cudaStreamBeginCaptureToGraph(s_, body, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      launch_level(a, D_, s_, hc_, 1);
      CK(cudaStreamEndCapture(s_, &body));
      CK(cudaGraphInstantiate(&gexec_, graph_, 0));
      gsig_ = sig;
    } catch (const CudaError&) {
      cudaStreamCaptureStatus cs;
      if (cudaStreamIsCapturing(s_, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(s_, &junk);
        if (junk) cudaGraphDestroy(junk);
      }
      cudaGetLastError();
      destroy_graph();
      use_graph_ = false;
    }
    launch_counter() = before;  // captured launches are counted when they execute
  }
  if (use_graph_) {
    CK(cudaGraphLaunch(gexec_, s_));
    return;
  }
  TravState* hs = static_cast<TravState*>(hst_);
  for (;;) {
    launch_level(a, D_, s_, 0, 0);
    CK(cudaMemcpyAsync(hs, a.st, sizeof(TravState), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    if (hs->overflow || hs->m[hs->cur] == 0) break;
  }
}

void Engine::traverse(const DevTree& qt, double h)
{
  const int K = qt.nodes;
  const int T = ser_.T;
  cudaStream_t s = s_;
  L_.reserve((size_t)K * T);
  for (DevBuf<int>* b : { &Lord_, &cntF_, &cntDT_, &cntB_ }) b->reserve(K);
  if (!hst_) {
    CK(cudaMallocHost(&hst_, sizeof(TravState)));
    dst_.reserve(sizeof(TravState));
  }
  TravState* hs = static_cast<TravState*>(hst_);
  TravState* ds = reinterpret_cast<TravState*>(dst_.p);
  if (capE_ == 0) {  // first guesses; overflow regrows (and the engine keeps the sizes)
    capE_ = std::max(4096, 2 * K);
    capP_ = std::max(1 << 16, 16 * K);
    capF_ = capDT_ = std::max(4096, 2 * K);
    capB_ = std::max(1 << 16, 16 * K);
  }
  for (int attempt = 0;; ++attempt) {
    for (int b = 0; b < 2; ++b) {
      fq_[b].reserve(capE_);
      foff_[b].reserve(capE_);
      flen_[b].reserve(capE_);
      fbase_[b].reserve(capE_);
      fr_[b].reserve(capP_);
    }
    pkmax_.reserve(capP_);
    pkmin_.reserve(capP_);
    dec_.reserve(capP_);
    cnt_.reserve(capE_);
    cntoff_.reserve(capE_);
    childlen_.reserve(capE_);
    newbase_.reserve(capE_);
    ctsum_.reserve(kScanTiles);
    ctoff_.reserve(kScanTiles);
    itF_.reserve(capF_);
    itDT_.reserve(capDT_);
    itB_.reserve(capB_);

    TravArgs a{};
    a.Q = view_of(qt);
    a.R = view_of(rt_);
    a.D = D_;
    a.pmax = ser_.pmax;
    a.cost = cfg_.cost_model;
    a.series = cfg_.mode == 1;
    a.T = T;
    a.st = ds;
    for (int b = 0; b < 2; ++b) {
      a.fq[b] = fq_[b].p;
      a.foff[b] = foff_[b].p;
      a.flen[b] = flen_[b].p;
      a.fr[b] = fr_[b].p;
      a.fbase[b] = fbase_[b].p;
    }
    a.pkmax = pkmax_.p;
    a.pkmin = pkmin_.p;
    a.dec = dec_.p;
    a.cnt = cnt_.p;
    a.cntoff = cntoff_.p;
    a.tsum = ctsum_.p;
    a.toff = ctoff_.p;
    a.childlen = childlen_.p;
    a.newbase = newbase_.p;
    a.L = L_.p;
    a.Lord = Lord_.p;
    a.itF = itF_.p;
    a.itDT = itDT_.p;
    a.itB = itB_.p;
    a.cntF = cntF_.p;
    a.cntDT = cntDT_.p;
    a.cntB = cntB_.p;
    const std::vector<const void*> sig = {
      a.Q.lo, a.Q.hi, a.Q.cen, a.Q.side, a.Q.left, a.Q.right, a.Q.count, a.Q.begin,
      a.R.lo, a.R.hi, a.R.side, a.R.left, a.R.right, a.R.count,
      a.st, a.fq[0], a.fq[1], a.foff[0], a.foff[1], a.flen[0], a.flen[1], a.fr[0], a.fr[1],
      a.fbase[0], a.fbase[1], a.pkmax, a.pkmin, a.dec, a.cnt, a.cntoff, a.tsum, a.toff,
      a.childlen, a.newbase, a.L, a.Lord, a.itF, a.itDT, a.itB, a.cntF, a.cntDT, a.cntB };

    CK(cudaMemsetAsync(L_.p, 0, sizeof(double) * K * T, s));
    for (DevBuf<int>* b : { &Lord_, &cntF_, &cntDT_, &cntB_ })
      CK(cudaMemsetAsync(b->p, 0, sizeof(int) * K, s));
    hs->h = h;
    hs->scale = -1.0 / (2.0 * h * h);
    hs->eps = cfg_.epsilon;
    hs->ntot = (double)n_;
    hs->capE = capE_;
    hs->capP = capP_;
    hs->capF = capF_;
    hs->capDT = capDT_;
    hs->capB = capB_;
    CK(cudaMemcpyAsync(ds, hs, sizeof(TravState), cudaMemcpyHostToDevice, s));
    k_trav_init<<<1, 1, 0, s>>>(a);
    CK_LAUNCH();
    run_levels(&a, sig);
    CK(cudaMemcpyAsync(hs, ds, sizeof(TravState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!use_persistent_ && use_graph_) launch_counter() += (uint64_t)hs->levels * kLevelKernels;
    if (!hs->overflow) break;
    if (attempt > 10) throw OutOfMemory("traversal buffers keep overflowing");
    const Cnt l = hs->lvl;
    auto grow = [](int cap, long long need) {
      if (need > INT32_MAX / 2) throw OutOfMemory("traversal exceeds 2^30 entries");
      return (int)std::max<long long>(cap, 2 * need);
    };
    capE_ = grow(capE_, l.e);
    capP_ = grow(capP_, l.p);
    capF_ = grow(capF_, (long long)hs->nF + l.f);
    capDT_ = grow(capDT_, (long long)hs->nDT + l.dt);
    capB_ = grow(capB_, (long long)hs->nB + l.b);
  }
  stats_ = Stats{};
  stats_.levels = hs->levels;
  stats_.pairs_visited = hs->pairs;
  stats_.prunes_finite_diff = hs->fd;
  stats_.prunes_farfield = hs->f;
  stats_.prunes_direct_local = hs->dt - hs->t;
  stats_.prunes_far_to_local = hs->t;
  stats_.base_cases = hs->b;
  stats_.kernel_evaluations = 2ull * hs->pairs + hs->kev;
  nF_ = hs->nF;
  nDT_ = hs->nDT;
  nB_ = hs->nB;

  // counting sort of the items by query node (stable: level order, then emit order)
  auto sort_items = [&](DevBuf<Item>& in, long long nitems, DevBuf<int>& cnt, DevBuf<int>& off,
                        DevBuf<Item>& out) {
    off.reserve((size_t)K + 1);
    if (nitems == 0) return;
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, cnt.p, off.p, K, s);
    scan_tmp_.reserve(need + 256);
    size_t have = scan_tmp_.cap;
    cub::DeviceScan::ExclusiveSum(scan_tmp_.p, have, cnt.p, off.p, K, s);
    out.reserve(nitems);
    k_scatter_items<<<ceil_div(nitems, 256), 256, 0, s>>>(in.p, (int)nitems, off.p, out.p);
    CK_LAUNCH();
  };
  sort_items(itF_, nF_, cntF_, offF_, sF_);
  sort_items(itDT_, nDT_, cntDT_, offDT_, sDT_);
  sort_items(itB_, nB_, cntB_, offB_, sB_);
}

// Unscaled moments of every reference node, once per tree (tables <= 4096 terms).
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
  DevBuf<int> dn, ds, dof;
  DevBuf<double> part;
  dn.reserve(nch);
  ds.reserve(nch);
  dof.reserve(K + 1);
  part.reserve((size_t)nch * T);
  CK(cudaMemcpyAsync(dn.p, cnode.data(), sizeof(int) * nch, cudaMemcpyHostToDevice, s_));
  CK(cudaMemcpyAsync(ds.p, cstart.data(), sizeof(int) * nch, cudaMemcpyHostToDevice, s_));
  CK(cudaMemcpyAsync(dof.p, coff.data(), sizeof(int) * (K + 1), cudaMemcpyHostToDevice, s_));
  Mt_.reserve((size_t)K * T);
  const DevSeries g = dev_series();
  const int smem = kMomChunk * D_ * ser_.pmax * (int)sizeof(double);
  k_moment_chunks<<<std::min(nch, 148 * 16), 128, smem, s_>>>(g, view_of(t), dn.p, ds.p, nch,
                                                               part.p);
  CK_LAUNCH();
  k_moment_reduce<<<std::min(K, 148 * 16), 128, 0, s_>>>(g, K, dof.p, part.p, Mt_.p);
  CK_LAUNCH();
  CK(cudaStreamSynchronize(s_));
}

void Engine::run_phases(const DevTree& qt, double h, double* d_out)
{
  cudaStream_t s = s_;
  const DevSeries g = dev_series();
  const double sc = inv_scale(h);
  const TreeView Q = view_of(qt), R = view_of(rt_);
  const int K = qt.nodes, T = ser_.T;
  CK(cudaEventRecord(ev_[2], s));
  traverse(qt, h);
  CK(cudaEventRecord(ev_[3], s));
  SPow sp;
  sp.v[0] = 1.0;
  for (int k = 1; k < 128; ++k) sp.v[k] = sp.v[k - 1] * sc;
  // moments of the reference nodes used by F/T items (large tables only; small
  // tables were computed for every node when the engine was built)
  const bool need_m = stats_.prunes_farfield + stats_.prunes_far_to_local > 0;
  if (need_m && !eager_) {
    mflag_.reserve(rt_.nodes);
    CK(cudaMemsetAsync(mflag_.p, 0, sizeof(int) * rt_.nodes, s));
    if (nF_) {
      k_mark_moments<<<ceil_div(nF_, 256), 256, 0, s>>>(sF_.p, (int)nF_, mflag_.p);
      CK_LAUNCH();
    }
    if (nDT_) {
      k_mark_moments<<<ceil_div(nDT_, 256), 256, 0, s>>>(sDT_.p, (int)nDT_, mflag_.p);
      CK_LAUNCH();
    }
    const int smem = 32 * D_ * ser_.pmax * (int)sizeof(double);
    k_moments<<<std::min(rt_.nodes, 148 * 8), 128, smem, s>>>(g, R, rt_.nodes, mflag_.p, mdone_.p,
                                                             Mt_.p);
    CK_LAUNCH();
  }
  CK(cudaEventRecord(ev_[4], s));
  // D/T items -> chunked partial tables -> per-query-node reduction
  if (nDT_) {
    lnch_.reserve(nDT_ + 1);
    lchoff_.reserve(nDT_ + 1);
    k_local_count<<<ceil_div(nDT_, 256), 256, 0, s>>>(sDT_.p, (int)nDT_, R, lnch_.p);
    CK_LAUNCH();
    CK(cudaMemsetAsync(lnch_.p + nDT_, 0, sizeof(int), s));
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, lnch_.p, lchoff_.p, (int)nDT_ + 1, s);
    scan_tmp_.reserve(need + 256);
    size_t have = scan_tmp_.cap;
    cub::DeviceScan::ExclusiveSum(scan_tmp_.p, have, lnch_.p, lchoff_.p, (int)nDT_ + 1, s);
    int nch = 0;
    CK(cudaMemcpyAsync(&nch, lchoff_.p + nDT_, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    lchunk_.reserve((size_t)nch * 3);
    LChunk* ch = reinterpret_cast<LChunk*>(lchunk_.p);
    k_local_fill<<<ceil_div(nDT_, 256), 256, 0, s>>>(sDT_.p, (int)nDT_, R, lchoff_.p, ch);
    CK_LAUNCH();
    lpart_.reserve((size_t)nch * T);
    const int smem = std::max(kLocSub * D_ * ser_.pmax, D_ * (2 * ser_.pmax)) * (int)sizeof(double);
    k_local_chunks<<<std::min(nch, 148 * 16), 64, smem, s>>>(g, Q, R, sDT_.p, ch, nch, Mt_.p, sp, sc,
                                                             lpart_.p);
    CK_LAUNCH();
    k_local_reduce<<<std::min(K, 148 * 16), 64, 0, s>>>(g, K, cntDT_.p, offDT_.p, sDT_.p,
                                                        lchoff_.p, lpart_.p, L_.p, Lord_.p);
    CK_LAUNCH();
  }
  if (cfg_.local_pushdown == 1 &&
      stats_.prunes_finite_diff + stats_.prunes_direct_local + stats_.prunes_far_to_local > 0) {
    const int smem = D_ * ser_.pmax * (int)sizeof(double);
    for (int d = 0; d + 1 < qt.height; ++d) {
      const int b = qt.depth_off[d], e = qt.depth_off[d + 1];
      k_l2l<<<std::min(e - b, 148 * 8), 64, smem, s>>>(g, Q, qt.by_depth.p + b, e - b, sc, L_.p,
                                                       Lord_.p);
      CK_LAUNCH();
    }
  }
  CK(cudaEventRecord(ev_[5], s));
  // base-case tasks
  const int nleaves = (int)qleaves_host_.size();
  int ntasks = 0;
  if (nB_) {
    ntask_.reserve(nleaves + 1);
    toff_.reserve(nleaves + 1);
    k_task_count<<<ceil_div(nleaves, 256), 256, 0, s>>>(leaves_.p, nleaves, cntB_.p, Q, ntask_.p);
    CK_LAUNCH();
    CK(cudaMemsetAsync(ntask_.p + nleaves, 0, sizeof(int), s));
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, ntask_.p, toff_.p, nleaves + 1, s);
    scan_tmp_.reserve(need + 256);
    size_t have = scan_tmp_.cap;
    cub::DeviceScan::ExclusiveSum(scan_tmp_.p, have, ntask_.p, toff_.p, nleaves + 1, s);
    CK(cudaMemcpyAsync(&ntasks, toff_.p + nleaves, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    tasks_.reserve((size_t)ntasks * 4);
    leaf_task_.reserve(K);
    k_task_fill<<<ceil_div(nleaves, 256), 256, 0, s>>>(leaves_.p, nleaves, cntB_.p, offB_.p, Q,
                                                       toff_.p, reinterpret_cast<BTask*>(tasks_.p),
                                                       leaf_task_.p);
    CK_LAUNCH();
    bpart_.reserve((size_t)ntasks * 32);
  } else {
    leaf_task_.reserve(K);
    bpart_.reserve(32);
  }
  const double* xq = nullptr;
  const double* xr = nullptr;
  if (ntasks) {  // scaled, centred, padded coordinates (Q and, if different, R)
    const int DP = padded_dim(D_);
    xq_.reserve((size_t)qt.n * DP);
    k_scale_points<<<ceil_div((long long)qt.n * DP, 256), 256, 0, s>>>(qt.xs.p, qt.n, D_, DP,
                                                                       rt_.centroid.p, sc, xq_.p);
    CK_LAUNCH();
    xq = xr = xq_.p;
    if (&qt != &rt_) {
      xr_.reserve((size_t)rt_.n * DP);
      k_scale_points<<<ceil_div((long long)rt_.n * DP, 256), 256, 0, s>>>(rt_.xs.p, rt_.n, D_, DP,
                                                                          rt_.centroid.p, sc, xr_.p);
      CK_LAUNCH();
      xr = xr_.p;
    }
  }
  CK(cudaEventRecord(ev_[9], s));
  if (ntasks)
    launch_base(D_, grid_warps(ntasks), s, Q, R, reinterpret_cast<const BTask*>(tasks_.p), ntasks,
                sB_.p, xq, xr, 1.0 / (2.0 * h * h), bpart_.p);
  CK(cudaEventRecord(ev_[6], s));
  s_ff_.reserve(qt.n);
  if (nF_) {
    const int gw = grid_warps(nleaves);
    const int pm = ser_.pmax;
#define FF_T(DD, PP)                                                                         \
  k_farfield_t<DD, PP><<<gw, kBlock, 0, s>>>(Q, R, leaves_.p, nleaves, cntF_.p, offF_.p, sF_.p, \
                                             Mt_.p, sp, sc, s_ff_.p)
    if (D_ == 1 && pm == 8) FF_T(1, 8);
    else if (D_ == 2 && pm == 6) FF_T(2, 6);
    else if (D_ == 3 && pm == 4) FF_T(3, 4);
    else if (D_ == 4 && pm == 2) FF_T(4, 2);
    else if (D_ == 5 && pm == 2) FF_T(5, 2);
    else
      k_farfield<<<gw, kBlock, 0, s>>>(g, Q, R, leaves_.p, nleaves, cntF_.p, offF_.p, sF_.p, Mt_.p,
                                      sp, sc, s_ff_.p);
#undef FF_T
    CK_LAUNCH();
  } else {
    CK(cudaMemsetAsync(s_ff_.p, 0, sizeof(double) * qt.n, s));
  }
  CK(cudaEventRecord(ev_[7], s));
  k_finalize<<<ceil_div(qt.n, 128), 128, 0, s>>>(g, Q, leaf_of_pos_.p, qt.perm.p, qt.n, L_.p,
                                                 Lord_.p, cntB_.p, leaf_task_.p, bpart_.p, s_ff_.p,
                                                 sc, cfg_.local_pushdown == 0, d_out);
  CK_LAUNCH();
  CK(cudaEventRecord(ev_[8], s));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventElapsedTime(&tim_.traverse_ms, ev_[2], ev_[3]));
  CK(cudaEventElapsedTime(&tim_.moments_ms, ev_[3], ev_[4]));
  CK(cudaEventElapsedTime(&tim_.local_ms, ev_[4], ev_[5]));
  CK(cudaEventElapsedTime(&tim_.base_ms, ev_[9], ev_[6]));
  CK(cudaEventElapsedTime(&tim_.farfield_ms, ev_[6], ev_[7]));
  CK(cudaEventElapsedTime(&tim_.final_ms, ev_[7], ev_[8]));
  CK(cudaEventElapsedTime(&tim_.total_ms, ev_[2], ev_[8]));
}

static void setup_leaves(const DevTree& t, DevBuf<int>& leaves, DevBuf<int>& leaf_of_pos,
                         std::vector<int>& host, cudaStream_t s)
{
  host.clear();
  for (int i = 0; i < t.nodes; ++i)
    if (t.h_left[i] < 0) host.push_back(i);
  leaves.reserve(host.size());
  CK(cudaMemcpyAsync(leaves.p, host.data(), sizeof(int) * host.size(), cudaMemcpyHostToDevice, s));
  leaf_of_pos.reserve(t.n);
  k_leaf_of_pos<<<(int)host.size(), 64, 0, s>>>(leaves.p, (int)host.size(), t.begin.p, t.count.p,
                                                leaf_of_pos.p);
  CK_LAUNCH();
  CK(cudaStreamSynchronize(s));
}

void Engine::compute_device(const double* d_queries, size_t nq, double h, double* d_out)
{
  if (!(h > 0.0)) throw InvalidArgument("bandwidth must be positive");
  if (!std::isfinite(h)) throw InvalidArgument("bandwidth must be positive and finite");
  const DevTree* qt = &rt_;
  if (d_queries) {
    if (nq == 0) throw InvalidArgument("PointSet requires N >= 1 and D >= 1");
    cudaEvent_t a = ev_[0], b = ev_[1];
    CK(cudaEventRecord(a, s_));
    build_tree(qt_tmp_, d_queries, (int)nq, D_, cfg_.leaf_threshold, s_);  // engine.cpp:417
    CK(cudaEventRecord(b, s_));
    qt = &qt_tmp_;
    setup_leaves(*qt, leaves_, leaf_of_pos_, qleaves_host_, s_);
  } else if (leaves_src_ != 0) {
    setup_leaves(rt_, leaves_, leaf_of_pos_, qleaves_host_, s_);
  }
  leaves_src_ = d_queries == nullptr ? 0 : 1;
  run_phases(*qt, h, d_out);
}

void Engine::compute_host(const double* h_queries, size_t nq, double h, double* h_out)
{
  const size_t n_out = h_queries ? nq : n_;
  DevBuf<double> out;
  out.reserve(n_out);
  if (h_queries) {
    qx_.reserve(nq * D_);
    CK(cudaMemcpyAsync(qx_.p, h_queries, sizeof(double) * nq * D_, cudaMemcpyHostToDevice, s_));
  }
  compute_device(h_queries ? qx_.p : nullptr, nq, h, out.p);
  CK(cudaMemcpyAsync(h_out, out.p, sizeof(double) * n_out, cudaMemcpyDeviceToHost, s_));
  CK(cudaStreamSynchronize(s_));
}

void Engine::cv_reduce(const double* d_sums, double h, const double* d_conv, double conv_h,
                       double* lk, int* clamped, double* ls)
{
  const size_t n = n_;
  if (n < 2) throw InvalidArgument("CV requires at least 2 points");
  const double two_pi = 6.283185307179586476925286766559;
  const double nh = (double)(n - 1) * std::pow(two_pi * h * h, 0.5 * D_);
  const double nc = d_conv ? (double)(n - 1) * std::pow(two_pi * conv_h * conv_h, 0.5 * D_) : 1.0;
  red_.reserve(kRedBlocks * 3);
  k_cv_partial<<<kRedBlocks, kBlock, 0, s_>>>(d_sums, d_conv, (int)n, nh, nc, red_.p);
  CK_LAUNCH();
  std::vector<double> part(kRedBlocks * 3);
  CK(cudaMemcpyAsync(part.data(), red_.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, s_));
  CK(cudaStreamSynchronize(s_));
  double a = 0, b = 0, c = 0;
  for (int k = 0; k < kRedBlocks; ++k) {
    a += part[k * 3];
    b += part[k * 3 + 1];
    c += part[k * 3 + 2];
  }
  if (lk) *lk = a / (double)n;
  if (clamped) *clamped = (int)c;
  if (ls) *ls = b / (double)n;
}

void naive_device(const double* d_q, size_t nq, const double* d_r, size_t nr, int D, double h,
                  double* d_out, cudaStream_t s)
{
  const int TR = 256;
  k_naive<<<ceil_div(nq, 128), 128, TR * D * sizeof(double), s>>>(d_q, (int)nq, d_r, (int)nr, D,
                                                                 -1.0 / (2.0 * h * h), d_out);
  CK_LAUNCH();
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
