// Level-synchronous dual-tree traversal on sm_100a (replaces the reference's
// recursive Traversal::recurse, engine.cpp:113-195, and choose_best_method,
// truncation.cpp:130-166).
//
// The frontier holds live (query node, reference node) pairs grouped by query node
// -- an antichain: each query node appears at most once per level -- and one warp
// classifies one query node's pairs.  A BATCH of bandwidths is traversed in lock
// step: an entry's key is slot * K + node, so every bandwidth of a CV sweep shares
// each level's launches and synchronisation.
//
// Error budget (the reference's proof, with a BFS lower bound):
// tau(Q, R) = eps |R| G^l(Q) / |R_total|, where G^l(Q) = the K(d_max) lower-bound
// mass of every pair retired at Q or an ancestor (pruned, summarised or sent to the
// base case) plus that of every live pair of Q.  Those pairs partition the reference
// set, so G^l(Q) <= G(q) for every q in Q and the errors of all retired pairs of q
// add up to <= eps G(q).
//
// Work items are appended per level with a per-(slot, node) rank and counting-sorted
// by key afterwards: every accumulation happens in a fixed order, results are
// bit-reproducible run to run.
#include "internal.cuh"

#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace dfgtb {
namespace cg = cooperative_groups;
using namespace detail;

namespace {

// ------------------------------------------------------------------ truncation
// Error bounds of truncation.cpp:40-81.  The reference tests, in increasing p
// (least_order, truncation.cpp:85-94),
//   bound(p) = count / (1-s)^(D*dpow) * S(p) <= tau,   S(p) = sum_{k<D} C(D,k) a^k b^(D-k).
// The fast test here is the division-free form count * S(p) <= tau * (1-s)^(D*dpow)
// ((1-s) > 0 wherever a bound is evaluated) with b = r^p * (1/sqrt(p!)) from a table:
// no FP64 divide per candidate order and no overflow of the prefactor.  Its result
// can differ from the reference's only when the two sides agree to ~(D+4) ulp, so
// within a relative margin of 1e-13 (or when tau (1-s)^n leaves the normal range) the
// reference's own expression is evaluated instead (division by sqrt(p!), prefactor,
// log-space fallback of truncation.cpp:46-52): the decisions are the reference's,
// bit for bit.  The ratios are formed exactly as the reference forms them:
// side / (2h) and side / (4h) are (side / h) * 0.5 and * 0.25 exactly.
__constant__ double c_isf[16];        // 1 / sqrt(p!)
__constant__ double c_sf[16];         // sqrt(p!)      (sqrt_factorial, truncation.cpp:20-27)
__constant__ double c_binom[17][17];  // C(n, k)       (binomial, truncation.cpp:11-18)
constexpr double kTieMargin = 1e-13;

__device__ __forceinline__ double d_ipow(double x, int n)
{  // int_pow, truncation.cpp:29-36
  double r = 1.0;
  for (int i = 0; i < n; ++i) r *= x;
  return r;
}

__device__ __forceinline__ double bound_sum_S(double a, double b, int dim)
{  // sum_{k<dim} C(dim,k) a^k b^(dim-k), same operation order as truncation.cpp:43-45
  double bp[kMaxDim + 1];
  bp[0] = 1.0;
  for (int k = 1; k <= dim; ++k) bp[k] = bp[k - 1] * b;
  double sum = 0.0, ak = 1.0;
  for (int k = 0; k < dim; ++k) {
    sum += c_binom[dim][k] * ak * bp[dim - k];
    ak *= a;
  }
  return sum;
}

// bound_sum (truncation.cpp:40-54) exactly as the reference evaluates it: explicit
// round-to-nearest products and sums (no FMA contraction, which the reference's x86-64
// build does not do either).  Only the log-space branch (prefactor overflow, i.e.
// 1 - s < ~1e-9) uses CUDA's log / exp / log1p, which may differ from glibc's by an ulp.
__device__ __noinline__ double ref_bound_sum(double count, double s, int dpow, double a, double b,
                                             int dim)
{
  double sum = 0.0;
  for (int k = 0; k < dim; ++k)
    sum = __dadd_rn(sum, __dmul_rn(__dmul_rn(c_binom[dim][k], d_ipow(a, k)), d_ipow(b, dim - k)));
  const double prefactor = count / d_ipow(1.0 - s, dim * dpow);
  double bound = __dmul_rn(prefactor, sum);
  if (!isfinite(bound) && count > 0.0 && sum > 0.0)
    bound = exp(__dadd_rn(__dsub_rn(log(count), __dmul_rn((double)(dim * dpow), log1p(-s))), log(sum)));
  return bound;
}

// One candidate order: fast test, the reference's expression near a tie.
__device__ __forceinline__ bool bound_ok(double count, double S, double thr, double tau, double s,
                                         int dpow, double a, double b_exact, int dim)
{
  const double lhs = count * S;
  if (thr > 1e-290) {
    if (lhs <= thr * (1.0 - kTieMargin)) return true;
    if (lhs > thr * (1.0 + kTieMargin)) return false;
  }
  return ref_bound_sum(count, s, dpow, a, b_exact, dim) <= tau;
}

// farfield_order / local_accum_order (truncation.cpp:98-112): least p <= pmax with
// the Lemma 3/4 bound <= tau, 0 if none or ratio >= 1.
__device__ int d_order_ff(double ratio, double count, double tau, int pmax, int dim)
{
  if (ratio >= 1.0) return 0;
  const double thr = tau * d_ipow(1.0 - ratio, dim);
  double rp = 1.0;  // int_pow(r, p): the same product sequence
  for (int p = 1; p <= pmax; ++p) {
    rp *= ratio;
    if (bound_ok(count, bound_sum_S(1.0 - rp, rp * c_isf[p], dim), thr, tau, ratio, 1, 1.0 - rp,
                 rp / c_sf[p], dim))
      return p;
  }
  return 0;
}

// f2l_order (truncation.cpp:114-128): Lemma 5 with s = 2r, power 2D; 0 if r >= 1/2.
__device__ int d_order_f2l(double ratio, double count, double tau, int pmax, int dim)
{
  if (ratio >= 0.5) return 0;
  const double s = 2.0 * ratio;
  const double thr = tau * d_ipow(1.0 - s, 2 * dim);
  double sp = 1.0;
  for (int p = 1; p <= pmax; ++p) {
    sp *= s;
    const double a = (1.0 - sp) * (1.0 - sp);
    if (bound_ok(count, bound_sum_S(a, sp * (2.0 - sp) * c_isf[p], dim), thr, tau, s, 2, a,
                 sp * (2.0 - sp) / c_sf[p], dim))
      return p;
  }
  return 0;
}

#ifndef DFGTB_ORDER_LB
#define DFGTB_ORDER_LB 1
#endif
// The three least-order searches of choose_best_method run interleaved, one candidate
// order of each per step: the same arithmetic per search as d_order_ff / d_order_f2l
// (identical orders), but three independent dependency chains instead of one three
// times as long (the method choice is a latency-bound phase of every traversal level).
__device__ __forceinline__ void orders3(double rF, double rD, double rT, double count, double tau, int pmax,
                                        int dim, int& pf, int& pd, int& pt)
{
  pf = pd = pt = 0;
  bool doneF = rF >= 1.0, doneD = rD >= 1.0, doneT = rT >= 0.5;
  const double sT = 2.0 * rT;
  const double thrF = doneF ? 0.0 : tau * d_ipow(1.0 - rF, dim);
  const double thrD = doneD ? 0.0 : tau * d_ipow(1.0 - rD, dim);
  const double thrT = doneT ? 0.0 : tau * d_ipow(1.0 - sT, 2 * dim);
#if DFGTB_ORDER_LB
  // Hopeless searches end before they start.  Every S(p) holds the term k = D - 1,
  //   S(p) >= D a_p^(D-1) b_p,
  // and over 1 <= p <= pmax: a_p >= a_1 (= 1 - r, resp. (1 - s)^2) and b_p >= b_pmax
  // (r^p / sqrt(p!) falls with p; x (2 - x) grows with x = s^p), so with the threshold's
  // own power of (1 - r) cancelled
  //   count D b_pmax > tau (1 - r)        (F, D)    count D b_pmax > tau (1 - s)^2   (T)
  // implies count S(p) > thr for every p: with the 1e-9 margin (roundings are ~1e-15)
  // bound_ok's fast test returns false for each of them, i.e. order 0 -- the reference's
  // decision.  Most pairs of a big level expand, and those ran all 3 pmax candidates.
  {
    const double cD = count * (double)dim * c_isf[pmax], tm = tau * (1.0 + 1e-9);
    if (!doneF && thrF > 1e-290 && cD * d_ipow(rF, pmax) > tm * (1.0 - rF)) doneF = true;
    if (!doneD && thrD > 1e-290 && cD * d_ipow(rD, pmax) > tm * (1.0 - rD)) doneD = true;
    if (!doneT && thrT > 1e-290) {
      const double x = d_ipow(sT, pmax);
      if (cD * x * (2.0 - x) > tm * (1.0 - sT) * (1.0 - sT)) doneT = true;
    }
  }
#endif
  double rpF = 1.0, rpD = 1.0, spT = 1.0;
  for (int p = 1; p <= pmax && !(doneF && doneD && doneT); ++p) {
    const double isf = c_isf[p], sf = c_sf[p];
    if (!doneF) {
      rpF *= rF;
      if (bound_ok(count, bound_sum_S(1.0 - rpF, rpF * isf, dim), thrF, tau, rF, 1, 1.0 - rpF, rpF / sf, dim)) {
        pf = p;
        doneF = true;
      }
    }
    if (!doneD) {
      rpD *= rD;
      if (bound_ok(count, bound_sum_S(1.0 - rpD, rpD * isf, dim), thrD, tau, rD, 1, 1.0 - rpD, rpD / sf, dim)) {
        pd = p;
        doneD = true;
      }
    }
    if (!doneT) {
      spT *= sT;
      const double aT = (1.0 - spT) * (1.0 - spT);
      if (bound_ok(count, bound_sum_S(aT, spT * (2.0 - spT) * isf, dim), thrT, tau, sT, 2, aT,
                   spT * (2.0 - spT) / sf, dim)) {
        pt = p;
        doneT = true;
      }
    }
  }
}

// choose_best_method, truncation.cpp:130-166 (ties F > D > T > E)
__device__ void dev_choose(double nq, double nr, double sq, double sr, double h, double tau,
                           int pmax, int dim, int cost, int& kind, int& order)
{
  const double uq = sq / h, ur = sr / h;  // side / (2h) = (side / h) * 0.5 exactly
  int pf, pd, pt;
  orders3(ur * 0.5, uq * 0.5, (uq < ur ? ur : uq) * 0.25, nr, tau, pmax, dim, pf, pd, pt);
  const double D = (double)dim;
  double cf = CUDART_INF, cd = CUDART_INF, ct = CUDART_INF;
  if (cost == 0) {  // exponential model; integer powers of D <= 5 are exact
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

// ------------------------------------------------------------------ state
// Device-resident traversal state: every kernel reads the frontier size here, so
// the level loop needs no host round trip.  Capacities are checked before anything
// is written; on overflow the loop stops and the host regrows the buffers and reruns.
// sCov: sum over retired pairs (FD, F, D, T, base case) of |Q| |R| -- every (q, r) pair
// is retired exactly once, so it must equal |Q| |R_total| (CoverageProbe, tests/probes.hpp:13-44)
enum SlotStat { sPairs = 0, sFD, sF, sD, sT, sB, sKev, sCov, sNStat };
constexpr int kMaxLevels = 1024;
constexpr int kNch = 4;               // chunks per CTA on big levels (cyclic deal)
#ifndef DFGTB_CYCLIC_PAIRS
#define DFGTB_CYCLIC_PAIRS 2000000000  // cyclic deal measured 3-5% slower on cfg3/cfg5: off
#endif
constexpr int kCyclicPairs = DFGTB_CYCLIC_PAIRS;  // levels with at least this many pairs
struct TravState {
  double eps, ntot;                    // per batch (host)
  int nslots, K;
  double h[kMaxSlots], scale[kMaxSlots];
  int capE, capP, capF, capDT, capB;   // buffer capacities (host)
  int cur;                             // frontier buffer of the current level
  int m[2], p[2];                      // entries / pairs in each frontier buffer
  int nF, nDT, nB;                     // items emitted so far
  int overflow, levels;
  int done;                            // CTAs finished with their tile sum (unused)
  Cnt lvl;                             // totals of the current level
  unsigned long long sst[kMaxSlots][sNStat];  // per-slot TraversalStats
};

struct TravArgs {
  TreeView Q, R;
  int D, pmax, cost, series, T;
  int selfq;  // Q = R: every query's sum is >= 1 (its own term)
  int f32;    // the FP32 base case may be flagged (order bit 2)
  TravState* st;
  int *fq[2], *foff[2], *flen[2], *fr[2];
  int* pent[2];  // entry index of every frontier pair (pair-balanced persistent path)
  double* fbase[2];
  double* glo;   // per entry lower bound G^l (persistent path)
  double *pkmax, *pkmin;
  int* dec;
  Cnt *cnt, *cntoff, *tsum, *toff;
  int* childlen;
  double* newbase;
  double* L;
  int* Lord;
  Item *itF, *itDT, *itB;
  int *cntF, *cntDT, *cntB;
  unsigned long long* trace;  // optional per-phase %globaltimer stamps (DFGTB_TRACE)
  const int* sq;              // start frontier: query nodes (nsq) x reference nodes (nsr)
  const int* sr;              //   (nullptr: the roots); see Engine::start_frontier
  int nsq, nsr;
  Cnt* lvlcnt;                // per-level output counters of k_traverse (zeroed per launch)
  unsigned long long* lvlep;  // per-level packed (entries << 32 | pairs) counters
};

__device__ __forceinline__ Cnt ldcg_cnt(const Cnt* p)
{
  const int* q = reinterpret_cast<const int*>(p);
  return Cnt{ __ldcg(q), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3), __ldcg(q + 4), __ldcg(q + 5),
              __ldcg(q + 6) };
}

// Collectives over aligned groups of W lanes (W = 32: the whole warp).  Every lane
// of the warp must call them (groups are segments of the shuffles' width).
template <int W>
__device__ __forceinline__ int warp_excl_scan(int v, int lane, int& total)
{
  int x = v;
#pragma unroll
  for (int o = 1; o < W; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o, W);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, W - 1, W);
  return x - v;
}
template <int W>
__device__ __forceinline__ double group_sum(double v)
{
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, W);
  return v;
}
template <int W, class I>
__device__ __forceinline__ I group_sum_i(I v)
{
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, W);
  return v;
}

struct CntSum {
  __host__ __device__ Cnt operator()(const Cnt& x, const Cnt& y) const
  {
    return Cnt{ x.e + y.e, x.p + y.p, x.f + y.f, x.dt + y.dt, x.t + y.t, x.b + y.b, x.fd + y.fd };
  }
};

// Root pairs (slot b: key b*K -> reference root) and a fresh state.
__global__ void k_trav_init(const __grid_constant__ TravArgs a)
{
  TravState& st = *a.st;
  const int nb = st.nslots;
  // start frontier: every (slot, query start node) entry pairs with every reference start
  // node (the roots unless a start depth is set: the levels above it are skipped -- a
  // valid dual-tree traversal whose first lower bounds already sum over many nodes)
  const int nq = a.sq ? a.nsq : 1, nr = a.sq ? a.nsr : 1;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  // the start frontier must fit the frontier buffers like any level: otherwise nothing is
  // written, the traversal finds an empty frontier and the host regrows and reruns
  const long long need_e = (long long)nb * nq, need_p = need_e * nr;
  const bool fits = need_e <= st.capE && need_p <= st.capP;
  if (!fits) {
    if (blockIdx.x == 0) {
      for (int b = threadIdx.x; b < nb; b += blockDim.x)
        for (int k = 0; k < sNStat; ++k) st.sst[b][k] = 0;
      if (threadIdx.x == 0) {
        st.cur = 0;
        st.m[0] = st.p[0] = st.m[1] = st.p[1] = 0;
        st.nF = st.nDT = st.nB = 0;
        st.levels = 0;
        st.done = 0;
        Cnt l{};
        l.e = (int)min(need_e, (long long)(INT32_MAX / 4));
        l.p = (int)min(need_p, (long long)(INT32_MAX / 4));
        st.lvl = l;
        st.overflow = 1;
      }
    }
    return;
  }
  for (int e = t0; e < nb * nq; e += nt) {
    const int b = e / nq, qi = e - b * nq;
    a.fq[0][e] = b * st.K + (a.sq ? a.sq[qi] : 0);
    a.foff[0][e] = e * nr;
    a.flen[0][e] = nr;
    a.fbase[0][e] = 0.0;
  }
  for (int j = t0; j < nb * nq * nr; j += nt) {
    a.fr[0][j] = a.sq ? a.sr[j % nr] : 0;
    a.pent[0][j] = j / nr;
  }
  if (blockIdx.x != 0) return;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    for (int k = 0; k < sNStat; ++k) st.sst[b][k] = 0;
  if (threadIdx.x == 0) {
    st.cur = 0;
    st.m[0] = nb * nq;
    st.p[0] = nb * nq * nr;
    st.m[1] = st.p[1] = 0;
    st.nF = st.nDT = st.nB = 0;
    st.overflow = 0;
    st.levels = 0;
    st.done = 0;
    st.lvl = Cnt{};
  }
}

// Base-case flags of a leaf pair (k_base_records, k_base_case).  Bit 0: every pair has
// y = d^2/2h^2 <= 708 (K(d_max) >= e^-707.97): the fast exp needs no underflow handling.
// Bit 1: terms below 2^-1021 may be dropped (absolute error <= |R| 2^-1021 against a sum
// >= 1 (Q = R) or >= G^l >= 1e-290: below 1e-280 relative); the MUFU fixed point also
// needs the query leaf's diameter <= 1000 in z units (sq sqrt(D) sqrt(log2 e) / (h sqrt 2),
// sqrt(log2 e / 2) < 0.8494).  Bit 2: the FP32 base case applies: diameter <= kF32Diam
// (every query within kF32Diam / 2 of the leaf's box centre), and the terms below 2^-190
// that its FP32 exp flushes to 0 cannot matter: Q != R needs sums >= G^l >= 1e-20
// (<= |R| 2^-190 / 1e-20 < 1e-30 relative); Q = R sums are >= 1 (the self term, added
// exactly in FP64: the FP32 partial sums hold only G - 1), so the dropped mass is
// <= |R| 2^-190 absolute, far below the 2^-53 resolution of the FP64 sum G the engine
// returns -- the CV scores' G - 1 is formed from that FP64 G (cv.cpp:17-25), so a
// leave-one-out mass below 2^-53 is invisible to them on the FP64 path as well.
__device__ __forceinline__ int base_flags(const TravArgs& a, double kmin, double glo, double sq, double h,
                                          int D)
{
  const double dz = sq * sqrt((double)D) * 0.8494;
#if defined(DFGTB_EXP_F32_DIAM)  // experiments only
  const double diam_x = DFGTB_EXP_F32_DIAM;
#else
  const double diam_x = kF32Diam;
#endif
  return (kmin >= 3.4e-308 ? 1 : 0) | ((a.selfq || glo >= 1e-290) && dz <= 1000.0 * h ? 2 : 0) |
         (a.f32 && (a.selfq || glo >= 1e-20) && dz <= diam_x * h ? 4 : 0);
}

// A group of W lanes, one frontier query node: kernel bounds of every live pair, the
// lower bound G^l, and the prune / summarise / base / expand decision per pair.  The
// whole warp calls it (valid = false: a group without an entry this round).
template <int DT, int W>
__device__ __forceinline__ void classify_entry(const TravArgs& a, TravState& st, int cur, int e,
                                               int lane, bool valid,
                                               unsigned long long (*sst)[sNStat] = nullptr)
{
  const int* fr = a.fr[cur];
  const int D = DT ? DT : a.D;
  const int key = valid ? a.fq[cur][e] : 0;
  const int slot = key / st.K;
  const int Q = key - slot * st.K;
  const double h = st.h[slot], scale = st.scale[slot], eps = st.eps, ntot = st.ntot;
  const int off = valid ? a.foff[cur][e] : 0, len = valid ? a.flen[cur][e] : 0;
  const double fb = valid ? a.fbase[cur][e] : 0.0;
  const double* qlo = a.Q.lo + (size_t)Q * D;
  const double* qhi = a.Q.hi + (size_t)Q * D;
  const bool qleaf = a.Q.left[Q] < 0;
  const double nq = (double)a.Q.count[Q];
  const double sq = a.Q.side[Q];
  // pass 1: kernel bounds and the lower-bound mass of every live pair
  double part = 0.0;
  for (int j = lane; j < len; j += W) {
    const int R = fr[off + j];
    double dl, du;
    box_bounds<DT>(qlo, qhi, a.R.lo + (size_t)R * D, a.R.hi + (size_t)R * D, D, dl, du);
    const double kmax = exp(scale * dl);  // kernel at closest approach
    const double kmin = exp(scale * du);
    a.pkmax[off + j] = kmax;
    a.pkmin[off + j] = kmin;
    part += (double)a.R.count[R] * kmin;
  }
  const double glo = fb + group_sum<W>(part);
  // pass 2: decisions
  double fd_dlo = 0.0, fd_const = 0.0, ret = 0.0;
  int nF = 0, nDT = 0, nT = 0, nB = 0, nFD = 0, slots = 0;
  unsigned long long kev = 0, cov = 0;
  for (int j = lane; j < len; j += W) {
    const int R = fr[off + j];
    const double kmax = a.pkmax[off + j], kmin = a.pkmin[off + j];
    const double nr = (double)a.R.count[R];
    const double dlo = nr * kmin;
    const double tau = (eps / ntot) * nr * glo;  // eps |R| G^l / N
    int kind = kX, order = 0;
    if (0.5 * nr * (kmax - kmin) <= tau) {  // kernel-difference prune, engine.cpp:137-148
      kind = kFD;
      fd_dlo += dlo;
      fd_const += 0.5 * nr * (kmax + kmin);
      ++nFD;
    } else {
      if (a.series) {
        dev_choose(nq, nr, sq, a.R.side[R], h, tau, a.pmax, D, a.cost, kind, order);
        if (kind == kE) kind = kX;
      }
      if (kind == kX && qleaf && a.R.left[R] < 0) {
        kind = kB;
        order = base_flags(a, kmin, glo, sq, h, D);
      }
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
    if (kind != kX) cov += (unsigned long long)a.Q.count[Q] * (unsigned long long)a.R.count[R];
    a.dec[off + j] = kind | (order << 8);
  }
  fd_dlo = group_sum<W>(fd_dlo);
  fd_const = group_sum<W>(fd_const);
  ret = group_sum<W>(ret);
  nF = group_sum_i<W>(nF);
  nDT = group_sum_i<W>(nDT);
  nT = group_sum_i<W>(nT);
  nB = group_sum_i<W>(nB);
  nFD = group_sum_i<W>(nFD);
  slots = group_sum_i<W>(slots);
  kev = group_sum_i<W>(kev);
  cov = group_sum_i<W>(cov);
  if (lane == 0 && valid) {
    const int ne = slots > 0 ? (qleaf ? 1 : 2) : 0;
    a.cnt[e] = Cnt{ ne, ne * slots, nF, nDT, nT, nB, nFD };
    a.childlen[e] = slots;
    a.newbase[e] = fb + (fd_dlo + ret);
    if (nFD) {
      a.L[(size_t)key * a.T] += fd_const;  // constant local term (order 1)
      if (a.Lord[key] < 1) a.Lord[key] = 1;
    }
    unsigned long long* ss = sst ? sst[slot] : st.sst[slot];
    atomicAdd(ss + sPairs, (unsigned long long)len);
    if (nFD) atomicAdd(ss + sFD, (unsigned long long)nFD);
    if (nF) atomicAdd(ss + sF, (unsigned long long)nF);
    if (nDT - nT) atomicAdd(ss + sD, (unsigned long long)(nDT - nT));
    if (nT) atomicAdd(ss + sT, (unsigned long long)nT);
    if (nB) atomicAdd(ss + sB, (unsigned long long)nB);
    if (kev) atomicAdd(ss + sKev, kev);
    if (cov) atomicAdd(ss + sCov, cov);
  }
}

template <int DT>
__global__ void __launch_bounds__(kBlock) k_classify(const __grid_constant__ TravArgs a)
{
  TravState& st = *a.st;
  const int cur = st.cur, m = st.m[cur];
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w0; e < m; e += nw) classify_entry<DT, 32>(a, st, cur, e, lane, true);
}

// Device-side exclusive scan of the per-entry counts (graph / host-loop paths):
// tile sums -> one-block scan of the tiles (+ capacity check) -> tile rescan.
constexpr int kScanTiles = 256;
__global__ void __launch_bounds__(256) k_scan_tiles(const __grid_constant__ TravArgs a)
{
  const TravState& st = *a.st;
  const int m = st.m[st.cur];
  const int per = (m + kScanTiles - 1) / kScanTiles;
  const int b0 = min(m, blockIdx.x * per), b1 = min(m, b0 + per);
  Cnt acc{};
  for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) acc = CntSum()(acc, a.cnt[i]);
  using BR = cub::BlockReduce<Cnt, 256>;
  __shared__ typename BR::TempStorage tmp;
  const Cnt tot = BR(tmp).Reduce(acc, CntSum());
  if (threadIdx.x == 0) a.tsum[blockIdx.x] = tot;
}

__device__ __forceinline__ bool over_capacity(const TravState& st, const Cnt& t, int gF, int gDT,
                                              int gB)
{
  return t.e > st.capE || t.p > st.capP || (long long)gF + t.f > st.capF ||
         (long long)gDT + t.dt > st.capDT || (long long)gB + t.b > st.capB;
}

__global__ void __launch_bounds__(kScanTiles) k_scan_top(const __grid_constant__ TravArgs a)
{
  TravState& st = *a.st;
  using BS = cub::BlockScan<Cnt, kScanTiles>;
  __shared__ typename BS::TempStorage tmp;
  Cnt agg, out;
  BS(tmp).ExclusiveScan(a.tsum[threadIdx.x], out, Cnt{}, CntSum(), agg);
  a.toff[threadIdx.x] = out;
  if (threadIdx.x == 0) {
    st.lvl = agg;
    if (over_capacity(st, agg, st.nF, st.nDT, st.nB)) st.overflow = 1;
  }
}

__global__ void __launch_bounds__(256) k_scan_local(const __grid_constant__ TravArgs a)
{
  const TravState& st = *a.st;
  const int m = st.m[st.cur];
  const int per = (m + kScanTiles - 1) / kScanTiles;
  const int b0 = min(m, blockIdx.x * per), b1 = min(m, b0 + per);
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

// A group of W lanes, one frontier query node: its part of the next frontier and its
// work items, at the offsets `o` (exclusive scan of the level's counts).  The whole
// warp calls it (valid = false: no entry for this group).
// cdec / cR (optional): the CTA's smem copies of the pairs' decisions and reference
// nodes, indexed by pair - cP0 (PairCache).
template <int W>
__device__ __forceinline__ void emit_entry(const TravArgs& a, int K, int cur, int gF, int gDT,
                                           int gB, int e, const Cnt& o, int lane, bool valid,
                                           const int* cdec = nullptr, const int* cR = nullptr, int cP0 = 0)
{
  const int nxt = cur ^ 1;
  const int* fr = a.fr[cur];
  int* nr = a.fr[nxt];
  const Cnt c = valid ? a.cnt[e] : Cnt{};
  const int key = valid ? a.fq[cur][e] : 0;
  const int slot = key / K;
  const int Q = key - slot * K;
  const int off = valid ? a.foff[cur][e] : 0, len = valid ? a.flen[cur][e] : 0;
  const bool qleaf = a.Q.left[Q] < 0;
  const int cl = valid ? a.childlen[e] : 0;
  // every group of the warp runs the same number of rounds (shuffles inside)
  const int rounds = W == 32 ? len : __reduce_max_sync(0xffffffffu, (unsigned)len);
  if (lane == 0 && c.e) {
    const double nb = a.newbase[e];
    if (qleaf) {
      a.fq[nxt][o.e] = key;
      a.fbase[nxt][o.e] = nb;
      a.foff[nxt][o.e] = o.p;
      a.flen[nxt][o.e] = cl;
    } else {
      a.fq[nxt][o.e] = slot * K + a.Q.left[Q];
      a.fq[nxt][o.e + 1] = slot * K + a.Q.right[Q];
      a.fbase[nxt][o.e] = nb;
      a.fbase[nxt][o.e + 1] = nb;
      a.foff[nxt][o.e] = o.p;
      a.foff[nxt][o.e + 1] = o.p + cl;
      a.flen[nxt][o.e] = cl;
      a.flen[nxt][o.e + 1] = cl;
    }
  }
  const int rF = valid ? a.cntF[key] : 0, rDT = valid ? a.cntDT[key] : 0,
            rB = valid ? a.cntB[key] : 0;
  int runX = 0, runF = 0, runDT = 0, runB = 0;
  for (int j0 = 0; j0 < rounds; j0 += W) {
    const int j = j0 + lane;
    int kind = kE, order = 0, R = 0;
    if (j < len) {
      const int dcode = cdec ? cdec[off - cP0 + j] : a.dec[off + j];
      kind = dcode & 0xff;
      order = dcode >> 8;
      R = cR ? cR[off - cP0 + j] : fr[off + j];
    }
    const bool rleaf = (j < len) ? a.R.left[R] < 0 : true;
    int tot;
    const int px = warp_excl_scan<W>(kind == kX ? (rleaf ? 1 : 2) : 0, lane, tot);
    if (kind == kX) {
      const int dst = o.p + runX + px;
      int* pe = a.pent[nxt];
      if (rleaf) {
        nr[dst] = R;
        pe[dst] = o.e;
        if (!qleaf) {
          nr[dst + cl] = R;
          pe[dst + cl] = o.e + 1;
        }
      } else {
        const int rl = a.R.left[R], rr = a.R.right[R];
        nr[dst] = rl;
        nr[dst + 1] = rr;
        pe[dst] = o.e;
        pe[dst + 1] = o.e;
        if (!qleaf) {
          nr[dst + cl] = rl;
          nr[dst + cl + 1] = rr;
          pe[dst + cl] = o.e + 1;
          pe[dst + cl + 1] = o.e + 1;
        }
      }
    }
    runX += tot;
    int t2;
    const int pf = warp_excl_scan<W>(kind == kF, lane, t2);
    if (kind == kF) a.itF[gF + o.f + runF + pf] = Item{ key, R, order | (kF << 8), rF + runF + pf };
    runF += t2;
    const int pd = warp_excl_scan<W>(kind == kD || kind == kT, lane, t2);
    if (kind == kD || kind == kT)
      a.itDT[gDT + o.dt + runDT + pd] = Item{ key, R, order | (kind << 8), rDT + runDT + pd };
    runDT += t2;
    const int pb = warp_excl_scan<W>(kind == kB, lane, t2);
    if (kind == kB) a.itB[gB + o.b + runB + pb] = Item{ key, R, (kB << 8) | order, rB + runB + pb };
    runB += t2;
  }
  if (lane == 0 && valid) {
    a.cntF[key] = rF + runF;
    a.cntDT[key] = rDT + runDT;
    a.cntB[key] = rB + runB;
  }
}

__global__ void __launch_bounds__(kBlock) k_emit(const __grid_constant__ TravArgs a)
{
  const TravState& st = *a.st;
  if (st.overflow) return;
  const int cur = st.cur, m = st.m[cur];
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w0; e < m; e += nw)
    emit_entry<32>(a, st.K, cur, st.nF, st.nDT, st.nB, e, a.cntoff[e], lane, true);
}

// Close a level (graph / host-loop paths): fold its totals into the state, flip the
// frontier buffers and tell the WHILE node whether another level follows.
__global__ void k_advance(const __grid_constant__ TravArgs a, cudaGraphConditionalHandle hc, int use_cond)
{
  TravState& st = *a.st;
  if (!st.overflow) {
    const Cnt l = st.lvl;
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

// The whole level loop in ONE cooperative launch (one CTA per SM).  Each level is a
// single phase: CTA b owns a contiguous, pair-balanced range of frontier entries; it
// classifies them, scans its counts, claims its output space with one atomic per
// counter on the level's totals, and emits -- then ONE grid-wide barrier makes the
// next frontier and the totals visible.  Every CTA advances an identical private copy
// of (cur, m, item offsets) and checks capacity itself; CTA 0 writes the state back.
#ifndef KPBLOCK
#define KPBLOCK 1024
#endif
constexpr int kPBlock = KPBLOCK;  // one CTA per SM: 32 warps to hide classify latency
constexpr int kTrAll = 4096 + 512 * 16 + 64 * 160 + 64;  // DFGTB_TRACE: per-level phase sums over CTAs
constexpr int kTrCta = kTrAll + 64 * 16;  // per level, per CTA: phase durations, pairs, entries
constexpr int kTrLen = kTrCta + 64 * 160 * 10;

template <int W>
__device__ __forceinline__ void emit_range(const TravArgs& a, int K, int cur, int gF, int gDT, int gB,
                                           int b0, int b1, const int* cdec = nullptr, const int* cR = nullptr,
                                           int cP0 = 0)
{
  const int g = threadIdx.x / W, lane = threadIdx.x % W;
  constexpr int ng = kPBlock / W;
  for (int base = b0; base < b1; base += ng) {
    const int e = base + g;
    if (__any_sync(0xffffffffu, e < b1))
      emit_entry<W>(a, K, cur, gF, gDT, gB, e, e < b1 ? a.cntoff[e] : Cnt{}, lane, e < b1, cdec, cR, cP0);
  }
}

// ---- shared-memory pair cache of a level's CTA range ------------------------------
// When a CTA's pair range [P0, P1) and entry range [e0, e1) fit, its pairs' reference
// node, count, kernel bounds and decision, and its entries' key, offset, length and G^l
// live in shared memory between the level's phases instead of round-tripping through
// L2 (the phases are latency-bound chains of dependent loads).  Same arithmetic, same
// lane-strided reduction order: identical results to the uncached phases.
#ifndef DFGTB_TRAV_CACHE
#define DFGTB_TRAV_CACHE 0  // measured: the level phases are not bound by these loads (0.80 vs 0.85 ms, cfg2)
#endif
constexpr bool kUseCache = DFGTB_TRAV_CACHE != 0;
constexpr int kCacheP = 4096;  // pairs
constexpr int kCacheE = 2048;  // entries
constexpr int kCacheBytes = kCacheP * (8 + 8 + 4 + 4 + 4 + 4) + kCacheE * (8 + 4 + 4 + 4);
struct PairCache {
  double *kmax, *kmin, *glo;
  int *R, *el, *cnt, *dec, *key, *off, *len;
  __device__ static PairCache at(unsigned char* p)
  {
    PairCache c;
    c.kmax = reinterpret_cast<double*>(p);
    c.kmin = c.kmax + kCacheP;
    c.glo = c.kmin + kCacheP;
    c.R = reinterpret_cast<int*>(c.glo + kCacheE);
    c.el = c.R + kCacheP;
    c.cnt = c.el + kCacheP;
    c.dec = c.cnt + kCacheP;
    c.key = c.dec + kCacheP;
    c.off = c.key + kCacheE;
    c.len = c.off + kCacheE;
    return c;
  }
};
// ---- pair-balanced level phases of k_traverse -------------------------------------
// CTA b owns the entries whose pair lists start in [b p / G, (b+1) p / G): a
// contiguous entry range holding ~p/G pairs (entry sizes differ by orders of
// magnitude, so equal ENTRY ranges left most CTAs idle at the grid barrier).  The
// heavy per-pair work (kernel bounds, method choice) runs flat over the CTA's pairs;
// the per-entry reductions run one warp per entry in the same lane-strided order as
// classify_entry, so the sums (and every decision) are bit-identical to it.

// Smallest entry e with foff[e] >= target (foff increasing, entries non-empty), for
// two targets at once, by a 1024-ary search with __syncthreads_count.
// The key is the entry's cost offset foff[e] + kEntryCost e (pairs plus a per-entry
// charge: the per-entry phases -- G^l, counts, emission -- run one warp per entry, so a
// range of many small entries costs more than its pairs say).
#ifndef DFGTB_ENTRY_COST
#define DFGTB_ENTRY_COST 16  // measured (cfg2 traversal ms, 640-thread build): 4 0.582, 8 0.557, 16 0.548, 24 0.558, 32 0.570
#endif
constexpr long long kEntryCost = DFGTB_ENTRY_COST;
__device__ __forceinline__ void entry_bounds(const int* foff, int m, long long t0, long long t1,
                                             int& e0, int& e1)
{
  int lo0 = 0, hi0 = m, lo1 = 0, hi1 = m;
  while (lo0 < hi0 || lo1 < hi1) {
    const int S0 = (hi0 - lo0 + kPBlock - 1) / kPBlock, S1 = (hi1 - lo1 + kPBlock - 1) / kPBlock;
    const int c0i = lo0 + (threadIdx.x + 1) * S0 - 1, c1i = lo1 + (threadIdx.x + 1) * S1 - 1;
    const bool p0 = lo0 < hi0 && c0i < hi0 && foff[c0i] + kEntryCost * c0i < t0;
    const bool p1 = lo1 < hi1 && c1i < hi1 && foff[c1i] + kEntryCost * c1i < t1;
    const int c0 = __syncthreads_count(p0), c1 = __syncthreads_count(p1);
    if (lo0 < hi0) {
      const int nlo = lo0 + c0 * S0;
      hi0 = min(hi0, lo0 + (c0 + 1) * S0 - 1);
      lo0 = nlo;
    }
    if (lo1 < hi1) {
      const int nlo = lo1 + c1 * S1;
      hi1 = min(hi1, lo1 + (c1 + 1) * S1 - 1);
      lo1 = nlo;
    }
  }
  e0 = lo0;
  e1 = lo1;
}

// Pass 1, one thread per pair: kernel bounds K(d_min), K(d_max).  kPU pairs per thread
// at a time with their loads issued back to back (the phase is latency-bound: each pair
// is a chain entry -> key -> boxes).
#ifndef DFGTB_TRAV_PU
#define DFGTB_TRAV_PU 1  // measured: 2 and 4 pairs per thread gain nothing (spills at 64 registers)
#endif
constexpr int kPU = DFGTB_TRAV_PU;
template <int DT>
__device__ __forceinline__ void pairs_bounds(const TravArgs& a, int cur, int K, int P0, int P1,
                                             const double* s_scale)
{
  const int D = DT ? DT : a.D;
  for (int j0 = P0 + threadIdx.x; j0 < P1; j0 += kPBlock * kPU) {
    int e[kPU], R[kPU], key[kPU];
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
      const int j = j0 + u * kPBlock;
      e[u] = j < P1 ? a.pent[cur][j] : -1;
      R[u] = j < P1 ? a.fr[cur][j] : 0;
    }
#pragma unroll
    for (int u = 0; u < kPU; ++u) key[u] = e[u] >= 0 ? a.fq[cur][e[u]] : 0;
#pragma unroll
    for (int u = 0; u < kPU; ++u) {
      const int j = j0 + u * kPBlock;
      if (j < P1) {
        const int slot = key[u] / K, Q = key[u] - slot * K;
        double dl, du;
        box_bounds<DT>(a.Q.lo + (size_t)Q * D, a.Q.hi + (size_t)Q * D, a.R.lo + (size_t)R[u] * D,
                       a.R.hi + (size_t)R[u] * D, D, dl, du);
        const double scale = s_scale[slot];
        a.pkmax[j] = exp(scale * dl);  // kernel at closest approach
        a.pkmin[j] = exp(scale * du);
      }
    }
  }
}

// One warp per entry: G^l = base + sum |R| K(d_max) over the entry's live pairs.
__device__ __forceinline__ void entries_glo(const TravArgs& a, int cur, int e0, int e1,
                                            unsigned long long* tr = nullptr)
{
  const int lane = threadIdx.x & 31;
  for (int e = e0 + (threadIdx.x >> 5); e < e1; e += kPBlock / 32) {
    const int off = a.foff[cur][e], len = a.flen[cur][e];
    if (tr && lane == 0) atomicMax(tr, (unsigned long long)len);
    double part = 0.0;
    for (int j = lane; j < len; j += 32)
      part += (double)a.R.count[a.fr[cur][off + j]] * a.pkmin[off + j];
    const double g = a.fbase[cur][e] + group_sum<32>(part);
    if (lane == 0) a.glo[e] = g;
  }
}

// Pass 2, one thread per pair: the prune / summarise / base / expand decision
// (engine.cpp:137-195 with choose_best_method, truncation.cpp:130-166).
template <int DT>
__device__ __forceinline__ void pairs_decide(const TravArgs& a, const TravState& st, int cur, int K,
                                             int P0, int P1, const double* s_h)
{
  const int D = DT ? DT : a.D;
  const double eps_nt = st.eps / st.ntot;
  for (int j0 = P0 + threadIdx.x; j0 < P1; j0 += kPBlock * kPU) {
  int ue[kPU], uR[kPU], ukey[kPU], ucnt[kPU];
  double uglo[kPU];
#pragma unroll
  for (int u = 0; u < kPU; ++u) {
    const int j = j0 + u * kPBlock;
    ue[u] = j < P1 ? a.pent[cur][j] : -1;
    uR[u] = j < P1 ? a.fr[cur][j] : 0;
  }
#pragma unroll
  for (int u = 0; u < kPU; ++u) {
    ukey[u] = ue[u] >= 0 ? a.fq[cur][ue[u]] : 0;
    uglo[u] = ue[u] >= 0 ? a.glo[ue[u]] : 0.0;
    ucnt[u] = a.R.count[uR[u]];
  }
#pragma unroll 1
  for (int u = 0; u < kPU; ++u) {
    const int j = j0 + u * kPBlock;
    if (j >= P1) break;
    const int e = ue[u];
    const int key = ukey[u];
    const int slot = key / K, Q = key - slot * K;
    const int R = uR[u];
    const double kmax = a.pkmax[j], kmin = a.pkmin[j];
    const double nr = (double)ucnt[u];
    const double tau = eps_nt * nr * uglo[u];  // eps |R| G^l / N
    int kind = kX, order = 0;
    if (0.5 * nr * (kmax - kmin) <= tau) {  // kernel-difference prune, engine.cpp:137-148
      kind = kFD;
    } else {
      if (a.series) {
        dev_choose((double)a.Q.count[Q], nr, a.Q.side[Q], a.R.side[R], s_h[slot], tau, a.pmax, D,
                   a.cost, kind, order);
        if (kind == kE) kind = kX;
      }
      if (kind == kX && a.Q.left[Q] < 0 && a.R.left[R] < 0) {
        kind = kB;
        order = base_flags(a, kmin, uglo[u], a.Q.side[Q], s_h[slot], D);
      }
    }
    a.dec[j] = kind | (order << 8);
    (void)e;
  }
  }
}

// One warp per entry: the entry's counts, next-level size and lower-bound base, the
// finite-difference constant, and the statistics (into the CTA's shared copy).
__device__ __forceinline__ void entries_reduce(const TravArgs& a, int cur, int K, int e0, int e1,
                                               unsigned long long (*s_sst)[sNStat])
{
  const int lane = threadIdx.x & 31;
  // statistics: lane k < sNStat keeps counter k of the warp's current slot in a register
  // and adds it to the CTA's shared copy when the slot changes and at the end of the
  // phase (one 8-lane atomic per warp and level instead of up to 8 serial ones per entry)
  int st_slot = -1;
  unsigned long long st_mine = 0;
  for (int e = e0 + (threadIdx.x >> 5); e < e1; e += kPBlock / 32) {
    const int key = a.fq[cur][e];
    const int slot = key / K, Q = key - slot * K;
    const int off = a.foff[cur][e], len = a.flen[cur][e];
    const bool qleaf = a.Q.left[Q] < 0;
    const unsigned long long nqi = (unsigned long long)a.Q.count[Q];
    double fd_dlo = 0.0, fd_const = 0.0, ret = 0.0;
    int nF = 0, nDT = 0, nT = 0, nB = 0, nFD = 0, slots = 0;
    unsigned long long kev = 0, cov = 0;
    for (int j = lane; j < len; j += 32) {
      const int R = a.fr[cur][off + j];
      const int kind = a.dec[off + j] & 0xff;
      const int cr = a.R.count[R];
      if (kind != kX) cov += nqi * (unsigned long long)cr;
      const double nr = (double)cr;
      const double kmin = a.pkmin[off + j];
      const double dlo = nr * kmin;
      if (kind == kFD) {
        fd_dlo += dlo;
        fd_const += 0.5 * nr * (a.pkmax[off + j] + kmin);
        ++nFD;
      } else if (kind == kX) {
        slots += a.R.left[R] < 0 ? 1 : 2;
      } else if (kind == kB) {
        ++nB;
        kev += nqi * (unsigned long long)cr;
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
    fd_dlo = group_sum<32>(fd_dlo);
    fd_const = group_sum<32>(fd_const);
    ret = group_sum<32>(ret);
    nF = group_sum_i<32>(nF);
    nDT = group_sum_i<32>(nDT);
    nT = group_sum_i<32>(nT);
    nB = group_sum_i<32>(nB);
    nFD = group_sum_i<32>(nFD);
    slots = group_sum_i<32>(slots);
    kev = group_sum_i<32>(kev);
    cov = group_sum_i<32>(cov);
    if (lane == 0) {
      const int ne = slots > 0 ? (qleaf ? 1 : 2) : 0;
      a.cnt[e] = Cnt{ ne, ne * slots, nF, nDT, nT, nB, nFD };
      a.childlen[e] = slots;
      a.newbase[e] = a.fbase[cur][e] + (fd_dlo + ret);
      if (nFD) {
        a.L[(size_t)key * a.T] += fd_const;  // constant local term (order 1)
        if (a.Lord[key] < 1) a.Lord[key] = 1;
      }
    }
    if (slot != st_slot) {
      if (st_mine && lane < sNStat) atomicAdd(s_sst[st_slot] + lane, st_mine);
      st_slot = slot;
      st_mine = 0;
    }
    st_mine += lane == sPairs ? (unsigned long long)len
               : lane == sFD  ? (unsigned long long)nFD
               : lane == sF   ? (unsigned long long)nF
               : lane == sD   ? (unsigned long long)(nDT - nT)
               : lane == sT   ? (unsigned long long)nT
               : lane == sB   ? (unsigned long long)nB
               : lane == sKev ? kev
                              : cov;
  }
  if (st_mine && lane < sNStat) atomicAdd(s_sst[st_slot] + lane, st_mine);
}

// Cached phases (PairCache): the same computations as pairs_bounds / entries_glo /
// pairs_decide / entries_reduce on the CTA's range [P0, P1) x [e0, e1).
template <int DT>
__device__ __forceinline__ void pairs_bounds_c(const TravArgs& a, int cur, int K, int P0, int P1, int e0,
                                               int e1, const double* s_scale, const PairCache& c)
{
  const int D = DT ? DT : a.D;
  for (int el = threadIdx.x; el < e1 - e0; el += kPBlock) {
    c.key[el] = a.fq[cur][e0 + el];
    c.off[el] = a.foff[cur][e0 + el] - P0;
    c.len[el] = a.flen[cur][e0 + el];
  }
  for (int j = P0 + threadIdx.x; j < P1; j += kPBlock) {
    const int e = a.pent[cur][j], R = a.fr[cur][j];
    const int key = a.fq[cur][e];
    const int slot = key / K, Q = key - slot * K;
    double dl, du;
    box_bounds<DT>(a.Q.lo + (size_t)Q * D, a.Q.hi + (size_t)Q * D, a.R.lo + (size_t)R * D,
                   a.R.hi + (size_t)R * D, D, dl, du);
    const double scale = s_scale[slot];
    const int l = j - P0;
    c.kmax[l] = exp(scale * dl);
    c.kmin[l] = exp(scale * du);
    c.R[l] = R;
    c.el[l] = e - e0;
    c.cnt[l] = a.R.count[R];
  }
}

__device__ __forceinline__ void entries_glo_c(const TravArgs& a, int cur, int e0, int e1, const PairCache& c)
{
  const int lane = threadIdx.x & 31;
  for (int el = threadIdx.x >> 5; el < e1 - e0; el += kPBlock / 32) {
    const int off = c.off[el], len = c.len[el];
    double part = 0.0;
    for (int j = lane; j < len; j += 32) part += (double)c.cnt[off + j] * c.kmin[off + j];
    const double g = a.fbase[cur][e0 + el] + group_sum<32>(part);
    if (lane == 0) c.glo[el] = g;
  }
}

template <int DT>
__device__ __forceinline__ void pairs_decide_c(const TravArgs& a, const TravState& st, int K, int P0, int P1,
                                               const double* s_h, const PairCache& c)
{
  const int D = DT ? DT : a.D;
  const double eps_nt = st.eps / st.ntot;
  for (int l = threadIdx.x; l < P1 - P0; l += kPBlock) {
    const int el = c.el[l];
    const int key = c.key[el];
    const int slot = key / K, Q = key - slot * K;
    const int R = c.R[l];
    const double kmax = c.kmax[l], kmin = c.kmin[l], glo = c.glo[el];
    const double nr = (double)c.cnt[l];
    const double tau = eps_nt * nr * glo;  // eps |R| G^l / N
    int kind = kX, order = 0;
    if (0.5 * nr * (kmax - kmin) <= tau) {  // kernel-difference prune, engine.cpp:137-148
      kind = kFD;
    } else {
      if (a.series) {
        dev_choose((double)a.Q.count[Q], nr, a.Q.side[Q], a.R.side[R], s_h[slot], tau, a.pmax, D, a.cost,
                   kind, order);
        if (kind == kE) kind = kX;
      }
      if (kind == kX && a.Q.left[Q] < 0 && a.R.left[R] < 0) {
        kind = kB;
        order = base_flags(a, kmin, glo, a.Q.side[Q], s_h[slot], D);
      }
    }
    c.dec[l] = kind | (order << 8);
  }
}

__device__ __forceinline__ void entries_reduce_c(const TravArgs& a, int cur, int K, int e0, int e1,
                                                 unsigned long long (*s_sst)[sNStat], const PairCache& c)
{
  const int lane = threadIdx.x & 31;
  for (int el = threadIdx.x >> 5; el < e1 - e0; el += kPBlock / 32) {
    const int e = e0 + el;
    const int key = c.key[el];
    const int slot = key / K, Q = key - slot * K;
    const int off = c.off[el], len = c.len[el];
    const bool qleaf = a.Q.left[Q] < 0;
    const unsigned long long nqi = (unsigned long long)a.Q.count[Q];
    double fd_dlo = 0.0, fd_const = 0.0, ret = 0.0;
    int nF = 0, nDT = 0, nT = 0, nB = 0, nFD = 0, slots = 0;
    unsigned long long kev = 0, cov = 0;
    for (int j = lane; j < len; j += 32) {
      const int kind = c.dec[off + j] & 0xff;
      const int cr = c.cnt[off + j];
      if (kind != kX) cov += nqi * (unsigned long long)cr;
      const double nr = (double)cr;
      const double kmin = c.kmin[off + j];
      const double dlo = nr * kmin;
      if (kind == kFD) {
        fd_dlo += dlo;
        fd_const += 0.5 * nr * (c.kmax[off + j] + kmin);
        ++nFD;
      } else if (kind == kX) {
        slots += a.R.left[c.R[off + j]] < 0 ? 1 : 2;
      } else if (kind == kB) {
        ++nB;
        kev += nqi * (unsigned long long)cr;
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
    fd_dlo = group_sum<32>(fd_dlo);
    fd_const = group_sum<32>(fd_const);
    ret = group_sum<32>(ret);
    nF = group_sum_i<32>(nF);
    nDT = group_sum_i<32>(nDT);
    nT = group_sum_i<32>(nT);
    nB = group_sum_i<32>(nB);
    nFD = group_sum_i<32>(nFD);
    slots = group_sum_i<32>(slots);
    kev = group_sum_i<32>(kev);
    cov = group_sum_i<32>(cov);
    if (lane == 0) {
      const int ne = slots > 0 ? (qleaf ? 1 : 2) : 0;
      a.cnt[e] = Cnt{ ne, ne * slots, nF, nDT, nT, nB, nFD };
      a.childlen[e] = slots;
      a.newbase[e] = a.fbase[cur][e] + (fd_dlo + ret);
      if (nFD) {
        a.L[(size_t)key * a.T] += fd_const;  // constant local term (order 1)
        if (a.Lord[key] < 1) a.Lord[key] = 1;
      }
      unsigned long long* ss = s_sst[slot];
      atomicAdd(ss + sPairs, (unsigned long long)len);
      if (nFD) atomicAdd(ss + sFD, (unsigned long long)nFD);
      if (nF) atomicAdd(ss + sF, (unsigned long long)nF);
      if (nDT - nT) atomicAdd(ss + sD, (unsigned long long)(nDT - nT));
      if (nT) atomicAdd(ss + sT, (unsigned long long)nT);
      if (nB) atomicAdd(ss + sB, (unsigned long long)nB);
      if (kev) atomicAdd(ss + sKev, kev);
      if (cov) atomicAdd(ss + sCov, cov);
    }
  }
}


#ifndef DFGTB_TRAV_CTAS_PER_SM
#define DFGTB_TRAV_CTAS_PER_SM 1
#endif
constexpr int kPerSM = DFGTB_TRAV_CTAS_PER_SM;  // co-resident traversal CTAs per SM
template <int DT>
__global__ void __launch_bounds__(kPBlock, kPerSM) k_traverse(const __grid_constant__ TravArgs a)
{
  cg::grid_group grid = cg::this_grid();
  TravState& st = *a.st;
  using BR = cub::BlockReduce<Cnt, kPBlock>;
  using BS = cub::BlockScan<Cnt, kPBlock>;
  __shared__ union {
    typename BR::TempStorage r;
    typename BS::TempStorage s;
  } tmp;
  __shared__ Cnt s_agg, s_excl;
  __shared__ int s_wsum[32][5];
  __shared__ double s_h[kMaxSlots], s_scale[kMaxSlots];
  __shared__ unsigned long long s_sst[kMaxSlots][sNStat];
  extern __shared__ __align__(16) unsigned char s_cache[];  // PairCache (kCacheBytes, dynamic)
  const PairCache pc = PairCache::at(s_cache);
  const int G = gridDim.x;
  const int K = st.K, nslots = st.nslots;
  for (int i = threadIdx.x; i < kMaxSlots * sNStat; i += kPBlock) (&s_sst[0][0])[i] = 0;
  for (int i = threadIdx.x; i < nslots; i += kPBlock) {
    s_h[i] = st.h[i];
    s_scale[i] = st.scale[i];
  }
  __syncthreads();
  int cur = 0, m = st.m[0], p = st.p[0], gF = 0, gDT = 0, gB = 0, levels = 0;
  // DFGTB_TRACE: per-phase %globaltimer stamps of CTA 0 (trace[4096 + 16 L + k])
  // and, from every CTA, the phase durations summed over CTAs (trace[kTrAll + 16 L + k])
  unsigned long long tph = 0;
#define PH(k)                                                                                   \
  if (a.trace && threadIdx.x == 0 && levels < 512) {                                           \
    unsigned long long t_;                                                                      \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
    if (blockIdx.x == 0) a.trace[4096 + levels * 16 + (k)] = t_;                                \
    if (levels < 64) atomicAdd(a.trace + kTrAll + levels * 16 + (k), t_ - tph);                 \
    if (levels < 64 && blockIdx.x < 160) a.trace[kTrCta + ((size_t)levels * 160 + blockIdx.x) * 10 + (k)] = t_ - tph; \
    tph = t_;                                                                                   \
  }
  for (;;) {
    if (a.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tph));
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && levels < 512) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[levels * 4] = t;
      a.trace[2048 + levels * 2] = (unsigned long long)m;
      a.trace[2048 + levels * 2 + 1] = (unsigned long long)p;
    }
    // Big levels are cut into nch * G pair-balanced chunks dealt CYCLICALLY (CTA b takes
    // chunks b, b + G, ..): per-pair cost depends strongly on the bandwidth slot, i.e.
    // on the position in the frontier, and interleaving averages it out.  A CTA's
    // output is the concatenation of its chunks (one scan, one claim), so nothing
    // downstream needs contiguous input ranges.
    const int nch = p >= kCyclicPairs ? kNch : 1;
    int cb0[kNch], cb1[kNch];
#pragma unroll
    for (int j = 0; j < kNch; ++j) {
      cb0[j] = cb1[j] = 0;
      if (j < nch) {
        const long long k = blockIdx.x + (long long)j * G, nk = (long long)G * nch;
        const long long tot = p + kEntryCost * m;  // cost of the level (see entry_bounds)
        entry_bounds(a.foff[cur], m, k * tot / nk, (k + 1) * tot / nk, cb0[j], cb1[j]);
      }
    }
    auto pofs = [&](int e) { return e < m ? a.foff[cur][e] : p; };
    const int cP0 = pofs(cb0[0]), cP1 = pofs(cb1[0]);
    const bool cached = kUseCache && nch == 1 && cP1 - cP0 <= kCacheP && cb1[0] - cb0[0] <= kCacheE;
    if (a.trace && threadIdx.x == 0 && levels < 64 && blockIdx.x < 160)
      a.trace[kTrCta + ((size_t)levels * 160 + blockIdx.x) * 10 + 9] =
        ((unsigned long long)(cb1[0] - cb0[0]) << 32) | (unsigned)(cP1 - cP0);
    PH(0);
    if (cached) {
      pairs_bounds_c<DT>(a, cur, K, cP0, cP1, cb0[0], cb1[0], s_scale, pc);
      __syncthreads();
      PH(1);
      entries_glo_c(a, cur, cb0[0], cb1[0], pc);
      __syncthreads();
      PH(2);
      pairs_decide_c<DT>(a, st, K, cP0, cP1, s_h, pc);
      __syncthreads();
      PH(3);
      entries_reduce_c(a, cur, K, cb0[0], cb1[0], s_sst, pc);
      __syncthreads();
    } else {
      for (int j = 0; j < nch; ++j) pairs_bounds<DT>(a, cur, K, pofs(cb0[j]), pofs(cb1[j]), s_scale);
      __syncthreads();
      PH(1);
      for (int j = 0; j < nch; ++j)
        entries_glo(a, cur, cb0[j], cb1[j], a.trace && levels < 64 ? a.trace + 4096 + 512 * 16 + 64 * 160 + levels : nullptr);
      __syncthreads();
      PH(2);
      for (int j = 0; j < nch; ++j) pairs_decide<DT>(a, st, cur, K, pofs(cb0[j]), pofs(cb1[j]), s_h);
      __syncthreads();
      PH(3);
      for (int j = 0; j < nch; ++j) entries_reduce(a, cur, K, cb0[j], cb1[j], s_sst);
      __syncthreads();
    }
    PH(4);
    // virtual index over the concatenated chunks -> frontier entry
    int nE = 0, cofs[kNch + 1];
#pragma unroll
    for (int j = 0; j < kNch; ++j) {
      cofs[j] = nE;
      nE += cb1[j] - cb0[j];
    }
    cofs[kNch] = nE;
    auto real = [&](int v) {
      int j = 0;
#pragma unroll
      for (int jj = 1; jj < kNch; ++jj)
        if (v >= cofs[jj]) j = jj;
      return cb0[j] + (v - cofs[j]);
    };
    // CTA scan of the entries' counts (e, p, f, dt, b): each thread sums a contiguous
    // segment, warp shuffle scan, scan of the 32 warp totals; the CTA total claims
    // output space with atomics (the order in which CTAs claim space only permutes the
    // next frontier; work items carry their per-key rank and are counting-sorted by
    // (key, rank) afterwards, so every result stays bit-reproducible).  Entries and
    // their pairs share ONE 64-bit atomic on the packed (e, p) totals, so pair offsets
    // grow with entry index (entry_bounds relies on it).
    const int per_t = (nE + kPBlock - 1) / kPBlock;
    const int s0 = min(nE, threadIdx.x * per_t), s1 = min(nE, (threadIdx.x + 1) * per_t);
    int v5[5] = { 0, 0, 0, 0, 0 };
    for (int v = s0; v < s1; ++v) {
      const Cnt c = a.cnt[real(v)];
      v5[0] += c.e;
      v5[1] += c.p;
      v5[2] += c.f;
      v5[3] += c.dt;
      v5[4] += c.b;
    }
    int x5[5];
    {
      const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        int x = v5[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        x5[k] = x - v5[k];  // exclusive within the warp
        if (lane == 31) s_wsum[wib][k] = x;
      }
      __syncthreads();
      if (wib == 0) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int w = lane < kPBlock / 32 ? s_wsum[lane][k] : 0;
          int x = w;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          s_wsum[lane][k] = x - w;  // exclusive warp prefix
          if (lane == 31) (&s_agg.e)[k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 3 : 5] = x;
        }
        if (lane == 0) s_agg.t = s_agg.fd = 0;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 5; ++k) x5[k] += s_wsum[wib][k];
    }
    if (threadIdx.x == 0) {
      const unsigned long long v =
        ((unsigned long long)(unsigned)s_agg.e << 32) | (unsigned)s_agg.p;
      const unsigned long long o = v ? atomicAdd(&a.lvlep[levels], v) : 0ull;
      s_excl.e = (int)(o >> 32);
      s_excl.p = (int)(o & 0xffffffffu);
      s_excl.t = s_excl.fd = 0;
    } else if (threadIdx.x < 4) {
      const int k = threadIdx.x == 1 ? 2 : threadIdx.x == 2 ? 3 : 5;  // f, dt, b
      const int v = (&s_agg.e)[k];
      (&s_excl.e)[k] = v ? atomicAdd(&a.lvlcnt[levels].e + k, v) : 0;
    }
    __syncthreads();
    if (a.trace && blockIdx.x == G - 1 && threadIdx.x == 0 && levels < 512) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[levels * 4 + 1] = t;
    }
    PH(5);
    const Cnt excl = s_excl;
    // everything this CTA writes ends below excl + agg: emit only if that fits (on
    // overflow the level is abandoned and the host reruns with larger buffers)
    if (!over_capacity(st, CntSum()(excl, s_agg), gF, gDT, gB)) {
      Cnt run{ excl.e + x5[0], excl.p + x5[1], excl.f + x5[2], excl.dt + x5[3], 0, excl.b + x5[4], 0 };
      for (int v = s0; v < s1; ++v) {
        const int i = real(v);
        a.cntoff[i] = run;
        const Cnt c = a.cnt[i];
        run.e += c.e;
        run.p += c.p;
        run.f += c.f;
        run.dt += c.dt;
        run.b += c.b;
      }
      __syncthreads();
      PH(6);
      if (cached) emit_range<32>(a, K, cur, gF, gDT, gB, cb0[0], cb1[0], pc.dec, pc.R, cP0);
      else
        for (int j = 0; j < nch; ++j) emit_range<32>(a, K, cur, gF, gDT, gB, cb0[j], cb1[j]);
    }
    PH(7);
    if (a.trace && threadIdx.x == 0 && levels < 64) {  // per-CTA busy time of the level
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      a.trace[4096 + 512 * 16 + levels * 160 + blockIdx.x] = t_;
    }
    grid.sync();
    PH(8);
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && levels < 512) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[levels * 4 + 2] = t;
      a.trace[(levels + 1) * 4 + 3] = t;
    }
    Cnt lv = ldcg_cnt(&a.lvlcnt[levels]);
    {
      const unsigned long long ep = __ldcg(&a.lvlep[levels]);
      lv.e = (int)(ep >> 32);
      lv.p = (int)(ep & 0xffffffffu);
    }
    if (over_capacity(st, lv, gF, gDT, gB)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        st.lvl = lv;
        st.overflow = 1;
      }
      break;
    }
    gF += lv.f;
    gDT += lv.dt;
    gB += lv.b;
    cur ^= 1;
    m = lv.e;
    p = lv.p;
    ++levels;
    if (m == 0) break;
    if (levels == kMaxLevels) {  // deeper than any kd-tree pair can go; report, don't spin
      if (blockIdx.x == 0 && threadIdx.x == 0) st.overflow = 2;
      break;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslots * sNStat; i += kPBlock) {
    const unsigned long long v = (&s_sst[0][0])[i];
    if (v) atomicAdd(&st.sst[0][0] + i, v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st.cur = cur;
    st.m[cur] = m;
    st.p[cur] = p;
    st.nF = gF;
    st.nDT = gDT;
    st.nB = gB;
    st.levels = levels;
  }
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

// The kernels of one level for the graph / host-loop paths.
constexpr int kLevelKernels = 6;
void launch_level(const TravArgs& a, int D, cudaStream_t s, cudaGraphConditionalHandle hc,
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



}  // namespace

// This file is compiled twice: as itself (1024-thread traversal CTAs, every host entry)
// and through traverse_small.cu (KPBLOCK = 640, DFGTB_TRAV_SMALL_TU: only the kernels,
// this upload into that unit's own __constant__ copies, and the kernel lookup below).
#ifdef DFGTB_TRAV_SMALL_TU
#define DFGTB_TRUNC_INIT init_truncation_tables_small
#else
#define DFGTB_TRUNC_INIT init_truncation_tables
#endif
void DFGTB_TRUNC_INIT(cudaStream_t s)
{
  double isf[16], sf[16], bin[17][17];
  double f = 1.0;
  for (int p = 0; p < 16; ++p) {
    if (p > 1) f *= p;  // sqrt_factorial, truncation.cpp:20-27
    sf[p] = std::sqrt(f);
    isf[p] = 1.0 / sf[p];
  }
  for (int n = 0; n <= 16; ++n)
    for (int k = 0; k <= 16; ++k) {
      double b = k > n ? 0.0 : 1.0;
      for (int i = 1; i <= k && k <= n; ++i) b *= (double)(n - k + i) / (double)i;  // truncation.cpp:11-18
      bin[n][k] = b;
    }
  CK(cudaMemcpyToSymbolAsync(c_isf, isf, sizeof(isf), 0, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyToSymbolAsync(c_sf, sf, sizeof(sf), 0, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyToSymbolAsync(c_binom, bin, sizeof(bin), 0, cudaMemcpyHostToDevice, s));
}

#ifdef DFGTB_TRAV_SMALL_TU
// k_traverse with kPBlock-thread CTAs (96 registers instead of 64: fewer spills, shorter
// dependent chains per level -- faster where the levels are latency-bound, slower where
// they are throughput-bound; Engine::run_levels chooses)
void* traverse_small_kernel(int D)
{
  switch (D) {
  case 1: return (void*)k_traverse<1>;
  case 2: return (void*)k_traverse<2>;
  case 3: return (void*)k_traverse<3>;
  case 4: return (void*)k_traverse<4>;
  case 5: return (void*)k_traverse<5>;
  default: return (void*)k_traverse<0>;
  }
}
int traverse_small_block() { return kPBlock; }
#else
// ------------------------------------------------------------------ test entries
namespace {
__global__ void k_choose_test(int n, const double* args, int* out)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* a = args + (size_t)9 * i;
  const int pmax = (int)a[6], dim = (int)a[7], cost = (int)a[8];
  int kind = kE, order = 0;
  dev_choose(a[0], a[1], a[2], a[3], a[4], a[5], pmax, dim, cost, kind, order);
  const double uq = a[2] / a[4], ur = a[3] / a[4];
  int* o = out + (size_t)5 * i;
  o[0] = kind;
  o[1] = order;
  o[2] = d_order_ff(ur * 0.5, a[1], a[5], pmax, dim);
  o[3] = d_order_ff(uq * 0.5, a[1], a[5], pmax, dim);
  o[4] = d_order_f2l((uq < ur ? ur : uq) * 0.25, a[1], a[5], pmax, dim);
}

__global__ void k_box_test(int n, int d, const double* boxes, double* out)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* b = boxes + (size_t)4 * d * i;
  box_bounds<0>(b, b + d, b + 2 * d, b + 3 * d, d, out[2 * i], out[2 * i + 1]);
}
}  // namespace

void choose_methods_device(size_t n, const double* args, int* out)
{
  if (n == 0) return;
  init_device_constants(0);
  DevBuf<double> da;
  DevBuf<int> dout;
  da.reserve(9 * n);
  dout.reserve(5 * n);
  CK(cudaMemcpy(da.p, args, sizeof(double) * 9 * n, cudaMemcpyHostToDevice));
  k_choose_test<<<ceil_div((long long)n, 128), 128>>>((int)n, da.p, dout.p);
  CK_LAUNCH();
  CK(cudaMemcpy(out, dout.p, sizeof(int) * 5 * n, cudaMemcpyDeviceToHost));
}

void box_bounds_device(size_t n, int d, const double* boxes, double* out)
{
  if (n == 0) return;
  DevBuf<double> db, dout;
  db.reserve(4 * (size_t)d * n);
  dout.reserve(2 * n);
  CK(cudaMemcpy(db.p, boxes, sizeof(double) * 4 * d * n, cudaMemcpyHostToDevice));
  k_box_test<<<ceil_div((long long)n, 128), 128>>>((int)n, d, db.p, dout.p);
  CK_LAUNCH();
  CK(cudaMemcpy(out, dout.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
}

void Engine::destroy_graph()
{
  if (gexec_) cudaGraphExecDestroy(gexec_);
  if (graph_) cudaGraphDestroy(graph_);
  gexec_ = nullptr;
  graph_ = nullptr;
  gsig_.clear();
}

// Runs the whole level loop: preferably one cooperative kernel; else one CUDA graph
// whose WHILE node repeats the level kernels until k_advance clears the condition;
// else the host launches levels and polls.
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
    // Small batches (slots x query points below kTravSmallWork) are latency-bound at every
    // level: the small-CTA build (traverse_small.cu: 640 threads, 96 registers) runs them
    // faster (cfg2, 0.9M: 0.637 -> 0.576 ms; cfg1: 0.320 -> 0.264 ms); bigger ones need the
    // 1024 threads (768 vs 1024 threads: cfg4, 1.4M: 23.6 vs 20.1 ms; cfg3, 3.6M: 12.3 vs
    // 10.9 ms; cfg5: 37.3 vs 32.4 ms).  DFGTB_TRAV_BLOCK = 640 / 1024 forces one.
    static const int blk_env = std::getenv("DFGTB_TRAV_BLOCK") ? std::atoi(std::getenv("DFGTB_TRAV_BLOCK")) : 0;
    const bool small = !kUseCache && (blk_env ? blk_env == traverse_small_block()
                                              : (long long)trav_nq_ * trav_nb_ < kTravSmallWork);
    int block = kPBlock;
    if (small) {
      fn = traverse_small_kernel(D_);
      block = traverse_small_block();
    }
    int dev = 0, nsm = 0, per_sm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int smem = kUseCache ? kCacheBytes : 0;
    if (smem) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
    if (per_sm >= 1) {
      TravArgs copy = a;
      void* kargs[] = { &copy };
      CK(cudaLaunchCooperativeKernel(fn, nsm * std::min(per_sm, kPerSM), block, kargs, smem, s_));
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

__global__ void k_trav_publish(const TravState* st, int* bc)
{  // BatchCounts: nF, nDT, nB, traversal overflow (an overflowed batch is rerun: its
   // item counts read as zero so nothing downstream follows a half-written list)
  const int ovf = st->overflow;
  bc[0] = ovf ? 0 : st->nF;
  bc[1] = ovf ? 0 : st->nDT;
  bc[2] = ovf ? 0 : st->nB;
  bc[3] = ovf;
  bc[8] = ovf ? 0 : st->nF;  // extents of the unsorted item arrays
  bc[9] = ovf ? 0 : st->nDT;
  bc[10] = ovf ? 0 : st->nB;
}

__global__ void k_trav_clear_on_overflow(const int* bc, int* cntF, int* cntDT, int* cntB, int KB)
{
  if (!bc[3]) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < KB; i += gridDim.x * blockDim.x)
    cntF[i] = cntDT[i] = cntB[i] = 0;
}

// Counting sort of the three item kinds by (key, rank).  scan = exclusive scan of the
// F | DT | B per-key counts (3 KB); n = the item totals (bc[8..10]).  Writes each kind's
// per-key offsets rebased to its segment start (offLoc, 3 segments of KB) and its items
// to sorted position (offset of its key + its rank).
__global__ void k_sort_items3(const int* scan, int KB, const int* n, const Item* inF, const Item* inDT,
                              const Item* inB, int capF, int capDT, int capB, int* offLoc, Item* outF,
                              Item* outDT, Item* outB)
{
  const int b1 = scan[KB], b2 = scan[2 * KB];  // segment starts (the first one is 0)
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = t0; i < 3 * KB; i += nt) offLoc[i] = scan[i] - (i < KB ? 0 : i < 2 * KB ? b1 : b2);
  const int mF = min(n[0], capF), mDT = min(n[1], capDT), mB = min(n[2], capB);
  for (int i = t0; i < mF + mDT + mB; i += nt) {
    if (i < mF) {
      const Item it = inF[i];
      if (it.key >= 0) outF[scan[it.key] + it.rank] = it;
    } else if (i < mF + mDT) {
      const Item it = inDT[i - mF];
      if (it.key >= 0) outDT[scan[KB + it.key] - b1 + it.rank] = it;
    } else {
      const Item it = inB[i - mF - mDT];
      if (it.key >= 0) outB[scan[2 * KB + it.key] - b2 + it.rank] = it;
    }
  }
}

// Start frontier of the traversal: the nodes at depth d0 (DFGTB_TRAV_START_DEPTH, default
// 5; 0 = the roots) and the leaves above it, of the query and of the reference tree.  The
// top levels of the level loop hold few pairs but cost a full level each (~15 us of
// barriers and dependent loads); starting below them is still a dual-tree traversal of a
// partition of Q x R, so the lower bounds and the eps guarantee hold unchanged.
static void frontier_nodes(const DevTree& t, int d0, std::vector<int>& out)
{
  out.clear();
  // preorder ids: the right child follows the left subtree; a node is in the frontier
  // if its depth is d0, or it is a leaf above that depth
  std::vector<std::pair<int, int>> stack{ { 0, 0 } };
  std::vector<int> sub(t.nodes, 1);
  for (int i = t.nodes - 1; i >= 0; --i)
    if (t.h_left[i] >= 0) sub[i] = 1 + sub[t.h_left[i]] + sub[t.h_left[i] + sub[t.h_left[i]]];
  while (!stack.empty()) {
    const auto [v, d] = stack.back();
    stack.pop_back();
    if (d == d0 || t.h_left[v] < 0) {
      out.push_back(v);
      continue;
    }
    const int l = t.h_left[v], r = l + sub[l];
    stack.push_back({ r, d + 1 });
    stack.push_back({ l, d + 1 });
  }
}

void Engine::start_frontier(const DevTree& qt, void* args)
{
  TravArgs& a = *static_cast<TravArgs*>(args);
  // measured (cfg2 sweep): depth 0 1.47 ms, 3 1.43, 4 1.39, 5 1.37, 6 1.38 with 1024-thread
  // CTAs; with the 640-thread small-batch build 4 1.135, 5 1.117, 6 1.105, 7 1.134; cfg3 neutral
  static const int d0 = std::getenv("DFGTB_TRAV_START_DEPTH") ? std::atoi(std::getenv("DFGTB_TRAV_START_DEPTH")) : 6;
  a.sq = a.sr = nullptr;
  a.nsq = a.nsr = 1;
  // only deep trees have top levels worth skipping (a shallow tree keeps the reference's
  // schedule, e.g. a loose eps still prunes the root pair alone)
  const int d = std::min(d0, std::min(qt.height, rt_.height) - 10);
  if (d <= 0) return;
  std::vector<int> qn, rn;
  frontier_nodes(qt, d, qn);
  frontier_nodes(rt_, d, rn);
  std::vector<int> both(qn);
  both.insert(both.end(), rn.begin(), rn.end());
  sfront_.reserve(both.size());
  CK(cudaMemcpyAsync(sfront_.p, both.data(), sizeof(int) * both.size(), cudaMemcpyHostToDevice, s_));
  a.sq = sfront_.p;
  a.sr = sfront_.p + qn.size();
  a.nsq = (int)qn.size();
  a.nsr = (int)rn.size();
}

// Launches the whole traversal of a batch and the counting sorts of its work items
// WITHOUT a host round trip: the counts stay on the device (bc_), the host reads them
// once at the end of the batch (traverse_finish) and reruns on overflow.
void Engine::traverse(const DevTree& qt, const double* h, int nb)
{
  const int K = qt.nodes;
  const int T = ser_.T;
  const long long KB = (long long)K * nb;
  if (KB > INT32_MAX / 2) throw OutOfMemory("batch too large: slots * nodes exceeds 2^30");
  cudaStream_t s = s_;
  L_.reserve((size_t)KB * T);
  Lord_.reserve(KB);
  cntAll_.reserve((size_t)3 * KB);
  cntF_.p = cntAll_.p;
  cntDT_.p = cntAll_.p + KB;
  cntB_.p = cntAll_.p + 2 * (size_t)KB;
  if (!hst_) {
    hst_ = pinned_alloc(sizeof(TravState));
    hst_bytes_ = sizeof(TravState);
    dst_.reserve(sizeof(TravState));
  }
  TravState* hs = static_cast<TravState*>(hst_);
  TravState* ds = reinterpret_cast<TravState*>(dst_.p);
  {  // first guesses; overflow regrows and the engine keeps the sizes
    // DFGTB_TINY_CAPS (tests): start from 64-element buffers, so first batches overflow,
    // regrow and rerun several times
    static const bool tiny = std::getenv("DFGTB_TINY_CAPS") != nullptr;
    const int kb = (int)std::min<long long>(KB, INT32_MAX / 64);
    capE_ = std::max(capE_, tiny ? 64 : std::max(4096, 2 * kb));
    capP_ = std::max(capP_, tiny ? 64 : std::max(1 << 16, 16 * kb));
    capF_ = std::max(capF_, tiny ? 64 : std::max(4096, 2 * kb));
    capDT_ = std::max(capDT_, tiny ? 64 : std::max(4096, 2 * kb));
    capB_ = std::max(capB_, tiny ? 64 : std::max(1 << 16, 16 * kb));
  }
  {
    for (int b = 0; b < 2; ++b) {
      fq_[b].reserve(capE_);
      foff_[b].reserve(capE_);
      flen_[b].reserve(capE_);
      fbase_[b].reserve(capE_);
      fr_[b].reserve(capP_);
      pent_[b].reserve(capP_);
    }
    pglo_.reserve(capE_);
    pkmax_.reserve(capP_);
    pkmin_.reserve(capP_);
    dec_.reserve(capP_);
    cnt_.reserve(capE_);
    cntoff_.reserve(capE_);
    childlen_.reserve(capE_);
    newbase_.reserve(capE_);
  }
  ctsum_.reserve(kScanTiles);
  ctoff_.reserve(kScanTiles);
  itF_.reserve(capF_);
  itDT_.reserve(capDT_);
  itB_.reserve(capB_);
  bc_.reserve(16);
  CK(cudaMemsetAsync(bc_.p, 0, sizeof(int) * 16, s));

  TravArgs a{};
  a.Q = view_of(qt);
  a.R = view_of(rt_);
  a.selfq = &qt == &rt_ ? 1 : 0;
  a.f32 = f32_ ? 1 : 0;
  a.D = D_;
  a.pmax = ser_.pmax;
  a.cost = cfg_.cost_model;
  a.series = cfg_.mode == 1;
  a.T = T;
  a.st = ds;
  for (int b = 0; b < 2; ++b) {
    const int bb = b;
    a.fq[b] = fq_[bb].p;
    a.foff[b] = foff_[bb].p;
    a.flen[b] = flen_[bb].p;
    a.fr[b] = fr_[bb].p;
    a.fbase[b] = fbase_[bb].p;
    a.pent[b] = pent_[bb].p;
  }
  a.glo = pglo_.p;
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
  lvlcnt_.reserve(kMaxLevels);
  CK(cudaMemsetAsync(lvlcnt_.p, 0, sizeof(Cnt) * kMaxLevels, s));
  a.lvlcnt = lvlcnt_.p;
  lvlep_.reserve(kMaxLevels);
  CK(cudaMemsetAsync(lvlep_.p, 0, sizeof(unsigned long long) * kMaxLevels, s));
  a.lvlep = lvlep_.p;
  static const bool tracing = std::getenv("DFGTB_TRACE") != nullptr;
  if (tracing) {
    trace_.reserve(kTrLen);
    CK(cudaMemsetAsync(trace_.p, 0, sizeof(unsigned long long) * (kTrLen), s));
    a.trace = trace_.p;
  }
  const std::vector<const void*> sig = {
    a.Q.lo, a.Q.hi, a.Q.cen, a.Q.side, a.Q.left, a.Q.right, a.Q.count, a.Q.begin,
    a.R.lo, a.R.hi, a.R.side, a.R.left, a.R.right, a.R.count,
    a.st, a.pent[0], a.pent[1], a.glo, a.fq[0], a.fq[1], a.foff[0], a.foff[1], a.flen[0], a.flen[1], a.fr[0], a.fr[1],
    a.fbase[0], a.fbase[1], a.pkmax, a.pkmin, a.dec, a.cnt, a.cntoff, a.tsum, a.toff,
    a.childlen, a.newbase, a.L, a.Lord, a.itF, a.itDT, a.itB, a.cntF, a.cntDT, a.cntB };

  CK(cudaMemsetAsync(L_.p, 0, sizeof(double) * KB * T, s));
  CK(cudaMemsetAsync(Lord_.p, 0, sizeof(int) * KB, s));
  CK(cudaMemsetAsync(cntAll_.p, 0, sizeof(int) * 3 * KB, s));
  hs->eps = cfg_.epsilon - exp_charge();  // the base case's reduced-precision exp is charged
  hs->ntot = (double)n_;
  hs->nslots = nb;
  hs->K = K;
  for (int b = 0; b < nb; ++b) {
    hs->h[b] = h[b];
    hs->scale[b] = -1.0 / (2.0 * h[b] * h[b]);
  }
  hs->capE = capE_;
  hs->capP = capP_;
  hs->capF = capF_;
  hs->capDT = capDT_;
  hs->capB = capB_;
  CK(cudaMemcpyAsync(ds, hs, sizeof(TravState), cudaMemcpyHostToDevice, s));
  start_frontier(qt, &a);
  k_trav_init<<<32, 256, 0, s>>>(a);
  CK_LAUNCH();
  trav_nq_ = qt.n;
  trav_nb_ = nb;
  run_levels(&a, sig);
  k_trav_publish<<<1, 1, 0, s>>>(ds, bc_.p);
  CK_LAUNCH();
  k_trav_clear_on_overflow<<<148, 256, 0, s>>>(bc_.p, cntF_.p, cntDT_.p, cntB_.p, (int)KB);
  CK_LAUNCH();
  trav_nb_ = nb;
  trav_trace_ = a.trace != nullptr;

  // counting sort of the items by key (stable: level order, then emit order)
  // all three kinds at once: one exclusive scan of the F | DT | B counts, then one kernel
  // rebases each segment's offsets to 0 and scatters the items to (key offset + rank)
  offAll_.reserve((size_t)3 * KB);
  offLoc_.reserve((size_t)3 * KB + 1);
  offF_.p = offLoc_.p;
  offDT_.p = offLoc_.p + KB;
  offB_.p = offLoc_.p + 2 * (size_t)KB;
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, cntAll_.p, offAll_.p, 3 * (int)KB, s);
  scan_tmp_.reserve(need + 256);
  size_t have = scan_tmp_.cap;
  cub::DeviceScan::ExclusiveSum(scan_tmp_.p, have, cntAll_.p, offAll_.p, 3 * (int)KB, s);
  sF_.reserve(capF_);
  sDT_.reserve(capDT_);
  sB_.reserve(capB_);
  k_sort_items3<<<148 * 4, 256, 0, s>>>(offAll_.p, (int)KB, bc_.p + 8, itF_.p, itDT_.p, itB_.p, capF_, capDT_,
                                        capB_, offLoc_.p, sF_.p, sDT_.p, sB_.p);
  CK_LAUNCH();
}

// After the batch's final synchronisation: statistics, and the traversal verdict
// (false: buffers overflowed and were regrown -- the batch must be rerun).
void Engine::traverse_fetch_async()
{
  CK(cudaMemcpyAsync(hst_, dst_.p, sizeof(TravState), cudaMemcpyDeviceToHost, s_));
}

bool Engine::traverse_finish(bool prefetched)
{
  TravState* hs = static_cast<TravState*>(hst_);
  const TravState* ds = reinterpret_cast<const TravState*>(dst_.p);
  if (!prefetched) CK(cudaMemcpy(hs, ds, sizeof(TravState), cudaMemcpyDeviceToHost));
  const int nb = trav_nb_;
  if (!use_persistent_ && use_graph_) launch_counter() += (uint64_t)hs->levels * kLevelKernels;
  if (trav_trace_) {  // per level: classify | scan | emit (microseconds)
    std::vector<unsigned long long> tr(kTrLen);
    CK(cudaMemcpy(tr.data(), trace_.p, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost));
    for (int L = 0; L < std::min(hs->levels, 511); ++L) {
      const unsigned long long* ph = tr.data() + 4096 + L * 16;
      const double d = 1e-3;
      std::fprintf(stderr, "DFGTB_TRACE level %d: entries %llu pairs %llu classify+lookback %.1f us, emit+sync %.1f us"
                   " | split %.1f bounds %.1f glo %.1f decide %.1f reduce %.1f offsets %.1f scan %.1f emit %.1f sync %.1f\n",
                   L, tr[2048 + L * 2], tr[2048 + L * 2 + 1], (tr[L * 4 + 1] - tr[L * 4]) * 1e-3,
                   (tr[L * 4 + 2] - tr[L * 4 + 1]) * 1e-3, (ph[0] - tr[L * 4]) * d, (ph[1] - ph[0]) * d,
                   (ph[2] - ph[1]) * d, (ph[3] - ph[2]) * d, (ph[4] - ph[3]) * d, (ph[5] - ph[4]) * d,
                   (ph[6] - ph[5]) * d, (ph[7] - ph[6]) * d, (ph[8] - ph[7]) * d);
      if (L < 64) {  // phase durations averaged over the CTAs
        const unsigned long long* pa = tr.data() + kTrAll + L * 16;
        const double g = 148.0;
        std::fprintf(stderr, "DFGTB_TRACE level %d: mean over CTAs us | split %.1f bounds %.1f glo %.1f decide %.1f "
                     "reduce %.1f offsets %.1f scan %.1f emit %.1f sync %.1f\n", L, pa[0] * d / g, pa[1] * d / g,
                     pa[2] * d / g, pa[3] * d / g, pa[4] * d / g, pa[5] * d / g, pa[6] * d / g, pa[7] * d / g,
                     pa[8] * d / g);
      }
      if (L < 64) {  // the slowest and the median CTA (sum of phases 0-7): phases, pairs, entries
        std::vector<std::pair<double, int>> bs;
        for (int b = 0; b < 148; ++b) {
          const unsigned long long* c = tr.data() + kTrCta + ((size_t)L * 160 + b) * 10;
          double t = 0;
          for (int k = 0; k < 8; ++k) t += c[k] * d;
          bs.push_back({ t, b });
        }
        std::sort(bs.begin(), bs.end());
        for (int w : { (int)bs.size() / 2, (int)bs.size() - 1 }) {
          const unsigned long long* c = tr.data() + kTrCta + ((size_t)L * 160 + bs[w].second) * 10;
          std::fprintf(stderr, "DFGTB_TRACE level %d: %s CTA %d busy %.1f us | split %.1f bounds %.1f glo %.1f decide %.1f "
                       "reduce %.1f offsets %.1f scan %.1f emit %.1f | pairs %llu entries %llu\n", L,
                       w == (int)bs.size() - 1 ? "slowest" : "median", bs[w].second, bs[w].first, c[0] * d, c[1] * d,
                       c[2] * d, c[3] * d, c[4] * d, c[5] * d, c[6] * d, c[7] * d, c[9] & 0xffffffffull, c[9] >> 32);
        }
      }
      if (L < 64) {  // CTA busy times: min / median / max (from the level start of CTA 0)
        std::vector<double> bt;
        for (int b = 0; b < 160; ++b) {
          const unsigned long long v = tr[4096 + 512 * 16 + L * 160 + b];
          if (v) bt.push_back((v - tr[L * 4]) * d);
        }
        std::sort(bt.begin(), bt.end());
        if (!bt.empty())
          std::fprintf(stderr, "DFGTB_TRACE level %d: CTA busy us min %.1f median %.1f p90 %.1f max %.1f; longest entry %llu pairs\n", L,
                       bt.front(), bt[bt.size() / 2], bt[bt.size() * 9 / 10], bt.back(),
                       tr[4096 + 512 * 16 + 64 * 160 + L]);
      }
    }
  }
  if (hs->overflow == 2) throw CudaError("traversal exceeded 1024 levels");
  if (hs->overflow) {
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
    return false;
  }
  slot_stats_.assign(nb, Stats{});
  for (int b = 0; b < nb; ++b) {
    Stats& st = slot_stats_[b];
    const unsigned long long* ss = hs->sst[b];
    st.levels = hs->levels;
    st.pairs_visited = ss[sPairs];
    st.prunes_finite_diff = ss[sFD];
    st.prunes_farfield = ss[sF];
    st.prunes_direct_local = ss[sD];
    st.prunes_far_to_local = ss[sT];
    st.base_cases = ss[sB];
    st.kernel_evaluations = 2ull * ss[sPairs] + ss[sKev];
    st.pairs_covered = ss[sCov];
  }
  nF_ = hs->nF;
  nDT_ = hs->nDT;
  nB_ = hs->nB;
  return true;
}

#endif  // DFGTB_TRAV_SMALL_TU

}  // namespace dfgtb
