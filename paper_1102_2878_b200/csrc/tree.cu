// Level-synchronous, bit-exact GPU build of the reference kd-tree.
//
// Reference: KdTree::build (kdtree.cpp:21-109).  Per level, for every node of the
// level at once:
//   1. bounds    : exact min/max per dimension over the node's points (ordered-key
//                  atomics, order independent);  centroid = 0.5*(lo+hi);
//                  widest = first dimension of maximal width (kdtree.cpp:49-71)
//   2. partition : std::partition(x[widest] <= mid) reproduced exactly.  libstdc++'s
//                  bidirectional __partition swaps the k-th failing element of the
//                  final left block with the k-th passing element (counted from the
//                  right) of the final right block; everything else stays.  A
//                  global prefix scan of the predicate gives both ranks directly.
//   3. fallback  : one-sided splits run a single-thread device restatement of
//                  libstdc++ 13's std::nth_element / __introselect (kdtree.cpp:85-94)
//                  on the node's segment; these nodes are rare (duplicates).
// Nodes are numbered in BFS order while building and renumbered to the reference's
// preorder ids at the end.
#include <chrono>
#include "tree.cuh"

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <numeric>

namespace dfgtb {
namespace cg = cooperative_groups;
namespace {

constexpr int kTile = 1024;
constexpr int kThreads = 256;

__device__ __forceinline__ unsigned long long dkey(double v)
{
  if (v == 0.0) v = 0.0;  // canonical +0 (reference compares with <, so +-0 tie)
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k)
{
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

struct LevelArgs {
  const double* x;     // original coordinates (row-major)
  int D;
  int* perm;
  const int* nbeg;     // per level node: begin
  const int* ncnt;     // per level node: count
  const int* tile_node;   // per tile: level-node index
  const int* tile_start;  // per tile: first sorted position
  unsigned long long* kmin;  // per level node * D
  unsigned long long* kmax;
};

__global__ void k_bounds_init(unsigned long long* kmin, unsigned long long* kmax, int m)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) {
    kmin[i] = ~0ull;
    kmax[i] = 0ull;
  }
}

// One CTA per tile of <= kTile points of one node.
__global__ void k_bounds_tiles(LevelArgs a)
{
  const int tile = blockIdx.x;
  const int j = a.tile_node[tile];
  const int start = a.tile_start[tile];
  const int end = min(a.nbeg[j] + a.ncnt[j], start + kTile);
  const int D = a.D;
  for (int d = 0; d < D; ++d) {
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int i = start + threadIdx.x; i < end; i += blockDim.x) {
      const unsigned long long k = dkey(a.x[(size_t)a.perm[i] * D + d]);
      mn = min(mn, k);
      mx = max(mx, k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&a.kmin[(size_t)j * D + d], mn);
      atomicMax(&a.kmax[(size_t)j * D + d], mx);
    }
  }
}

// Per level node: bounds, centroid, widest side, split midpoint (kdtree.cpp:49-78).
__global__ void k_decide(LevelArgs a, int m, int leaf, int base, double* lo, double* hi,
                         double* centroid, double* max_side, int* split_dim, double* mid_out,
                         int* do_split)
{
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int D = a.D;
  const size_t o = (size_t)(base + j) * D;
  int widest = 0;
  double width = 0.0;
  for (int d = 0; d < D; ++d) {
    const double l = dkey_inv(a.kmin[(size_t)j * D + d]);
    const double h = dkey_inv(a.kmax[(size_t)j * D + d]);
    lo[o + d] = l;
    hi[o + d] = h;
    centroid[o + d] = __dmul_rn(0.5, __dadd_rn(l, h));
    const double w = __dadd_rn(h, -l);
    if (d == 0 || w > width) {
      width = w;
      widest = d;
    }
  }
  max_side[base + j] = width;
  const int split = a.ncnt[j] > leaf;
  do_split[j] = split;
  split_dim[base + j] = split ? widest : -1;
  mid_out[j] = centroid[o + widest];  // 0.5*(lo+hi) of the widest dimension
}

// Predicate flags for every position of a splitting node.
__global__ void k_flags(LevelArgs a, const int* do_split, const int* split_dim_lvl,
                        const double* mid, int* flag)
{
  const int tile = blockIdx.x;
  const int j = a.tile_node[tile];
  if (!do_split[j]) return;
  const int start = a.tile_start[tile];
  const int end = min(a.nbeg[j] + a.ncnt[j], start + kTile);
  const int w = split_dim_lvl[j];
  const double m = mid[j];
  for (int i = start + threadIdx.x; i < end; i += blockDim.x)
    flag[i] = a.x[(size_t)a.perm[i] * a.D + w] <= m ? 1 : 0;
}

// Right-block passers register at slot (begin + rank-from-right).
__global__ void k_slots(LevelArgs a, const int* do_split, const int* flag, const int* P,
                        int* slot)
{
  const int tile = blockIdx.x;
  const int j = a.tile_node[tile];
  if (!do_split[j]) return;
  const int b = a.nbeg[j], e = b + a.ncnt[j];
  const int start = a.tile_start[tile];
  const int end = min(e, start + kTile);
  const int L = P[e] - P[b];
  for (int i = start + threadIdx.x; i < end; i += blockDim.x)
    if (i >= b + L && flag[i]) slot[b + (P[e] - P[i] - 1)] = i;
}

// Left-block failers swap with their partner (disjoint pairs -> race free).
__global__ void k_swap(LevelArgs a, const int* do_split, const int* flag, const int* P,
                       const int* slot)
{
  const int tile = blockIdx.x;
  const int j = a.tile_node[tile];
  if (!do_split[j]) return;
  const int b = a.nbeg[j], e = b + a.ncnt[j];
  const int start = a.tile_start[tile];
  const int end = min(e, start + kTile);
  const int L = P[e] - P[b];
  for (int i = start + threadIdx.x; i < end && i < b + L; i += blockDim.x) {
    if (!flag[i]) {
      const int k = (i - b) - (P[i] - P[b]);
      const int partner = slot[b + k];
      const int t = a.perm[i];
      a.perm[i] = a.perm[partner];
      a.perm[partner] = t;
    }
  }
}

// ---- single-thread restatement of libstdc++ 13 nth_element (stl_algo.h) ----
struct KeyCmp {
  const double* x;
  int D, w;
  __device__ double key(int idx) const { return x[(size_t)idx * D + w]; }
  __device__ bool operator()(int a, int b) const { return key(a) < key(b); }
};

__device__ void dswap(int* a, int* b)
{
  const int t = *a;
  *a = *b;
  *b = t;
}

__device__ void dev_median_to_first(int* res, int* a, int* b, int* c, const KeyCmp& cmp)
{
  if (cmp(*a, *b)) {
    if (cmp(*b, *c)) dswap(res, b);
    else if (cmp(*a, *c)) dswap(res, c);
    else dswap(res, a);
  } else if (cmp(*a, *c)) dswap(res, a);
  else if (cmp(*b, *c)) dswap(res, c);
  else dswap(res, b);
}

__device__ int* dev_unguarded_partition(int* first, int* last, int* pivot, const KeyCmp& cmp)
{
  for (;;) {
    while (cmp(*first, *pivot)) ++first;
    --last;
    while (cmp(*pivot, *last)) --last;
    if (!(first < last)) return first;
    dswap(first, last);
    ++first;
  }
}

__device__ void dev_insertion_sort(int* first, int* last, const KeyCmp& cmp)
{
  if (first == last) return;
  for (int* i = first + 1; i != last; ++i) {
    const int v = *i;
    if (cmp(v, *first)) {
      for (int* p = i; p != first; --p) *p = *(p - 1);
      *first = v;
    } else {
      int* l = i;
      int* nx = i - 1;
      while (cmp(v, *nx)) {
        *l = *nx;
        l = nx;
        --nx;
      }
      *l = v;
    }
  }
}

__device__ void dev_push_heap(int* first, long hole, long top, int v, const KeyCmp& cmp)
{
  long parent = (hole - 1) / 2;
  while (hole > top && cmp(first[parent], v)) {
    first[hole] = first[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  first[hole] = v;
}

__device__ void dev_adjust_heap(int* first, long hole, long len, int v, const KeyCmp& cmp)
{
  const long top = hole;
  long second = hole;
  while (second < (len - 1) / 2) {
    second = 2 * (second + 1);
    if (cmp(first[second], first[second - 1])) second--;
    first[hole] = first[second];
    hole = second;
  }
  if ((len & 1) == 0 && second == (len - 2) / 2) {
    second = 2 * (second + 1);
    first[hole] = first[second - 1];
    hole = second - 1;
  }
  dev_push_heap(first, hole, top, v, cmp);
}

__device__ void dev_heap_select(int* first, int* middle, int* last, const KeyCmp& cmp)
{
  const long len = middle - first;
  if (len >= 2) {
    long parent = (len - 2) / 2;
    for (;;) {
      dev_adjust_heap(first, parent, len, first[parent], cmp);
      if (parent == 0) break;
      parent--;
    }
  }
  for (int* i = middle; i < last; ++i) {
    if (cmp(*i, *first)) {
      const int v = *i;
      *i = *first;
      dev_adjust_heap(first, 0, len, v, cmp);
    }
  }
}

__device__ void dev_nth_element(int* first, int* nth, int* last, const KeyCmp& cmp)
{
  if (first == last || nth == last) return;
  long n = last - first;
  int lg = 0;
  while (n > 1) {
    n >>= 1;
    ++lg;
  }
  long depth = 2L * lg;
  while (last - first > 3) {
    if (depth == 0) {
      dev_heap_select(first, nth + 1, last, cmp);
      dswap(first, nth);
      return;
    }
    --depth;
    int* mid = first + (last - first) / 2;
    dev_median_to_first(first, first + 1, mid, last - 1, cmp);
    int* cut = dev_unguarded_partition(first + 1, last, first, cmp);
    if (cut <= nth) first = cut;
    else last = cut;
  }
  dev_insertion_sort(first, last, cmp);
}

// dev_nth_element on n EQUAL keys (a node of identical points, whose midpoint split is
// always one-sided) with the whole CTA: libstdc++'s introselect then does, per round,
// __move_median_to_first = swap(first, mid) and an __unguarded_partition that swaps
// (f + i, last - 1 - i) for i < (last - f) / 2 (f = first + 1) and returns f + that
// count; the closing insertion sort moves nothing.  Same swaps, in parallel per round.
template <int NT>
__device__ void par_equal_nth(int* q, int n, int tid)
{
  if (n <= 0) return;
  const int nth = n / 2;
  int first = 0, last = n;
  int lg = 0;
  for (int t = n; t > 1; t >>= 1) ++lg;
  int depth = 2 * lg;  // never exhausted: every round halves the range
  while (last - first > 3 && depth > 0) {
    --depth;
    const int mid = first + (last - first) / 2;
    __syncthreads();
    if (tid == 0) dswap(q + first, q + mid);
    __syncthreads();
    const int f = first + 1, ts = (last - f) / 2;
    for (int i = tid; i < ts; i += NT) dswap(q + f + i, q + last - 1 - i);
    const int cut = f + ts;
    if (cut <= nth) first = cut;
    else last = cut;
  }
  __syncthreads();
}

// One thread per splitting node: final left count / split coordinate, running the
// median fallback when the midpoint split is one-sided (kdtree.cpp:85-94).
__global__ void k_finish_split(LevelArgs a, int m, int base, const int* do_split,
                               const int* split_dim_lvl, const double* mid, const int* P,
                               int* left_count, double* split_coord)
{
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  if (!do_split[j]) {
    left_count[j] = 0;
    split_coord[base + j] = 0.0;
    return;
  }
  const int b = a.nbeg[j], c = a.ncnt[j];
  const int L = P[b + c] - P[b];
  if (L == 0 || L == c) {
    KeyCmp cmp{ a.x, a.D, split_dim_lvl[j] };
    int* p0 = a.perm + b;
    dev_nth_element(p0, p0 + c / 2, p0 + c, cmp);
    left_count[j] = c / 2;
    split_coord[base + j] = cmp.key(p0[c / 2]);
  } else {
    left_count[j] = L;
    split_coord[base + j] = mid[j];
  }
}

// Scatter BFS-indexed build arrays into preorder-indexed tree arrays.
__global__ void k_to_preorder(int K, int D, const int* bfs2pre, const double* blo,
                              const double* bhi, const double* bcen, const double* bside,
                              const double* bsc, const int* bsd, const int* bleft,
                              const int* bright, const int* bbeg, const int* bcnt,
                              const int* bpar, const int* bdep, double* lo, double* hi,
                              double* cen, double* side, double* sc, int* sd, int* left,
                              int* right, int* beg, int* cnt, int* par, int* dep, int* by_depth,
                              const int* rank)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int p = bfs2pre[i];
  for (int d = 0; d < D; ++d) {
    lo[(size_t)p * D + d] = blo[(size_t)i * D + d];
    hi[(size_t)p * D + d] = bhi[(size_t)i * D + d];
    cen[(size_t)p * D + d] = bcen[(size_t)i * D + d];
  }
  side[p] = bside[i];
  sc[p] = bsc[i];
  sd[p] = bsd[i];
  left[p] = bleft[i] < 0 ? -1 : bfs2pre[bleft[i]];
  right[p] = bright[i] < 0 ? -1 : bfs2pre[bright[i]];
  beg[p] = bbeg[i];
  cnt[p] = bcnt[i];
  par[p] = bpar[i] < 0 ? -1 : bfs2pre[bpar[i]];
  dep[p] = bdep[i];
  by_depth[rank ? rank[i] : i] = p;
}

// Ancestor chain of every node (root first), for nodes with depth < kMaxAnc: kernels
// that walk a leaf's ancestors read them with one coalesced load instead of a
// dependent parent-pointer chain.
__global__ void k_ancestors(int K, const int* parent, const int* depth, int* anc)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const int dp = depth[i];
  if (dp >= kMaxAnc) return;
  int a = i;
  for (int k = dp; k >= 0; --k) {
    anc[(size_t)i * kMaxAnc + k] = a;
    a = parent[a];
  }
}

__global__ void k_gather_points(const double* x, const int* perm, int n, int D, double* xs)
{
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)n * D) return;
  const size_t r = i / D, d = i % D;
  xs[i] = x[(size_t)perm[r] * D + d];
}

__global__ void k_iota(int* p, int n)
{
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

// ------------------------------------------------------------------------------
// Persistent build: every level in ONE cooperative launch (one CTA per SM), node
// bookkeeping on the device, no host round trip per level.  Same arithmetic and the
// same partition / nth_element semantics as the per-level kernels above; six grid
// barriers per level:
//   A bounds (ordered-key atomics)  | B decide  | C flags + chunk scans  |
//   D P and child ids               | E slots + one-sided fallback  | F swaps + next seg
// Positions are statically chunked over the CTAs (C scans its chunk locally, D adds
// the preceding chunks' totals), so the prefix P and the BFS child ids are exactly
// those of a sequential scan.
#ifndef DFGTB_TREE_PB
#define DFGTB_TREE_PB 1024
#endif
constexpr int kPB = DFGTB_TREE_PB;  // threads per CTA of k_build
constexpr int kMaxTreeLevels = 256;

struct BuildArgs {
  const double* x;
  int n, D, leaf;
  int *perm, *seg, *flag, *P, *slot;
  int *nbeg, *ncnt, *nleft, *nright, *npar, *ndep;  // BFS node ids
  double *blo, *bhi, *bcen, *bside, *bsc;
  int* bsd;
  unsigned long long *kmin, *kmax;  // bounds keys, two level buffers of 2n*D (level parity)
  int* pslot;                       // next-level node -> its slot 2j+side in the keys buffer
  double* mid;                      // per level node
  int *dosplit, *child, *lc;        // per level node
  int* ctot;                        // 2 * gridDim.x chunk totals
  int* lvl;                         // [0] = levels, [1..] = level base offsets
  unsigned long long* trace;        // DFGTB_TRACE: per level 8 %globaltimer stamps of CTA 0
  int* lvlmax;                      // per level: largest count of a splitting node
  int* kcount;                      // node count (ids handed out by the local phase)
  int local_S;                      // subtree size of the CTA-local phase (0: off)
  int* loc;                         // {base, m, level} of the local phase (m = 0: none)
};

__device__ __forceinline__ void chunk_of(int total, int b, int G, int& lo, int& hi)
{
  lo = (int)((long long)total * b / G);
  hi = (int)((long long)total * (b + 1) / G);
}

// ---- CTA-local subtrees ---------------------------------------------------------
// Once every splitting node of a level holds <= local_S points, each CTA builds whole
// subtrees (the level's nodes b, b + G, ..) in shared memory: the same bounds / split
// rule / partition pairing / nth_element fallback as the global phases, one local level
// per step with __syncthreads only.  Node ids of the new nodes come from an atomic
// counter (any labelling with children after parents works: the host renumbers to
// preorder and ranks nodes by depth).
constexpr int kLS = 4096;  // positions per subtree (shared memory)
constexpr int kLN = 256;   // nodes per local level
constexpr int kLMaxD = 8;  // dimensions the local phase supports
constexpr int kLEq = 64;      // identical-point nodes per local level handled by the whole CTA
constexpr int kLCacheD = 2;  // D <= 2: the subtree's coordinates are staged in shared memory
int local_smem_bytes(int D)
{
  return 5 * kLS * 4 + 4                          // sp, seg, flag, P (+1), slot
         + 2 * kLN * (6 * 4 + 8) + kLN * 2 * 4     // two node buffers, lc, rank
         + 2 * 2 * kLN * D * 8                     // child key min / max
         + (D <= kLCacheD ? kLS * (8 * D + 4) : 0);  // coordinates + point ids (local ids in sp)
}

template <int NT, class TS>
__device__ void local_subtrees(const BuildArgs& a, TS& tmp, unsigned char* lsm, int base, int m, int level,
                               const int* dsp, const double* mdp)
{
  constexpr int kPB = NT;  // threads of the calling CTA
  using BS = cub::BlockScan<int, kPB>;
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, D = a.D;
  int* sp = reinterpret_cast<int*>(lsm);
  int* sseg = sp + kLS;
  int* sflag = sseg + kLS;
  int* sP = sflag + kLS;  // kLS + 1
  int* sslot = sP + kLS + 1;
  int* nb0 = sslot + kLS;  // node buffers: id, bg, cn, ds, w (5 x kLN ints) each
  int* nb1 = nb0 + 5 * kLN;
  int* nlc = nb1 + 5 * kLN;
  int* nrk = nlc + kLN;
  double* nmid0 = reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(nrk + kLN + 1) & ~(uintptr_t)7);
  double* nmid1 = nmid0 + kLN;
  unsigned long long* kmn = reinterpret_cast<unsigned long long*>(nmid1 + kLN);
  unsigned long long* kmx = kmn + 2 * kLN * D;
  // D <= kLCacheD: sp holds LOCAL ids into the staged coordinates xl (the nth_element
  // swaps are the same, the keys compare equal): no global load per comparison
  const bool cache = D <= kLCacheD;
  double* xl = reinterpret_cast<double*>(kmx + 2 * kLN * D);
  int* gid = reinterpret_cast<int*>(xl + kLS * D);
  const double* X = cache ? xl : a.x;
  __shared__ int s_ns, s_cbase, s_neq;
  __shared__ int2 s_eq[kLEq];  // this local level's nodes of identical points
  if (tid == 0) s_neq = 0;
  for (int j = blockIdx.x; j < m; j += G) {
#ifdef DFGTB_TREE_DEBUG
    unsigned long long t0_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0_));
    int levels_ = 0, maxnodes_ = 0, eqn_ = 0;
#endif
    const int id0 = base + j, b0 = a.nbeg[id0], c = a.ncnt[id0];
    for (int k = tid; k < c; k += kPB) {
      const int g = a.perm[b0 + k];
      if (cache) {
        gid[k] = g;
        sp[k] = k;
        for (int d = 0; d < D; ++d) xl[(size_t)k * D + d] = a.x[(size_t)g * D + d];
      } else {
        sp[k] = g;
      }
      sseg[k] = 0;
    }
    int* cur = nb0;
    int* nxt = nb1;
    double* cmid = nmid0;
    double* xmid = nmid1;
    if (tid == 0) {
      cur[0] = id0;
      cur[kLN] = 0;
      cur[2 * kLN] = c;
      cur[3 * kLN] = dsp[j];
      cur[4 * kLN] = a.bsd[id0];
      cmid[0] = mdp[j];
    }
    int ncur = 1, lev = level;
    __syncthreads();
    while (ncur > 0) {
      const int* nid = cur;
      const int* nbg = cur + kLN;
      const int* ncn = cur + 2 * kLN;
      const int* nds = cur + 3 * kLN;
      const int* nw = cur + 4 * kLN;
      for (int i = tid; i < 2 * ncur * D; i += kPB) {
        kmn[i] = ~0ull;
        kmx[i] = 0ull;
      }
      __syncthreads();
      // predicate x_w <= mid (the children's bounds are reduced after the partition, over
      // their contiguous position ranges: no shared-memory atomics)
      for (int k = tid; k < c; k += kPB) {
        int f = 0;
        const int jj = sseg[k];
        if (jj >= 0 && nds[jj]) f = X[(size_t)sp[k] * D + nw[jj]] <= cmid[jj] ? 1 : 0;
        sflag[k] = f;
      }
      __syncthreads();
      // exclusive prefix of the flags over the subtree's positions
      {
        constexpr int IPT = kLS / kPB;
        int in[IPT], out[IPT], agg;
#pragma unroll
        for (int t = 0; t < IPT; ++t) {
          const int k = tid * IPT + t;
          in[t] = k < c ? sflag[k] : 0;
        }
        BS(tmp).ExclusiveSum(in, out, agg);
#pragma unroll
        for (int t = 0; t < IPT; ++t) {
          const int k = tid * IPT + t;
          if (k < c) sP[k] = out[t];
        }
        if (tid == 0) sP[c] = agg;
      }
      __syncthreads();
      // per node: final left count (median fallback for one-sided splits, kdtree.cpp:85-94);
      // per position: right-block passers register their slots
      for (int jj = tid; jj < ncur; jj += kPB) {
        const int id = nid[jj];
        if (!nds[jj]) {
          a.bsc[id] = 0.0;
          a.nleft[id] = a.nright[id] = -1;
          continue;
        }
        const int bg = nbg[jj], cn = ncn[jj];
        const int L = sP[bg + cn] - sP[bg];
        int l;
        if (L == 0 || L == cn) {
          KeyCmp cmp{ X, D, nw[jj] };
          int* q0 = sp + bg;
          if (a.bside[id] == 0.0 && cn > 3) {
            // identical points: both children's bounds are the node's, and the median
            // permutation is par_equal_nth's (run by the whole CTA below)
            const int k = atomicAdd(&s_neq, 1);
            if (k < kLEq) {
              s_eq[k] = make_int2(bg, cn);
              l = cn / 2;
              a.bsc[id] = cmp.key(q0[0]);
              nlc[jj] = l;
              continue;
            }
          }
          dev_nth_element(q0, q0 + cn / 2, q0 + cn, cmp);
          l = cn / 2;
          a.bsc[id] = cmp.key(q0[cn / 2]);
        } else {
          l = L;
          a.bsc[id] = cmid[jj];
        }
        nlc[jj] = l;
      }
      for (int k = tid; k < c; k += kPB) {
        const int jj = sseg[k];
        if (jj < 0 || !nds[jj] || !sflag[k]) continue;
        const int bg = nbg[jj], e = bg + ncn[jj];
        const int L = sP[e] - sP[bg];
        if (k >= bg + L) sslot[bg + (sP[e] - sP[k] - 1)] = k;
      }
      __syncthreads();
#ifdef DFGTB_TREE_DEBUG
      ++levels_;
      maxnodes_ = max(maxnodes_, ncur);
      eqn_ += min(s_neq, kLEq);
#endif
      const int neq = min(s_neq, kLEq);
      for (int e = 0; e < neq; ++e) par_equal_nth<kPB>(sp + s_eq[e].x, s_eq[e].y, tid);
      __syncthreads();
      if (tid == 0) s_neq = 0;
      // left-block failers swap with their partners (libstdc++ partition pairing)
      for (int k = tid; k < c; k += kPB) {
        const int jj = sseg[k];
        if (jj < 0 || !nds[jj] || sflag[k]) continue;
        const int bg = nbg[jj];
        const int L = sP[bg + ncn[jj]] - sP[bg];
        if (k < bg + L) {
          const int kk = (k - bg) - (sP[k] - sP[bg]);
          const int partner = sslot[bg + kk];
          const int t = sp[k];
          sp[k] = sp[partner];
          sp[partner] = t;
        }
      }
      // children: ranks among splitting nodes, ids, records, next-level node buffers
      if (tid < 32) {
        int run = 0;
        for (int j0 = 0; j0 < ncur; j0 += 32) {
          const int jj = j0 + lane;
          const int sflg = jj < ncur ? nds[jj] : 0;
          int x = sflg;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          if (jj < ncur) nrk[jj] = run + x - sflg;
          run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
          s_ns = run;
          s_cbase = run ? atomicAdd(a.kcount, 2 * run) : 0;
        }
      }
      __syncthreads();
      // children's bounds: one warp per child over its contiguous positions (after the
      // swaps above), the same min / max keys as the reference's bounds pass
      for (int c2 = tid >> 5; c2 < 2 * ncur; c2 += kPB / 32) {
        const int jj = c2 >> 1, side = c2 & 1;
        if (!nds[jj]) continue;
        const int bg = nbg[jj], cn = ncn[jj], l = nlc[jj];
        const int k0 = side ? bg + l : bg, k1 = side ? bg + cn : bg + l;
        for (int d = 0; d < D; ++d) {
          unsigned long long mn = ~0ull, mx = 0ull;
          for (int k = k0 + lane; k < k1; k += 32) {
            const unsigned long long kk = dkey(X[(size_t)sp[k] * D + d]);
            mn = min(mn, kk);
            mx = max(mx, kk);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          }
          if (lane == 0) {
            kmn[c2 * D + d] = mn;
            kmx[c2 * D + d] = mx;
          }
        }
      }
      __syncthreads();
      const int ns = s_ns, cbase = s_cbase;
      for (int jj = tid; jj < ncur; jj += kPB) {
        if (!nds[jj]) continue;
        const int id = nid[jj], bg = nbg[jj], cn = ncn[jj], l = nlc[jj], r = nrk[jj];
        const int cid = cbase + 2 * r;
        a.nleft[id] = cid;
        a.nright[id] = cid + 1;
        for (int side = 0; side < 2; ++side) {
          const int ch = cid + side, q = 2 * r + side;
          const int cb = side ? bg + l : bg, cc = side ? cn - l : l;
          a.npar[ch] = id;
          a.ndep[ch] = lev + 1;
          a.nbeg[ch] = b0 + cb;
          a.ncnt[ch] = cc;
          const size_t o = (size_t)ch * D;
          int widest = 0;
          double width = 0.0;
          for (int d = 0; d < D; ++d) {
            const double lo = dkey_inv(kmn[(2 * jj + side) * D + d]);
            const double hi = dkey_inv(kmx[(2 * jj + side) * D + d]);
            a.blo[o + d] = lo;
            a.bhi[o + d] = hi;
            a.bcen[o + d] = __dmul_rn(0.5, __dadd_rn(lo, hi));
            const double w = __dadd_rn(hi, -lo);
            if (d == 0 || w > width) {
              width = w;
              widest = d;
            }
          }
          a.bside[ch] = width;
          const int split = cc > a.leaf;
          a.bsd[ch] = split ? widest : -1;
          nxt[q] = ch;
          nxt[kLN + q] = cb;
          nxt[2 * kLN + q] = cc;
          nxt[3 * kLN + q] = split;
          nxt[4 * kLN + q] = split ? widest : -1;
          xmid[q] = a.bcen[o + widest];
        }
      }
      // positions move to their child (next-level index) or retire
      for (int k = tid; k < c; k += kPB) {
        const int jj = sseg[k];
        if (jj < 0) continue;
        sseg[k] = nds[jj] ? 2 * nrk[jj] + (k < nbg[jj] + nlc[jj] ? 0 : 1) : -1;
      }
      __syncthreads();
      int* t = cur;
      cur = nxt;
      nxt = t;
      double* tm = cmid;
      cmid = xmid;
      xmid = tm;
      ncur = 2 * ns;
      ++lev;
    }
#ifdef DFGTB_TREE_DEBUG
    unsigned long long t1_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1_));
    if (tid == 0) printf("TREEDBG subtree %d: %d points, %d local levels, max %d nodes/level, %d equal-key nodes, %.1f us\n", j, c, levels_, maxnodes_, eqn_, (t1_ - t0_) * 1e-3);
#endif
    for (int k = tid; k < c; k += kPB) a.perm[b0 + k] = cache ? gid[sp[k]] : sp[k];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kPB, 1) k_build(const __grid_constant__ BuildArgs a)
{
  cg::grid_group grid = cg::this_grid();
  using BS = cub::BlockScan<int, kPB>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int s_carry;
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int n = a.n, D = a.D;
  const size_t gt = (size_t)bid * kPB + tid, gs = (size_t)G * kPB;
  for (size_t i = gt; i < (size_t)n; i += gs) {
    a.perm[i] = (int)i;
    a.seg[i] = 0;
  }
  for (size_t i = gt; i < (size_t)D; i += gs) {
    a.kmin[i] = ~0ull;
    a.kmax[i] = 0ull;
  }
  if (gt == 0) {
    a.nbeg[0] = 0;
    a.ncnt[0] = n;
    a.npar[0] = -1;
    a.ndep[0] = 0;
  }
  int p0, p1;
  chunk_of(n, bid, G, p0, p1);
  int base = 0, m = 1, level = 0;
  grid.sync();
  const size_t KBUF = (size_t)2 * n * D;  // keys buffer stride (level parity)
  const size_t NBL = (size_t)n + 1;        // per-level node arrays stride (level parity)
  // B: bounds, centroid, widest side, split midpoint (kdtree.cpp:49-78) of the nodes of
  // level `lev`; resets the keys its children will collect.  Runs in the same phase as
  // the previous level's swaps (it only needs bounds, counts and child slots).
  auto decide = [&](int lev, int bs, int mm) {
    for (size_t jj = gt; jj < (size_t)mm; jj += gs) {
      const int j = (int)jj;
      const size_t o = (size_t)(bs + j) * D;
      int widest = 0;
      double width = 0.0;
      const size_t ks = (size_t)(lev == 0 ? j : a.pslot[j]) * D;
      for (int d = 0; d < D; ++d) {
        const double l = dkey_inv(a.kmin[(lev & 1) * KBUF + ks + d]);
        const double h = dkey_inv(a.kmax[(lev & 1) * KBUF + ks + d]);
        a.blo[o + d] = l;
        a.bhi[o + d] = h;
        a.bcen[o + d] = __dmul_rn(0.5, __dadd_rn(l, h));
        const double w = __dadd_rn(h, -l);
        if (d == 0 || w > width) {
          width = w;
          widest = d;
        }
      }
      a.bside[bs + j] = width;
      const int split = a.ncnt[bs + j] > a.leaf;
      if (split) atomicMax(&a.lvlmax[lev], a.ncnt[bs + j]);
      a.dosplit[(lev & 1) * NBL + j] = split;
      a.bsd[bs + j] = split ? widest : -1;
      a.mid[(lev & 1) * NBL + j] = a.bcen[o + widest];
    }
    for (size_t i = gt; i < (size_t)2 * mm * D; i += gs) {  // children's bounds keys
      a.kmin[((lev + 1) & 1) * KBUF + i] = ~0ull;
      a.kmax[((lev + 1) & 1) * KBUF + i] = 0ull;
    }
  };
  // A (root only): exact bounds.  Deeper levels get their bounds from the parent's
  // predicate pass (C) -- the left child is exactly {x_w <= mid} -- or, for one-sided
  // splits, from the median fallback (E).
  for (int i0 = p0; i0 < p1; i0 += kPB) {
    const int i = i0 + tid;
    const int j = i < p1 ? a.seg[i] : -1;
    const int j0 = __shfl_sync(0xffffffffu, j, 0);
    const bool uni = __all_sync(0xffffffffu, j == j0) && j0 >= 0;
    for (int d = 0; d < D; ++d) {
      const unsigned long long k = j >= 0 ? dkey(a.x[(size_t)a.perm[i] * D + d]) : 0ull;
      if (uni) {
        unsigned long long mn = k, mx = k;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
          atomicMin(&a.kmin[(size_t)j0 * D + d], mn);
          atomicMax(&a.kmax[(size_t)j0 * D + d], mx);
        }
      } else if (j >= 0) {
        atomicMin(&a.kmin[(size_t)j * D + d], k);
        atomicMax(&a.kmax[(size_t)j * D + d], k);
      }
    }
  }
  grid.sync();
  decide(0, 0, 1);
  grid.sync();
  bool local = false;
  for (;;) {
    if (gt == 0) a.lvl[1 + level] = base;
    if (a.trace && bid == 0 && tid == 0 && level < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); a.trace[level * 8] = t_; }
    const int* dsp = a.dosplit + (level & 1) * NBL;  // this level's split flags / midpoints
    const double* mdp = a.mid + (level & 1) * NBL;
    if (a.local_S > 0 && level > 0 && __ldcg(&a.lvlmax[level]) <= a.local_S) {
      // every subtree below this level fits one CTA's shared memory: k_build_local builds
      // them there, one subtree per CTA (more, smaller CTAs than this kernel's)
      if (gt == 0) {
        a.loc[0] = base;
        a.loc[1] = m;
        a.loc[2] = level;
      }
      local = true;
      break;
    }
    unsigned long long* cmin = a.kmin + ((level + 1) & 1) * KBUF;  // children's (next level)
    unsigned long long* cmax = a.kmax + ((level + 1) & 1) * KBUF;
    // C: predicate flags and the CTA's chunk scans (positions; splitting level nodes)
    {
      if (tid == 0) s_carry = 0;
      __syncthreads();
      for (int i0 = p0; i0 < p1; i0 += kPB) {
        const int i = i0 + tid;
        int f = 0, js = -1;  // js: the point's child slot 2j + (right) of a splitting node
        const double* xp = nullptr;
        if (i < p1) {
          const int j = a.seg[i];
          if (j >= 0 && dsp[j]) {
            xp = a.x + (size_t)a.perm[i] * D;
            f = xp[a.bsd[base + j]] <= mdp[j] ? 1 : 0;
            js = 2 * j + (f ? 0 : 1);
          }
          a.flag[i] = f;
        }
        // children's bounds: warp-reduced per (node, side) when the warp is one node
        {
          const int jn = js >= 0 ? js >> 1 : -1;
          const int j0 = __shfl_sync(0xffffffffu, jn, 0);
          const bool uni = __all_sync(0xffffffffu, jn == j0) && j0 >= 0;
          for (int d = 0; d < D; ++d) {
            const unsigned long long k = js >= 0 ? dkey(xp[d]) : 0ull;
            if (uni) {
#pragma unroll
              for (int side = 0; side < 2; ++side) {
                const bool mine = (js & 1) == side;
                if (!__any_sync(0xffffffffu, mine)) continue;
                unsigned long long mn = mine ? k : ~0ull, mx = mine ? k : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                  mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                  mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                if (lane == 0) {
                  atomicMin(&cmin[(size_t)(2 * j0 + side) * D + d], mn);
                  atomicMax(&cmax[(size_t)(2 * j0 + side) * D + d], mx);
                }
              }
            } else if (js >= 0) {
              atomicMin(&cmin[(size_t)js * D + d], k);
              atomicMax(&cmax[(size_t)js * D + d], k);
            }
          }
        }
        int ex, agg;
        BS(tmp).ExclusiveSum(f, ex, agg);
        if (i < p1) a.P[i] = s_carry + ex;  // chunk-local exclusive prefix
        __syncthreads();
        if (tid == 0) s_carry += agg;
        __syncthreads();
      }
      if (tid == 0) a.ctot[bid] = s_carry;
      int n0, n1;
      chunk_of(m, bid, G, n0, n1);
      if (tid == 0) s_carry = 0;
      __syncthreads();
      for (int j0 = n0; j0 < n1; j0 += kPB) {
        const int j = j0 + tid;
        const int f = j < n1 ? dsp[j] : 0;
        int ex, agg;
        BS(tmp).ExclusiveSum(f, ex, agg);
        if (j < n1) a.child[j] = s_carry + ex;  // chunk-local rank among splitting nodes
        __syncthreads();
        if (tid == 0) s_carry += agg;
        __syncthreads();
      }
      if (tid == 0) a.ctot[G + bid] = s_carry;
    }
    grid.sync();
    if (a.trace && bid == 0 && tid == 0 && level < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); a.trace[level * 8 + 2] = t_; }
    // D: global prefix P, child BFS ids and the children's records
    int poff = 0, noff = 0, nsplit = 0;
    {
      int v0 = 0, v1 = 0, v2 = 0;
      for (int b = lane; b < G; b += 32) {
        const int t0 = __ldcg(&a.ctot[b]), t1 = __ldcg(&a.ctot[G + b]);
        if (b < bid) {
          v0 += t0;
          v1 += t1;
        }
        v2 += t1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      poff = v0;
      noff = v1;
      nsplit = v2;
    }
    for (int i = p0 + tid; i < p1; i += kPB) a.P[i] += poff;

    if (bid == G - 1 && tid == 0) a.P[n] = poff + __ldcg(&a.ctot[bid]);
    {
      int n0, n1;
      chunk_of(m, bid, G, n0, n1);
      for (int j = n0 + tid; j < n1; j += kPB) {
        const int id = base + j;
        if (dsp[j]) {
          const int c = base + m + 2 * (noff + a.child[j]);
          a.child[j] = c;
          a.pslot[c - (base + m)] = 2 * j;          // next level: left child
          a.pslot[c - (base + m) + 1] = 2 * j + 1;  // right child
          a.nleft[id] = c;
          a.nright[id] = c + 1;
          a.npar[c] = a.npar[c + 1] = id;
          a.ndep[c] = a.ndep[c + 1] = a.ndep[id] + 1;
        } else {
          a.child[j] = -1;
          a.nleft[id] = a.nright[id] = -1;
          a.bsc[id] = 0.0;
        }
      }
    }
    grid.sync();
    if (a.trace && bid == 0 && tid == 0 && level < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); a.trace[level * 8 + 3] = t_; }
    // E: right-block passers register their slots; one-sided splits run the median
    // fallback (kdtree.cpp:85-94) on their own segment (no swaps happen there)
    for (int i = p0 + tid; i < p1; i += kPB) {
      const int j = a.seg[i];
      if (j < 0 || !dsp[j] || !a.flag[i]) continue;
      const int b = a.nbeg[base + j], e = b + a.ncnt[base + j];
      const int L = a.P[e] - a.P[b];
      if (i >= b + L) a.slot[b + (a.P[e] - a.P[i] - 1)] = i;
    }
    {
      int n0, n1;
      chunk_of(m, bid, G, n0, n1);
      for (int j = n0 + tid; j < n1; j += kPB) {
        if (!dsp[j]) continue;
        const int id = base + j;
        const int b = a.nbeg[id], c = a.ncnt[id];
        const int L = a.P[b + c] - a.P[b];
        int l;
        if (L == 0 || L == c) {
          KeyCmp cmp{ a.x, D, a.bsd[id] };
          int* q0 = a.perm + b;
          dev_nth_element(q0, q0 + c / 2, q0 + c, cmp);
          l = c / 2;
          a.bsc[id] = cmp.key(q0[c / 2]);
          // the children are the two halves of the segment: exact bounds by a scan
          for (int side = 0; side < 2; ++side) {
            const int k0 = side ? l : 0, k1 = side ? c : l;
            for (int d = 0; d < D; ++d) {
              unsigned long long mn = ~0ull, mx = 0ull;
              for (int k = k0; k < k1; ++k) {
                const unsigned long long kk = dkey(a.x[(size_t)q0[k] * D + d]);
                mn = min(mn, kk);
                mx = max(mx, kk);
              }
              cmin[(size_t)(2 * j + side) * D + d] = mn;
              cmax[(size_t)(2 * j + side) * D + d] = mx;
            }
          }
        } else {
          l = L;
          a.bsc[id] = mdp[j];
        }
        a.lc[j] = l;
        const int ch = a.child[j];
        a.nbeg[ch] = b;
        a.ncnt[ch] = l;
        a.nbeg[ch + 1] = b + l;
        a.ncnt[ch + 1] = c - l;
      }
    }
    grid.sync();
    if (a.trace && bid == 0 && tid == 0 && level < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); a.trace[level * 8 + 4] = t_; }
    // F: left-block failers swap with their partners; every position learns its
    // next-level node (its own CTA reads it next, in A)
    const int nbase = base + m;
    for (int i = p0 + tid; i < p1; i += kPB) {
      const int j = a.seg[i];
      if (j < 0) continue;
      if (!dsp[j]) {
        a.seg[i] = -1;
        continue;
      }
      const int b = a.nbeg[base + j];
      const int L = a.P[b + a.ncnt[base + j]] - a.P[b];
      if (i < b + L && !a.flag[i]) {
        const int k = (i - b) - (a.P[i] - a.P[b]);
        const int partner = a.slot[b + k];
        const int t = a.perm[i];
        a.perm[i] = a.perm[partner];
        a.perm[partner] = t;
      }
      a.seg[i] = a.child[j] - nbase + (i < b + a.lc[j] ? 0 : 1);
    }
    base = nbase;
    m = 2 * nsplit;
    ++level;
    if (m == 0 || level >= kMaxTreeLevels - 1) break;
    if (gt == 0) *a.kcount = base + m;  // ids the local phase hands out start here
    decide(level, base, m);  // same phase: needs only bounds / counts / slots of level-1
    grid.sync();
    if (a.trace && bid == 0 && tid == 0 && level < 64) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); a.trace[level * 8 + 5] = t_; }
  }
  if (gt == 0 && !local) {
    a.lvl[0] = level;
    a.lvl[1 + level] = base;
    *a.kcount = base;
  }
}

// The CTA-local subtree phase, launched after k_build (which stops at the level where
// every splitting node holds <= local_S points): one kLocalThreads CTA per subtree.
constexpr int kLocalThreads = 512;
__global__ void __launch_bounds__(kLocalThreads) k_build_local(const __grid_constant__ BuildArgs a)
{
  const int m = a.loc[1];
  if (m == 0) return;
  const int base = a.loc[0], level = a.loc[2];
  const size_t NBL = (size_t)a.n + 1;
  using BS = cub::BlockScan<int, kLocalThreads>;
  __shared__ typename BS::TempStorage tmp;
  extern __shared__ __align__(16) unsigned char lsm[];
  local_subtrees<kLocalThreads>(a, tmp, lsm, base, m, level, a.dosplit + (level & 1) * NBL,
                                a.mid + (level & 1) * NBL);
}

}  // namespace

// Preorder renumbering and the preorder device/host arrays, from BFS-indexed arrays.
static void finish_tree(DevTree& t, const double* d_x, int n, int D, int K,
                        const std::vector<int>& h_left, const std::vector<int>& h_right,
                        const std::vector<int>& h_beg, const std::vector<int>& h_cnt,
                        const std::vector<int>& level_off, const double* blo, const double* bhi,
                        const double* bcen, const double* bside, const double* bsc, const int* bsd,
                        const int* d_bleft, const int* d_bright, const int* d_bbeg, const int* d_bcnt,
                        const int* d_bpar, const int* d_bdep, cudaStream_t s,
                        const std::vector<int>* rank = nullptr);

static bool build_tree_persistent(DevTree& t, const double* d_x, int n, int D, int leaf,
                                  cudaStream_t s)
{
  int dev = 0, nsm = 0, per_sm = 0, coop = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // CTA-local subtree phase: subtrees of <= local_S points (kLN nodes per local level
  // bound it by the leaf size), D <= kLMaxD; DFGTB_TREE_LOCAL=0 turns it off
  static const int local_env = std::getenv("DFGTB_TREE_LOCAL") ? std::atoi(std::getenv("DFGTB_TREE_LOCAL")) : -1;
  const int local_cap = local_env >= 0 ? std::min(local_env, kLS) : kLS;
  const int local_S = (local_env == 0 || D > kLMaxD) ? 0 : (int)std::min<long long>(local_cap, (long long)kLN * (leaf + 1) / 2);
  const int lsmem = local_S >= 512 ? local_smem_bytes(D) : 0;  // k_build_local
  if (lsmem) CK(cudaFuncSetAttribute(k_build_local, cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem));
  const int smem = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_build, kPB, smem));
  if (!coop || per_sm < 1) return false;
  // CTAs: 64 for small sets (measured: cheaper grid barriers, enough threads), one
  // per SM from ~256k points; DFGTB_TREE_CTAS overrides (experiments)
  static const int env_g = std::getenv("DFGTB_TREE_CTAS") ? std::atoi(std::getenv("DFGTB_TREE_CTAS")) : 0;
  const int G = env_g > 0 ? std::min(env_g, nsm) : std::min(nsm, std::max(64, ceil_div(n, 4 * kPB)));
  const int maxK = 2 * n;
  DevBuf<double> blo, bhi, bcen, bside, bsc, mid;
  DevBuf<int> bsd, seg, flag, P, slot, nbeg, ncnt, nleft, nright, npar, ndep, dosplit, child, lc,
    ctot, lvl, pslot, lvlmax, kcount;
  DevBuf<unsigned long long> kmin, kmax;
  blo.reserve((size_t)maxK * D);
  bhi.reserve((size_t)maxK * D);
  bcen.reserve((size_t)maxK * D);
  bside.reserve(maxK);
  bsc.reserve(maxK);
  bsd.reserve(maxK);
  for (DevBuf<int>* b : { &nbeg, &ncnt, &nleft, &nright, &npar, &ndep }) b->reserve(maxK);
  for (DevBuf<int>* b : { &seg, &flag, &slot, &child, &lc }) b->reserve((size_t)n + 1);
  dosplit.reserve((size_t)2 * (n + 1));  // two level buffers
  P.reserve((size_t)n + 1);
  mid.reserve((size_t)2 * (n + 1));
  kmin.reserve((size_t)4 * n * D + D);  // two level buffers of 2n*D keys
  kmax.reserve((size_t)4 * n * D + D);
  pslot.reserve((size_t)n + 1);
  ctot.reserve(2 * G);
  lvl.reserve(kMaxTreeLevels + 2);
  t.perm.reserve(n);
  lvlmax.reserve(kMaxTreeLevels);
  kcount.reserve(1);
  CK(cudaMemsetAsync(lvlmax.p, 0, sizeof(int) * kMaxTreeLevels, s));
  BuildArgs a{ d_x, n, D, leaf, t.perm.p, seg.p, flag.p, P.p, slot.p, nbeg.p, ncnt.p, nleft.p,
               nright.p, npar.p, ndep.p, blo.p, bhi.p, bcen.p, bside.p, bsc.p, bsd.p, kmin.p,
               kmax.p, pslot.p, mid.p, dosplit.p, child.p, lc.p, ctot.p, lvl.p };
  a.lvlmax = lvlmax.p;
  a.kcount = kcount.p;
  a.local_S = lsmem ? local_S : 0;
  DevBuf<int> loc;
  loc.reserve(4);
  CK(cudaMemsetAsync(loc.p, 0, sizeof(int) * 4, s));
  a.loc = loc.p;
  static const bool tracing = std::getenv("DFGTB_TRACE") != nullptr;
  DevBuf<unsigned long long> trace;
  if (tracing) {
    trace.reserve(64 * 8);
    CK(cudaMemsetAsync(trace.p, 0, sizeof(unsigned long long) * 64 * 8, s));
    a.trace = trace.p;
  }
  void* kargs[] = { &a };
  const auto c0 = std::chrono::steady_clock::now();
  CK(cudaLaunchCooperativeKernel((void*)k_build, G, kPB, kargs, smem, s));
  CK_LAUNCH();
  if (lsmem) {
    static int lgrid = 0;
    if (!lgrid) {
      int lper = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lper, k_build_local, kLocalThreads, lsmem));
      lgrid = nsm * std::max(1, lper);
    }
    k_build_local<<<lgrid, kLocalThreads, lsmem, s>>>(a);
    CK_LAUNCH();
  }
  if (tracing) {
    std::vector<unsigned long long> tr(64 * 8);
    CK(cudaMemcpyAsync(tr.data(), trace.p, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int L = 0; L < 64 && tr[L * 8]; ++L) {
      std::fprintf(stderr, "DFGTB_TRACE tree level %d (us):", L);
      unsigned long long prev = tr[L * 8];
      for (int k = 1; k < 8; ++k)
        if (tr[L * 8 + k]) {
          std::fprintf(stderr, " p%d %.1f", k, (tr[L * 8 + k] - prev) * 1e-3);
          prev = tr[L * 8 + k];
        }
      if (L + 1 < 64 && tr[L * 8 + 8]) std::fprintf(stderr, " total %.1f", (tr[L * 8 + 8] - tr[L * 8]) * 1e-3);
      std::fprintf(stderr, "\n");
    }
  }
  // Node count and node arrays back in ONE round trip when the count fits the guess (the
  // last tree's count plus a margin, per process): a pinned block of the count and the
  // first `guess` entries of the four arrays; the remainder is fetched only on a miss.
  static std::atomic<int> last_K{ 0 };
  const int guess = std::min(maxK, std::max(1024, last_K.load() + last_K.load() / 8 + 64));
  size_t pin_cap = 4096;  // block sizes in powers of two: the pinned pool reuses them across trees
  while (pin_cap < (size_t)guess) pin_cap *= 2;
  const size_t pin_bytes = sizeof(int) * (4 * pin_cap + 16);
  int* pin = static_cast<int*>(pinned_alloc(pin_bytes));
  struct PinFree {
    int* p;
    size_t b;
    ~PinFree() { pinned_free(p, b); }
  } pin_free{ pin, pin_bytes };
  CK(cudaMemcpyAsync(pin, kcount.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  const int* d_arr[4] = { nleft.p, nright.p, nbeg.p, ncnt.p };
  for (int k = 0; k < 4; ++k)
    CK(cudaMemcpyAsync(pin + 16 + (size_t)k * guess, d_arr[k], sizeof(int) * guess, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int K = pin[0];
  last_K.store(K);
  std::vector<int> h_left(K), h_right(K), h_beg(K), h_cnt(K);
  std::vector<int>* h_arr[4] = { &h_left, &h_right, &h_beg, &h_cnt };
  for (int k = 0; k < 4; ++k)
    std::copy(pin + 16 + (size_t)k * guess, pin + 16 + (size_t)k * guess + std::min(K, guess), h_arr[k]->begin());
  if (K > guess) {
    for (int k = 0; k < 4; ++k)
      CK(cudaMemcpyAsync(h_arr[k]->data() + guess, d_arr[k] + guess, sizeof(int) * (K - guess),
                         cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  // depth of every node (children have larger ids than their parent), the depth-major
  // rank (BFS ids of the global levels keep their order) and the level offsets
  std::vector<int> h_dep(K, 0), cnt_d(1, 0);
  for (int i = 0; i < K; ++i) {
    if ((size_t)h_dep[i] >= cnt_d.size()) cnt_d.resize(h_dep[i] + 1, 0);
    ++cnt_d[h_dep[i]];
    if (h_left[i] >= 0) h_dep[h_left[i]] = h_dep[h_right[i]] = h_dep[i] + 1;
  }
  const int levels = (int)cnt_d.size();
  if (levels >= kMaxTreeLevels - 1) throw CudaError("kd-tree deeper than 255 levels");
  std::vector<int> level_off(levels + 1, 0), rank(K);
  for (int d = 0; d < levels; ++d) level_off[d + 1] = level_off[d] + cnt_d[d];
  {
    std::vector<int> fill(level_off.begin(), level_off.end() - 1);
    for (int i = 0; i < K; ++i) rank[i] = fill[h_dep[i]]++;
  }
  t.n = n;
  t.D = D;
  t.leaf = leaf;
  const auto c1 = std::chrono::steady_clock::now();
  finish_tree(t, d_x, n, D, K, h_left, h_right, h_beg, h_cnt, level_off, blo.p, bhi.p, bcen.p,
              bside.p, bsc.p, bsd.p, nleft.p, nright.p, nbeg.p, ncnt.p, npar.p, ndep.p, s, &rank);
  if (tracing) {
    const auto c2 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "DFGTB_TRACE tree host: build+copies %.1f us, finish %.1f us (G=%d, levels %d, K %d)\n",
                 std::chrono::duration<double, std::micro>(c1 - c0).count(),
                 std::chrono::duration<double, std::micro>(c2 - c1).count(), G, levels, K);
  }
  return true;
}

void build_tree(DevTree& t, const double* d_x, int n, int D, int leaf, cudaStream_t s)
{
  if (leaf < 1) throw InvalidArgument("leaf_threshold must be >= 1");
  if (n < 1 || D < 1) throw InvalidArgument("PointSet requires N >= 1 and D >= 1");
  static const bool host_levels = std::getenv("DFGTB_TREE_HOST_LEVELS") != nullptr;
  if (!host_levels && build_tree_persistent(t, d_x, n, D, leaf, s)) return;
  build_tree_levels(t, d_x, n, D, leaf, s);
}

// Host-driven level loop (fallback when one CTA per SM cannot be co-scheduled).
void build_tree_levels(DevTree& t, const double* d_x, int n, int D, int leaf, cudaStream_t s)
{
  t.n = n;
  t.D = D;
  t.leaf = leaf;
  const int maxK = 2 * n;  // nodes <= 2n - 1

  // BFS-indexed build arrays
  DevBuf<double> blo, bhi, bcen, bside, bsc;
  DevBuf<int> bsd;
  blo.reserve((size_t)maxK * D);
  bhi.reserve((size_t)maxK * D);
  bcen.reserve((size_t)maxK * D);
  bside.reserve(maxK);
  bsc.reserve(maxK);
  bsd.reserve(maxK);

  t.perm.reserve(n);
  k_iota<<<ceil_div(n, 256), 256, 0, s>>>(t.perm.p, n);
  CK_LAUNCH();  // (counts every launch below too)

  DevBuf<int> flag, P, slot;
  flag.reserve((size_t)n + 1);
  P.reserve((size_t)n + 1);
  slot.reserve(n);
  CK(cudaMemsetAsync(flag.p, 0, sizeof(int) * ((size_t)n + 1), s));

  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, flag.p, P.p, n + 1, s);
  DevBuf<unsigned char> scan_tmp;
  scan_tmp.reserve(scan_bytes + 16);

  // host bookkeeping (BFS ids)
  std::vector<int> h_beg{ 0 }, h_cnt{ n }, h_left, h_right, h_par{ -1 }, h_dep{ 0 };
  std::vector<int> level_off{ 0 };
  DevBuf<int> d_nbeg, d_ncnt, d_tnode, d_tstart, d_dosplit, d_sd_lvl, d_lc;
  DevBuf<double> d_mid;
  DevBuf<unsigned long long> d_kmin, d_kmax;

  int base = 0;
  while (base < (int)h_beg.size()) {
    const int m = (int)h_beg.size() - base;
    // tiles
    std::vector<int> tnode, tstart;
    for (int j = 0; j < m; ++j) {
      const int b = h_beg[base + j], c = h_cnt[base + j];
      for (int st = b; st < b + c; st += kTile) {
        tnode.push_back(j);
        tstart.push_back(st);
      }
    }
    const int ntiles = (int)tnode.size();
    d_nbeg.reserve(m);
    d_ncnt.reserve(m);
    d_tnode.reserve(ntiles);
    d_tstart.reserve(ntiles);
    d_dosplit.reserve(m);
    d_sd_lvl.reserve(m);
    d_lc.reserve(m);
    d_mid.reserve(m);
    d_kmin.reserve((size_t)m * D);
    d_kmax.reserve((size_t)m * D);
    CK(cudaMemcpyAsync(d_nbeg.p, h_beg.data() + base, sizeof(int) * m, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_ncnt.p, h_cnt.data() + base, sizeof(int) * m, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_tnode.p, tnode.data(), sizeof(int) * ntiles, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_tstart.p, tstart.data(), sizeof(int) * ntiles, cudaMemcpyHostToDevice, s));

    LevelArgs a{ d_x, D, t.perm.p, d_nbeg.p, d_ncnt.p, d_tnode.p, d_tstart.p, d_kmin.p, d_kmax.p };
    k_bounds_init<<<ceil_div((long long)m * D, 256), 256, 0, s>>>(d_kmin.p, d_kmax.p, m * D);
    CK_LAUNCH();
    k_bounds_tiles<<<ntiles, kThreads, 0, s>>>(a);
    CK_LAUNCH();
    k_decide<<<ceil_div(m, 128), 128, 0, s>>>(a, m, leaf, base, blo.p, bhi.p, bcen.p, bside.p,
                                              bsd.p, d_mid.p, d_dosplit.p);
    CK_LAUNCH();
    // split_dim per level node (for flags) = bsd[base + j]
    CK(cudaMemcpyAsync(d_sd_lvl.p, bsd.p + base, sizeof(int) * m, cudaMemcpyDeviceToDevice, s));
    k_flags<<<ntiles, kThreads, 0, s>>>(a, d_dosplit.p, d_sd_lvl.p, d_mid.p, flag.p);
    CK_LAUNCH();
    cub::DeviceScan::ExclusiveSum(scan_tmp.p, scan_bytes, flag.p, P.p, n + 1, s);
    k_slots<<<ntiles, kThreads, 0, s>>>(a, d_dosplit.p, flag.p, P.p, slot.p);
    CK_LAUNCH();
    k_swap<<<ntiles, kThreads, 0, s>>>(a, d_dosplit.p, flag.p, P.p, slot.p);
    CK_LAUNCH();
    k_finish_split<<<ceil_div(m, 64), 64, 0, s>>>(a, m, base, d_dosplit.p, d_sd_lvl.p, d_mid.p,
                                                  P.p, d_lc.p, bsc.p);
    CK_LAUNCH();
    // reset flags of this level's splitting segments (non-split positions stay 0)
    CK(cudaMemsetAsync(flag.p, 0, sizeof(int) * ((size_t)n + 1), s));

    std::vector<int> lc(m), ds(m);
    CK(cudaMemcpyAsync(lc.data(), d_lc.p, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ds.data(), d_dosplit.p, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));

    const int next_base = (int)h_beg.size();
    h_left.resize(h_beg.size(), -1);
    h_right.resize(h_beg.size(), -1);
    for (int j = 0; j < m; ++j) {
      if (!ds[j]) continue;
      const int id = base + j;
      const int b = h_beg[id], c = h_cnt[id];
      h_left[id] = (int)h_beg.size();
      h_beg.push_back(b);
      h_cnt.push_back(lc[j]);
      h_par.push_back(id);
      h_dep.push_back(h_dep[id] + 1);
      h_right[id] = (int)h_beg.size();
      h_beg.push_back(b + lc[j]);
      h_cnt.push_back(c - lc[j]);
      h_par.push_back(id);
      h_dep.push_back(h_dep[id] + 1);
    }
    base = next_base;
    level_off.push_back(base);
  }
  const int K = (int)h_beg.size();
  h_left.resize(K, -1);
  h_right.resize(K, -1);
  DevBuf<int> d_bleft, d_bright, d_bbeg, d_bcnt, d_bpar, d_bdep;
  auto up = [&](DevBuf<int>& b, const std::vector<int>& v) {
    b.reserve(v.size());
    CK(cudaMemcpyAsync(b.p, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice, s));
  };
  up(d_bleft, h_left);
  up(d_bright, h_right);
  up(d_bbeg, h_beg);
  up(d_bcnt, h_cnt);
  up(d_bpar, h_par);
  up(d_bdep, h_dep);
  finish_tree(t, d_x, n, D, K, h_left, h_right, h_beg, h_cnt, level_off, blo.p, bhi.p, bcen.p,
              bside.p, bsc.p, bsd.p, d_bleft.p, d_bright.p, d_bbeg.p, d_bcnt.p, d_bpar.p, d_bdep.p,
              s);
}

static void finish_tree(DevTree& t, const double* d_x, int n, int D, int K,
                        const std::vector<int>& h_left, const std::vector<int>& h_right,
                        const std::vector<int>& h_beg, const std::vector<int>& h_cnt,
                        const std::vector<int>& level_off, const double* blo, const double* bhi,
                        const double* bcen, const double* bside, const double* bsc, const int* bsd,
                        const int* d_bleft, const int* d_bright, const int* d_bbeg, const int* d_bcnt,
                        const int* d_bpar, const int* d_bdep, cudaStream_t s,
                        const std::vector<int>* rank)
{
  t.nodes = K;
  t.height = (int)level_off.size() - 1;
  t.depth_off = level_off;

  // preorder numbering: left = parent + 1, right = parent + 1 + size(left)
  std::vector<int> sub(K, 1);
  for (int i = K - 1; i >= 0; --i)
    if (h_left[i] >= 0) sub[i] = 1 + sub[h_left[i]] + sub[h_right[i]];
  // (kept in the tree: the source of an asynchronous upload must outlive this call)
  std::vector<int>& bfs2pre = t.h_pre;
  bfs2pre.assign(K, 0);
  bfs2pre[0] = 0;
  for (int i = 0; i < K; ++i)
    if (h_left[i] >= 0) {
      bfs2pre[h_left[i]] = bfs2pre[i] + 1;
      bfs2pre[h_right[i]] = bfs2pre[i] + 1 + sub[h_left[i]];
    }
  DevBuf<int> d_map, d_rank;
  d_map.reserve(K);
  CK(cudaMemcpyAsync(d_map.p, bfs2pre.data(), sizeof(int) * K, cudaMemcpyHostToDevice, s));
  if (rank) {
    t.h_rank = *rank;
    d_rank.reserve(K);
    CK(cudaMemcpyAsync(d_rank.p, t.h_rank.data(), sizeof(int) * K, cudaMemcpyHostToDevice, s));
  }
  t.lo.reserve((size_t)K * D);
  t.hi.reserve((size_t)K * D);
  t.centroid.reserve((size_t)K * D);
  t.max_side.reserve(K);
  t.split_coord.reserve(K);
  t.split_dim.reserve(K);
  t.left.reserve(K);
  t.right.reserve(K);
  t.begin.reserve(K);
  t.count.reserve(K);
  t.parent.reserve(K);
  t.depth.reserve(K);
  t.by_depth.reserve(K);
  k_to_preorder<<<ceil_div(K, 256), 256, 0, s>>>(
    K, D, d_map.p, blo, bhi, bcen, bside, bsc, bsd, d_bleft, d_bright, d_bbeg, d_bcnt, d_bpar,
    d_bdep, t.lo.p, t.hi.p, t.centroid.p, t.max_side.p, t.split_coord.p, t.split_dim.p, t.left.p,
    t.right.p, t.begin.p, t.count.p, t.parent.p, t.depth.p, t.by_depth.p, rank ? d_rank.p : nullptr);
  CK_LAUNCH();
  t.anc.reserve((size_t)K * kMaxAnc);
  k_ancestors<<<ceil_div(K, 256), 256, 0, s>>>(K, t.parent.p, t.depth.p, t.anc.p);
  CK_LAUNCH();
  t.xs.reserve((size_t)n * D);
  k_gather_points<<<ceil_div((long long)n * D, 256), 256, 0, s>>>(d_x, t.perm.p, n, D, t.xs.p);
  CK_LAUNCH();
  t.h_count.assign(K, 0);
  t.h_left.assign(K, -1);
  t.h_begin.assign(K, 0);
  for (int i = 0; i < K; ++i) {
    t.h_count[bfs2pre[i]] = h_cnt[i];
    t.h_begin[bfs2pre[i]] = h_beg[i];
    t.h_left[bfs2pre[i]] = h_left[i] < 0 ? -1 : bfs2pre[h_left[i]];
  }
  // no host wait: everything above is ordered on `s`; the temporaries of the build go to
  // the allocator's pending list, which is only reused after a device synchronisation
}

}  // namespace dfgtb
