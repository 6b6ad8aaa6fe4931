/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference DFGT path.
 *
 * This file is the checker used by tests/ (and the "port" CPU baseline in
 * bench.py); it is never linked into the product library.  Each function names
 * the reference file:line it restates (paths under /root/reference/proj/src).
 * The tree build restates libstdc++ 13's std::partition / std::nth_element
 * (bits/stl_algo.h:1469-1495, 85-102, 1631-1640, 1812-1900, 1957-1979;
 * bits/stl_heap.h:135-150, 224-265, 340-360), which the reference calls at
 * kdtree.cpp:80-94 and which therefore decide the point permutation.
 *
 * Parity pins: tests/test_oracle.py (reference unit-test goldens + the compiled
 * reference in oracle/_ref + fixtures in tests/golden/).
 */
#include "dfgt_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ dataset */

double orc_gaussian_normalizer(size_t dim, double h)
{ /* dataset.cpp:32-39 */
  const double two_pi = 6.283185307179586476925286766559;
  return pow(two_pi * h * h, 0.5 * (double)dim);
}

static double sqdist(const double* a, const double* b, size_t d)
{ /* dataset.cpp:41-49: sum of squared differences in dimension order */
  double s = 0.0;
  for (size_t k = 0; k < d; ++k) {
    const double t = a[k] - b[k];
    s += t * t;
  }
  return s;
}

void orc_naive_kde(const double* q, size_t nq, const double* r, size_t nr, size_t d, double h,
                   double* out)
{ /* engine.cpp:22-36, kernel dataset.hpp:55 / dataset.cpp:23-30 */
  const double scale = -1.0 / (2.0 * h * h);
  for (size_t i = 0; i < nq; ++i) {
    double g = 0.0;
    for (size_t j = 0; j < nr; ++j) g += exp(scale * sqdist(q + i * d, r + j * d, d));
    out[i] = g;
  }
}

void orc_box_bounds_sq(const double* alo, const double* ahi, const double* blo,
                       const double* bhi, size_t d, double* lo_sq, double* hi_sq)
{ /* kdtree.cpp:122-141 */
  double lo = 0.0, hi = 0.0;
  for (size_t k = 0; k < d; ++k) {
    const double g1 = blo[k] - ahi[k];
    const double g2 = alo[k] - bhi[k];
    const double l = 0.5 * (g1 + fabs(g1) + g2 + fabs(g2));
    lo += l * l;
    const double u1 = bhi[k] - alo[k], u2 = ahi[k] - blo[k];
    const double u = u1 > u2 ? u1 : u2; /* std::max returns the first on ties */
    hi += u * u;
  }
  *lo_sq = lo;
  *hi_sq = hi;
}

/* ------------------------------------------------------------------- kdtree */

typedef struct {
  const double* x;
  size_t d;
  int dim; /* comparison coordinate */
} key_ctx;

static inline double key(const key_ctx* c, int idx) { return c->x[(size_t)idx * c->d + c->dim]; }
static inline int less_idx(const key_ctx* c, int a, int b) { return key(c, a) < key(c, b); }
static inline void swp(int* a, int* b)
{
  int t = *a;
  *a = *b;
  *b = t;
}

/* std::__partition, bidirectional-iterator form (stl_algo.h:1469-1495) */
static int* part_le(int* first, int* last, const key_ctx* c, double mid)
{
  for (;;) {
    for (;;) {
      if (first == last) return first;
      if (key(c, *first) <= mid) ++first;
      else break;
    }
    --last;
    for (;;) {
      if (first == last) return first;
      if (!(key(c, *last) <= mid)) --last;
      else break;
    }
    swp(first, last);
    ++first;
  }
}

/* stl_algo.h:85-102 */
static void median_to_first(int* res, int* a, int* b, int* cc, const key_ctx* c)
{
  if (less_idx(c, *a, *b)) {
    if (less_idx(c, *b, *cc)) swp(res, b);
    else if (less_idx(c, *a, *cc)) swp(res, cc);
    else swp(res, a);
  } else if (less_idx(c, *a, *cc)) swp(res, a);
  else if (less_idx(c, *b, *cc)) swp(res, cc);
  else swp(res, b);
}

/* stl_algo.h:1871-1900 */
static int* unguarded_partition(int* first, int* last, int* pivot, const key_ctx* c)
{
  for (;;) {
    while (less_idx(c, *first, *pivot)) ++first;
    --last;
    while (less_idx(c, *pivot, *last)) --last;
    if (!(first < last)) return first;
    swp(first, last);
    ++first;
  }
}

static int* unguarded_partition_pivot(int* first, int* last, const key_ctx* c)
{
  int* mid = first + (last - first) / 2;
  median_to_first(first, first + 1, mid, last - 1, c);
  return unguarded_partition(first + 1, last, first, c);
}

/* stl_algo.h:1812-1840 */
static void insertion_sort(int* first, int* last, const key_ctx* c)
{
  if (first == last) return;
  for (int* i = first + 1; i != last; ++i) {
    if (less_idx(c, *i, *first)) {
      int v = *i;
      memmove(first + 1, first, (size_t)(i - first) * sizeof(int));
      *first = v;
    } else {
      int v = *i;
      int* l = i;
      int* nx = i - 1;
      while (less_idx(c, v, *nx)) {
        *l = *nx;
        l = nx;
        --nx;
      }
      *l = v;
    }
  }
}

/* stl_heap.h:135-150 */
static void push_heap(int* first, long hole, long top, int v, const key_ctx* c)
{
  long parent = (hole - 1) / 2;
  while (hole > top && less_idx(c, first[parent], v)) {
    first[hole] = first[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  first[hole] = v;
}

/* stl_heap.h:224-250 */
static void adjust_heap(int* first, long hole, long len, int v, const key_ctx* c)
{
  const long top = hole;
  long second = hole;
  while (second < (len - 1) / 2) {
    second = 2 * (second + 1);
    if (less_idx(c, first[second], first[second - 1])) second--;
    first[hole] = first[second];
    hole = second;
  }
  if ((len & 1) == 0 && second == (len - 2) / 2) {
    second = 2 * (second + 1);
    first[hole] = first[second - 1];
    hole = second - 1;
  }
  push_heap(first, hole, top, v, c);
}

/* stl_algo.h:1631-1640 with stl_heap.h:254-265 and 340-360 */
static void heap_select(int* first, int* middle, int* last, const key_ctx* c)
{
  const long len = middle - first;
  if (len >= 2) {
    long parent = (len - 2) / 2;
    for (;;) {
      adjust_heap(first, parent, len, first[parent], c);
      if (parent == 0) break;
      parent--;
    }
  }
  for (int* i = middle; i < last; ++i) {
    if (less_idx(c, *i, *first)) {
      int v = *i;
      *i = *first;
      adjust_heap(first, 0, len, v, c);
    }
  }
}

static int lg2(long n)
{
  int k = 0;
  while (n > 1) {
    n >>= 1;
    ++k;
  }
  return k;
}

/* std::nth_element -> __introselect (stl_algo.h:1957-1979, 4773-4791) */
static void nth_element(int* first, int* nth, int* last, const key_ctx* c)
{
  if (first == last || nth == last) return;
  long depth = 2L * lg2(last - first);
  while (last - first > 3) {
    if (depth == 0) {
      heap_select(first, nth + 1, last, c);
      swp(first, nth);
      return;
    }
    --depth;
    int* cut = unguarded_partition_pivot(first, last, c);
    if (cut <= nth) first = cut;
    else last = cut;
  }
  insertion_sort(first, last, c);
}

typedef struct {
  const double* x;
  size_t n, d;
  int leaf;
  orc_tree* t;
  int nodes;
} build_ctx;

static int build_node(build_ctx* b, int64_t begin, int count)
{ /* kdtree.cpp:36-105: preorder node ids, bounds over owned points, widest side
     (first maximum), midpoint split via std::partition, median fallback. */
  orc_tree* t = b->t;
  const size_t d = b->d;
  const int node = b->nodes++;
  t->begin[node] = begin;
  t->count[node] = count;
  t->left[node] = -1;
  t->right[node] = -1;
  t->split_dim[node] = -1;
  t->split_coord[node] = 0.0;
  double* lo = t->lo + (size_t)node * d;
  double* hi = t->hi + (size_t)node * d;
  for (size_t k = 0; k < d; ++k) {
    double l = b->x[(size_t)t->perm[begin] * d + k], h = l;
    for (int i = 1; i < count; ++i) {
      const double v = b->x[(size_t)t->perm[begin + i] * d + k];
      l = v < l ? v : l; /* std::min(l, v) keeps l unless v < l */
      h = h < v ? v : h; /* std::max(h, v) keeps h unless h < v */
    }
    lo[k] = l;
    hi[k] = h;
    t->centroid[(size_t)node * d + k] = 0.5 * (l + h);
  }
  int widest = 0;
  double width = hi[0] - lo[0];
  for (size_t k = 1; k < d; ++k) {
    const double w = hi[k] - lo[k];
    if (w > width) {
      width = w;
      widest = (int)k;
    }
  }
  t->max_side[node] = width;
  if (count <= b->leaf) return node;

  const double mid = 0.5 * (lo[widest] + hi[widest]);
  key_ctx c = { b->x, d, widest };
  int* p0 = t->perm + begin;
  int* split = part_le(p0, p0 + count, &c, mid);
  long left_count = split - p0;
  double split_coord = mid;
  if (left_count == 0 || left_count == count) {
    int* m = p0 + count / 2;
    nth_element(p0, m, p0 + count, &c);
    left_count = count / 2;
    split_coord = key(&c, *m);
  }
  t->split_dim[node] = widest;
  t->split_coord[node] = split_coord;
  t->left[node] = build_node(b, begin, (int)left_count);
  t->right[node] = build_node(b, begin + left_count, count - (int)left_count);
  return node;
}

int orc_tree_build(const double* x, size_t n, size_t d, int leaf, orc_tree* t)
{
  if (leaf < 1 || n == 0) return -1;
  for (size_t i = 0; i < n; ++i) t->perm[i] = (int)i;
  build_ctx b = { x, n, d, leaf, t, 0 };
  build_node(&b, 0, (int)n);
  return b.nodes;
}

/* --------------------------------------------------------------- truncation */

static double binomial(int n, int k)
{ /* truncation.cpp:11-18 */
  double b = 1.0;
  for (int i = 1; i <= k; ++i) b *= (double)(n - k + i) / (double)i;
  return b;
}

static double sqrt_factorial(int p)
{ /* truncation.cpp:20-27 */
  double f = 1.0;
  for (int k = 2; k <= p; ++k) f *= k;
  return sqrt(f);
}

static double ipow(double x, int n)
{
  double r = 1.0;
  for (int i = 0; i < n; ++i) r *= x;
  return r;
}

static double bound_sum(double count, double s, int dpow, double a, double b, int dim)
{ /* truncation.cpp:40-54 (log-space fallback when the prefactor overflows) */
  double sum = 0.0;
  for (int k = 0; k < dim; ++k) sum += binomial(dim, k) * ipow(a, k) * ipow(b, dim - k);
  const double pre = count / ipow(1.0 - s, dim * dpow);
  double bound = pre * sum;
  if (!isfinite(bound) && count > 0.0 && sum > 0.0)
    bound = exp(log(count) - (double)(dim * dpow) * log1p(-s) + log(sum));
  return bound;
}

double orc_farfield_error_bound(double count, double r, int p, int dim)
{ /* truncation.cpp:58-65 (local_error_bound is the same formula, :67-70) */
  if (count <= 0.0) return 0.0;
  const double rp = ipow(r, p);
  return bound_sum(count, r, 1, 1.0 - rp, rp / sqrt_factorial(p), dim);
}

double orc_f2l_error_bound(double count, double r, int p, int dim)
{ /* truncation.cpp:72-81 */
  if (count <= 0.0) return 0.0;
  const double s = 2.0 * r, sp = ipow(s, p);
  return bound_sum(count, s, 2, (1.0 - sp) * (1.0 - sp), sp * (2.0 - sp) / sqrt_factorial(p),
                   dim);
}

/* least_order (truncation.cpp:85-94) for the three methods (:98-128); 0 = none */
static int order_ff(double ratio, double count, double tau, int p_max, int dim)
{
  if (ratio >= 1.0) return 0;
  for (int p = 1; p <= p_max; ++p)
    if (orc_farfield_error_bound(count, ratio, p, dim) <= tau) return p;
  return 0;
}

static int order_f2l(double ratio, double count, double tau, int p_max, int dim)
{
  if (ratio >= 0.5) return 0;
  for (int p = 1; p <= p_max; ++p)
    if (orc_f2l_error_bound(count, ratio, p, dim) <= tau) return p;
  return 0;
}

void orc_choose_best_method(double nq, double nr, double side_q, double side_r, double h,
                            double tau, int p_max, int dim, int cost_model, int* kind,
                            int* order)
{ /* truncation.cpp:130-166 */
  const int pf = order_ff(side_r / (2.0 * h), nr, tau, p_max, dim);
  const int pd = order_ff(side_q / (2.0 * h), nr, tau, p_max, dim);
  /* std::max(a, b) == (a < b ? b : a) */
  const int pt = order_f2l((side_q < side_r ? side_r : side_q) / (4.0 * h), nr, tau, p_max, dim);
  const double D = (double)dim;
  double cf = INFINITY, cd = INFINITY, ct = INFINITY;
  if (cost_model == 0) {
    if (pf) cf = nq * pow(D, (double)(pf + 1));
    if (pd) cd = nr * pow(D, (double)(pd + 1));
    if (pt) ct = pow(D, 2.0 * pt + 1);
  } else {
    if (pf) cf = nq * pow((double)pf, D);
    if (pd) cd = nr * pow((double)pd, D);
    if (pt) ct = D * pow((double)pt, 2.0 * D);
  }
  const double ce = D * nq * nr;
  const double m1 = cd < cf ? cd : cf, m2 = ce < ct ? ce : ct;
  const double best = m2 < m1 ? m2 : m1;
  if (cf == best) { *kind = 1; *order = pf; }
  else if (cd == best) { *kind = 2; *order = pd; }
  else if (ct == best) { *kind = 3; *order = pt; }
  else { *kind = 0; *order = 0; }
}

int orc_default_p_max(int dim)
{ /* truncation.cpp:168-186 */
  static const int tab[6] = { 0, 8, 6, 4, 2, 2 };
  return dim >= 1 && dim <= 5 ? tab[dim] : 1;
}

/* ------------------------------------------------------------------- series */

typedef struct {
  int dim, pmax, size;
  int* pos;      /* term -> storage position */
  int* parent;   /* term -> parent term */
  int* pdim;     /* term -> grown coordinate */
  int* degree;   /* term -> |alpha| */
  double* invf;  /* term -> 1/alpha! */
  unsigned char* dig;  /* term*dim digits, dim 0 most significant */
  double* fact_pos;    /* position -> alpha! */
  double* invf_pos;    /* position -> 1/alpha! */
  double *expn, *contrib, *scaled, *H;
} geo;

static int block(const geo* g, int p)
{
  int s = 1;
  for (int k = 0; k < g->dim; ++k) s *= p;
  return s;
}

static void geo_init(geo* g, int dim, int pmax)
{ /* series.cpp:61-154: terms ordered by (max digit, position), i.e. a stable
     sort of positions by ring; parent = first nonzero digit decremented. */
  g->dim = dim;
  g->pmax = pmax;
  int T = 1;
  for (int k = 0; k < dim; ++k) T *= pmax;
  g->size = T;
  g->pos = malloc(sizeof(int) * T);
  g->parent = malloc(sizeof(int) * T);
  g->pdim = malloc(sizeof(int) * T);
  g->degree = malloc(sizeof(int) * T);
  g->invf = malloc(sizeof(double) * T);
  g->dig = malloc((size_t)T * dim);
  g->fact_pos = malloc(sizeof(double) * T);
  g->invf_pos = malloc(sizeof(double) * T);
  g->expn = calloc(T, sizeof(double));
  g->contrib = calloc(T, sizeof(double));
  g->scaled = calloc(dim, sizeof(double));
  g->H = calloc((size_t)dim * (2 * pmax), sizeof(double));
  int* ring = malloc(sizeof(int) * T);
  int* order_of_pos = malloc(sizeof(int) * T);
  double fac[16];
  fac[0] = 1.0;
  for (int k = 1; k < 16; ++k) fac[k] = fac[k - 1] * k;
  for (int p = 0; p < T; ++p) {
    int rest = p, mx = 0;
    double f = 1.0;
    for (int k = 0; k < dim; ++k) {
      const int dg = rest % pmax;
      rest /= pmax;
      if (dg > mx) mx = dg;
      f *= fac[dg];
    }
    ring[p] = mx;
    g->fact_pos[p] = f;
    g->invf_pos[p] = 1.0 / f;
  }
  int i = 0;
  for (int rg = 0; rg < pmax; ++rg)
    for (int p = 0; p < T; ++p)
      if (ring[p] == rg) {
        order_of_pos[p] = i;
        g->pos[i++] = p;
      }
  for (i = 0; i < T; ++i) {
    const int p = g->pos[i];
    unsigned char* dg = g->dig + (size_t)i * dim;
    int rest = p, deg = 0;
    for (int k = dim - 1; k >= 0; --k) {
      dg[k] = (unsigned char)(rest % pmax);
      rest /= pmax;
      deg += dg[k];
    }
    g->degree[i] = deg;
    g->invf[i] = g->invf_pos[p];
    if (deg == 0) {
      g->parent[i] = -1;
      g->pdim[i] = -1;
    } else {
      int j = 0;
      while (dg[j] == 0) ++j;
      int stride = 1;
      for (int k = j + 1; k < dim; ++k) stride *= pmax;
      g->parent[i] = order_of_pos[p - stride];
      g->pdim[i] = j;
    }
  }
  free(ring);
  free(order_of_pos);
}

static void geo_free(geo* g)
{
  free(g->pos); free(g->parent); free(g->pdim); free(g->degree); free(g->invf);
  free(g->dig); free(g->fact_pos); free(g->invf_pos); free(g->expn); free(g->contrib);
  free(g->scaled); free(g->H);
}

static void scale_off(const geo* g, const double* a, const double* b, double h)
{ /* series.cpp:208-217 */
  const double s = 1.0 / (h * 1.4142135623730951);
  for (int k = 0; k < g->dim; ++k) g->scaled[k] = (a[k] - b[k]) * s;
}

static void expand(const geo* g, int order, double* out)
{ /* series.cpp:222-232 */
  const int n = block(g, order);
  out[g->pos[0]] = 1.0;
  for (int i = 1; i < n; ++i)
    out[g->pos[i]] = out[g->pos[g->parent[i]]] * g->scaled[g->pdim[i]];
}

static void derivs(const geo* g, int orders)
{ /* series.cpp:163-177 */
  const int st = 2 * g->pmax;
  for (int k = 0; k < g->dim; ++k) {
    double* h = g->H + (size_t)k * st;
    const double t = g->scaled[k];
    h[0] = exp(-t * t);
    if (orders > 1) {
      h[1] = 2.0 * t * h[0];
      for (int j = 1; j + 1 < orders; ++j) h[j + 1] = 2.0 * t * h[j] - 2.0 * j * h[j - 1];
    }
  }
}

static double herm(const geo* g, const unsigned char* a)
{ /* series.cpp:188-195 */
  const int st = 2 * g->pmax;
  double f = 1.0;
  for (int k = 0; k < g->dim; ++k) f *= g->H[(size_t)k * st + a[k]];
  return f;
}

static double sgn(int deg) { return (deg & 1) ? -1.0 : 1.0; }

static void moments_acc(const geo* g, const double* x, size_t d, const int* idx, size_t n,
                        const double* c, double h, double* M)
{ /* series.cpp:238-254 */
  for (size_t r = 0; r < n; ++r) {
    scale_off(g, x + (size_t)(idx ? idx[r] : (int)r) * d, c, h);
    expand(g, g->pmax, g->expn);
    for (int i = 0; i < g->size; ++i) M[g->pos[i]] += g->expn[g->pos[i]];
  }
  for (int i = 0; i < g->size; ++i) M[g->pos[i]] *= g->invf[i];
}

static void f2f(const geo* g, const double* src, const double* sc, const double* dc, double h,
                double* dst)
{ /* series.cpp:256-287 */
  scale_off(g, sc, dc, h);
  expand(g, g->pmax, g->expn);
  for (int i = 0; i < g->size; ++i) {
    const unsigned char* gm = g->dig + (size_t)i * g->dim;
    double acc = 0.0;
    for (int j = 0; j < g->size; ++j) {
      const unsigned char* al = g->dig + (size_t)j * g->dim;
      int dp = 0, ok = 1;
      for (int k = 0; k < g->dim; ++k) {
        const int df = (int)gm[k] - (int)al[k];
        if (df < 0) { ok = 0; break; }
        dp = dp * g->pmax + df;
      }
      if (ok) acc += g->invf_pos[dp] * src[g->pos[j]] * g->expn[dp];
    }
    dst[g->pos[i]] += acc;
  }
}

static double eval_ff(const geo* g, const double* M, const double* c, const double* q, double h,
                      int order)
{ /* series.cpp:289-303 */
  scale_off(g, q, c, h);
  derivs(g, order);
  const int n = block(g, order);
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += M[g->pos[i]] * herm(g, g->dig + (size_t)i * g->dim);
  return s;
}

static void direct_local(const geo* g, const double* x, size_t d, const int* idx, size_t n,
                         const double* c, double h, int order, double* L)
{ /* series.cpp:305-326 */
  const int nt = block(g, order);
  for (int i = 0; i < nt; ++i) g->contrib[g->pos[i]] = 0.0;
  for (size_t r = 0; r < n; ++r) {
    scale_off(g, c, x + (size_t)(idx ? idx[r] : (int)r) * d, h);
    derivs(g, order);
    for (int i = 0; i < nt; ++i) g->contrib[g->pos[i]] += herm(g, g->dig + (size_t)i * g->dim);
  }
  for (int i = 0; i < nt; ++i)
    L[g->pos[i]] += sgn(g->degree[i]) * g->invf[i] * g->contrib[g->pos[i]];
}

static void f2l(const geo* g, const double* M, const double* sc, const double* dc, double h,
                int order, double* L)
{ /* series.cpp:328-353 */
  scale_off(g, dc, sc, h);
  derivs(g, 2 * order - 1);
  const int n = block(g, order), st = 2 * g->pmax;
  for (int i = 0; i < n; ++i) {
    const unsigned char* be = g->dig + (size_t)i * g->dim;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const unsigned char* al = g->dig + (size_t)j * g->dim;
      double f = 1.0;
      for (int k = 0; k < g->dim; ++k) f *= g->H[(size_t)k * st + al[k] + be[k]];
      acc += M[g->pos[j]] * f;
    }
    L[g->pos[i]] += sgn(g->degree[i]) * g->invf[i] * acc;
  }
}

static void l2l(const geo* g, const double* src, const double* sc, const double* dc, double h,
                int order, double* dst)
{ /* series.cpp:355-391 */
  scale_off(g, dc, sc, h);
  expand(g, order, g->expn);
  const int n = block(g, order);
  for (int i = 0; i < n; ++i) {
    const unsigned char* al = g->dig + (size_t)i * g->dim;
    const double ifa = g->invf[i];
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const unsigned char* be = g->dig + (size_t)j * g->dim;
      int dp = 0, ok = 1;
      for (int k = 0; k < g->dim; ++k) {
        const int df = (int)be[k] - (int)al[k];
        if (df < 0) { ok = 0; break; }
        dp = dp * g->pmax + df;
      }
      if (ok) {
        const double binom = g->fact_pos[g->pos[j]] * ifa * g->invf_pos[dp];
        acc += binom * src[g->pos[j]] * g->expn[dp];
      }
    }
    dst[g->pos[i]] += acc;
  }
}

static double eval_loc(const geo* g, const double* L, const double* c, const double* q,
                       double h, int order)
{ /* series.cpp:393-407 */
  scale_off(g, q, c, h);
  expand(g, order, g->expn);
  const int n = block(g, order);
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += L[g->pos[i]] * g->expn[g->pos[i]];
  return s;
}

/* public wrappers over the series primitives (one-shot geometry each call) */
int orc_series_table_size(int dim, int p_max)
{
  int T = 1;
  for (int k = 0; k < dim; ++k) T *= p_max;
  return T;
}

void orc_series_terms(int dim, int p_max, int* pos, int* parent, int* pdim, int* degree,
                      double* invf)
{
  geo g;
  geo_init(&g, dim, p_max);
  for (int i = 0; i < g.size; ++i) {
    pos[i] = g.pos[i];
    parent[i] = g.parent[i];
    pdim[i] = g.pdim[i];
    degree[i] = g.degree[i];
    invf[i] = g.invf[i];
  }
  geo_free(&g);
}

void orc_series_moments(int dim, int p_max, const double* pts, size_t n, const double* center,
                        double h, double* M)
{
  geo g;
  geo_init(&g, dim, p_max);
  moments_acc(&g, pts, (size_t)dim, NULL, n, center, h, M);
  geo_free(&g);
}

void orc_series_f2f(int dim, int p_max, const double* src, const double* sc, const double* dc,
                    double h, double* dst)
{
  geo g;
  geo_init(&g, dim, p_max);
  f2f(&g, src, sc, dc, h, dst);
  geo_free(&g);
}

double orc_series_eval_farfield(int dim, int p_max, const double* M, const double* c,
                                const double* q, double h, int order)
{
  geo g;
  geo_init(&g, dim, p_max);
  const double v = eval_ff(&g, M, c, q, h, order);
  geo_free(&g);
  return v;
}

void orc_series_direct_local(int dim, int p_max, const double* pts, size_t n,
                             const double* c, double h, int order, double* L)
{
  geo g;
  geo_init(&g, dim, p_max);
  direct_local(&g, pts, (size_t)dim, NULL, n, c, h, order, L);
  geo_free(&g);
}

void orc_series_f2l(int dim, int p_max, const double* M, const double* sc, const double* dc,
                    double h, int order, double* L)
{
  geo g;
  geo_init(&g, dim, p_max);
  f2l(&g, M, sc, dc, h, order, L);
  geo_free(&g);
}

void orc_series_l2l(int dim, int p_max, const double* src, const double* sc, const double* dc,
                    double h, int order, double* dst)
{
  geo g;
  geo_init(&g, dim, p_max);
  l2l(&g, src, sc, dc, h, order, dst);
  geo_free(&g);
}

double orc_series_eval_local(int dim, int p_max, const double* L, const double* c,
                             const double* q, double h, int order)
{
  geo g;
  geo_init(&g, dim, p_max);
  const double v = eval_loc(&g, L, c, q, h, order);
  geo_free(&g);
  return v;
}

/* ------------------------------------------------------------------- engine */

typedef struct {
  const double *qx, *rx;
  size_t d;
  const orc_tree *qt, *rt;
  geo* g;
  const double* M; /* ref moments, node-major */
  double h, scale, eps, nref_total;
  int series, cost_model;
  double *q_lo, *q_up, *s_ex, *s_ff, *s_loc;
  double *n_lo, *n_up, *n_dlo, *n_dup, *L;
  int* Lord;
  uint64_t st[7];
} trav;

static double kval(const trav* T, double d2) { return exp(T->scale * d2); }
static double* loc_of(trav* T, int n) { return T->L + (size_t)n * T->g->size; }

static void base_case(trav* T, int qn, int rn)
{ /* engine.cpp:239-269 */
  const orc_tree *qt = T->qt, *rt = T->rt;
  const size_t d = T->d;
  T->n_lo[qn] = INFINITY;
  T->n_up[qn] = -INFINITY;
  for (int a = 0; a < qt->count[qn]; ++a) {
    const int q = qt->perm[qt->begin[qn] + a];
    double lower = T->q_lo[q] + T->n_dlo[qn];
    double upper = T->q_up[q] + T->n_dup[qn];
    double ex = T->s_ex[q];
    for (int b = 0; b < rt->count[rn]; ++b) {
      const int r = rt->perm[rt->begin[rn] + b];
      const double v = kval(T, sqdist(T->qx + (size_t)q * d, T->rx + (size_t)r * d, d));
      lower += v;
      ex += v;
      upper += v - 1.0;
    }
    T->q_lo[q] = lower;
    T->q_up[q] = upper;
    T->s_ex[q] = ex;
    if (lower < T->n_lo[qn]) T->n_lo[qn] = lower;
    if (upper > T->n_up[qn]) T->n_up[qn] = upper;
  }
  T->n_dlo[qn] = 0.0;
  T->n_dup[qn] = 0.0;
  T->st[2]++;
  T->st[0] += (uint64_t)qt->count[qn] * (uint64_t)rt->count[rn];
}

static void summarize(trav* T, int qn, int rn, int kind, int order)
{ /* engine.cpp:197-237 */
  const orc_tree *qt = T->qt, *rt = T->rt;
  const size_t d = T->d;
  if (kind == 1) {
    for (int a = 0; a < qt->count[qn]; ++a) {
      const int q = qt->perm[qt->begin[qn] + a];
      T->s_ff[q] += eval_ff(T->g, T->M + (size_t)rn * T->g->size, rt->centroid + (size_t)rn * d,
                            T->qx + (size_t)q * d, T->h, order);
    }
    T->st[4]++;
  } else if (kind == 2) {
    direct_local(T->g, T->rx, d, rt->perm + rt->begin[rn], (size_t)rt->count[rn],
                 qt->centroid + (size_t)qn * d, T->h, order, loc_of(T, qn));
    if (order > T->Lord[qn]) T->Lord[qn] = order;
    T->st[5]++;
  } else if (kind == 3) {
    f2l(T->g, T->M + (size_t)rn * T->g->size, rt->centroid + (size_t)rn * d,
        qt->centroid + (size_t)qn * d, T->h, order, loc_of(T, qn));
    if (order > T->Lord[qn]) T->Lord[qn] = order;
    T->st[6]++;
  }
}

static void recurse(trav* T, int qn, int rn)
{ /* engine.cpp:113-195 */
  const orc_tree *qt = T->qt, *rt = T->rt;
  const size_t d = T->d;
  T->st[1]++;
  double dl, du;
  orc_box_bounds_sq(qt->lo + (size_t)qn * d, qt->hi + (size_t)qn * d, rt->lo + (size_t)rn * d,
                    rt->hi + (size_t)rn * d, d, &dl, &du);
  const double kmax = kval(T, dl), kmin = kval(T, du);
  T->st[0] += 2;
  const double nr = (double)rt->count[rn];
  const double dlo = nr * kmin, dup = nr * (kmax - 1.0);
  const double glo = T->n_lo[qn] + T->n_dlo[qn] + dlo;
  const double tau = T->eps * nr * glo / T->nref_total;
  if (0.5 * nr * (kmax - kmin) <= tau) {
    T->n_dlo[qn] += dlo;
    T->n_dup[qn] += dup;
    loc_of(T, qn)[0] += 0.5 * nr * (kmax + kmin);
    if (T->Lord[qn] < 1) T->Lord[qn] = 1;
    T->st[3]++;
    return;
  }
  if (T->series) {
    int kind, order;
    orc_choose_best_method((double)qt->count[qn], nr, qt->max_side[qn], rt->max_side[rn], T->h,
                           tau, T->g->pmax, (int)d, T->cost_model, &kind, &order);
    if (kind != 0) {
      T->n_dlo[qn] += dlo;
      T->n_dup[qn] += dup;
      summarize(T, qn, rn, kind, order);
      return;
    }
  }
  if (qt->left[qn] < 0) {
    if (rt->left[rn] < 0) base_case(T, qn, rn);
    else {
      recurse(T, qn, rt->left[rn]);
      recurse(T, qn, rt->right[rn]);
    }
    return;
  }
  const int ql = qt->left[qn], qr = qt->right[qn];
  T->n_dlo[ql] += T->n_dlo[qn];
  T->n_dlo[qr] += T->n_dlo[qn];
  T->n_dup[ql] += T->n_dup[qn];
  T->n_dup[qr] += T->n_dup[qn];
  T->n_dlo[qn] = 0.0;
  T->n_dup[qn] = 0.0;
  if (rt->left[rn] < 0) {
    recurse(T, ql, rn);
    recurse(T, qr, rn);
  } else {
    recurse(T, ql, rt->left[rn]);
    recurse(T, ql, rt->right[rn]);
    recurse(T, qr, rt->left[rn]);
    recurse(T, qr, rt->right[rn]);
  }
  const double a = T->n_lo[ql] + T->n_dlo[ql], b = T->n_lo[qr] + T->n_dlo[qr];
  T->n_lo[qn] = b < a ? b : a;
  const double c = T->n_up[ql] + T->n_dup[ql], e = T->n_up[qr] + T->n_dup[qr];
  T->n_up[qn] = c < e ? e : c;
}

static void post_process(trav* T, int qn)
{ /* engine.cpp:271-318 */
  const orc_tree* qt = T->qt;
  const size_t d = T->d;
  const int ts = T->g->size;
  if (qt->left[qn] < 0) {
    const int order = T->Lord[qn];
    for (int a = 0; a < qt->count[qn]; ++a) {
      const int q = qt->perm[qt->begin[qn] + a];
      T->q_lo[q] += T->n_dlo[qn];
      T->q_up[q] += T->n_dup[qn];
      if (order > 0)
        T->s_loc[q] = eval_loc(T->g, loc_of(T, qn), qt->centroid + (size_t)qn * d,
                               T->qx + (size_t)q * d, T->h, order);
    }
    T->n_dlo[qn] = 0.0;
    T->n_dup[qn] = 0.0;
    memset(loc_of(T, qn), 0, sizeof(double) * ts);
    return;
  }
  const int ql = qt->left[qn], qr = qt->right[qn];
  const int order = T->Lord[qn];
  if (order > 0) {
    l2l(T->g, loc_of(T, qn), qt->centroid + (size_t)qn * d, qt->centroid + (size_t)ql * d, T->h,
        order, loc_of(T, ql));
    l2l(T->g, loc_of(T, qn), qt->centroid + (size_t)qn * d, qt->centroid + (size_t)qr * d, T->h,
        order, loc_of(T, qr));
    if (T->Lord[ql] < order) T->Lord[ql] = order;
    if (T->Lord[qr] < order) T->Lord[qr] = order;
  }
  T->n_dlo[ql] += T->n_dlo[qn];
  T->n_dlo[qr] += T->n_dlo[qn];
  T->n_dup[ql] += T->n_dup[qn];
  T->n_dup[qr] += T->n_dup[qn];
  T->n_dlo[qn] = 0.0;
  T->n_dup[qn] = 0.0;
  memset(loc_of(T, qn), 0, sizeof(double) * ts);
  post_process(T, ql);
  post_process(T, qr);
}

static void tree_alloc(orc_tree* t, size_t n, size_t d)
{
  const size_t m = 2 * n;
  t->perm = malloc(sizeof(int) * n);
  t->lo = malloc(sizeof(double) * m * d);
  t->hi = malloc(sizeof(double) * m * d);
  t->centroid = malloc(sizeof(double) * m * d);
  t->max_side = malloc(sizeof(double) * m);
  t->left = malloc(sizeof(int) * m);
  t->right = malloc(sizeof(int) * m);
  t->split_dim = malloc(sizeof(int) * m);
  t->split_coord = malloc(sizeof(double) * m);
  t->begin = malloc(sizeof(int64_t) * m);
  t->count = malloc(sizeof(int) * m);
}

static void tree_free(orc_tree* t)
{
  free(t->perm); free(t->lo); free(t->hi); free(t->centroid); free(t->max_side);
  free(t->left); free(t->right); free(t->split_dim); free(t->split_coord);
  free(t->begin); free(t->count);
}

static void ref_moments(const orc_tree* rt, const double* rx, size_t d, geo* g, double h,
                        int node, double* M)
{ /* engine.cpp:368-403 (post-order: leaf moments, then F2F of both children) */
  double* Mn = M + (size_t)node * g->size;
  if (rt->left[node] < 0) {
    moments_acc(g, rx, d, rt->perm + rt->begin[node], (size_t)rt->count[node],
                rt->centroid + (size_t)node * d, h, Mn);
    return;
  }
  const int l = rt->left[node], r = rt->right[node];
  ref_moments(rt, rx, d, g, h, l, M);
  ref_moments(rt, rx, d, g, h, r, M);
  f2f(g, M + (size_t)l * g->size, rt->centroid + (size_t)l * d, rt->centroid + (size_t)node * d,
      h, Mn);
  f2f(g, M + (size_t)r * g->size, rt->centroid + (size_t)r * d, rt->centroid + (size_t)node * d,
      h, Mn);
}

int orc_dfgt(const double* r, size_t nr, const double* q, size_t nq, size_t d, double h,
             double eps, int leaf, int p_max, int cost_model, int mode, double* out,
             uint64_t* stats)
{ /* DualTreeEngine ctor + compute, engine.cpp:352-424 */
  if (!(h > 0.0) || eps < 0.0 || leaf < 1 || nr == 0 || d == 0) return 1;
  if (q == NULL) {
    q = r;
    nq = nr;
  }
  const int pm = mode == 0 ? 1 : (p_max > 0 ? p_max : orc_default_p_max((int)d));
  orc_tree rt, qt;
  tree_alloc(&rt, nr, d);
  orc_tree_build(r, nr, d, leaf, &rt);
  const int rnodes = 2 * (int)nr;
  geo g;
  geo_init(&g, (int)d, pm);
  double* M = NULL;
  if (mode == 1) {
    M = calloc((size_t)rnodes * g.size, sizeof(double));
    ref_moments(&rt, r, d, &g, h, 0, M);
  }
  tree_alloc(&qt, nq, d);
  const int qnodes = orc_tree_build(q, nq, d, leaf, &qt);
  trav T;
  memset(&T, 0, sizeof T);
  T.qx = q;
  T.rx = r;
  T.d = d;
  T.qt = &qt;
  T.rt = &rt;
  T.g = &g;
  T.M = M;
  T.h = h;
  T.scale = -1.0 / (2.0 * h * h);
  T.eps = eps;
  T.nref_total = (double)nr;
  T.series = mode == 1;
  T.cost_model = cost_model;
  T.q_lo = calloc(nq, sizeof(double));
  T.q_up = malloc(nq * sizeof(double));
  T.s_ex = calloc(nq, sizeof(double));
  T.s_ff = calloc(nq, sizeof(double));
  T.s_loc = calloc(nq, sizeof(double));
  T.n_lo = calloc(qnodes, sizeof(double));
  T.n_up = malloc(qnodes * sizeof(double));
  T.n_dlo = calloc(qnodes, sizeof(double));
  T.n_dup = calloc(qnodes, sizeof(double));
  T.L = calloc((size_t)qnodes * g.size, sizeof(double));
  T.Lord = calloc(qnodes, sizeof(int));
  for (size_t i = 0; i < nq; ++i) T.q_up[i] = (double)nr;
  for (int i = 0; i < qnodes; ++i) T.n_up[i] = (double)nr;
  recurse(&T, 0, 0);
  post_process(&T, 0);
  for (size_t i = 0; i < nq; ++i) out[i] = T.s_loc[i] + T.s_ff[i] + T.s_ex[i];
  if (stats) memcpy(stats, T.st, sizeof T.st);
  free(T.q_lo); free(T.q_up); free(T.s_ex); free(T.s_ff); free(T.s_loc);
  free(T.n_lo); free(T.n_up); free(T.n_dlo); free(T.n_dup); free(T.L); free(T.Lord);
  free(M);
  geo_free(&g);
  tree_free(&rt);
  tree_free(&qt);
  return 0;
}

/* ----------------------------------------------------------------------- cv */

double orc_lkcv(size_t n, size_t d, double h, const double* sums, int* clamped)
{ /* cv.cpp:17-25, 61-76 */
  const double norm = (double)(n - 1) * orc_gaussian_normalizer(d, h);
  double acc = 0.0;
  int cl = 0;
  for (size_t j = 0; j < n; ++j) {
    double loo = sums[j] - 1.0;
    if (loo <= 0.0) {
      loo = DBL_MIN;
      ++cl;
    }
    acc += log(loo / norm);
  }
  if (clamped) *clamped = cl;
  return acc / (double)n;
}

double orc_lscv(size_t n, size_t d, double h, const double* sums, double conv_h,
                const double* conv_sums)
{ /* cv.cpp:78-97 */
  const double nh = (double)(n - 1) * orc_gaussian_normalizer(d, h);
  const double nc = (double)(n - 1) * orc_gaussian_normalizer(d, conv_h);
  double acc = 0.0;
  for (size_t j = 0; j < n; ++j) {
    const double dens = (sums[j] - 1.0) / nh;
    const double cd = (conv_sums[j] - 1.0) / nc;
    acc += cd - 2.0 * dens;
  }
  return acc / (double)n;
}

double orc_pilot_bandwidth(const double* x, size_t n, size_t d)
{ /* cv.cpp:112-139 */
  double ss = 0.0;
  for (size_t k = 0; k < d; ++k) {
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += x[i * d + k];
    mean /= (double)n;
    double var = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double t = x[i * d + k] - mean;
      var += t * t;
    }
    ss += sqrt(var / (double)(n - 1));
  }
  const double sigma = ss / (double)d;
  return sigma * pow((double)n, -1.0 / ((double)d + 4.0));
}
