// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product path.
//
// C-ABI shim over the *unmodified* reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  It lets the Python tests,
// the golden-fixture generator and bench.py's CPU arms (`cpu_baseline`,
// `--impl reference`) call the reference implementation through ctypes.
// Every entry point forwards to one reference symbol; nothing is re-implemented.
//
//   ref_naive_kde            -> dfgt::naive_kde               engine.cpp:22-36
//   ref_tree_*               -> dfgt::KdTree::build + accessors kdtree.cpp:21-109
//   ref_box_bounds_sq        -> dfgt::box_distance_bounds_sq  kdtree.cpp:122-141
//   ref_engine_*             -> dfgt::DualTreeEngine          engine.cpp:352-424
//   ref_lkcv / ref_lscv      -> dfgt::lkcv_from_sums / lscv_from_sums  cv.cpp:61-97
//   ref_pilot_bandwidth      -> dfgt::pilot_bandwidth          cv.cpp:112-139
//   ref_*_error_bound, ref_choose_best_method, ref_default_p_max  truncation.cpp
//   ref_series_*             -> series.cpp primitives (moments, F2F, F2L, L2L, evals)
//   ref_gaussian_normalizer  -> dataset.cpp:32-39
//
// Return convention: 0 ok, 1 std::invalid_argument / out_of_range, 2 other exception.
#include "dfgt/cv.hpp"
#include "dfgt/engine.hpp"
#include "dfgt/kdtree.hpp"
#include "dfgt/series.hpp"
#include "dfgt/truncation.hpp"

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f)
{
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

dfgt::PointSet make_set(const double* x, size_t n, size_t d)
{
  return dfgt::PointSet(n, d, std::vector<double>(x, x + n * d));
}

struct RefEngine {
  dfgt::PointSet refs;
  dfgt::DualTreeEngine engine;
  RefEngine(dfgt::PointSet r, dfgt::DualTreeEngine::Mode m, dfgt::EngineConfig c)
    : refs(std::move(r))
    , engine(refs, m, c)
  {
  }
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_naive_kde(const double* q, size_t nq, const double* r, size_t nr, size_t d, double h,
                  double* out)
{
  return guard([&] {
    auto qs = make_set(q, nq, d);
    auto rs = make_set(r, nr, d);
    auto s = dfgt::naive_kde(qs, rs, h);
    std::memcpy(out, s.data(), s.size() * sizeof(double));
  });
}

double ref_gaussian_normalizer(size_t d, double h) { return dfgt::gaussian_normalizer(d, h); }

// ---- kd-tree -------------------------------------------------------------
void* ref_tree_build(const double* x, size_t n, size_t d, int leaf)
{
  dfgt::KdTree* t = nullptr;
  int rc = guard([&] {
    auto pts = make_set(x, n, d);
    t = new dfgt::KdTree(dfgt::KdTree::build(pts, leaf));
  });
  return rc == 0 ? t : nullptr;
}

int ref_tree_node_count(void* t) { return static_cast<dfgt::KdTree*>(t)->node_count(); }
int ref_tree_height(void* t) { return static_cast<dfgt::KdTree*>(t)->height(); }

void ref_tree_export(void* tp, size_t n, int* perm, double* lo, double* hi, double* centroid,
                     double* max_side, int* left, int* right, int* split_dim,
                     double* split_coord, long long* begin, int* count)
{
  auto* t = static_cast<dfgt::KdTree*>(tp);
  const size_t d = t->dim();
  const int* base = t->points_of(0).data();
  std::memcpy(perm, base, n * sizeof(int));
  for (int k = 0; k < t->node_count(); ++k) {
    for (size_t j = 0; j < d; ++j) {
      lo[k * d + j] = t->lower(k)[j];
      hi[k * d + j] = t->upper(k)[j];
      centroid[k * d + j] = t->centroid(k)[j];
    }
    max_side[k] = t->max_side(k);
    left[k] = t->left(k);
    right[k] = t->right(k);
    split_dim[k] = t->split_dim(k);
    split_coord[k] = t->split_coord(k);
    begin[k] = static_cast<long long>(t->points_of(k).data() - base);
    count[k] = t->count(k);
  }
}

void ref_tree_free(void* t) { delete static_cast<dfgt::KdTree*>(t); }

void ref_box_bounds_sq(const double* alo, const double* ahi, const double* blo,
                       const double* bhi, size_t d, double* out2)
{
  auto b = dfgt::box_distance_bounds_sq({ alo, d }, { ahi, d }, { blo, d }, { bhi, d });
  out2[0] = b.lower;
  out2[1] = b.upper;
}

// ---- engine ----------------------------------------------------------------
// mode: 0 = centroid (DFD), 1 = series (DFGT).  pmax <= 0 -> reference default.
void* ref_engine_create(const double* r, size_t n, size_t d, double eps, int leaf, int pmax,
                        int cost_model, int mode)
{
  RefEngine* e = nullptr;
  int rc = guard([&] {
    dfgt::EngineConfig c;
    c.epsilon = eps;
    c.leaf_threshold = leaf;
    if (pmax > 0) {
      c.p_max = pmax;
    }
    c.cost_model = cost_model == 1 ? dfgt::CostModel::term_count : dfgt::CostModel::exponential;
    e = new RefEngine(make_set(r, n, d),
                      mode == 0 ? dfgt::DualTreeEngine::Mode::centroid
                                : dfgt::DualTreeEngine::Mode::series,
                      c);
  });
  return rc == 0 ? e : nullptr;
}

// q == nullptr -> queries are the reference set (Q = R, as SumProvider does, cv.cpp:48).
// stats (nullable): kernel_evaluations, pairs_visited, base_cases, prunes_fd, prunes_F,
// prunes_D, prunes_T (TraversalStats order, engine.hpp:66-74).
int ref_engine_compute(void* ep, const double* q, size_t nq, double h, double* out,
                       unsigned long long* stats)
{
  auto* e = static_cast<RefEngine*>(ep);
  return guard([&] {
    std::vector<double> s;
    if (q == nullptr) {
      s = e->engine.compute(e->refs, h);
    } else {
      auto qs = make_set(q, nq, e->refs.dim());
      s = e->engine.compute(qs, h);
    }
    std::memcpy(out, s.data(), s.size() * sizeof(double));
    if (stats) {
      const auto& st = e->engine.last_stats();
      stats[0] = st.kernel_evaluations;
      stats[1] = st.pairs_visited;
      stats[2] = st.base_cases;
      stats[3] = st.prunes_finite_diff;
      stats[4] = st.prunes_farfield;
      stats[5] = st.prunes_direct_local;
      stats[6] = st.prunes_far_to_local;
    }
  });
}

int ref_engine_p_max(void* ep) { return static_cast<RefEngine*>(ep)->engine.p_max(); }
void ref_engine_free(void* ep) { delete static_cast<RefEngine*>(ep); }

// ---- CV --------------------------------------------------------------------
int ref_lkcv(const double* r, size_t n, size_t d, double h, const double* sums, double* score,
             int* clamped)
{
  return guard([&] {
    auto rs = make_set(r, n, d);
    auto res = dfgt::lkcv_from_sums(rs, h, { sums, n });
    *score = res.score;
    *clamped = res.clamped;
  });
}

int ref_lscv(const double* r, size_t n, size_t d, double h, const double* sums, double conv_h,
             const double* conv_sums, double* score)
{
  return guard([&] {
    auto rs = make_set(r, n, d);
    auto res = dfgt::lscv_from_sums(rs, h, { sums, n }, conv_h, { conv_sums, n });
    *score = res.score;
  });
}

int ref_pilot_bandwidth(const double* r, size_t n, size_t d, double* out)
{
  return guard([&] { *out = dfgt::pilot_bandwidth(make_set(r, n, d)); });
}

// ---- truncation ------------------------------------------------------------
double ref_farfield_error_bound(double c, double r, int p, int d)
{
  return dfgt::farfield_error_bound(c, r, p, d);
}
double ref_f2l_error_bound(double c, double r, int p, int d)
{
  return dfgt::f2l_error_bound(c, r, p, d);
}
// out2 = {kind (0=E,1=F,2=D,3=T), order}
void ref_choose_best_method(double nq, double nr, double sq, double sr, double h, double tau,
                            int pmax, int d, int cost_model, int* out2)
{
  auto c = dfgt::choose_best_method(
    nq, nr, sq, sr, h, tau, pmax, d,
    cost_model == 1 ? dfgt::CostModel::term_count : dfgt::CostModel::exponential);
  out2[0] = static_cast<int>(c.kind);
  out2[1] = c.order;
}
int ref_default_p_max(int d) { return dfgt::default_p_max(d); }

// ---- series primitives (tables in reference layout: p_max^D, base-p_max positions)
namespace {
struct Geo {
  dfgt::SeriesGeometry g;
  dfgt::SeriesWorkspace ws;
  explicit Geo(int d, int p)
    : g(d, p)
    , ws(g)
  {
  }
};
} // namespace

void* ref_series_geometry(int d, int pmax)
{
  Geo* g = nullptr;
  guard([&] { g = new Geo(d, pmax); });
  return g;
}
void ref_series_free(void* g) { delete static_cast<Geo*>(g); }
int ref_series_table_size(void* g) { return static_cast<Geo*>(g)->g.table_size(); }
// term enumeration: pos[i], parent[i], parent_dim[i], degree[i], inv_factorial[i]
void ref_series_terms(void* gp, int* pos, int* parent, int* pdim, int* degree, double* invf)
{
  const auto& t = static_cast<Geo*>(gp)->g.terms();
  for (size_t i = 0; i < t.size(); ++i) {
    pos[i] = t[i].pos;
    parent[i] = t[i].parent;
    pdim[i] = t[i].parent_dim;
    degree[i] = t[i].degree;
    invf[i] = t[i].inv_factorial;
  }
}

void ref_series_moments(void* gp, const double* pts, size_t n, size_t d, const double* center,
                        double h, double* moments)
{
  auto* G = static_cast<Geo*>(gp);
  auto ps = make_set(pts, n, d);
  std::vector<int> idx(n);
  for (size_t i = 0; i < n; ++i) idx[i] = static_cast<int>(i);
  dfgt::accumulate_farfield_moments(G->g, ps, idx, { center, d }, h, G->ws,
                                    { moments, static_cast<size_t>(G->g.table_size()) });
}

void ref_series_f2f(void* gp, const double* src, const double* src_c, const double* dst_c,
                    size_t d, double h, double* dst)
{
  auto* G = static_cast<Geo*>(gp);
  const size_t ts = static_cast<size_t>(G->g.table_size());
  dfgt::trans_far_to_far(G->g, { src, ts }, { src_c, d }, { dst_c, d }, h, G->ws, { dst, ts });
}

double ref_series_eval_farfield(void* gp, const double* moments, const double* center,
                                const double* q, size_t d, double h, int order)
{
  auto* G = static_cast<Geo*>(gp);
  const size_t ts = static_cast<size_t>(G->g.table_size());
  return dfgt::eval_farfield(G->g, { moments, ts }, { center, d }, { q, d }, h, order, G->ws);
}

void ref_series_direct_local(void* gp, const double* pts, size_t n, size_t d,
                             const double* center, double h, int order, double* local)
{
  auto* G = static_cast<Geo*>(gp);
  auto ps = make_set(pts, n, d);
  std::vector<int> idx(n);
  for (size_t i = 0; i < n; ++i) idx[i] = static_cast<int>(i);
  dfgt::accumulate_direct_local(G->g, ps, idx, { center, d }, h, order, G->ws,
                                { local, static_cast<size_t>(G->g.table_size()) });
}

void ref_series_f2l(void* gp, const double* moments, const double* src_c, const double* dst_c,
                    size_t d, double h, int order, double* local)
{
  auto* G = static_cast<Geo*>(gp);
  const size_t ts = static_cast<size_t>(G->g.table_size());
  dfgt::trans_far_to_local(G->g, { moments, ts }, { src_c, d }, { dst_c, d }, h, order, G->ws,
                           { local, ts });
}

void ref_series_l2l(void* gp, const double* src, const double* src_c, const double* dst_c,
                    size_t d, double h, int order, double* dst)
{
  auto* G = static_cast<Geo*>(gp);
  const size_t ts = static_cast<size_t>(G->g.table_size());
  dfgt::trans_local_to_local(G->g, { src, ts }, { src_c, d }, { dst_c, d }, h, order, G->ws,
                             { dst, ts });
}

double ref_series_eval_local(void* gp, const double* local, const double* center,
                             const double* q, size_t d, double h, int order)
{
  auto* G = static_cast<Geo*>(gp);
  const size_t ts = static_cast<size_t>(G->g.table_size());
  return dfgt::eval_local(G->g, { local, ts }, { center, d }, { q, d }, h, order, G->ws);
}

} // extern "C"
