// C ABI (include/dfgtb.h): the drop-in boundary for the reference's DFGT path.
// Exceptions map to return codes like the reference CLI maps them to exit codes
// (std::invalid_argument -> 1, cli.cpp:513-516); messages via dfgtb_last_error().
#include "../../include/dfgtb.h"
#include "engine.cuh"
#include "series_dev.cuh"

#include <cfloat>
#include <chrono>
#include <cstring>
#include <string>

using namespace dfgtb;

struct dfgtb_handle {
  std::unique_ptr<Engine> eng;
  DevBuf<double> s1, s2;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f)
{
  try {
    f();
    return DFGTB_OK;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return DFGTB_EINVAL;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DFGTB_EINVAL;
  } catch (const OutOfMemory& e) {
    g_err = e.what();
    return DFGTB_ENOMEM;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return DFGTB_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DFGTB_ECUDA;
  }
}

Config to_cfg(const dfgtb_config* c)
{
  Config k;
  if (c) {
    k.epsilon = c->epsilon;
    k.leaf_threshold = c->leaf_threshold;
    k.p_max = c->p_max;
    k.cost_model = c->cost_model;
    k.mode = c->mode;
    k.local_pushdown = c->local_pushdown;
  }
  return k;
}

void fill_stats(const Stats& s, dfgtb_stats* o)
{
  if (!o) return;
  o->kernel_evaluations = s.kernel_evaluations;
  o->pairs_visited = s.pairs_visited;
  o->base_cases = s.base_cases;
  o->prunes_finite_diff = s.prunes_finite_diff;
  o->prunes_farfield = s.prunes_farfield;
  o->prunes_direct_local = s.prunes_direct_local;
  o->prunes_far_to_local = s.prunes_far_to_local;
  o->levels = (uint64_t)s.levels;
  o->pairs_covered = s.pairs_covered;
}

void check_h(dfgtb_handle* h)
{
  if (!h || !h->eng) throw InvalidArgument("null dfgtb handle");
}

double normalizer(size_t d, double h)
{  // gaussian_normalizer, dataset.cpp:32-39
  if (d == 0 || !(h > 0.0)) throw InvalidArgument("gaussian_normalizer requires D >= 1 and h > 0");
  const double two_pi = 6.283185307179586476925286766559;
  return std::pow(two_pi * h * h, 0.5 * (double)d);
}

// ---------------------------------------------------------------- series test ops
__global__ void k_series_op(DevSeries g, int op, const double* in, int n, const double* a,
                            const double* b, double s, int order, double* out)
{
  extern __shared__ double sm[];
  switch (op) {
  case 0: dev_moments_block(g, in, n, a, s, out, sm); break;
  case 1:
    if (threadIdx.x == 0) out[0] = dev_eval_farfield(g, in, a, b, s, order);
    break;
  case 2: dev_direct_local_block(g, in, n, a, s, order, out, sm); break;
  case 3: dev_f2l_block(g, in, a, b, s, order, out, sm); break;
  case 4: dev_l2l_block(g, in, a, b, s, order, out, sm); break;
  case 5:
    if (threadIdx.x == 0) out[0] = dev_eval_local(g, in, a, b, s, order);
    break;
  }
}

}  // namespace

__global__ void k_widen(const float* in, size_t n, double* out)
{
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];  // exact
}

// float32 host points -> float64 device points (the H2D moves half the bytes).
static void widen_to_device(const float* h_in, size_t n, DevBuf<double>& out)
{
  DevBuf<float> f;
  f.reserve(n);
  out.reserve(n);
  CK(cudaMemcpy(f.p, h_in, sizeof(float) * n, cudaMemcpyHostToDevice));
  k_widen<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256>>>(f.p, n, out.p);
  CK_LAUNCH();
  CK(cudaDeviceSynchronize());
}

extern "C" {

void dfgtb_default_config(dfgtb_config* c)
{
  c->epsilon = 0.01;
  c->leaf_threshold = 20;
  c->p_max = 0;
  c->cost_model = 0;
  c->mode = 1;
  c->local_pushdown = 0;
}

const char* dfgtb_last_error(void) { return g_err.c_str(); }

int dfgtb_create(const double* refs, size_t n, size_t d, const dfgtb_config* cfg,
                 dfgtb_handle** out)
{
  return guard([&] {
    if (!out) throw InvalidArgument("null output handle");
    if (!refs && n) throw InvalidArgument("null reference points");
    auto* h = new dfgtb_handle;
    try {
      h->eng.reset(new Engine(refs, n, d, to_cfg(cfg), false));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int dfgtb_create_device(const double* d_refs, size_t n, size_t d, const dfgtb_config* cfg,
                        dfgtb_handle** out)
{
  return guard([&] {
    if (!out) throw InvalidArgument("null output handle");
    auto* h = new dfgtb_handle;
    try {
      h->eng.reset(new Engine(d_refs, n, d, to_cfg(cfg), true));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int dfgtb_create_f32(const float* refs, size_t n, size_t d, const dfgtb_config* cfg,
                     dfgtb_handle** out)
{
  return guard([&] {
    if (!out) throw InvalidArgument("null output handle");
    if (!refs && n) throw InvalidArgument("null reference points");
    if (n == 0 || d == 0) throw InvalidArgument("PointSet requires N >= 1 and D >= 1");
    DevBuf<double> wide;
    widen_to_device(refs, n * d, wide);
    auto* h = new dfgtb_handle;
    try {
      h->eng.reset(new Engine(wide.p, n, d, to_cfg(cfg), true));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void dfgtb_destroy(dfgtb_handle* h) { delete h; }

int dfgtb_compute(dfgtb_handle* h, const double* queries, size_t nq, double bw, double* out,
                  dfgtb_stats* st)
{
  return guard([&] {
    check_h(h);
    h->eng->compute_host(queries, nq, bw, out);
    fill_stats(h->eng->last_stats(), st);
  });
}

int dfgtb_compute_device(dfgtb_handle* h, const double* dq, size_t nq, double bw, double* dout,
                         dfgtb_stats* st)
{
  return guard([&] {
    check_h(h);
    h->eng->wait_legacy_stream();  // inputs produced on the legacy stream are ordered first
    h->eng->compute_device(dq, nq, bw, dout);
    fill_stats(h->eng->last_stats(), st);
  });
}

int dfgtb_last_stats(dfgtb_handle* h, dfgtb_stats* st)
{
  return guard([&] {
    check_h(h);
    fill_stats(h->eng->last_stats(), st);
  });
}

int dfgtb_last_timings(dfgtb_handle* h, dfgtb_timings* t)
{
  return guard([&] {
    check_h(h);
    const Timings& s = h->eng->last_timings();
    t->tree_ms = s.tree_ms;
    t->traverse_ms = s.traverse_ms;
    t->moments_ms = s.moments_ms;
    t->local_ms = s.local_ms;
    t->base_ms = s.base_ms;
    t->farfield_ms = s.farfield_ms;
    t->final_ms = s.final_ms;
    t->total_ms = s.total_ms;
    t->base_f32_ms = s.base_f32_ms;
    t->base_fp64_ms = s.base_fp64_ms;
    t->moments_build_ms = h->eng->moments_build_ms();
  });
}

int dfgtb_p_max(dfgtb_handle* h) { return h && h->eng ? h->eng->p_max() : -1; }

int dfgtb_base_exp_mode(dfgtb_handle* h)
{
  if (!h || !h->eng) return -1;
  return h->eng->f32_exp() ? 2 : h->eng->mufu_exp() ? 1 : 0;
}

// Batched CV: every bandwidth (and its convolution bandwidth) of `ns` scales goes
// through ONE lock-step traversal; sums stay in HBM; CV partial sums come back.
static void cv_rows(dfgtb_handle* h, const double* bws, const double* convs, int ns,
                    dfgtb_cv_row* rows)
{
  Engine& e = *h->eng;
  DeviceGuard dg(e.device());
  const size_t n = e.n();
  if (n < 2) throw InvalidArgument("likelihood CV requires at least 2 points");
  const bool ls = convs != nullptr;
  std::vector<double> hs(bws, bws + ns);
  if (ls) hs.insert(hs.end(), convs, convs + ns);
  const int nb = (int)hs.size();
  h->s1.reserve(n * (size_t)nb);
  std::vector<double> lk(ns), lsv(ns);
  std::vector<int> cl(ns);
  // the sums of every h (then every conv_h) and their CV partial sums: one host wait
  e.compute_batch_cv(hs.data(), nb, h->s1.p, bws, convs, ns, lk.data(), cl.data(), lsv.data());
  const Timings& t = e.last_timings();
  for (int k = 0; k < ns; ++k) {
    dfgtb_cv_row& r = rows[k];
    r.h = bws[k];
    r.conv_h = ls ? convs[k] : 0.0;
    r.lk_score = lk[k];
    r.lk_clamped = cl[k];
    r.ls_score = ls ? lsv[k] : 0.0;
    // the batch shares one traversal: its device time is split evenly over the rows
    r.seconds = t.total_ms * 1e-3 / ns;
    r.base_ms = t.base_ms / ns;
    r.base_pairs = r.kernel_evaluations = r.pairs_visited = 0;
    for (int slot : { k, ns + k }) {
      if (slot >= nb) continue;
      const Stats& st = e.last_stats(slot);
      r.base_pairs += st.kernel_evaluations - 2ull * st.pairs_visited;
      r.kernel_evaluations += st.kernel_evaluations;
      r.pairs_visited += st.pairs_visited;
    }
  }
}

int dfgtb_cv(dfgtb_handle* h, double bw, double conv_h, dfgtb_cv_row* row)
{
  return guard([&] {
    check_h(h);
    cv_rows(h, &bw, conv_h > 0.0 ? &conv_h : nullptr, 1, row);
  });
}

int dfgtb_sweep(dfgtb_handle* h, const double* scales, size_t ns, double base_h, int sqrt2,
                dfgtb_cv_row* rows)
{
  return guard([&] {
    check_h(h);
    if (!(base_h > 0.0)) throw InvalidArgument("base bandwidth must be positive");
    for (size_t i = 1; i < ns; ++i)
      if (!(scales[i] > scales[i - 1])) throw InvalidArgument("scales must be strictly increasing");
    const size_t chunk = kMaxSlots / 2;  // h and conv_h of up to 32 scales per batch
    for (size_t i0 = 0; i0 < ns; i0 += chunk) {
      const int m = (int)std::min(chunk, ns - i0);
      std::vector<double> bws(m), convs(m);
      for (int k = 0; k < m; ++k) {
        bws[k] = scales[i0 + k] * base_h;
        convs[k] = sqrt2 ? std::sqrt(2.0) * bws[k] : 2.0 * bws[k];  // cv.cpp:27-30
      }
      cv_rows(h, bws.data(), convs.data(), m, rows + i0);
      for (int k = 0; k < m; ++k) rows[i0 + k].scale = scales[i0 + k];
    }
  });
}

int dfgtb_sweep_best(const dfgtb_cv_row* rows, size_t ns, size_t* lk_best, size_t* ls_best)
{
  return guard([&] {
    if (ns == 0 || !rows) throw InvalidArgument("empty sweep");
    size_t bk = 0, bs = 0;
    for (size_t i = 1; i < ns; ++i) {
      if (rows[i].lk_score > rows[bk].lk_score) bk = i;
      if (rows[i].ls_score < rows[bs].ls_score) bs = i;
    }
    if (lk_best) *lk_best = bk;
    if (ls_best) *ls_best = bs;
  });
}

int dfgtb_compute_batch(dfgtb_handle* h, const double* queries, size_t nq, const double* bws,
                        size_t nb, double* out_sums, dfgtb_stats* stats)
{
  return guard([&] {
    check_h(h);
    Engine& e = *h->eng;
    const size_t n_out = queries ? nq : e.n();
    if (nb == 0) throw InvalidArgument("empty bandwidth batch");
    DevBuf<double> q, out;
    out.reserve(n_out * nb);
    DeviceGuard dg(e.device());
    // every copy is ordered on the engine's stream (pageable host memory: the async
    // copies are staged by the driver; the stream synchronisation ends the call)
    if (queries) {
      q.reserve(nq * e.dim());
      CK(cudaMemcpyAsync(q.p, queries, sizeof(double) * nq * e.dim(), cudaMemcpyHostToDevice,
                         e.stream()));
    }
    for (size_t b0 = 0; b0 < nb; b0 += kMaxSlots) {
      const int m = (int)std::min<size_t>(kMaxSlots, nb - b0);
      e.compute_batch(queries ? q.p : nullptr, nq, bws + b0, m, out.p);
      CK(cudaMemcpyAsync(out_sums + b0 * n_out, out.p, sizeof(double) * n_out * m,
                         cudaMemcpyDeviceToHost, e.stream()));
      CK(cudaStreamSynchronize(e.stream()));
      if (stats)
        for (int k = 0; k < m; ++k) fill_stats(e.last_stats(k), stats + b0 + k);
    }
  });
}

int dfgtb_compute_batch_f32(dfgtb_handle* h, const float* queries, size_t nq, const double* bws,
                            size_t nb, double* out_sums, dfgtb_stats* stats)
{
  return guard([&] {
    check_h(h);
    Engine& e = *h->eng;
    if (!queries) throw InvalidArgument("null query points");
    if (nb == 0) throw InvalidArgument("empty bandwidth batch");
    DeviceGuard dg(e.device());
    DevBuf<double> q, out;
    widen_to_device(queries, nq * e.dim(), q);
    out.reserve(nq * nb);
    for (size_t b0 = 0; b0 < nb; b0 += kMaxSlots) {
      const int m = (int)std::min<size_t>(kMaxSlots, nb - b0);
      e.compute_batch(q.p, nq, bws + b0, m, out.p);
      CK(cudaMemcpyAsync(out_sums + b0 * nq, out.p, sizeof(double) * nq * m, cudaMemcpyDeviceToHost,
                         e.stream()));
      CK(cudaStreamSynchronize(e.stream()));
      if (stats)
        for (int k = 0; k < m; ++k) fill_stats(e.last_stats(k), stats + b0 + k);
    }
  });
}

int dfgtb_lkcv_from_sums(size_t n, size_t d, double bw, const double* sums, double* score,
                         int* clamped)
{
  return guard([&] {
    if (n < 2) throw InvalidArgument("likelihood CV requires at least 2 points");
    const double norm = (double)(n - 1) * normalizer(d, bw);
    double acc = 0.0;
    int cl = 0;
    for (size_t j = 0; j < n; ++j) {
      double loo = sums[j] - 1.0;
      if (loo <= 0.0) {
        loo = DBL_MIN;
        ++cl;
      }
      acc += std::log(loo / norm);
    }
    *score = acc / (double)n;
    if (clamped) *clamped = cl;
  });
}

int dfgtb_lscv_from_sums(size_t n, size_t d, double bw, const double* sums, double conv_h,
                         const double* conv_sums, double* score)
{
  return guard([&] {
    if (n < 2) throw InvalidArgument("least-squares CV requires at least 2 points");
    const double nh = (double)(n - 1) * normalizer(d, bw);
    const double nc = (double)(n - 1) * normalizer(d, conv_h);
    double acc = 0.0;
    for (size_t j = 0; j < n; ++j) acc += (conv_sums[j] - 1.0) / nc - 2.0 * ((sums[j] - 1.0) / nh);
    *score = acc / (double)n;
  });
}

int dfgtb_tree_nodes(dfgtb_handle* h) { return h && h->eng ? h->eng->ref_tree().nodes : -1; }
int dfgtb_tree_height(dfgtb_handle* h) { return h && h->eng ? h->eng->ref_tree().height : -1; }

int dfgtb_export_tree(dfgtb_handle* h, int* perm, double* lo, double* hi, double* centroid,
                      double* max_side, int* left, int* right, int* split_dim,
                      double* split_coord, int64_t* begin, int* count)
{
  return guard([&] {
    check_h(h);
    DeviceGuard dg(h->eng->device());
    CK(cudaStreamSynchronize(h->eng->stream()));
    const DevTree& t = h->eng->ref_tree();
    const size_t K = t.nodes, D = t.D;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    cp(perm, t.perm.p, sizeof(int) * t.n);
    cp(lo, t.lo.p, sizeof(double) * K * D);
    cp(hi, t.hi.p, sizeof(double) * K * D);
    cp(centroid, t.centroid.p, sizeof(double) * K * D);
    cp(max_side, t.max_side.p, sizeof(double) * K);
    cp(left, t.left.p, sizeof(int) * K);
    cp(right, t.right.p, sizeof(int) * K);
    cp(split_dim, t.split_dim.p, sizeof(int) * K);
    cp(split_coord, t.split_coord.p, sizeof(double) * K);
    cp(count, t.count.p, sizeof(int) * K);
    if (begin) {
      std::vector<int> b(K);
      CK(cudaMemcpy(b.data(), t.begin.p, sizeof(int) * K, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < K; ++i) begin[i] = b[i];
    }
  });
}

int dfgtb_naive(const double* q, size_t nq, const double* r, size_t nr, size_t d, double bw,
                double* out)
{
  return guard([&] {
    if (!(bw > 0.0) || !std::isfinite(bw)) throw InvalidArgument("bandwidth must be positive and finite");
    if (d == 0 || d > (size_t)kMaxDim) throw InvalidArgument("dimension must be in [1, 16]");
    DevBuf<double> dq, dr, dout;
    dq.reserve(nq * d);
    dr.reserve(nr * d);
    dout.reserve(nq);
    CK(cudaMemcpy(dq.p, q, sizeof(double) * nq * d, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dr.p, r, sizeof(double) * nr * d, cudaMemcpyHostToDevice));
    naive_device(dq.p, nq, dr.p, nr, (int)d, bw, dout.p, 0);
    CK(cudaMemcpy(out, dout.p, sizeof(double) * nq, cudaMemcpyDeviceToHost));
  });
}

int dfgtb_series_op(int op, size_t d, int p_max, const double* in, size_t n, const double* a,
                    const double* b, double bw, int order, double* out)
{
  return guard([&] {
    if (op < 0 || op > 5) throw InvalidArgument("unknown series op");
    if (!(bw > 0.0)) throw InvalidArgument("bandwidth must be positive");
    SeriesTables t((int)d, p_max);
    if ((op != 0) && (order < 1 || order > p_max)) throw InvalidArgument("order outside [1, p_max]");
    DevBuf<unsigned char> blob;
    upload_series(t, blob, 0);
    const DevSeries g = series_view(t, blob);
    const size_t T = t.T;
    // position layout (reference) <-> term layout (device)
    auto to_terms = [&](const double* pos_tab) {
      std::vector<double> v(T);
      for (size_t i = 0; i < T; ++i) v[i] = pos_tab[t.pos[i]];
      return v;
    };
    DevBuf<double> din, da, db, dout;
    std::vector<double> hin;
    if (op == 0 || op == 2) hin.assign(in, in + n * d);
    else hin = to_terms(in);
    din.reserve(std::max<size_t>(hin.size(), 1));
    if (!hin.empty()) CK(cudaMemcpy(din.p, hin.data(), sizeof(double) * hin.size(), cudaMemcpyHostToDevice));
    da.reserve(d);
    db.reserve(d);
    CK(cudaMemcpy(da.p, a, sizeof(double) * d, cudaMemcpyHostToDevice));
    if (b) CK(cudaMemcpy(db.p, b, sizeof(double) * d, cudaMemcpyHostToDevice));
    const bool scalar = op == 1 || op == 5;
    std::vector<double> hout = scalar ? std::vector<double>(1, 0.0) : to_terms(out);
    dout.reserve(hout.size());
    CK(cudaMemcpy(dout.p, hout.data(), sizeof(double) * hout.size(), cudaMemcpyHostToDevice));
    const int smem = (int)sizeof(double) * std::max<int>(32 * (int)d * p_max, (int)d * (2 * p_max));
    k_series_op<<<1, 128, smem>>>(g, op, din.p, (int)n, da.p, db.p, inv_scale(bw), order, dout.p);
    CK_LAUNCH();
    CK(cudaMemcpy(hout.data(), dout.p, sizeof(double) * hout.size(), cudaMemcpyDeviceToHost));
    if (scalar) out[0] = hout[0];
    else
      for (size_t i = 0; i < T; ++i) out[t.pos[i]] = hout[i];
  });
}

int dfgtb_choose_methods(size_t n, const double* args, int* out)
{
  return guard([&] {
    if (n && (!args || !out)) throw InvalidArgument("dfgtb_choose_methods: null pointer");
    for (size_t i = 0; i < n; ++i) {
      const double* a = args + 9 * i;
      if (a[6] < 1 || a[6] > 15 || a[7] < 1 || a[7] > kMaxDim || (a[8] != 0 && a[8] != 1))
        throw InvalidArgument("dfgtb_choose_methods: p_max in [1, 15], dim in [1, 16], cost 0/1");
    }
    choose_methods_device(n, args, out);
  });
}

int dfgtb_box_bounds(size_t n, size_t d, const double* boxes, double* out)
{
  return guard([&] {
    if (d < 1 || d > (size_t)kMaxDim) throw InvalidArgument("dimension must be in [1, 16]");
    if (n && (!boxes || !out)) throw InvalidArgument("dfgtb_box_bounds: null pointer");
    box_bounds_device(n, (int)d, boxes, out);
  });
}

uintptr_t dfgtb_stream(dfgtb_handle* h)
{
  return h && h->eng ? (uintptr_t)h->eng->stream() : 0;
}

uint64_t dfgtb_launch_count(dfgtb_handle* h)
{
  (void)h;
  return launch_counter();
}

int dfgtb_device_count(void)
{
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void dfgtb_release_cached_memory(void) { cache_release_all(); }

int dfgtb_guard_check(void)
{
  try {
    return guard_check();
  } catch (...) {
    return -2;
  }
}

namespace {
__global__ void k_guard_poke(int* p, int at) { p[at] = 7; }  // one element past the end
}  // namespace

int dfgtb_guard_selftest(void)
{
  if (!guard_mode()) return -1;
  try {
    int detected = 0;
    {
      DevBuf<int> b;
      b.reserve(256);
      const int before = guard_check();
      k_guard_poke<<<1, 1>>>(b.p, (int)b.cap);
      CK_LAUNCH();
      detected = guard_check() > before ? 1 : 0;
      CK(cudaMemset(reinterpret_cast<unsigned char*>(b.p + b.cap), kGuardByte, kGuardBytes));  // repair
    }
    return detected;
  } catch (...) {
    return -2;
  }
}

double dfgtb_dfma_peak(void)
{
  double v = -1.0;
  guard([&] {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    v = measure_dfma_peak(dev);
  });
  return v;
}

double dfgtb_ex2_peak(void)
{
  double v = -1.0;
  guard([&] {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    v = measure_ex2_peak(dev);
  });
  return v;
}

double dfgtb_mufu_exp_error(void)
{
  double v = -1.0;
  guard([&] { v = mufu_exp_max_error(); });
  return v;
}

int dfgtb_last_base_split(dfgtb_handle* h, int* f32_tasks, int* fp64_tasks, uint64_t* f32_pairs,
                          uint64_t* fp64_pairs)
{
  return guard([&] {
    if (!h || !h->eng || !f32_tasks || !fp64_tasks) throw InvalidArgument("dfgtb_last_base_split: null argument");
    unsigned long long a = 0, b = 0;
    h->eng->base_split(*f32_tasks, *fp64_tasks, a, b);
    if (f32_pairs) *f32_pairs = a;
    if (fp64_pairs) *fp64_pairs = b;
  });
}

double dfgtb_f32_exp_error(void)
{
  double v = -1.0;
  guard([&] { v = f32_exp_max_error(); });
  return v;
}

int dfgtb_f32_terms(size_t d, const double* q, const double* r, const double* c, size_t n, double* out)
{
  return guard([&] {
    if (d < 1 || d > 5) throw InvalidArgument("dfgtb_f32_terms: d must be in 1..5");
    if (n == 0) return;
    if (!q || !r || !c || !out) throw InvalidArgument("dfgtb_f32_terms: null pointer");
    f32_terms_host((int)d, q, r, c, n, out);
  });
}

}  // extern "C"
