// dfgtb.hpp -- C++ host mirror of the reference's DFGT interface over the C ABI.
//
// Header-only.  Same names, argument meaning and exceptions as the reference
// (/root/reference/proj/include/dfgt/{dataset,engine,cv}.hpp), in namespace dfgtb,
// so a caller of dfgt::DualTreeEngine / compute_sums / bandwidth_sweep switches by
// changing the namespace and linking libdfgtb.so:
//
//   dfgt::PointSet                  -> dfgtb::PointSet           (dataset.hpp:15-41)
//   dfgt::EngineConfig              -> dfgtb::EngineConfig       (engine.hpp:17-26)
//   dfgt::DualTreeEngine            -> dfgtb::DualTreeEngine     (engine.hpp:86-111)
//   dfgt::naive_kde/dfd_kde/dfgt_kde, compute_sums               (engine.hpp:29,113-137)
//   dfgt::lkcv_from_sums/lscv_from_sums, bandwidth_sweep          (cv.hpp:35-62)
//   dfgt::gaussian_normalizer, load_points, write_values          (dataset.hpp:64-78)
//
// dfgtb::DualTreeEngine copies the reference points to the GPU (the reference
// borrows them); everything else follows the reference contract.
#pragma once

#include "dfgtb.h"

#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace dfgtb {

inline void check(int rc)
{
  if (rc == DFGTB_OK) return;
  const std::string msg = dfgtb_last_error();
  if (rc == DFGTB_EINVAL) throw std::invalid_argument(msg);
  if (rc == DFGTB_ENOMEM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

class PointSet {
public:
  PointSet(std::size_t n, std::size_t dim)
    : n_(n)
    , dim_(dim)
    , data_(n * dim, 0.0)
  {
  }
  PointSet(std::size_t n, std::size_t dim, std::vector<double> data)
    : n_(n)
    , dim_(dim)
    , data_(std::move(data))
  {
    if (n_ == 0 || dim_ == 0) throw std::invalid_argument("PointSet requires N >= 1 and D >= 1");
    if (data_.size() != n_ * dim_) throw std::invalid_argument("PointSet data size does not match N x D");
  }
  std::size_t size() const { return n_; }
  std::size_t dim() const { return dim_; }
  std::span<const double> row(std::size_t i) const { return { data_.data() + i * dim_, dim_ }; }
  std::span<double> row(std::size_t i) { return { data_.data() + i * dim_, dim_ }; }
  const std::vector<double>& data() const { return data_; }

private:
  std::size_t n_, dim_;
  std::vector<double> data_;
};

enum class CostModel { exponential, term_count };

struct EngineConfig {
  double epsilon = 0.01;
  int leaf_threshold = 20;
  std::optional<int> p_max;
  CostModel cost_model = CostModel::exponential;
};

using TraversalStats = dfgtb_stats;

inline double gaussian_normalizer(std::size_t dim, double h)
{
  if (dim == 0 || !(h > 0.0)) throw std::invalid_argument("gaussian_normalizer requires D >= 1 and h > 0");
  return std::pow(6.283185307179586476925286766559 * h * h, 0.5 * static_cast<double>(dim));
}

class DualTreeEngine {
public:
  enum class Mode { centroid, series };

  DualTreeEngine(const PointSet& refs, Mode mode, EngineConfig config = {})
    : n_(refs.size())
    , dim_(refs.dim())
  {
    dfgtb_config c;
    dfgtb_default_config(&c);
    c.epsilon = config.epsilon;
    c.leaf_threshold = config.leaf_threshold;
    c.p_max = config.p_max.value_or(0);
    c.cost_model = config.cost_model == CostModel::term_count ? 1 : 0;
    c.mode = mode == Mode::series ? 1 : 0;
    check(dfgtb_create(refs.data().data(), refs.size(), refs.dim(), &c, &h_));
  }
  ~DualTreeEngine()
  {
    if (h_) dfgtb_destroy(h_);
  }
  DualTreeEngine(const DualTreeEngine&) = delete;
  DualTreeEngine& operator=(const DualTreeEngine&) = delete;

  //! Per-query sums, |approx - exact| <= epsilon * exact (engine.hpp:93-95).
  std::vector<double> compute(const PointSet& queries, double h)
  {
    if (queries.dim() != dim_) throw std::invalid_argument("query and reference dimensions differ");
    std::vector<double> out(queries.size());
    check(dfgtb_compute(h_, queries.data().data(), queries.size(), h, out.data(), &stats_));
    return out;
  }
  //! Q = R fast path (the reference tree doubles as the query tree).
  std::vector<double> compute_self(double h)
  {
    std::vector<double> out(n_);
    check(dfgtb_compute(h_, nullptr, 0, h, out.data(), &stats_));
    return out;
  }
  const TraversalStats& last_stats() const { return stats_; }
  int p_max() const { return dfgtb_p_max(h_); }
  dfgtb_handle* handle() const { return h_; }

private:
  dfgtb_handle* h_ = nullptr;
  std::size_t n_, dim_;
  TraversalStats stats_{};
};

inline std::vector<double> naive_kde(const PointSet& q, const PointSet& r, double h)
{
  if (q.dim() != r.dim()) throw std::invalid_argument("query and reference dimensions differ");
  std::vector<double> out(q.size());
  check(dfgtb_naive(q.data().data(), q.size(), r.data().data(), r.size(), r.dim(), h, out.data()));
  return out;
}

inline std::vector<double> dfgt_kde(const PointSet& q, const PointSet& r, double h,
                                    const EngineConfig& config = {})
{
  if (q.dim() != r.dim()) throw std::invalid_argument("query and reference dimensions differ");
  DualTreeEngine e(r, DualTreeEngine::Mode::series, config);
  return &q == &r ? e.compute_self(h) : e.compute(q, h);
}

inline std::vector<double> dfd_kde(const PointSet& q, const PointSet& r, double h, double epsilon,
                                   int leaf_threshold = 20)
{
  if (q.dim() != r.dim()) throw std::invalid_argument("query and reference dimensions differ");
  EngineConfig c;
  c.epsilon = epsilon;
  c.leaf_threshold = leaf_threshold;
  DualTreeEngine e(r, DualTreeEngine::Mode::centroid, c);
  return &q == &r ? e.compute_self(h) : e.compute(q, h);
}

enum class Algorithm { naive, dfd, dfgt };

inline std::optional<Algorithm> parse_algorithm(std::string_view name)
{
  if (name == "naive") return Algorithm::naive;
  if (name == "dfd") return Algorithm::dfd;
  if (name == "dfgt") return Algorithm::dfgt;
  return std::nullopt;
}

inline std::vector<double> compute_sums(Algorithm a, const PointSet& q, const PointSet& r, double h,
                                        const EngineConfig& config = {})
{
  switch (a) {
  case Algorithm::naive: return naive_kde(q, r, h);
  case Algorithm::dfd: return dfd_kde(q, r, h, config.epsilon, config.leaf_threshold);
  case Algorithm::dfgt: return dfgt_kde(q, r, h, config);
  }
  throw std::invalid_argument("unknown algorithm");
}

struct ScoreResult {
  double score = 0.0;
  int clamped = 0;
};

inline ScoreResult lkcv_from_sums(const PointSet& refs, double h, std::span<const double> sums)
{
  ScoreResult r;
  check(dfgtb_lkcv_from_sums(refs.size(), refs.dim(), h, sums.data(), &r.score, &r.clamped));
  return r;
}

inline ScoreResult lscv_from_sums(const PointSet& refs, double h, std::span<const double> sums,
                                  double conv_h, std::span<const double> conv_sums)
{
  ScoreResult r;
  check(dfgtb_lscv_from_sums(refs.size(), refs.dim(), h, sums.data(), conv_h, conv_sums.data(),
                             &r.score));
  return r;
}

//! pilot_bandwidth (cv.cpp:112-139): mean per-dimension sample std * N^(-1/(D+4)).
inline double pilot_bandwidth(const PointSet& refs)
{
  const std::size_t n = refs.size(), dim = refs.dim();
  if (n < 2) throw std::invalid_argument("pilot bandwidth requires at least 2 points");
  double sigma_sum = 0.0;
  for (std::size_t d = 0; d < dim; ++d) {
    double mean = 0.0;
    for (std::size_t i = 0; i < n; ++i) mean += refs.row(i)[d];
    mean /= static_cast<double>(n);
    double var = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
      const double t = refs.row(i)[d] - mean;
      var += t * t;
    }
    sigma_sum += std::sqrt(var / static_cast<double>(n - 1));
  }
  const double sigma = sigma_sum / static_cast<double>(dim);
  if (!(sigma > 0.0)) throw std::invalid_argument("pilot bandwidth undefined for zero-variance data");
  return sigma * std::pow(static_cast<double>(n), -1.0 / (static_cast<double>(dim) + 4.0));
}

enum class CvScore { likelihood, least_squares };

struct CvRow {
  double scale = 0.0, h = 0.0, score = 0.0, seconds = 0.0;
  std::optional<double> max_rel_err;
  int clamped = 0;
};

//! bandwidth_sweep (cv.cpp:141-182) on the GPU engine; sums stay on the device.
inline std::vector<CvRow> bandwidth_sweep(const PointSet& refs, std::span<const double> scales,
                                          double base_h, CvScore kind, const EngineConfig& cfg = {},
                                          bool sqrt2_convolution = false)
{
  DualTreeEngine e(refs, DualTreeEngine::Mode::series, cfg);
  std::vector<dfgtb_cv_row> raw(scales.size());
  check(dfgtb_sweep(e.handle(), scales.data(), scales.size(), base_h, sqrt2_convolution ? 1 : 0,
                    raw.data()));
  std::vector<CvRow> rows;
  for (const auto& r : raw) {
    CvRow c;
    c.scale = r.scale;
    c.h = r.h;
    c.seconds = r.seconds;
    c.score = kind == CvScore::likelihood ? r.lk_score : r.ls_score;
    c.clamped = kind == CvScore::likelihood ? r.lk_clamped : 0;
    rows.push_back(c);
  }
  return rows;
}

//! load_points (dataset.cpp:95-138): comma or whitespace separated, delimiter
//! auto-detected from the first non-empty line; ragged rows, bad fields and
//! non-finite values are errors with their line number.
inline PointSet load_points(const std::string& path, std::optional<char> delimiter = {})
{
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open '" + path + "'");
  std::vector<double> data;
  std::size_t dim = 0, rows = 0, line_no = 0;
  std::string line;
  char delim = delimiter.value_or('\0');
  while (std::getline(in, line)) {
    ++line_no;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    if (delim == '\0') delim = line.find(',') != std::string::npos ? ',' : ' ';
    std::vector<std::string> fields;
    std::istringstream ss(line);
    std::string tok;
    if (delim == ' ') {
      while (ss >> tok) fields.push_back(tok);
    } else {
      while (std::getline(ss, tok, delim)) fields.push_back(tok);
    }
    if (fields.empty()) continue;
    if (dim == 0) dim = fields.size();
    else if (fields.size() != dim)
      throw std::runtime_error("line " + std::to_string(line_no) + ": expected " +
                               std::to_string(dim) + " fields, got " + std::to_string(fields.size()));
    for (const auto& f : fields) {
      const auto b = f.find_first_not_of(" \t\r");
      const auto e = f.find_last_not_of(" \t\r");
      if (b == std::string::npos) throw std::runtime_error("line " + std::to_string(line_no) + ": empty field");
      double v = 0.0;
      const char* first = f.data() + b;
      const char* last = f.data() + e + 1;
      auto res = std::from_chars(first, last, v);
      if (res.ec != std::errc{} || res.ptr != last)
        throw std::runtime_error("line " + std::to_string(line_no) + ": unparseable numeric field '" +
                                 f.substr(b, e - b + 1) + "'");
      if (!std::isfinite(v)) throw std::runtime_error("line " + std::to_string(line_no) + ": non-finite value");
      data.push_back(v);
    }
    ++rows;
  }
  if (rows == 0) throw std::runtime_error("'" + path + "' contains no points");
  return PointSet(rows, dim, std::move(data));
}

//! write_values (dataset.cpp:140-154): one value per line, %.17g.
inline void write_values(const std::string& path, std::span<const double> values)
{
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write '" + path + "'");
  char buf[64];
  for (double v : values) {
    std::snprintf(buf, sizeof(buf), "%.17g\n", v);
    out << buf;
  }
  if (!out) throw std::runtime_error("write failed for '" + path + "'");
}

}  // namespace dfgtb
