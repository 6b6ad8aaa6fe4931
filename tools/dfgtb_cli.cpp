// dfgtb_cli -- command-line driver of the GPU engine with the reference CLI's
// `kde` / `cv` semantics (cli.cpp:128-199): same file formats (load_points /
// write_values), density normalisation and CV table, so outputs diff file-to-file
// against the reference.  Exit codes: 0 ok, 2 usage / IO / invalid argument.
//
//   dfgtb_cli kde --refs R.csv [--queries Q.csv] --bandwidth H --out OUT
//                 [--algorithm dfgt|dfd|naive] [--epsilon E] [--leaf-threshold L]
//                 [--pmax P] [--cost-model exponential|term-count] [--raw-sums]
//   dfgtb_cli cv  --refs R.csv --out TABLE.csv [--score lscv|lkcv] [--scales a,b,..]
//                 [--base-h H] [--convolution-bandwidth 2x|sqrt2] [--epsilon E] ...
#include "dfgtb.hpp"

#include <cstring>
#include <fstream>
#include <iostream>
#include <map>

namespace {

std::string fmt(double v, const char* f)
{
  char b[64];
  std::snprintf(b, sizeof b, f, v);
  return b;
}

std::vector<double> parse_list(const std::string& s)
{
  std::vector<double> v;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) v.push_back(std::stod(t));
  return v;
}

int run(int argc, char** argv)
{
  if (argc < 2) {
    std::cerr << "usage: dfgtb_cli kde|cv [options]\n";
    return 2;
  }
  const std::string cmd = argv[1];
  std::map<std::string, std::string> opt;
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) {
      std::cerr << "error: unexpected argument " << k << "\n";
      return 2;
    }
    if (k == "--raw-sums") {
      opt[k] = "1";
      continue;
    }
    if (i + 1 >= argc) {
      std::cerr << "error: missing value for " << k << "\n";
      return 2;
    }
    opt[k] = argv[++i];
  }
  dfgtb::EngineConfig cfg;
  if (opt.count("--epsilon")) cfg.epsilon = std::stod(opt["--epsilon"]);
  if (opt.count("--leaf-threshold")) cfg.leaf_threshold = std::stoi(opt["--leaf-threshold"]);
  if (opt.count("--pmax")) cfg.p_max = std::stoi(opt["--pmax"]);
  if (opt.count("--cost-model"))
    cfg.cost_model = opt["--cost-model"] == "term-count" ? dfgtb::CostModel::term_count
                                                         : dfgtb::CostModel::exponential;
  if (!opt.count("--refs") || !opt.count("--out")) {
    std::cerr << "error: --refs and --out are required\n";
    return 2;
  }
  const dfgtb::PointSet refs = dfgtb::load_points(opt["--refs"]);
  if (cmd == "kde") {
    if (!opt.count("--bandwidth")) {
      std::cerr << "error: --bandwidth is required\n";
      return 2;
    }
    const double h = std::stod(opt["--bandwidth"]);
    const auto algo = dfgtb::parse_algorithm(opt.count("--algorithm") ? opt["--algorithm"] : "dfgt");
    if (!algo) {
      std::cerr << "error: unknown algorithm\n";
      return 2;
    }
    std::vector<double> sums;
    if (opt.count("--queries")) {
      const dfgtb::PointSet q = dfgtb::load_points(opt["--queries"]);
      sums = dfgtb::compute_sums(*algo, q, refs, h, cfg);
    } else {
      sums = dfgtb::compute_sums(*algo, refs, refs, h, cfg);
    }
    if (!opt.count("--raw-sums")) {  // cli.cpp:141-147
      const double norm = static_cast<double>(refs.size()) * dfgtb::gaussian_normalizer(refs.dim(), h);
      for (double& s : sums) s /= norm;
    }
    dfgtb::write_values(opt["--out"], sums);
    return 0;
  }
  if (cmd == "cv") {
    const std::string score = opt.count("--score") ? opt["--score"] : "lscv";
    if (score != "lscv" && score != "lkcv") {
      std::cerr << "error: --score must be lscv or lkcv\n";
      return 2;
    }
    const std::string conv = opt.count("--convolution-bandwidth") ? opt["--convolution-bandwidth"] : "2x";
    if (conv != "2x" && conv != "sqrt2") {
      std::cerr << "error: --convolution-bandwidth must be 2x or sqrt2\n";
      return 2;
    }
    std::vector<double> scales = opt.count("--scales") ? parse_list(opt["--scales"])
                                                       : std::vector<double>{ 1e-3, 1e-2, 1e-1, 1.0, 10.0, 100.0, 1e3 };
    double base_h = opt.count("--base-h") ? std::stod(opt["--base-h"]) : 0.0;
    if (base_h <= 0.0) base_h = dfgtb::pilot_bandwidth(refs);
    const auto rows = dfgtb::bandwidth_sweep(
      refs, scales, base_h, score == "lkcv" ? dfgtb::CvScore::likelihood : dfgtb::CvScore::least_squares,
      cfg, conv == "sqrt2");
    std::ofstream table(opt["--out"]);
    if (!table) throw std::runtime_error("cannot write '" + opt["--out"] + "'");
    table << "scale,h,score,seconds,max_rel_err\n";
    for (const auto& r : rows) {
      table << fmt(r.scale, "%.6g") << ',' << fmt(r.h, "%.10g") << ',' << fmt(r.score, "%.10g") << ','
            << fmt(r.seconds, "%.3f") << ",\n";
      if (r.clamped > 0)
        std::cerr << "warning: h=" << r.h << ": " << r.clamped
                  << " leave-one-out sums clamped to the smallest positive double\n";
    }
    return 0;
  }
  std::cerr << "error: unknown subcommand " << cmd << "\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv)
{
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
