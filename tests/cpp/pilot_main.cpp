// Test driver for the host mirror's pilot_bandwidth (include/dfgtb.hpp, cv.cpp:112-139):
// reads "n d" then n*d raw float64 values (binary, row-major) from a file and prints
// the bandwidth with %.17g.  Header-only use: no libdfgtb.so needed.
#include "dfgtb.hpp"

#include <cstdio>
#include <vector>

int main(int argc, char** argv)
{
  if (argc != 2) return 2;
  std::FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  unsigned long long nd[2];
  if (std::fread(nd, sizeof(nd), 1, f) != 1) return 2;
  std::vector<double> v(nd[0] * nd[1]);
  if (std::fread(v.data(), sizeof(double), v.size(), f) != v.size()) return 2;
  std::fclose(f);
  try {
    dfgtb::PointSet p(nd[0], nd[1], std::move(v));
    std::printf("%.17g\n", dfgtb::pilot_bandwidth(p));
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  return 0;
}
