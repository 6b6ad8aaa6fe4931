// Hermite / Taylor series machinery for the DFGT (device side + host term tables).
//
// Term enumeration follows the reference's SeriesGeometry (series.cpp:61-154):
// multi-indices alpha with every digit < p_max, ordered by (max digit, base-p_max
// position with dimension 0 most significant), so the first p^D terms are exactly
// the order-p truncation.  Unlike the reference, device tables are stored in TERM
// order (the truncated prefix is contiguous); the C-ABI converts to the reference's
// position layout at the boundary (dfgtb_series_* entry points).
#pragma once

#include "common.cuh"

#include <cmath>

namespace dfgtb {

struct SeriesTables {
  int D = 0, pmax = 0, T = 0;
  std::vector<int> pos;          // term -> base-p_max position
  std::vector<int> term_of_pos;  // position -> term
  std::vector<int> parent;       // term -> parent term (-1 for alpha = 0)
  std::vector<int> pdim;         // term -> coordinate grown from the parent
  std::vector<int> degree;       // |alpha|
  std::vector<double> invf;      // 1/alpha!
  std::vector<double> fact;      // alpha!
  std::vector<uint64_t> dig;     // packed digits, 4 bits per dimension

  SeriesTables() = default;
  SeriesTables(int dim, int p_max)
  {
    if (dim < 1 || p_max < 1 || p_max > 15) throw InvalidArgument("SeriesGeometry requires dim >= 1 and 1 <= p_max <= 15");
    long long size = 1;
    for (int d = 0; d < dim; ++d) {
      size *= p_max;
      if (size > 100000000LL) throw InvalidArgument("p_max^dim coefficient table is too large");
    }
    if (p_max > 1 && dim > kMaxDim) throw InvalidArgument("dimension > 16 requires p_max == 1");
    D = dim;
    pmax = p_max;
    T = (int)size;
    pos.resize(T);
    term_of_pos.resize(T);
    parent.resize(T);
    pdim.resize(T);
    degree.resize(T);
    invf.resize(T);
    fact.resize(T);
    dig.resize(T);
    double fac[16];
    fac[0] = 1.0;
    for (int k = 1; k < 16; ++k) fac[k] = fac[k - 1] * k;
    // ring = max digit; terms are positions grouped by ring, ascending position within
    std::vector<int> ring(T);
    for (int p = 0; p < T; ++p) {
      int rest = p, mx = 0;
      for (int d = 0; d < D; ++d) {
        mx = std::max(mx, rest % pmax);
        rest /= pmax;
      }
      ring[p] = mx;
    }
    int i = 0;
    for (int rg = 0; rg < pmax; ++rg)
      for (int p = 0; p < T; ++p)
        if (ring[p] == rg) {
          term_of_pos[p] = i;
          pos[i++] = p;
        }
    for (i = 0; i < T; ++i) {
      int rest = pos[i], deg = 0;
      double f = 1.0;
      uint64_t packed = 0;
      int digits[64] = {0};
      for (int d = D - 1; d >= 0; --d) {
        const int g = rest % pmax;
        rest /= pmax;
        if (d < 64) digits[d] = g;
        deg += g;
        f *= fac[g];
        if (d < kMaxDim) packed |= (uint64_t)g << (4 * d);
      }
      degree[i] = deg;
      fact[i] = f;
      invf[i] = 1.0 / f;
      dig[i] = packed;
      if (deg == 0) {
        parent[i] = -1;
        pdim[i] = -1;
      } else {
        int j = 0;
        while (digits[j] == 0) ++j;
        int stride = 1;
        for (int d = j + 1; d < D; ++d) stride *= pmax;
        parent[i] = term_of_pos[pos[i] - stride];
        pdim[i] = j;
      }
    }
  }
  int block(int p) const
  {
    int s = 1;
    for (int d = 0; d < D; ++d) s *= p;
    return s;
  }
};

// Device view of the term tables (one allocation owned by the engine).
struct DevSeries {
  int D, pmax, T;
  const uint64_t* dig;
  const double* invf;
  const double* fact;
  const int* degree;
  const int* term_of_pos;
  const int* pos;  // term -> base-p_max position (the reference's table layout)
};

__host__ __device__ constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }

__host__ __device__ inline int ipow_i(int b, int e)
{
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// 1-D Hermite functions h_k(t), k < orders (series.cpp:163-177).
__device__ inline void hermite_row(double t, int orders, double* h)
{
  h[0] = exp(-t * t);
  if (orders > 1) {
    h[1] = 2.0 * t * h[0];
    for (int k = 1; k + 1 < orders; ++k) h[k + 1] = 2.0 * t * h[k] - 2.0 * k * h[k - 1];
  }
}

// Product prod_d H[d][alpha_d (+ beta_d)] over packed digits; H stride = hs.
__device__ inline double herm_prod(const double* H, int hs, int D, uint64_t a)
{
  double f = 1.0;
  for (int d = 0; d < D; ++d) f *= H[d * hs + digit_of(a, d)];
  return f;
}
__device__ inline double herm_prod2(const double* H, int hs, int D, uint64_t a, uint64_t b)
{
  double f = 1.0;
  for (int d = 0; d < D; ++d) f *= H[d * hs + digit_of(a, d) + digit_of(b, d)];
  return f;
}
// Monomial prod_d P[d][alpha_d] with P[d][k] = u_d^k.
__device__ inline double mono(const double* P, int ps, int D, uint64_t a)
{
  double f = 1.0;
  for (int d = 0; d < D; ++d) f *= P[d * ps + digit_of(a, d)];
  return f;
}

__host__ __device__ inline double inv_scale(double h) { return 1.0 / (h * 1.4142135623730951); }

}  // namespace dfgtb
