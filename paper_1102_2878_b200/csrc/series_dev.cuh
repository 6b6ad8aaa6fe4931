// Device series primitives shared by the traversal kernels and the parity-test
// entry points.  Each restates one reference primitive (series.cpp) on TERM-order
// tables: the first order^D entries of a table are its order-`order` truncation.
#pragma once

#include "series.cuh"

namespace dfgtb {

constexpr int kPMaxDev = 15;

// Block-cooperative: M[i] = (1/alpha_i!) sum_r prod_d ((x_r - c)*s)_d^{alpha_i,d}
// over the full table (accumulate_farfield_moments, series.cpp:238-254).
// `pts` are the node's points (row-major, contiguous).  smem: 32*D*pmax doubles.
__device__ inline void dev_moments_block(const DevSeries& g, const double* pts, int npts,
                                         const double* c, double s, double* Mout, double* smem,
                                         const int* opos = nullptr)
{
  // opos != nullptr: write the table in the reference's POSITION layout
  auto M = [&](int i) -> double& { return Mout[opos ? opos[i] : i]; };
  const int D = g.D, pm = g.pmax, T = g.T;
  const int per = D * pm;
  double acc[8];
  const int nmine = (T - (int)threadIdx.x + (int)blockDim.x - 1) / (int)blockDim.x;
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  // tables beyond 8*blockDim terms fall back to global accumulation
  const bool reg = nmine <= 8;
  if (!reg)
    for (int i = threadIdx.x; i < T; i += blockDim.x) M(i) = 0.0;
  for (int base = 0; base < npts; base += 32) {
    const int m = min(32, npts - base);
    __syncthreads();
    for (int w = threadIdx.x; w < m * D; w += blockDim.x) {
      const int pt = w / D, d = w % D;
      const double u = (pts[(size_t)(base + pt) * D + d] - c[d]) * s;
      double* P = smem + pt * per + d * pm;
      P[0] = 1.0;
      for (int k = 1; k < pm; ++k) P[k] = P[k - 1] * u;
    }
    __syncthreads();
    int slot = 0;
    for (int i = threadIdx.x; i < T; i += blockDim.x, ++slot) {
      const uint64_t a = g.dig[i];
      double sum = 0.0;
      for (int pt = 0; pt < m; ++pt) sum += mono(smem + pt * per, pm, D, a);
      if (reg) acc[slot] += sum;
      else M(i) += sum;
    }
  }
  int slot = 0;
  for (int i = threadIdx.x; i < T; i += blockDim.x, ++slot)
    M(i) = (reg ? acc[slot] : M(i)) * g.invf[i];
}

// Per thread: sum_{i < order^D} M[i] h_alpha_i((q - c)*s)   (eval_farfield, series.cpp:289-303)
// spow != nullptr: M holds UNSCALED moments (h-independent) and M[i] * s^|alpha_i|
// is the reference's scaled moment.
__device__ inline double dev_eval_farfield(const DevSeries& g, const double* M, const double* c,
                                           const double* q, double s, int order,
                                           const double* spow = nullptr,
                                           const int* mpos = nullptr)
{
  const int D = g.D;
  double H[kMaxDim * kPMaxDev];
  for (int d = 0; d < D; ++d) hermite_row((q[d] - c[d]) * s, order, H + d * kPMaxDev);
  const int n = ipow_i(order, D);
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    const double mi = M[mpos ? mpos[i] : i];  // mpos: table stored in position layout
    const double m = spow ? mi * spow[g.degree[i]] : mi;
    sum += m * herm_prod(H, kPMaxDev, D, g.dig[i]);
  }
  return sum;
}

// Block-cooperative direct local accumulation of `npts` points into L (terms < order^D)
// (accumulate_direct_local, series.cpp:305-326).  smem: 32*D*order doubles.
__device__ inline void dev_direct_local_block(const DevSeries& g, const double* pts, int npts,
                                              const double* c, double s, int order, double* L,
                                              double* smem)
{
  const int D = g.D;
  const int n = ipow_i(order, D);
  const int per = D * order;
  const bool reg = n <= 8 * (int)blockDim.x;
  double acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  for (int base = 0; base < npts; base += 32) {
    const int m = min(32, npts - base);
    __syncthreads();
    for (int w = threadIdx.x; w < m * D; w += blockDim.x) {
      const int pt = w / D, d = w % D;
      hermite_row((c[d] - pts[(size_t)(base + pt) * D + d]) * s, order, smem + pt * per + d * order);
    }
    __syncthreads();
    int slot = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x, ++slot) {
      const uint64_t a = g.dig[i];
      double sum = 0.0;
      for (int pt = 0; pt < m; ++pt) sum += herm_prod(smem + pt * per, order, D, a);
      if (reg) acc[slot] += sum;
      else L[i] += ((g.degree[i] & 1) ? -1.0 : 1.0) * g.invf[i] * sum;  // huge tables
    }
  }
  __syncthreads();
  if (!reg) return;
  int slot = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x, ++slot) {
    const double sg = (g.degree[i] & 1) ? -1.0 : 1.0;
    L[i] += sg * g.invf[i] * acc[slot];
  }
}

// Block-cooperative F2L: L[b] += (-1)^|b|/b! sum_a M[a] h_{a+b}((c_dst - c_src)*s)
// (trans_far_to_local, series.cpp:328-353).  smem: D*(2*order-1) doubles.
// With raw != 0 the unsigned sum is written to L[i] instead (partial tables that
// are reduced and signed later); spow as in dev_eval_farfield.
__device__ inline void dev_f2l_block(const DevSeries& g, const double* M, const double* src_c,
                                     const double* dst_c, double s, int order, double* L,
                                     double* smem, const double* spow = nullptr, int raw = 0,
                                     const int* mpos = nullptr)
{
  const int D = g.D;
  const int n = ipow_i(order, D);
  const int ho = 2 * order - 1;
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    hermite_row((dst_c[d] - src_c[d]) * s, ho, smem + d * ho);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t b = g.dig[i];
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const double mj = M[mpos ? mpos[j] : j];
      const double m = spow ? mj * spow[g.degree[j]] : mj;
      acc += m * herm_prod2(smem, ho, D, g.dig[j], b);
    }
    if (raw) {
      L[i] = acc;
    } else {
      const double sg = (g.degree[i] & 1) ? -1.0 : 1.0;
      L[i] += sg * g.invf[i] * acc;
    }
  }
}

// Unsigned direct-local partial: P[i] = sum_{r in pts} prod_d h_{alpha_i,d}((c - r)*s)
// for i < order^D (one chunk of a D item; sign and 1/alpha! applied at reduction).
// smem: npts*D*order doubles (npts <= blockDim-sized chunk).
__device__ inline void dev_direct_local_partial(const DevSeries& g, const double* pts, int npts,
                                                const double* c, double s, int order, double* P,
                                                double* smem, bool accumulate = false)
{
  const int D = g.D;
  const int n = ipow_i(order, D);
  const int per = D * order;
  __syncthreads();
  for (int w = threadIdx.x; w < npts * D; w += blockDim.x) {
    const int pt = w / D, d = w % D;
    hermite_row((c[d] - pts[(size_t)pt * D + d]) * s, order, smem + pt * per + d * order);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t a = g.dig[i];
    double sum = 0.0;
    for (int pt = 0; pt < npts; ++pt) sum += herm_prod(smem + pt * per, order, D, a);
    P[i] = accumulate ? P[i] + sum : sum;
  }
}

// Block-cooperative L2L: dst[a] += sum_{b >= a} b!/(a!(b-a)!) src[b] ((c_dst - c_src)*s)^(b-a)
// (trans_local_to_local, series.cpp:355-391).  smem: D*order doubles.
__device__ inline void dev_l2l_block(const DevSeries& g, const double* src, const double* src_c,
                                     const double* dst_c, double s, int order, double* dst,
                                     double* smem)
{
  const int D = g.D;
  const int n = ipow_i(order, D);
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const double u = (dst_c[d] - src_c[d]) * s;
    double* P = smem + d * order;
    P[0] = 1.0;
    for (int k = 1; k < order; ++k) P[k] = P[k - 1] * u;
  }
  __syncthreads();
  double fac[kPMaxDev + 1];
  fac[0] = 1.0;
  for (int k = 1; k <= kPMaxDev; ++k) fac[k] = fac[k - 1] * k;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t a = g.dig[i];
    const double ifa = g.invf[i];
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const uint64_t b = g.dig[j];
      bool dom = true;
      double fd = 1.0, mo = 1.0;
      for (int d = 0; d < D; ++d) {
        const int df = digit_of(b, d) - digit_of(a, d);
        if (df < 0) {
          dom = false;
          break;
        }
        fd *= fac[df];
        mo *= smem[d * order + df];
      }
      if (dom) acc += g.fact[j] * ifa * (1.0 / fd) * src[j] * mo;
    }
    dst[i] += acc;
  }
}

// Per thread: sum_{i < order^D} L[i] ((q - c)*s)^alpha_i   (eval_local, series.cpp:393-407)
__device__ inline double dev_eval_local(const DevSeries& g, const double* L, const double* c,
                                        const double* q, double s, int order)
{
  const int D = g.D;
  double P[kMaxDim * kPMaxDev];
  for (int d = 0; d < D; ++d) {
    const double u = (q[d] - c[d]) * s;
    double* p = P + d * kPMaxDev;
    p[0] = 1.0;
    for (int k = 1; k < order; ++k) p[k] = p[k - 1] * u;
  }
  const int n = ipow_i(order, D);
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += L[i] * mono(P, kPMaxDev, D, g.dig[i]);
  return sum;
}

}  // namespace dfgtb
