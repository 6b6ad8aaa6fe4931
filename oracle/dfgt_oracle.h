/* TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's DFGT hot path
 * (/root/reference/proj/src/{dataset,kdtree,series,truncation,engine,cv}.cpp),
 * used by tests/ and by bench.py's cpu_baseline leg as the CHECKER.  The product
 * path (paper_1102_2878_b200/) never links or calls this library.
 *
 * Pinning: tests/test_oracle.py checks every function here against the goldens
 * in the reference's own unit tests (proj/tests/test_*.cpp) and, where the
 * compiled reference (oracle/_ref/libdfgt_ref.so) is available, against the
 * reference itself on seeded inputs and the committed fixtures in tests/golden/.
 */
#ifndef DFGT_ORACLE_H
#define DFGT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dataset.cpp:32-39 */
double orc_gaussian_normalizer(size_t dim, double h);
/* engine.cpp:22-36  (row-major N x D) */
void orc_naive_kde(const double* q, size_t nq, const double* r, size_t nr, size_t d, double h,
                   double* out);
/* kdtree.cpp:122-141 */
void orc_box_bounds_sq(const double* alo, const double* ahi, const double* blo,
                       const double* bhi, size_t d, double* lo_sq, double* hi_sq);

/* kdtree.cpp:21-109.  Node arrays sized for 2n-1 nodes by the caller.
 * Returns the node count. */
typedef struct {
  int* perm;           /* n */
  double* lo;          /* nodes*d */
  double* hi;          /* nodes*d */
  double* centroid;    /* nodes*d */
  double* max_side;    /* nodes */
  int* left;           /* nodes */
  int* right;          /* nodes */
  int* split_dim;      /* nodes */
  double* split_coord; /* nodes */
  int64_t* begin;      /* nodes */
  int* count;          /* nodes */
} orc_tree;
int orc_tree_build(const double* x, size_t n, size_t d, int leaf, orc_tree* t);

/* truncation.cpp */
double orc_farfield_error_bound(double count, double r, int p, int dim);
double orc_f2l_error_bound(double count, double r, int p, int dim);
/* kind: 0=E, 1=F, 2=D, 3=T  (ApproxChoice::Kind order, truncation.hpp:199-204) */
void orc_choose_best_method(double nq, double nr, double side_q, double side_r, double h,
                            double tau, int p_max, int dim, int cost_model, int* kind,
                            int* order);
int orc_default_p_max(int dim);

/* series.cpp -- tables in the reference layout (p_max^D, base-p_max positions,
 * dimension 0 most significant). */
int orc_series_table_size(int dim, int p_max);
void orc_series_terms(int dim, int p_max, int* pos, int* parent, int* parent_dim,
                      int* degree, double* inv_factorial);
void orc_series_moments(int dim, int p_max, const double* pts, size_t n,
                        const double* center, double h, double* moments);
void orc_series_f2f(int dim, int p_max, const double* src, const double* src_c,
                    const double* dst_c, double h, double* dst);
double orc_series_eval_farfield(int dim, int p_max, const double* moments,
                                const double* center, const double* q, double h, int order);
void orc_series_direct_local(int dim, int p_max, const double* pts, size_t n,
                             const double* center, double h, int order, double* local);
void orc_series_f2l(int dim, int p_max, const double* moments, const double* src_c,
                    const double* dst_c, double h, int order, double* local);
void orc_series_l2l(int dim, int p_max, const double* src, const double* src_c,
                    const double* dst_c, double h, int order, double* dst);
double orc_series_eval_local(int dim, int p_max, const double* local, const double* center,
                             const double* q, double h, int order);

/* engine.cpp:43-424: full depth-first DFGT (mode 1) / DFD (mode 0) traversal.
 * q == NULL -> Q = R.  stats[7] as TraversalStats (engine.hpp:66-74).
 * Returns 0 on success, 1 on invalid argument. */
int orc_dfgt(const double* r, size_t nr, const double* q, size_t nq, size_t d, double h,
             double eps, int leaf, int p_max, int cost_model, int mode, double* out,
             uint64_t* stats);

/* cv.cpp:17-25, 61-97, 112-139 */
double orc_lkcv(size_t n, size_t d, double h, const double* sums, int* clamped);
double orc_lscv(size_t n, size_t d, double h, const double* sums, double conv_h,
                const double* conv_sums);
double orc_pilot_bandwidth(const double* x, size_t n, size_t d);

#ifdef __cplusplus
}
#endif
#endif
