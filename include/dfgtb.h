/* dfgtb -- B200-native (sm_100a) dual-tree fast Gauss transform: C ABI.
 *
 * Drop-in boundary for the reference's DFGT kernel-summation path
 * (/root/reference/proj).  Each entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; no C++ or torch types.  Points are
 * N x D row-major float64 (PointSet, dataset.hpp:15-41).  Host pointers unless a
 * function name ends in _device.
 *
 * Return codes: DFGTB_OK 0, DFGTB_EINVAL 1 (the reference's std::invalid_argument),
 * DFGTB_ECUDA 2 (CUDA/runtime error), DFGTB_ENOMEM 3.  dfgtb_last_error() gives the
 * message (thread local).  A handle owns one CUDA stream and is not thread-safe,
 * like DualTreeEngine (engine.hpp:85).
 */
#ifndef DFGTB_H
#define DFGTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFGTB_OK 0
#define DFGTB_EINVAL 1
#define DFGTB_ECUDA 2
#define DFGTB_ENOMEM 3

/* EngineConfig (engine.hpp:17-26) + DualTreeEngine::Mode (engine.hpp:89). */
typedef struct dfgtb_config {
  double epsilon;     /* relative error bound, >= 0                       (default 0.01) */
  int leaf_threshold; /* kd-tree leaf size, >= 1                          (default 20)   */
  int p_max;          /* series order limit; 0 = default_p_max(D)         (truncation.cpp:168) */
  int cost_model;     /* 0 exponential, 1 term_count                      (truncation.hpp:216) */
  int mode;           /* 0 centroid (DFD), 1 series (DFGT)                (engine.hpp:89) */
  int local_pushdown; /* 0: evaluate ancestors' local expansions at each query (default);
                         1: the reference's L2L push-down chain (engine.cpp:294-304).
                         Identical mathematics (exact polynomial re-centering). */
} dfgtb_config;

/* TraversalStats (engine.hpp:66-74) + level count of the BFS traversal. */
typedef struct dfgtb_stats {
  uint64_t kernel_evaluations;
  uint64_t pairs_visited;
  uint64_t base_cases;
  uint64_t prunes_finite_diff;
  uint64_t prunes_farfield;
  uint64_t prunes_direct_local;
  uint64_t prunes_far_to_local;
  uint64_t levels;
  /* Coverage (the reference's CoverageProbe, tests/probes.hpp:13-44): sum over every
   * retired node pair (finite-difference prune, F, D, T, base case) of |Q| * |R|.
   * Every (query, reference) pair is retired exactly once, so this equals
   * n_queries * n_refs. */
  uint64_t pairs_covered;
} dfgtb_stats;

/* Device time (ms, CUDA events on the handle's stream) of the last compute. */
typedef struct dfgtb_timings {
  float tree_ms, traverse_ms, moments_ms, local_ms, base_ms, farfield_ms, final_ms, total_ms;
  float base_f32_ms, base_fp64_ms; /* base_ms split: FP32 kernel | FP64 kernel */
  float moments_build_ms;           /* the handle's one-time unscaled moments (K2/K3) */
} dfgtb_timings;

/* One bandwidth of a CV sweep (CvRow, cv.hpp:49-56 + ScoreResult cv.hpp:25-32). */
typedef struct dfgtb_cv_row {
  double scale, h, conv_h;
  double lk_score;  /* lkcv_from_sums  (cv.cpp:61-76) */
  int lk_clamped;
  double ls_score;  /* lscv_from_sums  (cv.cpp:78-97) */
  double seconds;   /* device time of this row's computes.  dfgtb_sweep runs all rows'
                       bandwidths through ONE batched traversal, so this is the batch's
                       device time divided evenly over the rows (a share, not a per-h
                       measurement); dfgtb_cv rows are measured individually. */
  double base_ms;   /* device time of the base-case kernel launches of this row */
  uint64_t base_pairs;          /* (q, r) kernel evaluations in those base cases */
  uint64_t kernel_evaluations;  /* TraversalStats::kernel_evaluations, summed */
  uint64_t pairs_visited;       /* TraversalStats::pairs_visited, summed */
} dfgtb_cv_row;

typedef struct dfgtb_handle dfgtb_handle;

void dfgtb_default_config(dfgtb_config* cfg);

/* DualTreeEngine(refs, mode, config)  engine.cpp:352-366 / engine.hpp:91.
 * Uploads the reference points and builds the kd-tree on the GPU (KdTree::build). */
int dfgtb_create(const double* refs, size_t n, size_t d, const dfgtb_config* cfg,
                 dfgtb_handle** out);
/* Same with refs already in device memory. */
int dfgtb_create_device(const double* d_refs, size_t n, size_t d, const dfgtb_config* cfg,
                        dfgtb_handle** out);
/* float32 points (BASELINE config 5: fp32 inputs, fp64 accumulation): widened exactly
 * to float64 on the device; identical results to dfgtb_create on the widened values. */
int dfgtb_create_f32(const float* refs, size_t n, size_t d, const dfgtb_config* cfg,
                     dfgtb_handle** out);
void dfgtb_destroy(dfgtb_handle* h);

/* DualTreeEngine::compute(queries, h)  engine.cpp:405-424 / engine.hpp:94-95.
 * queries == NULL -> Q = R (the reference tree is reused as query tree).
 * out_sums: nq (or n when Q = R) sums in input order.  stats nullable. */
int dfgtb_compute(dfgtb_handle* h, const double* queries, size_t nq, double bandwidth,
                  double* out_sums, dfgtb_stats* stats);
int dfgtb_compute_device(dfgtb_handle* h, const double* d_queries, size_t nq, double bandwidth,
                         double* d_out_sums, dfgtb_stats* stats);

/* Several bandwidths in ONE lock-step GPU traversal (what a CV sweep does with its
 * h and 2h passes, cv.cpp:156-180): out_sums[b * n_out + i] is the sum at bws[b];
 * stats (nullable) receives nb entries.  Equivalent to nb dfgtb_compute calls. */
int dfgtb_compute_batch(dfgtb_handle* h, const double* queries, size_t nq, const double* bws,
                        size_t nb, double* out_sums, dfgtb_stats* stats);

/* DualTreeEngine::last_stats / p_max  engine.hpp:97-99. */
/* dfgtb_compute_batch with float32 queries (widened exactly on the device; Q != R). */
int dfgtb_compute_batch_f32(dfgtb_handle* h, const float* queries, size_t nq, const double* bws,
                            size_t nb, double* out_sums, dfgtb_stats* stats);
int dfgtb_last_stats(dfgtb_handle* h, dfgtb_stats* stats);
int dfgtb_last_timings(dfgtb_handle* h, dfgtb_timings* t);
int dfgtb_p_max(dfgtb_handle* h);

/* Base-case exp of this handle: 2 = FP32 distance / ex2 / partial sums for the leaf
 * pairs that qualify, MUFU ex2 with FP64 distance and sums for the rest (epsilon >=
 * 5e-3, 3e-4 charged against epsilon); 1 = MUFU ex2 only (epsilon >= 1e-4, 4e-6
 * charged); 0 = FP64 exp (<= ~1 ulp); -1 on a bad handle. */
int dfgtb_base_exp_mode(dfgtb_handle* h);

/* lkcv_from_sums + lscv_from_sums on Q = R sums computed on the device at h and
 * conv_h (cv.cpp:61-97; conv_h = 2h or sqrt(2)h, cv.cpp:27-30).  conv_h <= 0 skips
 * the least-squares score.  Sums never leave the device. */
int dfgtb_cv(dfgtb_handle* h, double bandwidth, double conv_h, dfgtb_cv_row* row);

/* bandwidth_sweep (cv.cpp:141-182) for both scores: rows[i] at scale[i]*base_h.
 * scales must be strictly increasing.  sqrt2 != 0 -> conv_h = sqrt(2) h. */
int dfgtb_sweep(dfgtb_handle* h, const double* scales, size_t ns, double base_h, int sqrt2,
                dfgtb_cv_row* rows);

/* h* of a sweep: lk_best = argmax lk_score, ls_best = argmin ls_score over the rows
 * (first index on ties, the argmin of acceptance.cpp:633-641).
 * Either output pointer may be NULL. */
int dfgtb_sweep_best(const dfgtb_cv_row* rows, size_t ns, size_t* lk_best, size_t* ls_best);

/* CV scores from host sums (lkcv_from_sums / lscv_from_sums, cv.cpp:61-97). */
int dfgtb_lkcv_from_sums(size_t n, size_t d, double bandwidth, const double* sums,
                         double* score, int* clamped);
int dfgtb_lscv_from_sums(size_t n, size_t d, double bandwidth, const double* sums,
                         double conv_h, const double* conv_sums, double* score);

/* Reference tree export for the bit-exact check (KdTree accessors, kdtree.hpp:22-57).
 * Arrays sized by dfgtb_tree_nodes(); begin is int64 like the reference's size_t. */
int dfgtb_tree_nodes(dfgtb_handle* h);
int dfgtb_tree_height(dfgtb_handle* h);
int dfgtb_export_tree(dfgtb_handle* h, int* perm, double* lo, double* hi, double* centroid,
                      double* max_side, int* left, int* right, int* split_dim,
                      double* split_coord, int64_t* begin, int* count);

/* naive_kde (engine.cpp:22-36): exhaustive FP64 sums on the GPU (K12). */
int dfgtb_naive(const double* queries, size_t nq, const double* refs, size_t nr, size_t d,
                double bandwidth, double* out);

/* Series primitives on the GPU (series.cpp), tables in the reference's position
 * layout (p_max^D entries, base-p_max digits, dimension 0 most significant).
 * op: 0 moments(pts n, center a)            -> out table        (series.cpp:238-254)
 *     1 eval_farfield(table in, center a, q b) -> out[0]        (series.cpp:289-303)
 *     2 direct_local(pts n, center a, order) -> out table += ... (series.cpp:305-326)
 *     3 far_to_local(table in, src a, dst b) -> out table += ... (series.cpp:328-353)
 *     4 local_to_local(table in, src a, dst b) -> out table += ...(series.cpp:355-391)
 *     5 eval_local(table in, center a, q b)  -> out[0]          (series.cpp:393-407)
 * For op 0/2 `in` holds n points; otherwise `in` is a table.  `out` is read-modify-
 * written for 2/3/4 like the reference's accumulate-into semantics. */
int dfgtb_series_op(int op, size_t d, int p_max, const double* in, size_t n, const double* a,
                    const double* b, double bandwidth, int order, double* out);

/* choose_best_method (truncation.cpp:130-166) and the least orders farfield_order /
 * local_accum_order / f2l_order (truncation.cpp:98-128) exactly as the traversal
 * evaluates them on the device, for n tuples.  args: n x 9 doubles (n_query, n_ref,
 * max_side_query, max_side_ref, h, tau, p_max, dim, cost_model); out: n x 5 ints
 * (kind: 0 exhaustive, 1 farfield, 2 direct_local, 3 far_to_local -- ApproxChoice::Kind
 * truncation.hpp:43-48; order; p_F; p_D; p_T, 0 = none).  Test entry. */
int dfgtb_choose_methods(size_t n, const double* args, int* out);

/* box_distance_bounds_sq (kdtree.cpp:122-141) as the traversal evaluates it on the
 * device.  boxes: n x 4d doubles (a_lo, a_hi, b_lo, b_hi); out: n x 2 (lo^2, hi^2). */
int dfgtb_box_bounds(size_t n, size_t d, const double* boxes, double* out);

/* Measured FP64 FMA instruction throughput of the device (instr/s); bench roofline. */
double dfgtb_dfma_peak(void);

/* Measured MUFU ex2.approx.f32 throughput (ex2/s); roofline of the MUFU base case. */
double dfgtb_ex2_peak(void);

/* Max relative error of the base case's MUFU exp (used when epsilon >= 1e-4; its
 * bound is charged against epsilon) over every argument it can form; test entry. */
double dfgtb_mufu_exp_error(void);

/* Base-case tasks (32-query chunk x run of reference leaves) of the handle's last
 * compute that ran on the FP32 kernel and on the FP64 kernel, and their (q, r) pairs
 * (pair pointers may be NULL; synchronises). */
int dfgtb_last_base_split(dfgtb_handle* h, int* f32_tasks, int* fp64_tasks, uint64_t* f32_pairs,
                          uint64_t* fp64_pairs);

/* Max relative error of ex2.approx.ftz.f32 -- the FP32 base case's exp (used when
 * epsilon >= 5e-3; kF32Charge) -- over every FP32 argument in [-126, 2^-10]; test entry. */
double dfgtb_f32_exp_error(void);

/* The FP32 base case's term for n (query q_i, reference r_i) pairs, exactly as the
 * kernel forms it: points are D-dimensional, already in z units (|q - r|^2 = z, the
 * term approximates 2^-z), centred on c (D doubles) before rounding to FP32.  out[i]
 * receives the term (test entry for the kF32Charge bound; d in 1..5). */
int dfgtb_f32_terms(size_t d, const double* q, const double* r, const double* c, size_t n, double* out);

/* Device (and pinned host) memory of destroyed handles is cached for reuse by later
 * handles, like PyTorch's caching allocator; this returns it to the driver. */
void dfgtb_release_cached_memory(void);

/* Guard mode (environment variable DFGTB_GUARD set before the first allocation): every
 * device block carries a 4 KB guard band past its end; dfgtb_guard_check() synchronises
 * and returns how many bands were written into (0: no out-of-bounds write seen), -1 when
 * guard mode is off.  dfgtb_guard_selftest() writes one element past a block and returns
 * 1 if the check caught it (test entry).  A debug aid, not part of the reference ABI. */
int dfgtb_guard_check(void);
int dfgtb_guard_selftest(void);

/* Number of visible CUDA devices (0 when none; never raises). */
int dfgtb_device_count(void);

/* The handle's CUDA stream (cudaStream_t as an integer) -- for timing with CUDA
 * events on the stream the kernels run on -- and the number of this library's
 * kernels launched on it since creation. */
uintptr_t dfgtb_stream(dfgtb_handle* h);
uint64_t dfgtb_launch_count(dfgtb_handle* h);

const char* dfgtb_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
