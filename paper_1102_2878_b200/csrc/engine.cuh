// DFGT engine: level-synchronous dual-tree traversal + series/base-case kernels.
#pragma once

#include "series.cuh"
#include "tree.cuh"

#include <functional>
#include <memory>

namespace dfgtb {

struct Config {
  double epsilon = 0.01;
  int leaf_threshold = 20;   // reference default (engine.hpp:19)
  int p_max = 0;             // 0 -> default_p_max(D)
  int cost_model = 0;        // 0 exponential, 1 term_count (truncation.hpp:216)
  int mode = 1;              // 0 centroid (DFD), 1 series (DFGT)
  // 0: every query evaluates the local expansions of all its ancestors directly
  //    (exact re-centering, one kernel); 1: the reference's L2L push-down chain
  //    (post_process, engine.cpp:294-304), one launch per tree level.
  int local_pushdown = 0;
};

// Mirrors TraversalStats (engine.hpp:66-74).
struct Stats {
  unsigned long long kernel_evaluations = 0, pairs_visited = 0, base_cases = 0,
                     prunes_finite_diff = 0, prunes_farfield = 0, prunes_direct_local = 0,
                     prunes_far_to_local = 0;
  int levels = 0;
  unsigned long long pairs_covered = 0;  // sum of |Q| |R| over retired pairs (== |Q| |R_total|)
};

// Device milliseconds of the last compute batch, per phase (CUDA events on the
// engine stream).
struct Timings {
  float tree_ms = 0, traverse_ms = 0, moments_ms = 0, local_ms = 0, base_ms = 0, farfield_ms = 0,
        final_ms = 0, total_ms = 0, base_f32_ms = 0, base_fp64_ms = 0;
};

struct Cnt {
  int e, p, f, dt, t, b, fd;
};

// A work item.  key = slot * K + query node (slot = bandwidth of the batch, K =
// query-tree node count); code = order | kind << 8 (kind 1 F, 2 D, 3 T, 4 base).
struct Item {
  int key, r, code, rank;
};

constexpr int kMaxSlots = 64;  // bandwidths per batch

// Base-case exp on the MUFU (ex2.approx.f32 on an exactly reduced argument, FP64
// distance and accumulation): per-term relative error < kMufuCharge, which the
// traversal pays for by running at eps - kMufuCharge.  Used when eps >= kMufuMinEps
// (the charge is then <= 4% of the budget) unless DFGTB_EXACT_EXP is set; smaller eps
// keep the FP64 exp (<= ~1 ulp).
constexpr double kMufuMinEps = 1e-4;
constexpr double kMufuCharge = 4e-6;
// FP32 base case (execute.cu FPt / base_tile_f32x2): FP32 differences, distance and
// partial sums, ex2.approx.f32 of the whole (shifted) argument.  Applies to leaf pairs whose
// query leaf's box diagonal is <= kF32Diam in units where |q - r|^2 = z = log2 e |q - r|^2 / 2h^2
// and whose sums are >= 1e-20 (Q != R) or >= 1 (Q = R, the self term; see base_flags);
// per-term relative error < kF32Charge (derivation at FPt).  Terms are formed as
// 2^(kF32Shift - z) and scaled back by kF32Unshift per tile.  Used when eps >= kF32MinEps
// (the charge is then <= 5% of the budget) unless DFGTB_NO_F32 is set.
constexpr double kF32MinEps = 5e-3;
constexpr double kF32Charge = 2e-4;
constexpr double kF32Diam = 150.0;
constexpr float kF32Shift = 64.0f;
constexpr double kF32Unshift = 0x1p-64;

int default_p_max(int D);

class Engine {
public:
  Engine(const double* h_refs, size_t n, size_t d, const Config& cfg, bool refs_on_device = false);
  ~Engine();

  // Sums for `nb` bandwidths at once (one lock-step traversal, batched kernels):
  // d_out[b * nq + i] = G_{h_b}(q_i) in input order.  d_queries nullptr -> Q = R.
  void compute_batch(const double* d_queries, size_t nq, const double* h, int nb, double* d_out);
  void compute_device(const double* d_queries, size_t nq, double h, double* d_out)
  {
    compute_batch(d_queries, nq, &h, 1, d_out);
  }
  void compute_host(const double* h_queries, size_t nq, double h, double* h_out);

  // CV reductions of Q = R sums on device, for `ns` scales at once:
  // lk[k], clamped[k] from d_sums + k*n at h[k]; ls[k] uses d_conv + k*n at conv_h[k]
  // (d_conv may be nullptr -> no LS).
  void cv_reduce(const double* d_sums, const double* h, const double* d_conv, const double* conv_h,
                 int ns, double* lk, int* clamped, double* ls);
  // compute_batch (Q = R) with the CV reduction queued behind it: one host wait for both
  void compute_batch_cv(const double* h, int nb, double* d_out, const double* bw, const double* conv_h,
                        int ns, double* lk, int* clamped, double* ls);
  void cv_enqueue(const double* d_sums, const double* h, const double* d_conv, const double* conv_h, int ns);
  void cv_collect(int ns, double* lk, int* clamped, double* ls) const;

  const Stats& last_stats(int slot = 0) const { return slot_stats_[slot]; }
  const Timings& last_timings() const { return tim_; }
  // device time of the engine's one-time moment kernels (K2/K3; waits for them)
  float moments_build_ms();
  const DevTree& ref_tree() const { return rt_; }
  int p_max() const { return ser_.pmax; }
  bool mufu_exp() const { return mufu_; }
  bool f32_exp() const { return f32_; }
  // tasks of the last batch's base case on the FP32 / FP64 kernels (synchronises)
  void base_split(int& f32_tasks, int& fp64_tasks, unsigned long long& f32_pairs,
                  unsigned long long& fp64_pairs);
  // the share of eps the base case's reduced-precision exp is charged
  double exp_charge() const { return f32_ ? kF32Charge : mufu_ ? kMufuCharge : 0.0; }
  int dim() const { return D_; }
  size_t n() const { return n_; }
  cudaStream_t stream() const { return s_; }
  int device() const { return dev_; }
  // Make the engine's stream wait for everything queued so far on the legacy default
  // stream (where callers of the *_device entry points typically produced their inputs).
  void wait_legacy_stream();
  const SeriesTables& series() const { return ser_; }
  DevSeries dev_series() const;
  const double* d_refs() const { return x_.p; }

private:
  void traverse(const DevTree& qt, const double* h, int nb);
  void traverse_fetch_async();  // the traversal state to the pinned host copy, on s_
  bool traverse_finish(bool prefetched = false);
  void run_levels(const void* trav_args, const std::vector<const void*>& sig);
  void destroy_graph();
  void run_phases(const DevTree& qt, const double* h, int nb, double* d_out);
  void launch_phases(const DevTree& qt, const double* h, int nb, double* d_out);
  void eager_moments();
  void setup_leaves(const DevTree& t);
  void start_frontier(const DevTree& qt, void* trav_args);

  Config cfg_;
  int dev_ = -1;  // device the engine was created on (made current by every entry point)
  int D_ = 0;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
  cudaStream_t s2_ = nullptr;  // local expansions + far field run beside the base case
  int base_cta_slack_ = 0;     // base-case CTA slots per SM left to s2_ (DFGTB_BASE_SLACK; 0 measured best)
  bool one_stream_ = false;    // DFGTB_ONE_STREAM: the s2_ chain on s_ too (serialised; per-kernel timings
                               // without SM sharing; measured 10% slower on cfg2 than the overlap)
  DevBuf<double> x_;        // reference points (original order)
  DevTree rt_;              // reference tree
  DevTree qt_tmp_;          // query tree (Q != R)
  DevBuf<double> qx_;       // query points (Q != R)
  SeriesTables ser_;
  DevBuf<unsigned char> ser_dev_;
  std::vector<unsigned char> ser_blob_;  // host source of ser_dev_'s upload
  DevBuf<int> leaves_, leaf_of_pos_;  // of the current query tree
  DevBuf<int> mom_node_, mom_start_, mom_off_;  // eager moments: chunk lists
  DevBuf<double> mom_part_;                     // eager moments: chunk partials
  std::vector<int> qleaves_host_;
  int leaves_src_ = -1;     // 0: leaves_ describe the reference tree, 1: a query tree
  // per batch (node-indexed arrays are slot-major: key = slot * K + node)
  DevBuf<double> L_, Mt_, s_ff_;      // Mt_: UNSCALED reference moments (h-independent)
  DevBuf<int> Lord_, mflag_, mdone_;
  // per-key item counts and their exclusive scans, F | DT | B back to back (one scan and
  // one scatter launch sort all three item kinds); the names view the three segments
  DevBuf<int> cntAll_, offAll_, offLoc_;
  struct IntView {
    int* p = nullptr;
  } cntF_, cntDT_, cntB_, offF_, offDT_, offB_;
  bool eager_ = false;                // Mt_ holds every node (tables <= 4096 terms)
  DevBuf<int> lnch_, lchoff_, lchunk_, tasks_, leaf_task_, leaf_runs_, brec_, bnext_;
  DevBuf<double> lpart_, bpart_, xq_, xr_, slotp_;
  // frontier (double buffered) and per-level scratch
  DevBuf<int> fq_[2], foff_[2], flen_[2], fr_[2], pent_[2];
  DevBuf<double> fbase_[2];
  DevBuf<double> pkmax_, pkmin_;
  DevBuf<int> dec_, childlen_;
  DevBuf<double> newbase_, pglo_;
  DevBuf<Cnt> cnt_, cntoff_, ctsum_, ctoff_, lvlcnt_;
  DevBuf<Item> itF_, itDT_, itB_, sF_, sDT_, sB_;
  DevBuf<unsigned char> scan_tmp_, scan_tmp2_;
  DevBuf<double> red_;
  DevBuf<unsigned long long> trace_;  // DFGTB_TRACE=1: per-level phase timestamps
  DevBuf<unsigned long long> lvlep_;  // per-level packed entry/pair counters (traversal)
  // device-driven level loop: state (device + pinned host mirror), capacities, graph
  void* hst_ = nullptr;
  void* hpin_ = nullptr;  // pinned: the batch's device counts (8 ints) | CV partial sums (run_phases, cv_*)
  std::function<void()> post_batch_;  // queued after a batch's last kernel, before its one host wait
  size_t hst_bytes_ = 0;
  DevBuf<unsigned char> dst_;
  int capE_ = 0, capP_ = 0, capF_ = 0, capDT_ = 0, capB_ = 0;
  DevBuf<int> sfront_;           // start frontier node lists (DFGTB_TRAV_START_DEPTH)
  bool use_persistent_ = true;  // one cooperative kernel runs every level
  bool use_graph_ = true;       // else: CUDA-graph WHILE loop; else host loop
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t gexec_ = nullptr;
  cudaGraphConditionalHandle hc_ = 0;
  std::vector<const void*> gsig_;
  cudaEvent_t ev_[16];
  cudaStream_t s3_ = nullptr;  // the FP64 base-case kernel beside the FP32 one
  cudaEvent_t fork3_ = nullptr, join3_ = nullptr;
  cudaStream_t s4_ = nullptr;  // the base case's preparation kernels (highest priority)
  cudaEvent_t prep_ev_ = nullptr;
  cudaEvent_t fork_ = nullptr, join_ = nullptr;
  cudaEvent_t legacy_ev_ = nullptr;
  cudaEvent_t mom_ev_[2] = { nullptr, nullptr };  // around the eager moment kernels (s2_)  // orders s_ after the legacy stream (wait_legacy_stream)
  std::vector<Stats> slot_stats_;
  Timings tim_;
  long long nF_ = 0, nDT_ = 0, nB_ = 0;
  int nb_ = 1;
  bool mufu_ = false;
  bool f32_ = false;
  bool base_conc_ = false;  // the last batch ran the two base-case kernels side by side
  const DevTree* last_q_ = nullptr;  // query tree and node count of the last batch (diagnostics)
  int last_K_ = 0;
  // device-side counts of a batch (no host round trip until its end):
  // [0] nF [1] nDT [2] nB [3] traversal overflow [4] local chunks [5] base tasks
  DevBuf<int> bc_;
  int trav_nb_ = 0;
  int trav_nq_ = 0;  // query points of the batch being traversed
  bool trav_trace_ = false;
  int capCh_ = 0, capTask_ = 0;  // local chunks / base tasks (grown on overflow)
};

// Exhaustive FP64 sums on the device (K12, naive_kde engine.cpp:22-36).
void naive_device(const double* d_q, size_t nq, const double* d_r, size_t nr, int D, double h,
                  double* d_out, cudaStream_t s);

// Measured FP64 FMA throughput (instr/s) -- roofline denominator for bench.py.
double measure_dfma_peak(int device);
// Measured MUFU ex2.approx.f32 throughput (ex2/s) -- the MUFU base case's roofline.
double measure_ex2_peak(int device);
// Max relative error of the base case's MUFU exp over every argument it can form.
double mufu_exp_max_error();
// Per leaf of t: the largest squared distance of a point to its nearest other point in
// the leaf (+inf for internal nodes and 1-point leaves).
// Max relative error of ex2.approx.ftz.f32 over every FP32 argument in [-126, 2^-10].
double f32_exp_max_error();
// The FP32 base case's term for host pairs (test entry; points in z units, stride d).
void f32_terms_host(int d, const double* q, const double* r, const double* c, size_t n, double* out);

// Series term tables -> one device blob, and the device view over it.
void upload_series(const SeriesTables& t, DevBuf<unsigned char>& dev, cudaStream_t s,
                   std::vector<unsigned char>* keep = nullptr);
DevSeries series_view(const SeriesTables& t, const DevBuf<unsigned char>& dev);

// Pinned host blocks (cached like device memory; engine.cu).
constexpr size_t kHostPinBytes = 64 + sizeof(double) * 148 * 3 * kMaxSlots;  // Engine::hpin_
void* pinned_alloc(size_t bytes);
void pinned_free(void* p, size_t bytes);

// Constant-bank coefficients of the base case's exp (execute.cu).
void init_exp_constants(cudaStream_t s);
// Constant tables of the error bounds (traverse.cu).
void init_truncation_tables(cudaStream_t s);
void init_truncation_tables_small(cudaStream_t s);  // traverse_small.cu's copies
void* traverse_small_kernel(int D);
int traverse_small_block();
// batches with fewer slot x query points than this run the 768-thread traversal
constexpr long long kTravSmallWork = 1000000;
// Both of the above, once per device and process (engine.cu).
void init_device_constants(cudaStream_t s);
// Test entries (traverse.cu): choose_best_method / the least orders and
// box_distance_bounds_sq exactly as the traversal evaluates them on the device.
//   args: n x 9 (nq, nr, sq, sr, h, tau, p_max, d, cost) -> out: n x 5 (kind, order, pf, pd, pt)
void choose_methods_device(size_t n, const double* args, int* out);
//   boxes: n x 4d (alo, ahi, blo, bhi) -> out: n x 2 (lo^2, hi^2)
void box_bounds_device(size_t n, int d, const double* boxes, double* out);

}  // namespace dfgtb
