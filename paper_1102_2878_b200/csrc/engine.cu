// DFGT engine host side: construction (GPU tree, moments), batched compute, CV.
//
// Reference: DualTreeEngine (engine.cpp:352-424).  The engine builds the reference
// tree once (KdTree::build, bit-exact on the GPU) and -- unlike the reference, which
// recomputes moments per bandwidth (moments_for, engine.cpp:368-403) -- computes the
// h-independent unscaled moments once.  compute_batch runs any number of bandwidths
// through ONE lock-step traversal (traverse.cu) and batched execution kernels
// (execute.cu); a single compute() is a batch of one.
#include "internal.cuh"

#include <cstdlib>

#include <cstring>
#include <mutex>
#include <unordered_map>

namespace dfgtb {

uint64_t& launch_counter()
{
  static uint64_t n = 0;
  return n;
}

// ---------------------------------------------------------- caching allocators
// Device blocks are cached per (device, size).  A freed block may still be in use by
// work queued on its owner's streams, so frees go to a pending list and become
// reusable after ONE device synchronisation, taken only when an allocation could
// reuse them (not one synchronisation per free: an engine releases ~40 buffers).
namespace {
std::mutex g_cache_mu;
std::unordered_map<uint64_t, std::vector<void*>>& dev_cache()
{
  static auto* c = new std::unordered_map<uint64_t, std::vector<void*>>();  // never destroyed
  return *c;
}
std::vector<std::pair<uint64_t, void*>>& dev_pending()
{
  static auto* c = new std::vector<std::pair<uint64_t, void*>>();
  return *c;
}
std::unordered_map<size_t, std::vector<void*>>& host_cache()
{
  static auto* c = new std::unordered_map<size_t, std::vector<void*>>();
  return *c;
}
uint64_t cache_key(size_t bytes, int dev) { return ((uint64_t)bytes << 8) | (uint64_t)(dev & 0xff); }
std::unordered_map<void*, std::pair<size_t, int>>& guard_blocks()  // block -> (bytes, device)
{
  static auto* c = new std::unordered_map<void*, std::pair<size_t, int>>();
  return *c;
}
void* take_cached(uint64_t key)  // g_cache_mu held
{
  auto it = dev_cache().find(key);
  if (it == dev_cache().end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  return p;
}
}  // namespace

int current_device()
{
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return dev;
}

void* cache_alloc(size_t bytes)
{
  const int dev = current_device();
  const uint64_t key = cache_key(bytes, dev);
  {
    std::unique_lock<std::mutex> g(g_cache_mu);
    if (void* p = take_cached(key)) return p;
    bool match = false;
    for (const auto& e : dev_pending()) match = match || e.first == key;
    if (match) {
      // Only the blocks of THIS device pending before the synchronisation are known
      // idle afterwards (cudaDeviceSynchronize covers the current device only).
      std::vector<std::pair<uint64_t, void*>> idle, keep;
      for (auto& e : dev_pending()) ((int)(e.first & 0xff) == (dev & 0xff) ? idle : keep).push_back(e);
      dev_pending().swap(keep);
      g.unlock();
      if (cudaDeviceSynchronize() != cudaSuccess) cudaGetLastError();
      g.lock();
      for (auto& e : idle) dev_cache()[e.first].push_back(e.second);
      if (void* p = take_cached(key)) return p;
    }
  }
  void* p = nullptr;
  const size_t extra = guard_mode() ? kGuardBytes : 0;
  cudaError_t e = cudaMalloc(&p, bytes + extra);
  if (e == cudaErrorMemoryAllocation) {  // give the cache back and retry once
    cudaGetLastError();
    cache_release_all();
    e = cudaMalloc(&p, bytes + extra);
  }
  CK(e);
  if (extra) {
    CK(cudaMemset(static_cast<unsigned char*>(p) + bytes, kGuardByte, kGuardBytes));
    std::lock_guard<std::mutex> g(g_cache_mu);
    guard_blocks()[p] = { bytes, dev };
  }
  return p;
}

bool sync_launch_mode()
{
  static const bool on = std::getenv("DFGTB_SYNC_LAUNCH") != nullptr;
  return on;
}

bool guard_mode()
{
  static const bool on = std::getenv("DFGTB_GUARD") != nullptr;
  return on;
}

int guard_check()
{
  if (!guard_mode()) return -1;
  std::vector<std::pair<void*, std::pair<size_t, int>>> blocks;
  {
    std::lock_guard<std::mutex> g(g_cache_mu);
    blocks.assign(guard_blocks().begin(), guard_blocks().end());
  }
  const int cur = current_device();
  std::vector<unsigned char> band(kGuardBytes);
  int bad = 0;
  for (const auto& b : blocks) {
    CK(cudaSetDevice(b.second.second));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(band.data(), static_cast<unsigned char*>(b.first) + b.second.first, kGuardBytes,
                  cudaMemcpyDeviceToHost));
    for (unsigned char c : band)
      if (c != kGuardByte) {
        ++bad;
        break;
      }
  }
  CK(cudaSetDevice(cur));
  return bad;
}

void cache_free(void* p, size_t bytes, int device)
{
  const uint64_t key = cache_key(bytes, device >= 0 ? device : current_device());
  std::lock_guard<std::mutex> g(g_cache_mu);
  dev_pending().emplace_back(key, p);
}

void cache_release_all()
{
  std::lock_guard<std::mutex> g(g_cache_mu);
  const int cur = current_device();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) cudaGetLastError();
  for (int d = 0; d < ndev; ++d)  // every device's queued work must be idle first
    if (cudaSetDevice(d) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) cudaGetLastError();
  auto free_on = [](uint64_t key, void* p) {
    if (cudaSetDevice((int)(key & 0xff)) != cudaSuccess) cudaGetLastError();
    cudaFree(p);
    guard_blocks().erase(p);
  };
  for (auto& kv : dev_cache())
    for (void* p : kv.second) free_on(kv.first, p);
  dev_cache().clear();
  for (auto& e : dev_pending()) free_on(e.first, e.second);
  dev_pending().clear();
  if (ndev > 0 && cudaSetDevice(cur) != cudaSuccess) cudaGetLastError();
  for (auto& kv : host_cache())
    for (void* p : kv.second) cudaFreeHost(p);
  host_cache().clear();
}

void* pinned_alloc(size_t bytes)
{
  {
    std::lock_guard<std::mutex> g(g_cache_mu);
    auto it = host_cache().find(bytes);
    if (it != host_cache().end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  CK(cudaMallocHost(&p, bytes));
  return p;
}

void pinned_free(void* p, size_t bytes)
{
  std::lock_guard<std::mutex> g(g_cache_mu);
  host_cache()[bytes].push_back(p);
}

// Streams and events are pooled per device like memory: creating / destroying them
// costs ~0.1-0.2 ms per engine, which a CV call that builds an engine per dataset pays
// every time.
struct StreamSet {
  cudaStream_t s = nullptr, s2 = nullptr, s3 = nullptr, s4 = nullptr;
  cudaEvent_t ev[16] = {}, fork = nullptr, join = nullptr, fork3 = nullptr, join3 = nullptr, prep = nullptr,
              legacy = nullptr, mom0 = nullptr, mom1 = nullptr;
};
static std::unordered_map<int, std::vector<StreamSet>>& stream_pool()
{
  static auto* p = new std::unordered_map<int, std::vector<StreamSet>>();
  return *p;
}

static StreamSet acquire_streams()
{
  int dev = 0;
  CK(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> g(g_cache_mu);
    auto& v = stream_pool()[dev];
    if (!v.empty()) {
      StreamSet r = v.back();
      v.pop_back();
      return r;
    }
  }
  StreamSet r;
  // Stream priorities.  After the traversal three chains run side by side: the local
  // expansions (s2: chunks -> reduce; the longest chain, it ends the batch), the far field
  // (s3) and the base case (s).  Default (2): s2 above the others, so the critical chain
  // is never queued behind the base-case kernels' CTAs (measured: cfg2 sweep -2%, cfg3
  // -1.8% against equal priorities; the base-case kernels then run at their isolated
  // rates).  DFGTB_STREAM_PRIO: 0 = equal, 1 = s high, 2 = s2 high, 3 = s2 > s3 > s,
  // 4 = s2 > s > s3.
  static const int prio = std::getenv("DFGTB_STREAM_PRIO") ? std::atoi(std::getenv("DFGTB_STREAM_PRIO")) : 2;
  int plo = 0, phi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&plo, &phi));  // phi = greatest priority (lowest number)
  const int pmid = plo > phi ? plo - 1 : plo;
  const int ps = prio == 1 ? phi : prio == 4 ? pmid : plo;
  const int ps2 = prio >= 2 ? phi : plo;
  const int ps3 = prio == 3 ? pmid : plo;
  CK(cudaStreamCreateWithPriority(&r.s, cudaStreamNonBlocking, ps));
  CK(cudaStreamCreateWithPriority(&r.s2, cudaStreamNonBlocking, ps2));
  CK(cudaStreamCreateWithPriority(&r.s3, cudaStreamNonBlocking, ps3));
  // s4: the base case's short preparation kernels (task lists, records, scaled points),
  // above everything so they are not queued behind the expansion kernels' CTAs
  CK(cudaStreamCreateWithPriority(&r.s4, cudaStreamNonBlocking, phi));
  CK(cudaEventCreateWithFlags(&r.prep, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&r.fork3, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&r.join3, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&r.legacy, cudaEventDisableTiming));
  CK(cudaEventCreate(&r.mom0));
  CK(cudaEventCreate(&r.mom1));
  for (auto& e : r.ev) CK(cudaEventCreate(&e));
  return r;
}

static void release_streams(const StreamSet& r)
{
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> g(g_cache_mu);
  stream_pool()[dev].push_back(r);
}

// __constant__ tables (exp coefficients, truncation bounds) are per device and
// h-independent: uploaded once per device and process.
void init_device_constants(cudaStream_t s)
{
  static std::mutex mu;
  static std::unordered_map<int, bool> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return;
  init_exp_constants(s);
  init_truncation_tables(s);
  init_truncation_tables_small(s);
  CK(cudaStreamSynchronize(s));
  done[dev] = true;
}

int default_p_max(int D)
{  // truncation.cpp:168-186
  switch (D) {
  case 1: return 8;
  case 2: return 6;
  case 3: return 4;
  case 4:
  case 5: return 2;
  default: return 1;
  }
}

Engine::Engine(const double* refs, size_t n, size_t d, const Config& cfg, bool on_device)
  : cfg_(cfg)
{
  // argument checks first: they must not depend on a GPU being present
  if (n == 0 || d == 0) throw InvalidArgument("PointSet requires N >= 1 and D >= 1");
  if (n > (size_t)INT32_MAX / 2) throw InvalidArgument("N too large for 32-bit node ids");
  if (cfg.epsilon < 0.0) throw InvalidArgument("epsilon must be >= 0");
  if (cfg.leaf_threshold < 1) throw InvalidArgument("leaf_threshold must be >= 1");
  if (cfg.p_max < 0 || (cfg.mode == 1 && cfg.p_max > 15))
    throw InvalidArgument("SeriesGeometry requires dim >= 1 and 1 <= p_max <= 15");
  D_ = (int)d;
  n_ = n;
  dev_ = current_device();
  if (const char* sl = std::getenv("DFGTB_BASE_SLACK")) base_cta_slack_ = std::atoi(sl);
  one_stream_ = std::getenv("DFGTB_ONE_STREAM") != nullptr;
  mufu_ = cfg.epsilon >= kMufuMinEps && D_ <= 5 && std::getenv("DFGTB_EXACT_EXP") == nullptr;
  f32_ = mufu_ && cfg.epsilon >= kF32MinEps && std::getenv("DFGTB_NO_F32") == nullptr;
  const int pm = cfg.mode == 0 ? 1 : (cfg.p_max > 0 ? cfg.p_max : default_p_max(D_));
  ser_ = SeriesTables(D_, pm);
  if (D_ * (pm - 1) >= 128) throw InvalidArgument("D * (p_max - 1) must be < 128");
  if (D_ > kMaxDim) throw InvalidArgument("dimension > 16 is not supported by the device engine");
  {
    const StreamSet ss = acquire_streams();
    s_ = ss.s;
    s2_ = ss.s2;
    fork_ = ss.fork;
    join_ = ss.join;
    for (int i = 0; i < 16; ++i) ev_[i] = ss.ev[i];
    s3_ = ss.s3;
    s4_ = ss.s4;
    prep_ev_ = ss.prep;
    fork3_ = ss.fork3;
    join3_ = ss.join3;
    legacy_ev_ = ss.legacy;
    mom_ev_[0] = ss.mom0;
    mom_ev_[1] = ss.mom1;
  }
  x_.reserve(n * d);
  if (on_device) wait_legacy_stream();  // the caller's producer of refs
  CK(cudaMemcpyAsync(x_.p, refs, sizeof(double) * n * d,
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s_));
  upload_series(ser_, ser_dev_, s_, &ser_blob_);
  init_device_constants(s_);
  CK(cudaEventRecord(ev_[0], s_));
  build_tree(rt_, x_.p, (int)n, D_, cfg.leaf_threshold, s_);
  CK(cudaEventRecord(ev_[1], s_));  // tree_ms: the tree build (the upload precedes ev_[0])
  if (std::getenv("DFGTB_TRACE")) {
    CK(cudaEventRecord(ev_[2], s_));
    CK(cudaEventSynchronize(ev_[2]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev_[0], ev_[2]));
    std::fprintf(stderr, "DFGTB_TRACE create: upload+tree %.3f ms\n", ms);
  }
  if (cfg.mode == 1) {
    if (ser_.T <= 4096) {
      eager_ = true;
      eager_moments();
    } else {
      Mt_.reserve((size_t)rt_.nodes * ser_.T);
      mdone_.reserve(rt_.nodes);
      CK(cudaMemsetAsync(mdone_.p, 0, sizeof(int) * rt_.nodes, s_));
    }
  }
  // the Q = R leaf list now, while the device builds the moments (the first batch finds it
  // ready; a Q != R batch replaces it)
  setup_leaves(rt_);
  leaves_src_ = 0;
  CK(cudaStreamSynchronize(s_));
  CK(cudaEventElapsedTime(&tim_.tree_ms, ev_[0], ev_[1]));
  slot_stats_.assign(1, Stats{});
}

Engine::~Engine()
{
  DeviceGuard dg(dev_);  // streams go back to this device's pool
  if (s_) cudaStreamSynchronize(s_);
  destroy_graph();
  if (hst_) pinned_free(hst_, hst_bytes_);
  if (hpin_) pinned_free(hpin_, kHostPinBytes);
  if (s2_) cudaStreamSynchronize(s2_);
  if (s_) {
    StreamSet ss;
    ss.s = s_;
    ss.s2 = s2_;
    ss.fork = fork_;
    ss.join = join_;
    for (int i = 0; i < 16; ++i) ss.ev[i] = ev_[i];
    ss.s3 = s3_;
    ss.s4 = s4_;
    ss.prep = prep_ev_;
    ss.fork3 = fork3_;
    ss.join3 = join3_;
    ss.legacy = legacy_ev_;
    ss.mom0 = mom_ev_[0];
    ss.mom1 = mom_ev_[1];
    release_streams(ss);  // pooled for the next engine on this device
  }
}

DevSeries Engine::dev_series() const { return series_view(ser_, ser_dev_); }

void upload_series(const SeriesTables& t, DevBuf<unsigned char>& dev, cudaStream_t s,
                   std::vector<unsigned char>* keep)
{
  const int T = t.T;
  const size_t bytes = sizeof(uint64_t) * T + sizeof(double) * 2 * T + sizeof(int) * 3 * T;
  dev.reserve(bytes);
  // keep != nullptr: the caller owns the upload's source and orders itself on `s` (no
  // host wait here: the engine's point upload is in flight on the same stream)
  std::vector<unsigned char> local;
  std::vector<unsigned char>& blob = keep ? *keep : local;
  blob.assign(bytes, 0);
  unsigned char* p = blob.data();
  std::memcpy(p, t.dig.data(), sizeof(uint64_t) * T);
  p += sizeof(uint64_t) * T;
  std::memcpy(p, t.invf.data(), sizeof(double) * T);
  p += sizeof(double) * T;
  std::memcpy(p, t.fact.data(), sizeof(double) * T);
  p += sizeof(double) * T;
  std::memcpy(p, t.degree.data(), sizeof(int) * T);
  p += sizeof(int) * T;
  std::memcpy(p, t.term_of_pos.data(), sizeof(int) * T);
  p += sizeof(int) * T;
  std::memcpy(p, t.pos.data(), sizeof(int) * T);
  CK(cudaMemcpyAsync(dev.p, blob.data(), bytes, cudaMemcpyHostToDevice, s));
  if (!keep) CK(cudaStreamSynchronize(s));
}

DevSeries series_view(const SeriesTables& t, const DevBuf<unsigned char>& dev)
{
  const int T = t.T;
  const unsigned char* p = dev.p;
  DevSeries g;
  g.D = t.D;
  g.pmax = t.pmax;
  g.T = T;
  g.dig = (const uint64_t*)p;
  p += sizeof(uint64_t) * T;
  g.invf = (const double*)p;
  p += sizeof(double) * T;
  g.fact = (const double*)p;
  p += sizeof(double) * T;
  g.degree = (const int*)p;
  p += sizeof(int) * T;
  g.term_of_pos = (const int*)p;
  p += sizeof(int) * T;
  g.pos = (const int*)p;
  return g;
}

void Engine::wait_legacy_stream()
{
  DeviceGuard dg(dev_);
  CK(cudaEventRecord(legacy_ev_, cudaStreamLegacy));
  CK(cudaStreamWaitEvent(s_, legacy_ev_, 0));
}

void Engine::compute_batch(const double* d_queries, size_t nq, const double* h, int nb,
                           double* d_out)
{
  DeviceGuard dg(dev_);
  if (nb < 1 || nb > kMaxSlots) throw InvalidArgument("batch size outside [1, 64]");
  for (int b = 0; b < nb; ++b) {
    if (!(h[b] > 0.0)) throw InvalidArgument("bandwidth must be positive");
    if (!std::isfinite(h[b])) throw InvalidArgument("bandwidth must be positive and finite");
  }
  const DevTree* qt = &rt_;
  if (d_queries) {
    if (nq == 0) throw InvalidArgument("PointSet requires N >= 1 and D >= 1");
    build_tree(qt_tmp_, d_queries, (int)nq, D_, cfg_.leaf_threshold, s_);  // engine.cpp:417
    qt = &qt_tmp_;
    setup_leaves(*qt);
    leaves_src_ = 1;
  } else if (leaves_src_ != 0) {
    setup_leaves(rt_);  // Q = R: the reference tree doubles as the query tree
    leaves_src_ = 0;
  }
  run_phases(*qt, h, nb, d_out);
}

float Engine::moments_build_ms()
{
  if (!eager_) return 0.f;
  DeviceGuard dg(dev_);
  float ms = 0.f;
  CK(cudaEventSynchronize(mom_ev_[1]));
  CK(cudaEventElapsedTime(&ms, mom_ev_[0], mom_ev_[1]));
  return ms;
}

void Engine::compute_host(const double* h_queries, size_t nq, double h, double* h_out)
{
  DeviceGuard dg(dev_);
  const size_t n_out = h_queries ? nq : n_;
  DevBuf<double> out;
  out.reserve(n_out);
  if (h_queries) {
    qx_.reserve(nq * D_);
    CK(cudaMemcpyAsync(qx_.p, h_queries, sizeof(double) * nq * D_, cudaMemcpyHostToDevice, s_));
  }
  compute_device(h_queries ? qx_.p : nullptr, nq, h, out.p);
  CK(cudaMemcpyAsync(h_out, out.p, sizeof(double) * n_out, cudaMemcpyDeviceToHost, s_));
  CK(cudaStreamSynchronize(s_));
}

}  // namespace dfgtb
