// Shared helpers for the DFGT sm_100a library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace dfgtb {

constexpr int kMaxDim = 16;   // digits packed 4 bits/dim in a uint64
constexpr int kWarp = 32;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct OutOfMemory : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line)
{
  if (e == cudaSuccess) return;
  std::string msg = std::string(what) + " failed at " + file + ":" + std::to_string(line) +
                    ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) throw OutOfMemory(msg);
  throw CudaError(msg);
}
#define CK(x) ::dfgtb::cuda_check((x), #x, __FILE__, __LINE__)
// Every kernel launch of this library is followed by CK_LAUNCH(): it checks the
// launch and counts it (dfgtb_launch_count reports the process-wide total).
uint64_t& launch_counter();
// DFGTB_SYNC_LAUNCH=1 (debugging): wait for the device after every launch, so a faulting
// kernel is reported at its own launch site instead of at the batch's final wait.
bool sync_launch_mode();
#define CK_LAUNCH()                                                                    \
  do {                                                                                 \
    ::dfgtb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);      \
    ++::dfgtb::launch_counter();                                                       \
    if (::dfgtb::sync_launch_mode())                                                   \
      ::dfgtb::cuda_check(cudaDeviceSynchronize(), "kernel execution", __FILE__, __LINE__); \
  } while (0)

// Process-wide caching device allocator (power-of-two size classes, like PyTorch's
// caching allocator): engines created and destroyed in a loop reuse their memory
// instead of paying cudaMalloc/cudaFree each time.  A block returned to the cache
// may still be read by queued kernels, so returning synchronises the device first
// (the guarantee cudaFree gave).  dfgtb_release_cached_memory() empties the cache.
// Blocks are keyed by the device they were allocated on (DevBuf records it), so a
// buffer freed while another device is current returns to its own device's pool.
void* cache_alloc(size_t bytes);
void cache_free(void* p, size_t bytes, int device);
// pinned host blocks, pooled like device memory (engine.cu)
void* pinned_alloc(size_t bytes);
void pinned_free(void* p, size_t bytes);
void cache_release_all();
// Guard mode (DFGTB_GUARD set when the library first allocates): every device block gets a
// kGuardBytes band past its end filled with kGuardByte; guard_check() synchronises and
// counts the bands some kernel wrote into (an out-of-bounds-write detector standing in
// for compute-sanitizer memcheck, which this pool does not run).
bool guard_mode();
int guard_check();
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;
int current_device();

// Makes `dev` current for a scope and restores the previous device afterwards.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev)
  {
    if (dev < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
      return;
    }
    if (prev != dev && cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
  }
  ~DeviceGuard()
  {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Growable device buffer (capacity only ever grows; contents not preserved on growth).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  int dev = -1;  // device the block was allocated on
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release()
  {
    if (p) cache_free(p, cap * sizeof(T), dev);
    p = nullptr;
    cap = 0;
  }
  // ensure room for n elements; growth is geometric
  T* reserve(size_t n)
  {
    if (n <= cap && p) return p;
    size_t c = cap ? cap : 1;
    while (c < n) c *= 2;
    if (c < 256) c = 256;
    release();
    p = static_cast<T*>(cache_alloc(c * sizeof(T)));
    cap = c;
    dev = current_device();
    return p;
  }
};

__host__ __device__ inline int digit_of(uint64_t packed, int d)
{
  return d < kMaxDim ? (int)((packed >> (4 * d)) & 15ull) : 0;
}

// Deterministic warp sum (xor butterfly; identical order on every call).
__device__ inline double warp_sum(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline int warp_sum_i(int v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace dfgtb
