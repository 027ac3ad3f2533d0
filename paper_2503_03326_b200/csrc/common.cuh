// common.cuh — shared host/device infrastructure of libocean_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ocean_b200.h"

// NVTX v3 (header-only; a no-op unless a tool such as Nsight attaches)
#include <nvtx3/nvToolsExt.h>

namespace ocn {

constexpr double kPi = 3.14159265358979323846;
constexpr double kGravity = 9.80665;

// Status-carrying exception used inside the library; every extern "C" entry
// converts it to an int status + ocn_last_error message (abi.cu).
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Error(status, buf);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    fail(OCN_ERR_CUDA, "CUDA error in %s (%s:%d): %s", what, file, line, cudaGetErrorString(e));
}
#define OCN_CUDA(x) ::ocn::cuda_check((x), #x, __FILE__, __LINE__)
// After every kernel launch: catches missing kernel images / bad configs.
#define OCN_LAUNCHED(ctx)                                                       \
  do {                                                                          \
    ::ocn::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
    (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                    \
  } while (0)

// Device allocation owned by RAII.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p, n = o.n;
    o.p = nullptr, o.n = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    OCN_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Pinned host staging buffer.
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void* ensure(size_t b) {
    if (b > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      OCN_CUDA(cudaMallocHost(&p, b));
      bytes = b;
    }
    return p;
  }
};


// Opt a kernel into `bytes` of dynamic shared memory on the current device,
// once per (device, kernel, size): the attribute lives in the device context,
// so a process-wide flag would leave a second device's context without it.
// Thread-safe (spectral.cu).
void smem_opt_in(const void* func, int bytes);
template <class F>
inline void smem_opt_in(F* func, size_t bytes) {
  smem_opt_in(reinterpret_cast<const void*>(func), (int)bytes);
}

}  // namespace ocn

// The context: one device, one stream, reusable scratch.
struct ocn_prof_window {
  cudaEvent_t start, stop;
  int cat;
};
struct ocn_ctx {
  bool profiling = false;
  int prof_mode = 0;  // 1: per-kernel windows (eager), 2: stage windows (graphs kept)
  std::vector<ocn_prof_window> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  double prof_ms[OCN_PROF_COUNT] = {0};
  uint64_t prof_count[OCN_PROF_COUNT] = {0};
  int device = 0;
  std::atomic<int> refs{1};  // owner + every handle created on it (freed at zero)
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  int priority = 0;  // ocn_ctx_create_priority: -1 low (work beside a higher-priority stream), 0, 1
  std::string last_error;
  std::atomic<uint64_t> launches{0};
  ocn::PinnedBuf pinned;
  ocn::DevBuf<unsigned char> scratch;  // generic per-call device scratch
};

namespace ocn {

// Scoped device guard for a context.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const ocn_ctx* c) {
    // never throws: also used on destruction paths (handles freed at exit)
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != c->device) cudaSetDevice(c->device);
    cudaGetLastError();
  }
  ~DeviceScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// RAII profiling window over a stretch of launches on ctx->stream.
struct ProfWindow {
  ocn_ctx* ctx;
  int cat;
  cudaEvent_t stop = nullptr;
  static cudaEvent_t get(ocn_ctx* c) {
    if (!c->prof_pool.empty()) {
      cudaEvent_t e = c->prof_pool.back();
      c->prof_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    OCN_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t start = nullptr;
  ProfWindow(ocn_ctx* c, int k) : ctx(c), cat(k) {
    if (!ctx->profiling || k < 0) return;
    start = get(ctx);
    OCN_CUDA(cudaEventRecord(start, ctx->stream));
  }
  ~ProfWindow() {
    if (!start) return;
    stop = get(ctx);
    cudaEventRecord(stop, ctx->stream);
    ctx->prof_pending.push_back({start, stop, cat});
  }
};

inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
inline int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// true when p is device (or managed) memory.
inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Input staging for the batched samplers: host or device pointer in, device pointer out.
struct InStage {
  const void* dev = nullptr;
  DevBuf<unsigned char> own;
  InStage(ocn_ctx* ctx, const void* p, size_t bytes) {
    if (is_device_ptr(p)) {
      dev = p;
    } else {
      own.alloc(bytes);
      OCN_CUDA(cudaMemcpyAsync(own.p, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
      dev = own.p;
    }
  }
};

struct OutStage {
  void* user;
  void* dev = nullptr;
  size_t bytes;
  bool host;
  DevBuf<unsigned char> own;
  ocn_ctx* ctx;
  OutStage(ocn_ctx* c, void* p, size_t b) : user(p), bytes(b), ctx(c) {
    host = !is_device_ptr(p);
    if (host) {
      own.alloc(b);
      dev = own.p;
    } else {
      dev = p;
    }
  }
  // copies back (and synchronizes) for host outputs
  void finish() {
    if (host) {
      OCN_CUDA(cudaMemcpyAsync(user, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  }
};

}  // namespace ocn

namespace ocn {
// NVTX range over a C-ABI stage (names follow the reference's stages:
// sim.hpp:50-54 surface / velocity / hydro / zones / integrate)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace ocn
