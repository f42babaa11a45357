// Context, device buffers and tensor handles.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace ctdgpu {

struct Ctx;
// Contexts alive in this process.  A buffer owned by an object the caller
// destroys after its context (e.g. at interpreter shutdown) is then left to
// process teardown instead of being freed through a dead stream.
inline std::mutex& ctx_registry_mutex() {
  static std::mutex m;
  return m;
}
inline std::set<const Ctx*>& ctx_registry() {
  static std::set<const Ctx*> s;
  return s;
}
inline void ctx_register(const Ctx* c, bool live) {
  std::lock_guard<std::mutex> lk(ctx_registry_mutex());
  if (live) ctx_registry().insert(c);
  else ctx_registry().erase(c);
}
inline bool ctx_alive(const Ctx* c) {
  std::lock_guard<std::mutex> lk(ctx_registry_mutex());
  return ctx_registry().count(c) != 0;
}

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  unsigned* d_flags = nullptr;   // kernel-raised error flags (FLAG_*)
  unsigned* d_bar = nullptr;     // grid-barrier words for persistent kernels
  int64_t launches = 0;          // kernels launched on this context

  // Buffers of kBigBytes or more come from a per-context cache of cudaMalloc
  // blocks instead of the stream-ordered pool: growing the pool costs ~12 ms
  // per GB on a B200 against ~0.6 ms for cudaMalloc (tools/alloc_probe.cu),
  // and C5's ~60 GB of per-call temporaries made a cold call ~4x slower.
  // Reuse is stream-ordered because every kernel of a context runs on its
  // one stream (set_stream synchronizes the old stream first).
  // Cached free bytes are capped (a quarter of the device, at most 48 GB, or
  // CTD_GPU_CACHE_GB; the excess is returned at once); ctd_gpu_ctx_trim
  // returns the rest (like torch.cuda.empty_cache).
  static constexpr size_t kBigBytes = size_t(64) << 20;
  std::multimap<size_t, void*> big_free;
  std::unordered_map<void*, size_t> big_live;
  size_t big_free_bytes = 0, big_cap = 0;
  std::mutex big_mu;

  void* big_alloc(size_t n) {
    n = (n + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    std::lock_guard<std::mutex> lk(big_mu);
    // the smallest cached block that fits, if within 25 % (+64 MB)
    auto it = big_free.lower_bound(n);
    if (it != big_free.end() && it->first <= n + n / 4 + (size_t(64) << 20)) {
      void* p = it->second;
      big_live.emplace(p, it->first);
      big_free_bytes -= it->first;
      big_free.erase(it);
      return p;
    }
    void* p = nullptr;
    static const bool trace = getenv("CTD_ALLOC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (cudaMalloc(&p, n) != cudaSuccess) {
      cudaGetLastError();
      big_trim_locked();  // give the cached blocks and the pool's reserve back, retry
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
      CUDA_OK(cudaMalloc(&p, n));
    }
    if (trace) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 1.0) fprintf(stderr, "[alloc] cudaMalloc %zu MB %.2f ms (cached free %zu MB)\n", n >> 20, ms,
                            big_free_bytes >> 20);
    }
    big_live.emplace(p, n);
    return p;
  }
  void big_trim_locked() {
    if (big_free.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto& b : big_free) cudaFree(b.second);
    big_free.clear();
    big_free_bytes = 0;
  }
  void big_trim() {
    std::lock_guard<std::mutex> lk(big_mu);
    big_trim_locked();
  }
  // context teardown: every cached and live block
  void big_release_all() {
    std::lock_guard<std::mutex> lk(big_mu);
    big_trim_locked();
    for (auto& b : big_live) cudaFree(b.first);
    big_live.clear();
  }

  void* alloc_bytes(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 16;
    if (n >= kBigBytes) return big_alloc(n);
    CUDA_OK(cudaMallocAsync(&p, n, stream));
    return p;
  }
  template <typename T>
  T* alloc(size_t n) { return static_cast<T*>(alloc_bytes(n * sizeof(T))); }
  void release(void* p) {
    if (!p) return;
    {
      std::lock_guard<std::mutex> lk(big_mu);
      auto it = big_live.find(p);
      if (it != big_live.end()) {
        const size_t n = it->second;
        big_live.erase(it);
        if (big_cap == 0) {
          size_t fr = 0, tot = 0;
          big_cap = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? std::min(tot / 4, size_t(48) << 30)
                                                              : (size_t(32) << 30);
          if (const char* e = getenv("CTD_GPU_CACHE_GB")) big_cap = (size_t)atoll(e) << 30;
        }
        if (big_free_bytes + n > big_cap) {
          if (getenv("CTD_ALLOC_TRACE")) fprintf(stderr, "[alloc] over cap: free %zu MB\n", n >> 20);
          cudaStreamSynchronize(stream);  // queued kernels may still use it
          cudaFree(p);
        } else {
          big_free.emplace(n, p);
          big_free_bytes += n;
        }
        return;
      }
    }
    cudaFreeAsync(p, stream);
  }
  void sync() { CUDA_OK(cudaStreamSynchronize(stream)); }
  void zero(void* p, size_t bytes) { CUDA_OK(cudaMemsetAsync(p, 0, bytes, stream)); }
  template <typename T>
  void to_host(T* dst, const T* src, size_t n) {
    if (n) CUDA_OK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, stream));
  }
  template <typename T>
  void to_dev(T* dst, const T* src, size_t n) {
    if (n) CUDA_OK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, stream));
  }
  template <typename T>
  T read1(const T* src) {
    T v;
    to_host(&v, src, 1);
    sync();
    return v;
  }
  // Reads and clears the kernel error flags; raises the mapped status.
  void check_flags(const char* where);

  // Optional live phase timing with CUDA events on `stream` (bench.py).
  static constexpr int kPhases = 8;
  bool timing = false;
  double phase_ms[kPhases] = {0};
  int64_t phase_n[kPhases] = {0};
  struct Mark {
    int ph;
    cudaEvent_t a, b;
  };
  std::vector<Mark> marks;
  int open_ph = -1;
  cudaEvent_t open_ev = nullptr;
  void phase_begin(int ph) {
    if (!timing) return;
    CUDA_OK(cudaEventCreate(&open_ev));
    CUDA_OK(cudaEventRecord(open_ev, stream));
    open_ph = ph;
  }
  void phase_end() {
    if (!timing || open_ph < 0) return;
    cudaEvent_t b;
    CUDA_OK(cudaEventCreate(&b));
    CUDA_OK(cudaEventRecord(b, stream));
    marks.push_back(Mark{open_ph, open_ev, b});
    open_ph = -1;
  }
  void phase_flush() {
    for (auto& m : marks) {
      CUDA_OK(cudaEventSynchronize(m.b));
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, m.a, m.b));
      phase_ms[m.ph] += ms;
      phase_n[m.ph] += 1;
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    marks.clear();
  }
};

enum Phase { PH_MATRICIZE = 0, PH_LAW, PH_SAMPLE, PH_FILTER_PREP, PH_FILTER, PH_ERROR, PH_H2D, PH_CORE };

// Scoped phase marker (no-op unless ctx->timing).
struct PhaseScope {
  Ctx* c;
  PhaseScope(Ctx* ctx, int ph) : c(ctx) { c->phase_begin(ph); }
  ~PhaseScope() { c->phase_end(); }
};

// RAII device buffer (stream-ordered allocation on the context stream).
template <typename T>
struct Buf {
  Ctx* c = nullptr;
  T* p = nullptr;
  size_t n = 0;
  Buf() = default;
  Buf(Ctx* ctx, size_t count) : c(ctx), p(ctx->alloc<T>(count)), n(count) {}
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : c(o.c), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) { reset(); c = o.c; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~Buf() { reset(); }
  void reset() {
    if (p && c && ctx_alive(c)) c->release(p);
    p = nullptr;
    n = 0;
  }
  void alloc(Ctx* ctx, size_t count) { reset(); c = ctx; p = ctx->alloc<T>(count); n = count; }
  void ensure(Ctx* ctx, size_t count) { if (n < count || !p) alloc(ctx, count); }
  void zero() { if (p) c->zero(p, n * sizeof(T)); }
  T* get() const { return p; }
};

constexpr int kMaxOrder = 16;

// SparseTensor (sparse_tensor.hpp:17-60) resident in HBM as SoA int32
// coordinates + fp64 values, lexicographically sorted and coalesced.
struct Tensor {
  Ctx* ctx = nullptr;
  int order = 0;
  int64_t shape[kMaxOrder] = {0};
  int64_t nnz = 0;
  const int32_t* idx[kMaxOrder] = {nullptr};
  const double* val = nullptr;
  Buf<int32_t> own_idx;  // owned storage when built from host
  Buf<double> own_val;
};

// Launch helper: counts launches and checks launch errors.
#define LAUNCH(ctx, kern, grid, block, smem, ...)                                   \
  do {                                                                              \
    kern<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);                  \
    (ctx)->launches++;                                                              \
    CUDA_OK(cudaGetLastError());                                                    \
  } while (0)

}  // namespace ctdgpu
