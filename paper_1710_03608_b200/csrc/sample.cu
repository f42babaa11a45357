// Inverse-CDF fiber sampling (sample_with_replacement, sampling.cpp:33-64)
// and first-occurrence dedup (unique_first_occurrence, sampling.cpp:66-78).
//
// The uniform stream is std::mt19937_64(seed) (sampling.cpp:56) with
// u = (r >> 11) * 2^-53 (:15-17), generated on the device by one CTA: the
// 312-word twist runs as three dependency-ordered parallel phases, tempering
// is elementwise.  Each draw is an independent upper_bound binary search
// (:59-61) over the clamped cumulative array of the nonempty fibers (columns
// with zero probability can never be returned by upper_bound, so restricting
// the search to nonempty fibers returns the same column).  Dedup sorts
// (fiber, position) pairs with the stable block radix sort and keeps the
// first position of each run, then compacts in draw order.
#include "radix.cuh"
#include "sample.cuh"

namespace ctdgpu {

namespace {

constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t y = (a & 0xFFFFFFFF80000000ULL) | (b & 0x7FFFFFFFULL);
  return c ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// One CTA of 320 threads; writes `count` raw outputs of mt19937_64(seed).
__global__ void k_mt19937_64(uint64_t seed, long long count, uint64_t* out) {
  __shared__ uint64_t mt[kMtN];
  const int t = threadIdx.x;
  if (t == 0) {  // seeding recurrence is inherently sequential (312 steps)
    mt[0] = seed;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  }
  __syncthreads();
  for (long long base = 0; base < count; base += kMtN) {
    // twist: k in [0,156) reads old k, k+1, k+156
    uint64_t v = 0;
    if (t < kMtM) v = mt_mix(mt[t], mt[t + 1], mt[t + kMtM]);
    __syncthreads();
    if (t < kMtM) mt[t] = v;
    __syncthreads();
    // k in [156,311): reads old k, k+1 and new k-156
    if (t >= kMtM && t < kMtN - 1) v = mt_mix(mt[t], mt[t + 1], mt[t - kMtM]);
    __syncthreads();
    if (t >= kMtM && t < kMtN - 1) mt[t] = v;
    __syncthreads();
    if (t == kMtN - 1) mt[t] = mt_mix(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
    __syncthreads();
    if (t < kMtN && base + t < count) out[base + t] = mt_temper(mt[t]);
    __syncthreads();
  }
}

// upper_bound of u over cum[0..F) -> fiber index.
__global__ void k_draw(const uint64_t* raw, long long count, const double* cum, long long F,
                       int32_t* fiber_out) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double u = (double)(raw[k] >> 11) * 0x1.0p-53;
  long long lo = 0, hi = F;
  while (lo < hi) {
    const long long mid = lo + ((hi - lo) >> 1);
    if (u < cum[mid]) hi = mid;
    else lo = mid + 1;
  }
  CTD_CHECK(lo < F);  // the clamped CDF ends at 1.0 > u
  fiber_out[k] = (int32_t)lo;
}

// Single CTA: dedup `count` fiber ids in draw order.
constexpr int kDedupThreads = 1024;
__global__ void __launch_bounds__(kDedupThreads) k_dedup(const int32_t* drawn, int count,
                                                         uint32_t* ka, uint32_t* kb, uint32_t* ia,
                                                         uint32_t* ib, int32_t* keep,
                                                         int32_t* unique_out, int* n_unique) {
  __shared__ uint32_t hist[(kDedupThreads / 32) * kRadix];
  __shared__ uint32_t sh[33];
  __shared__ int shi[33];
  for (int p = threadIdx.x; p < count; p += blockDim.x) {
    ka[p] = (uint32_t)drawn[p];
    ia[p] = (uint32_t)p;
    keep[p] = 0;
  }
  __syncthreads();
  const bool inb = block_radix_sort<uint32_t>(ka, kb, ia, ib, count, 32, hist, sh);
  const uint32_t* K = inb ? kb : ka;
  const uint32_t* I = inb ? ib : ia;
  for (int p = threadIdx.x; p < count; p += blockDim.x)
    if (p == 0 || K[p - 1] != K[p]) keep[I[p]] = 1;  // stable: first position of each run
  __syncthreads();
  // ordered compaction
  const int per = (count + blockDim.x - 1) / blockDim.x;
  const int c0 = min((int)threadIdx.x * per, count), c1 = min(c0 + per, count);
  int nk = 0;
  for (int p = c0; p < c1; ++p) nk += keep[p];
  int tot;
  int pos = block_excl_sum<int>(nk, shi, &tot);
  for (int p = c0; p < c1; ++p)
    if (keep[p]) {
      CTD_CHECK(pos < count);
      unique_out[pos++] = drawn[p];
    }
  if (threadIdx.x == 0) *n_unique = tot;
}

// Dedup of arbitrary int64 ids: stable sort by (hi, lo) via two 32-bit
// passes, first position of each run of equal values kept.
__global__ void __launch_bounds__(kDedupThreads) k_dedup64(const int64_t* in, int count, uint32_t* ka,
                                                           uint32_t* kb, uint32_t* ia, uint32_t* ib,
                                                           int32_t* keep, int64_t* out, int* n_unique) {
  __shared__ uint32_t hist[(kDedupThreads / 32) * kRadix];
  __shared__ uint32_t sh[33];
  __shared__ int shi[33];
  for (int p = threadIdx.x; p < count; p += blockDim.x) {
    ka[p] = (uint32_t)((uint64_t)in[p] & 0xffffffffu);
    ia[p] = (uint32_t)p;
    keep[p] = 0;
  }
  __syncthreads();
  bool inb = block_radix_sort<uint32_t>(ka, kb, ia, ib, count, 32, hist, sh);
  uint32_t* K2 = inb ? kb : ka;
  uint32_t* I2 = inb ? ib : ia;
  uint32_t* K3 = inb ? ka : kb;
  uint32_t* I3 = inb ? ia : ib;
  for (int p = threadIdx.x; p < count; p += blockDim.x) {
    K3[p] = (uint32_t)((uint64_t)in[I2[p]] >> 32);
    I3[p] = I2[p];
  }
  __syncthreads();
  inb = block_radix_sort<uint32_t>(K3, K2, I3, I2, count, 32, hist, sh);
  const uint32_t* I = inb ? I2 : I3;
  for (int p = threadIdx.x; p < count; p += blockDim.x)
    if (p == 0 || in[I[p - 1]] != in[I[p]]) keep[I[p]] = 1;
  __syncthreads();
  const int per = (count + blockDim.x - 1) / blockDim.x;
  const int c0 = min((int)threadIdx.x * per, count), c1 = min(c0 + per, count);
  int nk = 0;
  for (int p = c0; p < c1; ++p) nk += keep[p];
  int tot;
  int pos = block_excl_sum<int>(nk, shi, &tot);
  for (int p = c0; p < c1; ++p)
    if (keep[p]) out[pos++] = in[p];
  if (threadIdx.x == 0) *n_unique = tot;
}

// upper_bound over an arbitrary cumulative array -> column index (int64).
__global__ void k_draw64(const uint64_t* raw, long long count, const double* cum, long long n,
                         int64_t* out) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double u = (double)(raw[k] >> 11) * 0x1.0p-53;
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = lo + ((hi - lo) >> 1);
    if (u < cum[mid]) hi = mid;
    else lo = mid + 1;
  }
  out[k] = lo;
}

}  // namespace

void draw_columns(Ctx* ctx, const double* cum, int64_t n, int64_t count, uint64_t seed, int64_t* d_out) {
  if (count <= 0) return;
  Buf<uint64_t> raw(ctx, count);
  mt19937_64(ctx, seed, count, raw.p);
  LAUNCH(ctx, k_draw64, ceil_div(count, 256), 256, 0, raw.p, (long long)count, cum, (long long)n, d_out);
}

void dedup_first64(Ctx* ctx, const int64_t* d_in, int64_t count, int64_t* d_out, int* d_n_unique) {
  if (count <= 0) {
    ctx->zero(d_n_unique, sizeof(int));
    return;
  }
  if (count > (1ll << 30)) fail(CTD_ERR_ARGUMENT, "list too large");
  Buf<uint32_t> ka(ctx, count), kb(ctx, count), ia(ctx, count), ib(ctx, count);
  Buf<int32_t> keep(ctx, count);
  LAUNCH(ctx, k_dedup64, 1, kDedupThreads, 0, d_in, (int)count, ka.p, kb.p, ia.p, ib.p, keep.p, d_out,
         d_n_unique);
}

void mt19937_64(Ctx* ctx, uint64_t seed, int64_t count, uint64_t* d_out) {
  if (count <= 0) return;
  LAUNCH(ctx, k_mt19937_64, 1, 320, 0, seed, (long long)count, d_out);
}

void draw_fibers(Ctx* ctx, const double* cum, int64_t F, int64_t count, uint64_t seed,
                 int32_t* d_fibers) {
  if (count <= 0) return;
  Buf<uint64_t> raw(ctx, count);
  mt19937_64(ctx, seed, count, raw.p);
  LAUNCH(ctx, k_draw, ceil_div(count, 256), 256, 0, raw.p, (long long)count, cum, (long long)F,
         d_fibers);
}

void dedup_first(Ctx* ctx, const int32_t* d_drawn, int64_t count, int32_t* d_unique,
                 int* d_n_unique) {
  if (count <= 0) {
    ctx->zero(d_n_unique, sizeof(int));
    return;
  }
  if (count > (1ll << 30)) fail(CTD_ERR_ARGUMENT, "sample size too large");
  Buf<uint32_t> ka(ctx, count), kb(ctx, count), ia(ctx, count), ib(ctx, count);
  Buf<int32_t> keep(ctx, count);
  LAUNCH(ctx, k_dedup, 1, kDedupThreads, 0, d_drawn, (int)count, ka.p, kb.p, ia.p, ib.p, keep.p,
         d_unique, d_n_unique);
}

}  // namespace ctdgpu
