// COO -> mode-alpha fiber bucketing: the GPU form of matricize
// (tensor_ops.cpp:118-135) + the SparseMatrix COO constructor
// (sparse_matrix.cpp:22-67) + column_sq_norms (tensor_ops.cpp:194-202).
//
// Layout: every entry gets the composite key (column j, row i_alpha).  Keys
// are unique for a normalized SparseTensor, so sorting them yields exactly
// the reference's (col,row) order.  Three HBM passes:
//   1. histogram of buckets  b = j >> wbits  (W = 2^wbits consecutive columns)
//   2. scatter every entry to its bucket as a 32-bit key
//      (j - b*W) << rowbits | row  plus its value; validates the input
//   3. one CTA per bucket: stable block radix sort of the bucket's keys in
//      shared memory (global memory for the rare oversize bucket), then a
//      coalesced write of rows/values, fiber heads ranked across buckets with
//      a decoupled look-back, and each fiber's squared norm summed in
//      ascending-row order (bit-identical to the reference loop).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cub/cub.cuh>

#include "bucket.cuh"
#include "radix.cuh"

namespace ctdgpu {

namespace {

constexpr int kSortThreads = 512;
constexpr int kCap = 8192;  // bucket capacity of the shared-memory path

struct CooView {
  int order;
  int mode;
  long long nnz;
  const int32_t* idx[kMaxOrder];
  const double* val;
  long long stride[kMaxOrder];
  long long shape[kMaxOrder];
};

__device__ __forceinline__ long long col_of(const CooView& c, long long i, int* row, bool* oob) {
  long long j = 0;
  bool bad = false;
  int r = 0;
  for (int k = 0; k < c.order; ++k) {
    const long long v = c.idx[k][i];
    bad |= (v < 0) | (v >= c.shape[k]);
    if (k == c.mode) r = (int)v;
    else j += v * c.stride[k];
  }
  *row = r;
  *oob = bad;
  return j;
}

__global__ void k_hist(CooView c, int wbits, unsigned* count, unsigned* flags) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const unsigned long long kNone = ~0ull;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < c.nnz; base += stride) {
    const long long i = base + threadIdx.x;
    const bool act = i < c.nnz;
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    if (!act) continue;
    int row;
    bool oob;
    const long long j = col_of(c, i, &row, &oob);
    if (oob) atomicOr(flags, FLAG_BOUNDS);
    const unsigned long long b = oob ? kNone : (unsigned long long)(j >> wbits);
    const unsigned peers = __match_any_sync(amask, b);
    if (b != kNone && (int)(threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&count[b], (unsigned)__popc(peers));
  }
}

__global__ void k_excl_scan_u32(const unsigned* cnt, long long n, unsigned long long* off,
                                unsigned* maxc) {
  __shared__ unsigned long long sh[33];
  unsigned long long carry = 0;
  unsigned mx = 0;
  for (long long b0 = 0; b0 < n; b0 += (long long)blockDim.x * 4) {
    unsigned long long v[4], s = 0;
    const long long base = b0 + (long long)threadIdx.x * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = (base + k < n) ? cnt[base + k] : 0ull;
      s += v[k];
      mx = max(mx, (unsigned)v[k]);
    }
    unsigned long long tot;
    unsigned long long pre = block_excl_sum<unsigned long long>(s, sh, &tot) + carry;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (base + k < n) off[base + k] = pre;
      pre += v[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = carry;
  atomicMax(maxc, mx);
}

struct ScatterOut {
  unsigned long long* cursor;
  uint32_t* tkey;
  double* tval;
  int* integer_ok;   // cleared when a value is not a small integer
  double* sum_sq;    // sum of v^2, any order
};

__global__ void k_scatter(CooView c, int wbits, int rowbits, ScatterOut o, unsigned* flags) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const unsigned long long wmask = (1ull << wbits) - 1ull;
  double sq = 0.0;
  bool intok = true;
  const unsigned long long kNone = ~0ull;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < c.nnz; base += stride) {
    const long long i = base + threadIdx.x;
    const bool act = i < c.nnz;
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    if (!act) continue;
    int row;
    bool oob;
    const long long j = col_of(c, i, &row, &oob);
    const double v = c.val[i];
    if (!oob) {
      if (v == 0.0) atomicOr(flags, FLAG_ZERO);
      intok &= (v == rint(v)) && (fabs(v) <= 67108864.0);
      sq += v * v;
    }
    const unsigned long long b = oob ? kNone : (unsigned long long)(j >> wbits);
    const unsigned peers = __match_any_sync(amask, b);
    const int leader = __ffs(peers) - 1;
    unsigned long long basepos = 0;
    if (b != kNone && (int)(threadIdx.x & 31) == leader)
      basepos = atomicAdd(&o.cursor[b], (unsigned long long)__popc(peers));
    basepos = __shfl_sync(peers, basepos, leader);
    if (b == kNone) continue;
    const unsigned long long pos = basepos + __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
    o.tkey[pos] = (uint32_t)((((unsigned long long)j & wmask) << rowbits) | (unsigned)row);
    o.tval[pos] = v;
  }
  sq = warp_sum(sq);
  const bool all_ok = __all_sync(0xffffffffu, intok);
  if ((threadIdx.x & 31) == 0) {
    if (sq != 0.0) atomicAdd(o.sum_sq, sq);
    if (!all_ok) atomicExch(o.integer_ok, 0);
  }
}

struct SortArgs {
  int cap;                        // shared-memory bucket capacity of this launch
  const unsigned long long* off;  // [nb+1]
  uint32_t* tkey;                 // [nnz] scattered keys (reused as sort buffer A)
  const double* tval;             // [nnz]
  uint32_t* gkey2;                // [nnz] global sort buffer B (oversize buckets)
  uint32_t* gidx1;                // [nnz]
  uint32_t* gidx2;                // [nnz]
  int32_t* out_row;
  double* out_val;
  int64_t* fcol;
  int64_t* fptr;
  double* norm;
  unsigned long long* status;     // look-back words, [nb]
  unsigned* ticket;
  long long nb;
  long long nnz;
  int wbits, rowbits;
  long long* F_out;
  unsigned* flags;
  int presorted;                  // oversize buckets already sorted (gkey2 keys, out_val values)
};

// Decoupled look-back over the buckets' fiber counts.  The count (distinct
// columns) can be published early (lookback_publish, from a bitmap of the
// bucket's columns, before the sort) so later buckets never wait on a slow
// one; lookback() then only walks back and publishes the inclusive prefix.
__device__ void lookback_publish(unsigned long long* st, long long b, long long agg) {
  const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62;
  atomicExch(&st[b], (b == 0 ? kInc : kAgg) | (unsigned long long)agg);
}

__device__ long long lookback(unsigned long long* st, long long b, long long agg, bool published) {
  const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1;
  if (b == 0) {
    if (!published) atomicExch(&st[0], kInc | (unsigned long long)agg);
    return 0;
  }
  if (!published) atomicExch(&st[b], kAgg | (unsigned long long)agg);
  long long prefix = 0;
  long long i = b - 1;
  while (true) {
    const unsigned long long s = *((volatile unsigned long long*)&st[i]);
    const unsigned long long f = s >> 62;
    if (f == 0) {
      __nanosleep(40);
      continue;
    }
    prefix += (long long)(s & kVal);
    if (f == 2) break;
    --i;
  }
  atomicExch(&st[b], kInc | (unsigned long long)(prefix + agg));
  return prefix;
}

__global__ void __launch_bounds__(kSortThreads) k_bucket_sort(SortArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* ska = (uint32_t*)smem;
  const int cap = a.cap;
  uint32_t* skb = ska + cap;
  uint16_t* sia = (uint16_t*)(skb + cap);
  uint16_t* sib = sia + cap;
  double* sv = (double*)(sib + cap);
  uint32_t* hist = (uint32_t*)(sv + cap);
  __shared__ uint32_t sh32[33];
  __shared__ long long sh64[33];
  __shared__ long long s_b, s_fbase;
  if (threadIdx.x == 0) s_b = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const long long b = s_b;
  if (b >= a.nb) return;
  const long long start = (long long)a.off[b];
  const int m = (int)((long long)a.off[b + 1] - start);
  const int T = blockDim.x, t = threadIdx.x;
  const int keybits = a.wbits + a.rowbits;
  const uint32_t rowmask = a.rowbits ? (0xffffffffu >> (32 - a.rowbits)) : 0u;
  // early publication of the bucket's fiber count (distinct columns)
  constexpr int kBmWords = 1024;  // columns per bucket <= 32768
  __shared__ unsigned bm[kBmWords];
  __shared__ int s_cnt;
  const bool early = a.wbits <= 15;
  if (early) {
    const int words = ((1 << a.wbits) + 31) >> 5;
    for (int w = t; w < words; w += T) bm[w] = 0u;
    if (t == 0) s_cnt = 0;
    __syncthreads();
    for (int p = t; p < m; p += T) {
      const uint32_t jl = a.rowbits < 32 ? (a.tkey[start + p] >> a.rowbits) : 0u;
      atomicOr(&bm[jl >> 5], 1u << (jl & 31));
    }
    __syncthreads();
    int c = 0;
    for (int w = t; w < words; w += T) c += __popc(bm[w]);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((t & 31) == 0 && c) atomicAdd(&s_cnt, c);
    __syncthreads();
    if (t == 0) lookback_publish(a.status, b, s_cnt);
  }
  const bool small = m <= cap;
  const uint32_t* K;
  const double* V;
  if (small) {
    for (int p = t; p < m; p += T) {
      ska[p] = a.tkey[start + p];
      sia[p] = (uint16_t)p;
    }
    __syncthreads();
    const bool inb = block_radix_sort<uint16_t>(ska, skb, sia, sib, m, keybits, hist, sh32);
    K = inb ? skb : ska;
    const uint16_t* I = inb ? sib : sia;
    for (int p = t; p < m; p += T) sv[p] = a.tval[start + I[p]];
    V = sv;
  } else if (a.presorted) {
    K = a.gkey2 + start;
    V = a.out_val + start;
  } else {
    uint32_t* ka = a.tkey + start;
    uint32_t* kb = a.gkey2 + start;
    uint32_t* ia = a.gidx1 + start;
    uint32_t* ib = a.gidx2 + start;
    for (int p = t; p < m; p += T) ia[p] = (uint32_t)p;
    __syncthreads();
    const bool inb = block_radix_sort<uint32_t>(ka, kb, ia, ib, m, keybits, hist, sh32);
    K = inb ? kb : ka;
    const uint32_t* I = inb ? ib : ia;
    for (int p = t; p < m; p += T) a.out_val[start + p] = a.tval[start + I[p]];
    V = a.out_val + start;
  }
  __syncthreads();
  // Contiguous chunk per thread: write rows/values, find fiber heads.
  const int per = (m + T - 1) / T;
  const int c0 = min(t * per, m), c1 = min(c0 + per, m);
  long long nh = 0;
  bool dup = false;
  for (int p = c0; p < c1; ++p) {
    const uint32_t key = K[p];
    a.out_row[start + p] = (int32_t)(key & rowmask);
    if (small) a.out_val[start + p] = V[p];
    const bool head = (p == 0) || ((K[p - 1] >> a.rowbits) != (key >> a.rowbits));
    dup |= (p > 0) && (K[p - 1] == key);
    nh += head;
  }
  if (dup) atomicOr(a.flags, FLAG_DUPLICATE);
  long long agg;
  long long rank = block_excl_sum<long long>(nh, sh64, &agg);
  if (t == 0) {
    if (early && agg != (long long)s_cnt) atomicOr(a.flags, FLAG_OVERFLOW);  // cannot happen
    s_fbase = lookback(a.status, b, agg, early);
    if (b == a.nb - 1) {
      *a.F_out = s_fbase + agg;
      a.fptr[s_fbase + agg] = a.nnz;
    }
  }
  __syncthreads();
  const long long fbase = s_fbase;
  for (int p = c0; p < c1; ++p) {
    const uint32_t key = K[p];
    const uint32_t jl = a.rowbits < 32 ? (key >> a.rowbits) : 0u;
    const bool head = (p == 0) || ((K[p - 1] >> a.rowbits) != jl);
    if (!head) continue;
    const long long f = fbase + rank++;
    a.fcol[f] = ((long long)b << a.wbits) + (long long)jl;
    a.fptr[f] = start + p;
    // column_sq_norms: s += v*v in ascending row order (tensor_ops.cpp:197-198).
    // The fiber's end first (keys are sorted: binary search for long fibers),
    // so the value loads do not wait on the loop condition.
    int e = p + 1;
    {
      const int lim = min(m, p + 16);
      while (e < lim && (K[e] >> a.rowbits) == jl) ++e;
      if (e == lim && e < m && (K[e] >> a.rowbits) == jl) {
        int lo = e, hi = m;  // first index in [lo, hi) with a larger column
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((K[mid] >> a.rowbits) == jl) lo = mid + 1;
          else hi = mid;
        }
        e = lo;
      }
    }
    double s = 0.0;
    int q = p;
    if (e - p >= 64) {  // long fiber: L1 prefetch 16 lines ahead of the 16-value batches
      for (; q + 16 <= e; q += 16) {
        if (q + 256 < e) asm volatile("prefetch.global.L1 [%0];" ::"l"(V + q + 256));
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = V[q + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) s = dadd(s, dsqr(v[u]));
      }
    }
    for (; q < e; ++q) s = dadd(s, dsqr(V[q]));
    a.norm[f] = s;
  }
}

// Oversize buckets (more entries than one CTA's shared memory holds: a heavy
// Zipf column) are sorted together by a device-wide radix sort instead of one
// CTA per bucket.  Their entries are compacted with 64-bit keys
// (rank of the bucket among the oversize ones, 32-bit in-bucket key); after
// the sort the compacted array is the concatenation of the sorted buckets in
// bucket order, so each entry goes back to its bucket's range.
// Buckets above each power-of-two size 256..8192 (cap selection).
__global__ void k_size_dist(const unsigned* count, long long nb, unsigned long long* above) {
  __shared__ unsigned long long sh[6];
  if (threadIdx.x < 6) sh[threadIdx.x] = 0;
  __syncthreads();
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (long long)gridDim.x * blockDim.x) {
    const unsigned c = count[b];
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if (c > (256u << k)) atomicAdd(&sh[k], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < 6 && sh[threadIdx.x]) atomicAdd(&above[threadIdx.x], sh[threadIdx.x]);
}

__global__ void k_over_count(const unsigned* count, long long nb, int cap, unsigned long long* ocnt,
                             unsigned* is_over) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const bool ov = count[b] > (unsigned)cap;
  ocnt[b] = ov ? count[b] : 0ull;
  is_over[b] = ov ? 1u : 0u;
}

__global__ void k_over_list(const unsigned* is_over, const unsigned* orank, long long nb,
                            long long* olist) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb && is_over[b]) olist[orank[b]] = b;
}

__global__ void k_over_pack(const long long* olist, const unsigned long long* off,
                            const unsigned long long* ooff, const uint32_t* tkey, int keybits,
                            unsigned long long* okey, uint32_t* oidx) {
  const long long r = blockIdx.x;
  const long long b = olist[r];
  const long long start = (long long)off[b], m = (long long)off[b + 1] - start;
  const long long o = (long long)ooff[b];
  for (long long p = threadIdx.x; p < m; p += blockDim.x) {
    okey[o + p] = ((unsigned long long)r << keybits) | tkey[start + p];
    oidx[o + p] = (uint32_t)(start + p);
  }
}

__global__ void k_over_unpack(const long long* olist, const unsigned long long* off,
                              const unsigned long long* ooff, const unsigned long long* skey,
                              const uint32_t* sidx, const double* tval, int keybits,
                              uint32_t* gkey2, double* out_val) {
  const long long b = olist[blockIdx.x];
  const long long start = (long long)off[b], m = (long long)off[b + 1] - start;
  const long long o = (long long)ooff[b];
  const unsigned long long kmask = keybits >= 32 ? 0xffffffffull : ((1ull << keybits) - 1ull);
  for (long long p = threadIdx.x; p < m; p += blockDim.x) {
    gkey2[start + p] = (uint32_t)(skey[o + p] & kmask);
    out_val[start + p] = tval[sidx[o + p]];
  }
}

int bits_for(long long n) {  // bits needed to represent 0..n-1
  int b = 0;
  while (b < 63 && (1ll << b) < n) ++b;
  return b;
}

}  // namespace

// The general path: any entry order (bucket scatter + per-bucket radix sort
// by (column, row)).  matricize() uses it when the input's rows are not
// ascending inside its columns (onesweep.cu needs that order).
static void matricize_sort(Ctx* ctx, const Tensor& x, int mode, Fibers& out) {
  static const bool htrace = getenv("CTD_HOST_TRACE") != nullptr;
  std::chrono::steady_clock::time_point ht[8];
  int nht = 0;
#define HT() \
  if (htrace) ht[nht++] = std::chrono::steady_clock::now();
  HT()
  if (mode < 0 || mode >= x.order)
    fail(CTD_ERR_ARGUMENT, "mode " + std::to_string(mode) + " out of range for order " +
                               std::to_string(x.order));
  CooView c{};
  c.order = x.order;
  c.mode = mode;
  c.nnz = x.nnz;
  c.val = x.val;
  long long acc = 1;
  for (int k = 0; k < x.order; ++k) {  // fiber_strides, tensor_ops.cpp:106-116
    c.idx[k] = x.idx[k];
    c.shape[k] = x.shape[k];
    if (k == mode) {
      c.stride[k] = 0;
      continue;
    }
    c.stride[k] = acc;
    acc *= x.shape[k];
  }
  out.rows = x.shape[mode];
  out.cols = acc;
  out.nnz = x.nnz;
  out.mode = mode;
  const int rowbits = bits_for(out.rows);
  if (rowbits > 31) fail(CTD_ERR_SHAPE, "mode extent exceeds 2^31");
  // Bucket width: ~2048 expected entries per bucket, key must fit 32 bits.
  int wbits = 0;
  {
    const double per_col = out.cols > 0 ? (double)x.nnz / (double)out.cols : 1.0;
    const double want = 1024.0 / (per_col > 0 ? per_col : 1.0);
    while (wbits < 32 - rowbits && (double)(1ll << (wbits + 1)) <= want) ++wbits;
    wbits = std::min(wbits, 32 - rowbits);
  }
  long long nb = out.cols > 0 ? ((out.cols - 1) >> wbits) + 1 : 1;
  if (nb > (1ll << 28)) fail(CTD_ERR_SHAPE, "matricized column count too large for bucketing");
  const long long nnz = x.nnz;
  out.row.alloc(ctx, nnz);
  out.val.alloc(ctx, nnz);
  out.col.alloc(ctx, nnz + 1);
  out.ptr.alloc(ctx, nnz + 1);
  out.norm.alloc(ctx, nnz + 1);
  Buf<long long> dF(ctx, 1);
  if (nnz == 0) {
    out.F = 0;
    ctx->zero(out.ptr.p, sizeof(int64_t));
    return;
  }
  HT()
  Buf<unsigned> count(ctx, nb);
  count.zero();
  Buf<unsigned long long> off(ctx, nb + 1), cursor(ctx, nb + 1), status(ctx, nb);
  status.zero();
  Buf<uint32_t> tkey(ctx, nnz);
  Buf<double> tval(ctx, nnz);
  Buf<int> intok(ctx, 1);
  Buf<double> sumsq(ctx, 1);
  Buf<unsigned> ticket(ctx, 1);
  ticket.zero();
  sumsq.zero();
  {
    const int one = 1;
    ctx->to_dev(intok.p, &one, 1);
  }
  const unsigned grid = (unsigned)std::min<long long>((nnz + 255) / 256, (long long)ctx->sm_count * 16);
  HT()
  LAUNCH(ctx, k_hist, grid, 256, 0, c, wbits, count.p, ctx->d_flags);
  Buf<unsigned> maxc(ctx, 1);
  maxc.zero();
  LAUNCH(ctx, k_excl_scan_u32, 1, 1024, 0, count.p, nb, off.p, maxc.p);
  CUDA_OK(cudaMemcpyAsync(cursor.p, off.p, (nb + 1) * sizeof(unsigned long long),
                          cudaMemcpyDeviceToDevice, ctx->stream));
  ScatterOut so{cursor.p, tkey.p, tval.p, intok.p, sumsq.p};
  LAUNCH(ctx, k_scatter, grid, 256, 0, c, wbits, rowbits, so, ctx->d_flags);
  // Oversize buckets need global sort buffers (sized nnz so every bucket owns
  // its slice), allocated below only when some bucket exceeds the capacity.
  Buf<uint32_t> gkey2, gidx1, gidx2;
  // Shared-memory capacity sized to the largest bucket (more CTAs per SM).
  const unsigned mx = ctx->read1(maxc.p);
  if (htrace) {
    std::vector<unsigned> hc(nb);
    ctx->to_host(hc.data(), count.p, nb);
    ctx->sync();
    long long nover = 0, eover = 0;
    for (long long b = 0; b < nb; ++b)
      if (hc[b] > (unsigned)kCap) ++nover, eover += hc[b];
    fprintf(stderr, "[matricize] nnz=%lld cols=%lld rowbits=%d wbits=%d buckets=%lld max=%u "
            "oversize=%lld (%lld entries)\n", nnz, (long long)out.cols, rowbits, wbits, nb, mx,
            nover, eover);
  }
  HT()
  // Shared-memory capacity: the smallest power of two holding the largest
  // bucket (<= kCap).  With many buckets, a large cap costs occupancy on every
  // CTA (kCap: one CTA per SM), so when few buckets (< 10%) are
  // above twice the mean size, cap is sized for the rest and the outliers go
  // through the device-wide sort below.
  int cap = 256;
  while (cap < (int)mx && cap < kCap) cap <<= 1;
  if (nb > 16ll * ctx->sm_count && nnz < (1ll << 32)) {
    Buf<unsigned long long> above(ctx, 6);
    above.zero();
    LAUNCH(ctx, k_size_dist, (unsigned)std::min<long long>(ceil_div(nb, 256), ctx->sm_count * 4), 256,
           0, count.p, nb, above.p);
    unsigned long long ab[6];
    ctx->to_host(ab, above.p, 6);
    ctx->sync();
    const double mean = (double)nnz / (double)nb;
    int small = 256;
    while (small < kCap && (double)small < 2.0 * mean) small <<= 1;
    int k = 0;
    while ((256 << k) < small) ++k;
    if (small < cap && (double)ab[k] < 0.1 * (double)nb) cap = small;
    if (htrace)
      fprintf(stderr, "[matricize] buckets above 256..8192: %llu %llu %llu %llu %llu %llu; cap %d\n",
              ab[0], ab[1], ab[2], ab[3], ab[4], ab[5], cap);
  }
  const int threads = cap <= 2048 ? 256 : kSortThreads;
  int presorted = 0;
  if ((int)mx > cap) {
    gkey2.alloc(ctx, nnz);  // presorted oversize keys (or the in-kernel sort's second buffer)
    if (nnz >= (1ll << 32)) {  // the in-kernel global-memory sort of oversize buckets
      gidx1.alloc(ctx, nnz);
      gidx2.alloc(ctx, nnz);
    }
  }
  if ((int)mx > cap && nnz < (1ll << 32)) {
    // oversize buckets: one device-wide radix sort over all of them
    Buf<unsigned long long> ocnt(ctx, nb), ooff(ctx, nb + 1);
    Buf<unsigned> isov(ctx, nb), orank(ctx, nb + 1);
    LAUNCH(ctx, k_over_count, ceil_div(nb, 256), 256, 0, count.p, nb, cap, ocnt.p, isov.p);
    size_t tb1 = 0, tb2 = 0;
    CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, tb1, ocnt.p, ooff.p, nb + 1, ctx->stream));
    CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, isov.p, orank.p, nb + 1, ctx->stream));
    Buf<unsigned char> tmp(ctx, std::max(tb1, tb2));
    CUDA_OK(cub::DeviceScan::ExclusiveSum(tmp.p, tb1, ocnt.p, ooff.p, nb, ctx->stream));
    CUDA_OK(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, isov.p, orank.p, nb, ctx->stream));
    ctx->launches += 4;  // two cub scans (init + scan kernels each)
    unsigned long long last_off = 0, last_cnt = 0;
    unsigned last_rank = 0, last_ov = 0;
    ctx->to_host(&last_off, ooff.p + nb - 1, 1);
    ctx->to_host(&last_cnt, ocnt.p + nb - 1, 1);
    ctx->to_host(&last_rank, orank.p + nb - 1, 1);
    ctx->to_host(&last_ov, isov.p + nb - 1, 1);
    ctx->sync();
    const long long n_over = (long long)last_rank + last_ov;
    const long long e_over = (long long)(last_off + last_cnt);
    if (n_over > 0) {
      Buf<long long> olist(ctx, n_over);
      LAUNCH(ctx, k_over_list, ceil_div(nb, 256), 256, 0, isov.p, orank.p, nb, olist.p);
      const int keybits = wbits + rowbits;
      const int obits = keybits + bits_for(n_over);
      Buf<unsigned long long> k1(ctx, e_over), k2(ctx, e_over);
      Buf<uint32_t> i1(ctx, e_over), i2(ctx, e_over);
      LAUNCH(ctx, k_over_pack, (unsigned)n_over, 256, 0, olist.p, off.p, ooff.p, tkey.p, keybits,
             k1.p, i1.p);
      size_t tb3 = 0;
      CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tb3, k1.p, k2.p, i1.p, i2.p, e_over, 0, obits,
                                              ctx->stream));
      Buf<unsigned char> tmp3(ctx, tb3);
      CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp3.p, tb3, k1.p, k2.p, i1.p, i2.p, e_over, 0, obits,
                                              ctx->stream));
      ctx->launches += 1 + (obits + 7) / 8;  // cub onesweep: histogram + one pass per 8 bits
      LAUNCH(ctx, k_over_unpack, (unsigned)n_over, 256, 0, olist.p, off.p, ooff.p, k2.p, i2.p,
             tval.p, keybits, gkey2.p, out.val.p);
      presorted = 1;
    }
  }
  SortArgs sa{cap, off.p, tkey.p, tval.p, gkey2.p, gidx1.p, gidx2.p, out.row.p, out.val.p,
              out.col.p, out.ptr.p, out.norm.p, status.p, ticket.p, nb, nnz, wbits, rowbits,
              dF.p, ctx->d_flags, presorted};
  const size_t smem = (size_t)cap * (4 + 4 + 2 + 2 + 8) + (threads / 32) * kRadix * 4;
  static unsigned long long attr_done = 0;
  if (first_on_device(&attr_done, ctx->device)) {
    const size_t smax = (size_t)kCap * (4 + 4 + 2 + 2 + 8) + (kSortThreads / 32) * kRadix * 4;
    CUDA_OK(cudaFuncSetAttribute(k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smax));
  }
  LAUNCH(ctx, k_bucket_sort, (unsigned)nb, threads, smem, sa);
  HT()
  long long F = 0;
  int iok = 0;
  double ssq = 0.0;
  ctx->to_host(&F, dF.p, 1);
  ctx->to_host(&iok, intok.p, 1);
  ctx->to_host(&ssq, sumsq.p, 1);
  ctx->sync();
  out.F = F;
  out.sum_sq = ssq;
  out.integer_exact = iok && ssq < 4503599627370496.0;  // 2^52
  ctx->check_flags("matricize");
  HT()
  if (htrace) {
    fprintf(stderr, "[matricize host]");
    for (int i = 1; i < nht; ++i)
      fprintf(stderr, " %.3f", std::chrono::duration<double, std::milli>(ht[i] - ht[i - 1]).count());
    fprintf(stderr, " ms\n");
  }
#undef HT
}

void matricize(Ctx* ctx, const Tensor& x, int mode, Fibers& out) {
  if (mode < 0 || mode >= x.order)
    fail(CTD_ERR_ARGUMENT, "mode " + std::to_string(mode) + " out of range for order " +
                               std::to_string(x.order));
  static const bool legacy = getenv("CTD_BUCKET_LEGACY") != nullptr;  // A/B hook
  if (!legacy && matricize_onesweep(ctx, x, mode, out)) return;
  out = Fibers{};
  matricize_sort(ctx, x, mode, out);
}

}  // namespace ctdgpu
