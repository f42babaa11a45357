// COO -> mode-alpha fiber bucketing for a normalized (lexicographically
// sorted) SparseTensor: the HBM-bound form of matricize (tensor_ops.cpp:
// 118-135) + the SparseMatrix COO constructor (sparse_matrix.cpp:22-67) +
// column_sq_norms (tensor_ops.cpp:194-202).
//
// In a lexicographically sorted COO every mode-alpha column (all other
// coordinates fixed) already lists its rows in ascending order, so the
// reference's (col, row) order is a STABLE sort by the column id j alone.
// That is an LSD radix sort of 32-bit keys with (row, value) payload, done as
// single-pass "onesweep" partitions of <= 9 bits each (C5: 27 bits, 3 passes;
// C2: 24 bits, 3; C4: 17 bits, 2):
//   k_os_hist   one read of the COO: the digit histograms of every pass, plus
//               the input checks (bounds, stored zeros, integrality, sum v^2)
//   k_os_pass   per 4096-entry tile: stable rank of every entry among equal
//               digits (warp match + per-warp counters), the tile's digit
//               counts published and prefixed across tiles by a decoupled
//               look-back, the tile reordered by digit in shared memory and
//               written out in contiguous per-digit runs
//   k_os_heads* fiber heads (j changes) -> fiber ids and offsets; rows must
//               strictly ascend inside a column (duplicates -> ArgumentError;
//               an unsorted input falls back to the general bucket sort)
//   norms       each fiber's squared norm summed in ascending-row order: a
//               thread per fiber (<= 32 entries), a warp (<= 1024), or the
//               block-wide exact sequential sum (seqsum.cuh): bit-identical
//               to the reference.
// Traffic per entry: 12 B (histogram) + 20 B read / 16 B write (first pass) +
// 32 B per further pass + 12 B (heads/norms), no atomics on the data path and
// no partial-sector scatter (bucket.cu's atomic scatter moved 3.3x its bytes).
#include <cstdlib>
#include <vector>

#include "bucket.cuh"
#include "seqsum.cuh"

namespace ctdgpu {

namespace {

constexpr int kOsThreads = 512;
constexpr int kOsItems = 8;
constexpr int kOsTile = kOsThreads * kOsItems;  // entries per tile
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsMaxBits = 9;
constexpr int kOsMaxPass = 4;
constexpr int kOsHeadsPer = 1024;  // entries per block in the heads kernels
constexpr int kOsShort = 32;       // fibers up to this long: norm summed by one thread
constexpr int kOsLong = 1024;      // fibers longer than this: block-wide exact norm

struct Coo {
  int order, mode;
  long long nnz;
  const int32_t* idx[kMaxOrder];
  const double* val;
  long long stride[kMaxOrder];
  long long shape[kMaxOrder];
};

__device__ __forceinline__ uint32_t coo_col(const Coo& c, long long i, int* row, bool* oob) {
  unsigned long long j = 0;
  bool bad = false;
  int r = 0;
  for (int k = 0; k < c.order; ++k) {
    const long long v = c.idx[k][i];
    bad |= (v < 0) | (v >= c.shape[k]);
    if (k == c.mode) r = (int)v;
    else j += (unsigned long long)v * (unsigned long long)c.stride[k];
  }
  *row = r;
  *oob = bad;
  return (uint32_t)j;
}

__global__ void k_os_hist(Coo c, int npass, int dbits, unsigned long long* hist, unsigned* flags, int* intok,
                          double* sumsq) {
  __shared__ unsigned sh[kOsMaxPass << kOsMaxBits];
  const int bins = 1 << dbits;
  for (int t = threadIdx.x; t < npass * bins; t += blockDim.x) sh[t] = 0u;
  __syncthreads();
  double sq = 0.0;
  bool iok = true, oobf = false, zf = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < c.nnz;
       i += (long long)gridDim.x * blockDim.x) {
    int row;
    bool oob;
    const uint32_t j = coo_col(c, i, &row, &oob);
    const double v = c.val[i];
    oobf |= oob;
    zf |= (v == 0.0);
    iok &= (v == rint(v)) && (fabs(v) <= 67108864.0);
    sq += v * v;
    for (int p = 0; p < npass; ++p) atomicAdd(&sh[p * bins + ((j >> (p * dbits)) & (bins - 1))], 1u);
  }
  sq = warp_sum(sq);
  const bool all_ok = __all_sync(0xffffffffu, iok);
  const bool any_oob = __any_sync(0xffffffffu, oobf), any_zero = __any_sync(0xffffffffu, zf);
  if ((threadIdx.x & 31) == 0) {
    if (sq != 0.0) atomicAdd(sumsq, sq);
    if (!all_ok) atomicExch(intok, 0);
    if (any_oob) atomicOr(flags, FLAG_BOUNDS);
    if (any_zero) atomicOr(flags, FLAG_ZERO);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < npass * bins; t += blockDim.x)
    if (sh[t]) atomicAdd(&hist[t], (unsigned long long)sh[t]);
}

// Exclusive scan of every pass's histogram (one block).
__global__ void k_os_scan_hist(const unsigned long long* hist, int npass, int bins, unsigned long long* base) {
  __shared__ unsigned long long sh[33];
  for (int p = 0; p < npass; ++p) {
    const unsigned long long v = threadIdx.x < bins ? hist[p * bins + threadIdx.x] : 0ull;
    const unsigned long long e = block_excl_sum<unsigned long long>(v, sh, nullptr);
    if (threadIdx.x < bins) base[p * bins + threadIdx.x] = e;
  }
}

struct PassArgs {
  Coo c;
  int first, last;
  const uint32_t* jin;
  const int32_t* rin;
  const double* vin;
  uint32_t* jout;
  int32_t* rout;
  double* vout;
  long long n;
  int shift, dbits;
  const unsigned long long* digit_base;  // [bins] global start of each digit
  unsigned long long* status;            // [tiles][bins] look-back words
  unsigned* ticket;
  int bulk;  // 1: every source array 16-byte aligned, full tiles arrive by bulk copy; 2: also the COO index columns
  int ka, kb;     // first pass, order 3: the two non-mode coordinates, j = i_ka + i_kb * mulb
  uint32_t mulb;
};

#ifndef CTD_OS_LEGACY
// 1-D bulk copies (TMA, cp.async.bulk) completing on a shared-memory mbarrier:
// the whole tile (keys, rows, values) is in flight from the CTA's first
// instruction, no registers held, one memory latency per tile.
__device__ __forceinline__ uint32_t os_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void os_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(os_smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void os_mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(os_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void os_bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   os_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(os_smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void os_mbar_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(os_smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

__global__ void __launch_bounds__(kOsThreads, 2) k_os_pass(PassArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int bins = 1 << a.dbits;
  // the tile in INPUT order (bulk-copied), permuted on the way out through sidx
  double* sv = reinterpret_cast<double*>(smem);                                      // [tile]
  uint32_t* sj = reinterpret_cast<uint32_t*>(sv + kOsTile);                          // [tile]
  int32_t* sr = reinterpret_cast<int32_t*>(sj + kOsTile);                            // [tile]
  unsigned long long* gbase = reinterpret_cast<unsigned long long*>(sr + kOsTile);   // [bins]
  unsigned* whist = reinterpret_cast<unsigned*>(gbase + bins);                       // [warps][bins]
  unsigned* doff = whist + kOsWarps * bins;                                          // [bins]
  uint16_t* sidx = reinterpret_cast<uint16_t*>(doff + bins);                         // [tile] slot -> item
  __shared__ long long s_tile;
  __shared__ unsigned sh32[33];
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) {
    const long long t0 = atomicAdd(a.ticket, 1u);
    s_tile = t0;
    const long long st0 = t0 * kOsTile;
    if (a.bulk && a.n - st0 >= kOsTile) {
      os_mbar_init(&s_bar, 1);
      const bool c3 = a.first && a.bulk == 2;  // order-3 COO: the index columns come by bulk copy too
      os_mbar_expect_tx(&s_bar, a.first ? (c3 ? kOsTile * 12u : kOsTile * 8u) : kOsTile * 16u);
      if (!c3) os_bulk_load(sv, (a.first ? a.c.val : a.vin) + st0, kOsTile * 8u, &s_bar);
      if (!a.first) {
        os_bulk_load(sj, a.jin + st0, kOsTile * 4u, &s_bar);
        os_bulk_load(sr, a.rin + st0, kOsTile * 4u, &s_bar);
      } else if (c3) {
        os_bulk_load(sr, a.c.idx[a.c.mode] + st0, kOsTile * 4u, &s_bar);
        os_bulk_load(sj, a.c.idx[a.ka] + st0, kOsTile * 4u, &s_bar);
        os_bulk_load(sv, a.c.idx[a.kb] + st0, kOsTile * 4u, &s_bar);  // parked in the value area; values follow
      }
    }
  }
  // (the counters are cleared while thread 0's ticket and copies are in flight;
  // scalar stores: 16-byte zeroing measured slower at C5, 15.2 vs 13.5 ms per pass)
  for (int t = threadIdx.x; t < kOsWarps * bins; t += blockDim.x) whist[t] = 0u;
  __syncthreads();
  const long long tile = s_tile;
  const long long start = tile * kOsTile;
  const int tn = (int)min((long long)kOsTile, a.n - start);
  const bool bulk = a.bulk && tn == kOsTile;
  const bool c3 = bulk && a.first && a.bulk == 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned mask = (unsigned)bins - 1u;
  unsigned* wh = whist + warp * bins;
  uint32_t jv[kOsItems];
  unsigned lr[kOsItems];
  // warp w owns the contiguous items [w*256, w*256+256) of the tile, 32 per
  // round: ranks follow the item order (stable).
  const int li0 = warp * (32 * kOsItems) + lane;
  if (c3) {
    // j = i_a + i_b * shape_a (fiber_strides, tensor_ops.cpp:106-116; < 2^32)
    // (one warp polls the mbarrier, the others sleep at the CTA barrier: 512
    // polling threads cost the co-resident CTA its issue slots)
    if (warp == 0) os_mbar_wait(&s_bar, 0);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
      const int li = li0 + r * 32;
      jv[r] = sj[li] + reinterpret_cast<const uint32_t*>(sv)[li] * a.mulb;
      sj[li] = jv[r];
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // the values, second phase of the mbarrier (waited for before the write-out)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      os_mbar_expect_tx(&s_bar, kOsTile * 8u);
      os_bulk_load(sv, a.c.val + start, kOsTile * 8u, &s_bar);
    }
  } else if (bulk) {
#ifdef CTD_OS_ALLPOLL
    os_mbar_wait(&s_bar, 0);
#else
    if (warp == 0) os_mbar_wait(&s_bar, 0);
    __syncthreads();
#endif
  }
  if (a.first && !c3) {
    // keys and rows from the COO's index columns (all rounds in flight)
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
      const int li = li0 + r * 32;
      uint32_t j = 0;
      int row = 0;
      if (li < tn) {
        bool oob;
        j = coo_col(a.c, start + li, &row, &oob);
      }
      jv[r] = j;
      sj[li] = j;
      sr[li] = row;
    }
    if (!bulk)
      for (int s = threadIdx.x; s < tn; s += blockDim.x) sv[s] = __ldcs(a.c.val + start + s);
  } else if (!a.first && !bulk) {
    for (int s = threadIdx.x; s < tn; s += blockDim.x) {
      sj[s] = __ldcs(a.jin + start + s);
      sr[s] = __ldcs(a.rin + start + s);
      sv[s] = __ldcs(a.vin + start + s);
    }
    __syncthreads();
  }
  if (!a.first) {
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) jv[r] = sj[li0 + r * 32];
  }
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const bool act = li0 + r * 32 < tn;
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    if (act) {
      const unsigned d = (jv[r] >> a.shift) & mask;
      // lanes with the same digit: one ballot per digit bit (cheaper than
      // MATCH.ANY on this part)
      // (all kOsMaxBits bits, unrolled: the bits above dbits are 0 in every
      // lane and leave peers unchanged)
      unsigned peers = amask;
#pragma unroll
      for (int b = 0; b < kOsMaxBits; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(amask, bit);
        peers &= bal ^ (bit ? 0u : 0xffffffffu);
      }
      const unsigned b0 = wh[d];
      lr[r] = b0 + __popc(peers & ((1u << lane) - 1u));
      __syncwarp(amask);
      if (lane == __ffs(peers) - 1) wh[d] = b0 + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive offsets of the warps, and the tile's total
  unsigned tot = 0;
  if ((int)threadIdx.x < bins) {
    const int d = threadIdx.x;
    for (int w = 0; w < kOsWarps; ++w) {
      const unsigned cnt = whist[w * bins + d];
      whist[w * bins + d] = tot;
      tot += cnt;
    }
  }
  const unsigned excl = block_excl_sum<unsigned>(tot, sh32, nullptr);
  if ((int)threadIdx.x < bins) {
    const int d = threadIdx.x;
    doff[d] = excl;
    // decoupled look-back over the tiles' counts of digit d
    const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = kAgg - 1ull;
    unsigned long long* st = a.status + tile * bins + d;
    if (tile == 0) {
      atomicExch(st, kInc | (unsigned long long)tot);
      gbase[d] = a.digit_base[d] - excl;  // global start of the digit's run minus its tile offset
    } else {
      atomicExch(st, kAgg | (unsigned long long)tot);
      // walk back 8 tiles per round trip (independent loads): a wave of
      // resident tiles otherwise serializes on one load latency per tile
      unsigned long long prefix = 0;
      long long i = tile - 1;
      bool done = false;
      while (!done) {
        unsigned long long w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          w[k] = (i - k >= 0) ? *((volatile unsigned long long*)(a.status + (i - k) * bins + d)) : kInc;
        // common case: all 8 published their aggregate only
        unsigned long long andw = w[0], orw = w[0], sum = w[0] & kVal;
#pragma unroll
        for (int k = 1; k < 8; ++k) {
          andw &= w[k];
          orw |= w[k];
          sum += w[k] & kVal;
        }
        if ((andw >> 62) == 1ull && (orw >> 62) == 1ull) {
          prefix += sum;
          i -= 8;
          continue;
        }
        int k = 0;
        for (; k < 8; ++k) {
          const unsigned long long f = w[k] >> 62;
          if (f == 0) break;  // not published yet: re-read from this tile
          prefix += w[k] & kVal;
          if (f == 2) {
            done = true;
            break;
          }
        }
        if (!done) {
          i -= k;
          if (k < 8) __nanosleep(32);
        }
      }
      atomicExch(st, kInc | (prefix + tot));
      gbase[d] = a.digit_base[d] + prefix - excl;
      CTD_CHECK(prefix + tot <= (unsigned long long)a.n);  // look-back total within the pass
    }
  }
  __syncthreads();
  // slot -> item map of the tile reordered by digit (stable)
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const int li = li0 + r * 32;
    if (li < tn) {
      const unsigned d = (jv[r] >> a.shift) & mask;
      const unsigned pos = doff[d] + whist[warp * bins + d] + lr[r];
      CTD_CHECK(pos < (unsigned)kOsTile);
      sidx[pos] = (uint16_t)li;
    }
  }
  if (c3 && warp == 0) os_mbar_wait(&s_bar, 1);
  __syncthreads();
  // contiguous per-digit runs to global memory
  for (int s = threadIdx.x; s < tn; s += blockDim.x) {
    const int src = sidx[s];
    const uint32_t j = sj[src];
    const unsigned d = (j >> a.shift) & mask;
    const unsigned long long gp = gbase[d] + (unsigned long long)s;
    CTD_CHECK(gp < (unsigned long long)a.n && s >= (int)doff[d]);
    if (a.last) {  // read next by the heads / norms (and, at C2 size, from L2)
      a.jout[gp] = j;
      a.rout[gp] = sr[src];
      a.vout[gp] = sv[src];
    } else {  // consumed by the next pass only: streaming stores
      __stcs(a.jout + gp, j);
      __stcs(a.rout + gp, sr[src]);
      __stcs(a.vout + gp, sv[src]);
    }
  }
}
#else  // CTD_OS_LEGACY: register/LDG staging (round-2 A/B baseline)
__global__ void __launch_bounds__(kOsThreads, 2) k_os_pass(PassArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int bins = 1 << a.dbits;
  double* tv = reinterpret_cast<double*>(smem);                                  // [tile]
  unsigned long long* gbase = reinterpret_cast<unsigned long long*>(tv + kOsTile);  // [bins]
  uint32_t* tj = reinterpret_cast<uint32_t*>(gbase + bins);                      // [tile]
  int32_t* tr = reinterpret_cast<int32_t*>(tj + kOsTile);                        // [tile]
  unsigned* whist = reinterpret_cast<unsigned*>(tr + kOsTile);                   // [warps][bins]
  unsigned* doff = whist + kOsWarps * bins;                                      // [bins]
  __shared__ long long s_tile;
  __shared__ unsigned sh32[33];
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  for (int t = threadIdx.x; t < kOsWarps * bins; t += blockDim.x) whist[t] = 0u;
  __syncthreads();
  const long long tile = s_tile;
  const long long start = tile * kOsTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned mask = (unsigned)bins - 1u;
  unsigned* wh = whist + warp * bins;
  uint32_t jv[kOsItems];
  int32_t rv[kOsItems];  // first pass: the row comes with j from the COO
  unsigned lr[kOsItems];
  // warp w owns the contiguous items [w*256, w*256+256) of the tile, 32 per
  // round: ranks follow the item order (stable).  Only the keys are loaded
  // now (all rounds in flight together); rows and values are read in the
  // scatter below, which keeps the item state in registers (no spills).
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const long long i = start + (long long)warp * (32 * kOsItems) + r * 32 + lane;
    uint32_t j = 0;
    int row = 0;
    if (i < a.n) {
      if (a.first) {
        bool oob;
        j = coo_col(a.c, i, &row, &oob);
      } else {
        j = __ldcs(a.jin + i);
      }
    }
    jv[r] = j;
    rv[r] = row;
  }
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const long long i = start + (long long)warp * (32 * kOsItems) + r * 32 + lane;
    const bool act = i < a.n;
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    if (act) {
      const unsigned d = (jv[r] >> a.shift) & mask;
      // lanes with the same digit: one ballot per digit bit (cheaper than
      // MATCH.ANY on this part)
      unsigned peers = amask;
      for (int b = 0; b < a.dbits; ++b) {
        const unsigned bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(amask, bit);
        peers &= bit ? bal : ~bal;
      }
      const unsigned b0 = wh[d];
      lr[r] = b0 + __popc(peers & ((1u << lane) - 1u));
      __syncwarp(amask);
      if (lane == __ffs(peers) - 1) wh[d] = b0 + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive offsets of the warps, and the tile's total
  unsigned tot = 0;
  if ((int)threadIdx.x < bins) {
    const int d = threadIdx.x;
    for (int w = 0; w < kOsWarps; ++w) {
      const unsigned cnt = whist[w * bins + d];
      whist[w * bins + d] = tot;
      tot += cnt;
    }
  }
  const unsigned excl = block_excl_sum<unsigned>(tot, sh32, nullptr);
  if ((int)threadIdx.x < bins) {
    const int d = threadIdx.x;
    doff[d] = excl;
    // decoupled look-back over the tiles' counts of digit d
    const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = kAgg - 1ull;
    unsigned long long* st = a.status + tile * bins + d;
    if (tile == 0) {
      atomicExch(st, kInc | (unsigned long long)tot);
      gbase[d] = a.digit_base[d];
    } else {
      atomicExch(st, kAgg | (unsigned long long)tot);
      // walk back 8 tiles per round trip (independent loads): a wave of
      // resident tiles otherwise serializes on one load latency per tile
      unsigned long long prefix = 0;
      long long i = tile - 1;
      bool done = false;
      while (!done) {
        unsigned long long w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          w[k] = (i - k >= 0) ? *((volatile unsigned long long*)(a.status + (i - k) * bins + d)) : kInc;
        int k = 0;
        for (; k < 8; ++k) {
          const unsigned long long f = w[k] >> 62;
          if (f == 0) break;  // not published yet: re-read from this tile
          prefix += w[k] & kVal;
          if (f == 2) {
            done = true;
            break;
          }
        }
        if (!done) {
          i -= k;
          if (k < 8) __nanosleep(32);
        }
      }
      atomicExch(st, kInc | (prefix + tot));
      gbase[d] = a.digit_base[d] + prefix;
      CTD_CHECK(prefix + tot <= (unsigned long long)a.n);  // look-back total within the pass
    }
  }
  __syncthreads();
  // the tile reordered by digit (stable) in shared memory
#pragma unroll
  for (int r = 0; r < kOsItems; ++r) {
    const long long i = start + (long long)warp * (32 * kOsItems) + r * 32 + lane;
    if (i < a.n) {
      const unsigned d = (jv[r] >> a.shift) & mask;
      const unsigned pos = doff[d] + whist[warp * bins + d] + lr[r];
      CTD_CHECK(pos < (unsigned)kOsTile);
      tj[pos] = jv[r];
      tr[pos] = a.first ? rv[r] : __ldcs(a.rin + i);
      tv[pos] = a.first ? a.c.val[i] : __ldcs(a.vin + i);
    }
  }
  __syncthreads();
  // contiguous per-digit runs to global memory
  const int tn = (int)min((long long)kOsTile, a.n - start);
  for (int s = threadIdx.x; s < tn; s += blockDim.x) {
    const uint32_t j = tj[s];
    const unsigned d = (j >> a.shift) & mask;
    const unsigned long long gp = gbase[d] + (unsigned long long)(s - (int)doff[d]);
    CTD_CHECK(gp < (unsigned long long)a.n && s >= (int)doff[d]);
    if (a.last) {  // read next by the heads / norms (and, at C2 size, from L2)
      a.jout[gp] = j;
      a.rout[gp] = tr[s];
      a.vout[gp] = tv[s];
    } else {  // consumed by the next pass only: streaming stores
      __stcs(a.jout + gp, j);
      __stcs(a.rout + gp, tr[s]);
      __stcs(a.vout + gp, tv[s]);
    }
  }
}

#endif  // CTD_OS_LEGACY

// Fiber heads: a head where j changes.  Inside a column rows must strictly
// ascend: equal -> duplicate coordinates, descending -> the input was not
// lexicographically sorted (the caller falls back to the general sort).
__device__ __forceinline__ bool os_head(const uint32_t* j, long long p) { return p == 0 || j[p] != j[p - 1]; }

__global__ void k_os_heads_count(const uint32_t* j, const int32_t* row, long long n, unsigned* bcnt, unsigned* flags,
                                 unsigned* unsorted) {
  __shared__ unsigned sh[33];
  const long long b0 = (long long)blockIdx.x * kOsHeadsPer;
  unsigned c = 0;
  bool dup = false, bad = false;
  for (int t = threadIdx.x; t < kOsHeadsPer; t += blockDim.x) {
    const long long p = b0 + t;
    if (p >= n) break;
    if (os_head(j, p)) {
      ++c;
    } else {
      const int r0 = row[p - 1], r1 = row[p];
      dup |= (r1 == r0);
      bad |= (r1 < r0);
    }
  }
  unsigned tot;
  block_excl_sum<unsigned>(c, sh, &tot);
  if (threadIdx.x == 0) bcnt[blockIdx.x] = tot;
  if (__any_sync(0xffffffffu, dup) && (threadIdx.x & 31) == 0) atomicOr(flags, FLAG_DUPLICATE);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(unsorted, 1u);
}

__global__ void k_os_scan_blocks(const unsigned* bcnt, long long nb, unsigned long long* bbase, long long* F_out,
                                 int64_t* fptr, long long n) {
  __shared__ unsigned long long sh[33];
  unsigned long long carry = 0;
  for (long long b0 = 0; b0 < nb; b0 += blockDim.x) {
    const long long b = b0 + threadIdx.x;
    const unsigned long long v = b < nb ? bcnt[b] : 0ull;
    unsigned long long tot;
    const unsigned long long e = block_excl_sum<unsigned long long>(v, sh, &tot);
    if (b < nb) bbase[b] = carry + e;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    *F_out = (long long)carry;
    fptr[carry] = n;
  }
}

__global__ void k_os_heads_write(const uint32_t* j, long long n, const unsigned long long* bbase, int64_t* fcol,
                                 int64_t* fptr) {
  __shared__ unsigned sh[33];
  const long long b0 = (long long)blockIdx.x * kOsHeadsPer;
  // consecutive entries per thread so the block scan follows entry order
  constexpr int kPer = kOsHeadsPer / 256;
  const long long p0 = b0 + (long long)threadIdx.x * kPer;
  unsigned c = 0;
  for (int u = 0; u < kPer; ++u)
    if (p0 + u < n && os_head(j, p0 + u)) ++c;
  unsigned f = block_excl_sum<unsigned>(c, sh, nullptr);
  const unsigned long long base = bbase[blockIdx.x];
  for (int u = 0; u < kPer; ++u) {
    const long long p = p0 + u;
    if (p < n && os_head(j, p)) {
      CTD_CHECK(base + f < (unsigned long long)n);
      fcol[base + f] = j[p];
      fptr[base + f] = p;
      ++f;
    }
  }
}

// column_sq_norms (tensor_ops.cpp:197-198): each fiber's v^2 summed in
// ascending row order.  Fibers up to kOsShort entries: a thread each; longer
// ones are listed for a warp each (k_os_norms_mid) or, beyond kOsLong, the
// block-wide exact sequential sum (k_os_norms_long).
__global__ void k_os_norms(const int64_t* fptr, const long long* F_in, const double* val, double* norm, int* midl,
                           int* nmid) {
  const long long F = *F_in;
  const int lane = threadIdx.x & 31;
  // whole warps iterate together: the list of longer fibers is appended to once
  // per warp (one atomic per listed fiber serialises on nmid at C5)
  for (long long f0 = (long long)blockIdx.x * blockDim.x + threadIdx.x - lane; f0 < F;
       f0 += (long long)gridDim.x * blockDim.x) {
    const long long f = f0 + lane;
    const bool valid = f < F;
    const long long b = valid ? fptr[f] : 0, e = valid ? fptr[f + 1] : 0;
    const bool mid = e - b > kOsShort;
    const unsigned m = __ballot_sync(0xffffffffu, mid);
    if (m) {
      int base = 0;
      if (lane == 0) base = atomicAdd(nmid, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (mid) midl[base + __popc(m & ((1u << lane) - 1u))] = (int)f;
    }
    if (!valid || mid) continue;
    double s = 0.0;
    for (long long q = b; q < e; ++q) s = dadd(s, dsqr(val[q]));
    norm[f] = s;
  }
}

// A warp per listed fiber: 32 values loaded per round (the next round's in
// flight), then added in order by every lane through shuffles.
// Integer tensors (every |v| <= 2^26 and integral, from k_os_hist): squares are
// exact integers, and because they are non-negative every partial sum in ANY
// order is at most the fiber's total.  A fiber whose parallel sum comes out
// below 2^52 therefore had only exactly representable partial sums: the
// result equals the reference's sequential sum bit for bit.  (A true total of
// 2^52 or more cannot round to less, so such fibers are always caught and take
// the sequential path.)  The tensor-wide sum of squares need not be small:
// C5's is ~1e16, its heaviest fiber's ~1e13.
constexpr double kOsExactLimit = 4503599627370496.0;  // 2^52
__device__ __forceinline__ bool os_int_exact(const int* intok) { return intok != nullptr && *intok != 0; }

__global__ void k_os_norms_mid(const int64_t* fptr, const int* list, const int* nlist, const double* val,
                               double* norm, int* longl, int* nlong, const int* intok) {
  const int nl = *nlist;
  const bool exact = os_int_exact(intok);
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  // the next fiber's bounds are fetched while this one is summed (list -> ptr ->
  // values is three dependent latencies per fiber otherwise)
  long long fn = 0, bn = 0, en = 0;
  if (warp < nl) {
    fn = list[warp];
    bn = fptr[fn];
    en = fptr[fn + 1];
  }
  for (long long q0 = warp; q0 < nl; q0 += nw) {
    const long long f = fn, b = bn, e = en;
    if (q0 + nw < nl) {
      fn = list[q0 + nw];
      bn = fptr[fn];
      en = fptr[fn + 1];
    }
    if (e - b > kOsLong) {
      if (lane == 0) longl[atomicAdd(nlong, 1)] = (int)f;
      continue;
    }
    if (exact) {
      double p = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
      long long q = b + lane;
      for (; q + 96 < e; q += 128) {  // four loads in flight per lane
        const double v0 = val[q], v1 = val[q + 32], v2 = val[q + 64], v3 = val[q + 96];
        p = dadd(p, dsqr(v0));
        p1 = dadd(p1, dsqr(v1));
        p2 = dadd(p2, dsqr(v2));
        p3 = dadd(p3, dsqr(v3));
      }
      for (; q < e; q += 32) p = dadd(p, dsqr(val[q]));
      p = warp_sum(dadd(dadd(p, p1), dadd(p2, p3)));
      if (p < kOsExactLimit) {  // warp-uniform
        if (lane == 0) norm[f] = p;
        continue;
      }
    }
    double s = 0.0;
    double cur = (b + lane < e) ? val[b + lane] : 0.0;
    for (long long base = b; base < e; base += 32) {
      const double nxt = (base + 32 + lane < e) ? val[base + 32 + lane] : 0.0;
      const double sq = dsqr(cur);
      const int cnt = (int)min(32ll, e - base);
      for (int t = 0; t < cnt; ++t) s = dadd(s, __shfl_sync(0xffffffffu, sq, t));
      cur = nxt;
    }
    if (lane == 0) norm[f] = s;
  }
}

// Integer-exact long fibers (see os_int_exact): a block per fiber, any order.
__global__ void __launch_bounds__(256, 8) k_os_norms_long_int(const int64_t* fptr, const int* longl, const int* nlong,
                                                              const double* val, double* norm, const int* intok,
                                                              int* longl2, int* nlong2) {
  __shared__ double s_part[2][8];
  if (!os_int_exact(intok)) return;
  const int nl = *nlong;
  int par = 0;
  for (int q = blockIdx.x; q < nl; q += gridDim.x, par ^= 1) {
    const long long f = longl[q];
    const long long b = fptr[f], len = fptr[f + 1] - b;
    const double* v = val + b;
    double p = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    long long i = threadIdx.x;
    const long long B = blockDim.x;
    for (; i + 3 * B < len; i += 4 * B) {  // four loads in flight per thread
      const double v0 = v[i], v1 = v[i + B], v2 = v[i + 2 * B], v3 = v[i + 3 * B];
      p = dadd(p, dsqr(v0));
      p1 = dadd(p1, dsqr(v1));
      p2 = dadd(p2, dsqr(v2));
      p3 = dadd(p3, dsqr(v3));
    }
    for (; i < len; i += B) p = dadd(p, dsqr(v[i]));
    p = warp_sum(dadd(dadd(p, p1), dadd(p2, p3)));
    if ((threadIdx.x & 31) == 0) s_part[par][threadIdx.x >> 5] = p;
    __syncthreads();  // (the slots alternate, so one barrier per fiber is enough)
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = dadd(t, s_part[par][w]);
      if (t < kOsExactLimit) norm[f] = t;
      else longl2[atomicAdd(nlong2, 1)] = (int)f;  // sequential path (k_os_norms_long)
    }
  }
}

__global__ void __launch_bounds__(256) k_os_norms_long(const int64_t* fptr, const int* longl, const int* nlong,
                                                       const double* val, double* norm, unsigned* flags,
                                                       const int* intok, const int* longl2, const int* nlong2) {
  __shared__ SeqSumSmem S;
  // integer tensors: only the fibers k_os_norms_long_int passed on
  const bool ints = os_int_exact(intok);
  if (ints) longl = longl2;
  const int nl = ints ? *nlong2 : *nlong;
  for (int q = blockIdx.x; q < nl; q += gridDim.x) {
    const long long f = longl[q];
    const double* v = val + fptr[f];
    auto get = [v](long long i) { return dsqr(v[i]); };
    bool bad = false;
    const double s = block_exact_sum(get, fptr[f + 1] - fptr[f], S, &bad);
    if (threadIdx.x == 0) {
      norm[f] = s;
      if (bad) atomicOr(flags, FLAG_SEQSUM);
    }
    __syncthreads();
  }
}

int os_bits_for(unsigned long long n) {
  int b = 0;
  while (b < 63 && (1ull << b) < n) ++b;
  return b;
}

}  // namespace

void fiber_norms(Ctx* ctx, Fibers& fb) {
  const long long nnz = fb.nnz, F = fb.F;
  fb.norm.alloc(ctx, F + 1);
  if (F == 0) return;
  Buf<long long> dF(ctx, 1);
  ctx->to_dev(dF.p, &F, 1);
  Buf<int> midl(ctx, nnz / kOsShort + 2), nmid(ctx, 1), longl(ctx, nnz / kOsLong + 2), nlong(ctx, 1);
  nmid.zero();
  nlong.zero();
  const unsigned ngrid = (unsigned)std::min<long long>((F + 255) / 256, (long long)ctx->sm_count * 16);
  LAUNCH(ctx, k_os_norms, ngrid, 256, 0, fb.ptr.p, dF.p, fb.val.p, fb.norm.p, midl.p, nmid.p);
  LAUNCH(ctx, k_os_norms_mid, (unsigned)ctx->sm_count * 8, 256, 0, fb.ptr.p, midl.p, nmid.p, fb.val.p, fb.norm.p,
         longl.p, nlong.p, (const int*)nullptr);
  LAUNCH(ctx, k_os_norms_long, (unsigned)ctx->sm_count * 4, 256, 0, fb.ptr.p, longl.p, nlong.p, fb.val.p, fb.norm.p,
         ctx->d_flags, (const int*)nullptr, (const int*)nullptr, (const int*)nullptr);
}

bool matricize_onesweep(Ctx* ctx, const Tensor& x, int mode, Fibers& out) {
  Coo c{};
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
  const long long nnz = x.nnz;
  if (acc > (1ll << 32) || nnz >= (1ll << 40) || nnz == 0) return false;
  out.rows = x.shape[mode];
  out.cols = acc;
  out.nnz = nnz;
  out.mode = mode;
  const int bits = std::max(1, os_bits_for((unsigned long long)acc));
  const int npass = (bits + kOsMaxBits - 1) / kOsMaxBits;
  const int dbits = (bits + npass - 1) / npass;
  const int bins = 1 << dbits;
  // validation, histograms
  Buf<unsigned long long> hist(ctx, (size_t)npass * bins), dbase(ctx, (size_t)npass * bins);
  hist.zero();
  Buf<int> intok(ctx, 1);
  Buf<double> sumsq(ctx, 1);
  sumsq.zero();
  {
    const int one = 1;
    ctx->to_dev(intok.p, &one, 1);
  }
  const unsigned hgrid = (unsigned)std::min<long long>((nnz + 255) / 256, (long long)ctx->sm_count * 8);
  LAUNCH(ctx, k_os_hist, hgrid, 256, 0, c, npass, dbits, hist.p, ctx->d_flags, intok.p, sumsq.p);
  LAUNCH(ctx, k_os_scan_hist, 1, 512, 0, hist.p, npass, bins, dbase.p);
  // LSD passes: ping-pong, the last one into the output arrays
  out.row.alloc(ctx, nnz);
  out.val.alloc(ctx, nnz);
  Buf<uint32_t> ja(ctx, nnz), jb(ctx, npass > 1 ? nnz : 1);
  Buf<int32_t> ra(ctx, npass > 1 ? nnz : 1);
  Buf<double> va(ctx, npass > 1 ? nnz : 1);
  const long long tiles = (nnz + kOsTile - 1) / kOsTile;
  Buf<unsigned long long> status(ctx, (size_t)tiles * bins);
  Buf<unsigned> ticket(ctx, 1);
#ifndef CTD_OS_LEGACY
  constexpr size_t kOsSlot = 2;  // the slot -> item map
#else
  constexpr size_t kOsSlot = 0;
#endif
  const size_t smem = (size_t)kOsTile * (8 + 4 + 4 + kOsSlot) + (size_t)bins * 8 + (size_t)(kOsWarps + 1) * bins * 4;
  static unsigned long long attr_done = 0;
  if (first_on_device(&attr_done, ctx->device)) {
    const size_t smax = (size_t)kOsTile * (16 + kOsSlot) + ((size_t)1 << kOsMaxBits) * (8 + (kOsWarps + 1) * 4);
    CUDA_OK(cudaFuncSetAttribute(k_os_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
  }
  for (int p = 0; p < npass; ++p) {
    // pass p reads the previous pass's output; the destinations alternate so
    // that the last pass lands in (jfinal, out.row, out.val)
    const bool last = p == npass - 1;
    PassArgs pa{};
    pa.c = c;
    pa.first = p == 0;
    const bool to_a = ((npass - 1 - p) & 1) == 0;  // last pass -> the "a"/output side
    uint32_t* jdst = to_a ? ja.p : jb.p;
    const uint32_t* jsrc = to_a ? jb.p : ja.p;
    pa.jin = jsrc;
    pa.rin = to_a ? ra.p : out.row.p;
    pa.vin = to_a ? va.p : out.val.p;
    pa.jout = jdst;
    pa.rout = to_a ? out.row.p : ra.p;
    pa.vout = to_a ? out.val.p : va.p;
    pa.last = last ? 1 : 0;
    pa.n = nnz;
    pa.shift = p * dbits;
    pa.dbits = dbits;
    pa.digit_base = dbase.p + (size_t)p * bins;
    pa.status = status.p;
    pa.ticket = ticket.p;
    pa.bulk = (((uintptr_t)(pa.first ? (const void*)c.val : (const void*)pa.vin) | (uintptr_t)pa.jin | (uintptr_t)pa.rin) & 15) == 0;
    if (pa.first && pa.bulk && c.order == 3 &&
        (((uintptr_t)c.idx[0] | (uintptr_t)c.idx[1] | (uintptr_t)c.idx[2]) & 15) == 0) {
      pa.ka = mode == 0 ? 1 : 0;
      pa.kb = mode == 2 ? 1 : 2;
      pa.mulb = (uint32_t)c.shape[pa.ka];
      pa.bulk = 2;
    }
    status.zero();
    ticket.zero();
    LAUNCH(ctx, k_os_pass, (unsigned)tiles, kOsThreads, smem, pa);
  }
  // fibers: heads, offsets, norms
  const uint32_t* jf = ja.p;
  const long long hb = (nnz + kOsHeadsPer - 1) / kOsHeadsPer;
  Buf<unsigned> bcnt(ctx, hb), uns(ctx, 1);
  Buf<unsigned long long> bbase(ctx, hb);
  uns.zero();
  Buf<long long> dF(ctx, 1);
  out.col.alloc(ctx, nnz + 1);
  out.ptr.alloc(ctx, nnz + 1);
  out.norm.alloc(ctx, nnz + 1);
  LAUNCH(ctx, k_os_heads_count, (unsigned)hb, 256, 0, jf, out.row.p, nnz, bcnt.p, ctx->d_flags, uns.p);
  LAUNCH(ctx, k_os_scan_blocks, 1, 1024, 0, bcnt.p, hb, bbase.p, dF.p, out.ptr.p, nnz);
  LAUNCH(ctx, k_os_heads_write, (unsigned)hb, 256, 0, jf, nnz, bbase.p, out.col.p, out.ptr.p);
  Buf<int> midl(ctx, nnz / kOsShort + 2), nmid(ctx, 1), longl(ctx, nnz / kOsLong + 2), nlong(ctx, 1);
  Buf<int> longl2(ctx, nnz / kOsLong + 2), nlong2(ctx, 1);
  nmid.zero();
  nlong.zero();
  nlong2.zero();
  const unsigned ngrid = (unsigned)std::min<long long>((nnz + 255) / 256, (long long)ctx->sm_count * 16);
  LAUNCH(ctx, k_os_norms, ngrid, 256, 0, out.ptr.p, dF.p, out.val.p, out.norm.p, midl.p, nmid.p);
  LAUNCH(ctx, k_os_norms_mid, (unsigned)ctx->sm_count * 8, 256, 0, out.ptr.p, midl.p, nmid.p, out.val.p, out.norm.p,
         longl.p, nlong.p, (const int*)intok.p);
  LAUNCH(ctx, k_os_norms_long_int, (unsigned)ctx->sm_count * 8, 256, 0, out.ptr.p, longl.p, nlong.p, out.val.p,
         out.norm.p, (const int*)intok.p, longl2.p, nlong2.p);
  LAUNCH(ctx, k_os_norms_long, (unsigned)ctx->sm_count * 4, 256, 0, out.ptr.p, longl.p, nlong.p, out.val.p,
         out.norm.p, ctx->d_flags, (const int*)intok.p, (const int*)longl2.p, (const int*)nlong2.p);
  long long F = 0;
  int iok = 0;
  double ssq = 0.0;
  unsigned unsorted = 0;
  ctx->to_host(&F, dF.p, 1);
  ctx->to_host(&iok, intok.p, 1);
  ctx->to_host(&ssq, sumsq.p, 1);
  ctx->to_host(&unsorted, uns.p, 1);
  ctx->sync();
  if (unsorted) return false;  // rows not ascending inside a column: general sort
  out.F = F;
  out.sum_sq = ssq;
  out.integer_exact = iok && ssq < 4503599627370496.0;  // 2^52
  ctx->check_flags("matricize");
  return true;
}

}  // namespace ctdgpu
