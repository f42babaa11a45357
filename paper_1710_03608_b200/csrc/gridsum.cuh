// Grid-distributed exact sequential sum of non-negative terms (the residual
// of try_append_fiber, fiber_basis.cpp:66-77) inside the persistent filter
// kernel.  Same algorithm as seqsum.cuh's block version, split over CTAs:
//   A (every CTA) classify one contiguous slice of the terms: approximate
//     prefix before the slice (a redundant strided read of the earlier terms),
//     binade classification, run monoids, the slice's segmented aggregate and
//     its direct elements -> published to global memory;
//   -- grid barrier --
//   B (every CTA, redundantly) segmented scan of the slice aggregates, then
//     one thread walks the few direct elements in order.  Every CTA derives
//     the same total, so no barrier follows.
// A failed self-check (direct-list overflow, run leaving its binade) falls
// back to a plain sequential sum, so the result is always the sequential one.
#pragma once
#include "seqsum.cuh"

namespace ctdgpu {

constexpr int kSliceDirects = 64;     // per-slice direct capacity before fallback
constexpr int kMaxDirectsTotal = 2048; // shared-memory walker capacity (64 KB)

struct SliceDirect {
  double x;
  Mono m;     // run monoid before it (within the slice, or from slice start)
  int inh;    // 1: no head before it inside the slice (prepend the carry)
  short e;    // e of the element before it; 0x7ffe: the previous slice's last
};

struct SliceSum {
  Seg agg;
  int nd;       // directs, -1 = overflow
  short last_e; // class/e of the slice's last element; 0x7fff: empty slice
  double head;  // slice 0: its exact sequential sum (summarized as one direct block)
};
static_assert(sizeof(SliceSum) % 8 == 0 && sizeof(SliceDirect) % 8 == 0, "8-byte words");

// Cross-CTA data is read through L2 (ld.global.cg): L1 is not coherent.
template <typename T>
__device__ __forceinline__ T ldcg_struct(const T* p) {
  T out;
  const long long* s = reinterpret_cast<const long long*>(p);
  long long* d = reinterpret_cast<long long*>(&out);
#pragma unroll
  for (int k = 0; k < (int)(sizeof(T) / 8); ++k) d[k] = __ldcg(s + k);
  return out;
}

// Step A.  `get(i)` returns term i (global index).  All threads of every CTA
// participate.
template <typename Get>
__device__ void slice_summarize(const Get& get, long long nt, SliceSum* ps, SliceDirect* pd,
                                SeqSumSmem& S) {
  const int T = blockDim.x, t = threadIdx.x;
  const long long nbk = gridDim.x, b = blockIdx.x;
  const long long per_slice = (nt + nbk - 1) / nbk;
  const long long s0 = min(b * per_slice, nt), s1 = min(s0 + per_slice, nt);
  // approximate prefix before the slice (any order)
  double part = 0.0;
  {
    long long i = t;
    for (; i + 3 * T < s0; i += 4 * T) {
      const double v0 = get(i), v1 = get(i + T), v2 = get(i + 2 * T), v3 = get(i + 3 * T);
      part += (v0 + v1) + (v2 + v3);
    }
    for (; i < s0; i += T) part += get(i);
  }
  const double P0 = block_sum<double>(part, S.dsh);
  const long long n = s1 - s0;
  const long long per = (n + T - 1) / T;
  const long long b0 = s0 + min((long long)t * per, n), b1 = s0 + min((long long)(t + 1) * per, n);
  double xv[4];
  double cs = 0.0;
  for (long long i = b0; i < b1; ++i) {
    const double v = get(i);
    if (i - b0 < 4) xv[i - b0] = v;
    cs += v;
  }
  const double pre = block_excl_sum<double>(cs, S.dsh, nullptr) + P0;
  const double mg = seq_margin(nt);
  auto term = [&](long long i) -> double { return (i - b0 < 4) ? xv[i - b0] : get(i); };
  Seg agg{0, mono_id()};
  int nd = 0;
  short le = (short)0x7fff;
  int fe = 0;
  const bool fast = (b0 > 0) && (b0 < b1) && seq_chunk_regular(pre, pre + cs, mg, &fe);
  if (fast) {
    for (long long i = b0; i < b1; ++i) {
      Mono m;
      seq_mono(term(i), fe, &m);
      agg.m = mono_cat(agg.m, m);
    }
    le = (short)fe;
  } else {
    double P = pre;
    for (long long i = b0; i < b1; ++i) {
      const double x = term(i);
      const double Pc = P + x;
      int e = 0;
      Mono m;
      const int c = seq_classify(i == 0, P, Pc, x, mg, &e, &m);
      if (c == CLS_REG) {
        agg.m = mono_cat(agg.m, m);
        le = (short)e;
      } else {
        agg.h = 1;
        agg.m = mono_id();
        if (c == CLS_DIRECT) ++nd;
        le = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
      }
      P = Pc;
    }
  }
  S.last_e[t] = (b0 < b1) ? le : (short)0x7fff;
  Seg tot;
  const Seg carry = block_seg_excl(agg, S.ssh, &tot);
  int ntot;
  int dpos = block_excl_sum<int>(nd, S.ish, &ntot);
  const bool over = ntot > kSliceDirects;
  if (!over && !fast && nd > 0) {
    // e of the element before my chunk: the previous chunk (chunks fill in
    // thread order), else the previous slice (resolved by the walker).
    short prev_e = (t > 0) ? S.last_e[t - 1] : (short)0x7ffe;
    double P = pre;
    Mono M = carry.m;
    int inh = carry.h ? 0 : 1;
    for (long long i = b0; i < b1; ++i) {
      const double x = term(i);
      const double Pc = P + x;
      int e = 0;
      Mono m;
      const int c = seq_classify(i == 0, P, Pc, x, mg, &e, &m);
      if (c == CLS_REG) {
        M = mono_cat(M, m);
        prev_e = (short)e;
      } else {
        if (c == CLS_DIRECT) {
          SliceDirect d;
          d.x = x;
          d.m = M;
          d.inh = inh;
          d.e = prev_e;
          pd[b * kSliceDirects + dpos] = d;
          ++dpos;
        }
        M = mono_id();
        inh = 0;
        prev_e = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
      }
      P = Pc;
    }
  }
  // the slice summary, published by the owner of the slice's last element
  const long long tlast = n > 0 ? (n - 1) / per : 0;
  if (t == tlast) {
    SliceSum s;
    s.agg = tot;
    s.nd = over ? -1 : ntot;
    s.last_e = (n > 0) ? le : (short)0x7fff;
    ps[b] = s;
  }
}

// Step B (after a grid barrier).  Returns the exact sequential total; *fail
// when the fallback was needed.  `scratch` is shared memory for up to
// gridDim.x slices and their directs.
template <typename Get>
__device__ double slice_combine(const Get& get, long long nt, const SliceSum* ps, const SliceDirect* pd,
                                SeqSumSmem& S, double* scratch, bool* fail) {
  const int T = blockDim.x, t = threadIdx.x;
  const int nbk = gridDim.x;
  Seg* sagg = reinterpret_cast<Seg*>(scratch);                 // [nbk]
  Mono* scin = reinterpret_cast<Mono*>(sagg + nbk);            // [nbk]
  int* snd = reinterpret_cast<int*>(scin + nbk);               // [nbk]
  int* sdoff = snd + nbk;                                      // [nbk]
  short* slast = reinterpret_cast<short*>(sdoff + nbk);        // [nbk]
  // slast + nbk holds sprev[nbk]; then the ordered directs and their slices
  SliceDirect* sdir = reinterpret_cast<SliceDirect*>(
      (reinterpret_cast<uintptr_t>(slast + 2 * nbk) + 15) & ~uintptr_t(15));  // [kMaxDirectsTotal]
  __syncthreads();
  int any_over = 0;
  Seg v{0, mono_id()};
  int ndv = 0;
  if (t < nbk) {
    const SliceSum s = ldcg_struct(ps + t);
    v = s.agg;
    ndv = s.nd < 0 ? 0 : s.nd;
    any_over = s.nd < 0;
    sagg[t] = s.agg;
    snd[t] = ndv;
    slast[t] = s.last_e;
  }
  const Seg cin = block_seg_excl(v, S.ssh, nullptr);
  int total_d;
  const int off = block_excl_sum<int>(ndv, S.ish, &total_d);
  const int over = __syncthreads_or(any_over || total_d > kMaxDirectsTotal);
  if (t < nbk) {
    scin[t] = cin.m;
    sdoff[t] = off;
  }
  __syncthreads();
  // class/e of the element before slice t (last non-empty earlier slice)
  short* sprev = slast + nbk;  // reuse: [nbk] after slast (fits before sdir alignment pad)
  if (t < nbk) {
    short p = E_ZERO;
    for (int q = t - 1; q >= 0; --q)
      if (slast[q] != (short)0x7fff) { p = slast[q]; break; }
    sprev[t] = p;
  }
  // cooperative copy of the directs into one ordered list
  if (!over) {
    for (int idx = t; idx < total_d; idx += T) {
      int lo = 0, hi = nbk - 1;  // last slice with sdoff <= idx and snd > 0
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sdoff[mid] <= idx) lo = mid;
        else hi = mid - 1;
      }
      while (snd[lo] == 0 || sdoff[lo] + snd[lo] <= idx) ++lo;
      SliceDirect d = ldcg_struct(pd + (long long)lo * kSliceDirects + (idx - sdoff[lo]));
      d.e = (d.e == (short)0x7ffe) ? (short)(-32000) : d.e;  // mark "previous slice"
      sdir[idx] = d;
      reinterpret_cast<int*>(sdir + kMaxDirectsTotal)[idx] = lo;
    }
  }
  __syncthreads();
  if (t == 0) {
    bool ok = !over;
    double acc = 0.0, head = 0.0;
    const int* sslice = reinterpret_cast<const int*>(sdir + kMaxDirectsTotal);
    short prev_last = E_ZERO;
    if (ok) {
      for (int idx = 0; idx < total_d && ok; ++idx) {
        const SliceDirect d = sdir[idx];
        const int s = sslice[idx];
        const Mono M = d.inh ? mono_cat(scin[s], d.m) : d.m;
        const short eb = (d.e == (short)(-32000)) ? sprev[s] : d.e;
        acc = head;
        if (eb >= -1100 && eb <= 1100) ok = seq_apply_run(head, eb, M, &acc);
        acc = dadd(acc, d.x);
        head = acc;
      }
      for (int q = nbk - 1; q >= 0; --q)
        if (slast[q] != (short)0x7fff) { prev_last = slast[q]; break; }
      acc = head;
      if (ok && prev_last >= -1100 && prev_last <= 1100) {
        // run from the last head to the end: carry through the last slice
        const Seg fin = seg_cat(Seg{0, scin[nbk - 1]}, sagg[nbk - 1]);
        ok = seq_apply_run(head, prev_last, fin.m, &acc);
      }
    }
    if (!ok) {  // sequential fallback: always the reference order
      acc = 0.0;
      for (long long i = 0; i < nt; ++i) acc = dadd(acc, get(i));
    }
    S.result = acc;
    S.bad = ok ? 0 : 1;
  }
  __syncthreads();
  const double r = S.result;
  if (fail) *fail = S.bad != 0;
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// Single-warp-per-CTA variant used by the filter: the same slice algorithm,
// but every scan is a warp shuffle scan (no CTA barriers), the approximate
// prefix before a slice comes from the earlier slices' published local sums
// (each CTA publishes its own, so nothing chains), and the slice summaries are
// published with per-slice epoch flags that the combiners wait on instead of
// a grid barrier.  Called by warp 0 of every CTA; all CTAs are co-resident.
// One 128-byte line per slice for the published sums and flags, so the
// pollers of different slices never share an L2 line.
struct SliceLoc {
  double s;
  unsigned epoch;
  unsigned pad[29];
};
static_assert(sizeof(SliceLoc) == 128, "one line per slice");
constexpr int kFlagStride = 32;  // unsigned per slice flag (128 bytes)

// Polls with a short back-off so that many waiting warps do not saturate the
// L2 slice holding the flag.
__device__ __forceinline__ void wait_epoch(const unsigned* f, unsigned epoch);
constexpr int kMaxSlices = 256;
constexpr int kWarpCache = 4;  // terms cached in registers per lane

constexpr int kCombineBar = 8;  // named barrier of the combine warps
struct WarpSumSmem {
  Seg rt_seg[kMaxSlices / 32];   // per-round (32 slices) totals of the combine
  int rt_nd[kMaxSlices / 32];
  int rt_last[kMaxSlices / 32];
  int rt_over[kMaxSlices / 32];
  SliceSum ss[kMaxSlices];
  Mono cin[kMaxSlices];
  int doff[kMaxSlices];
  int nd[kMaxSlices];
  short sprev[kMaxSlices];
  Mono finm;
  short prev_last;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void wait_epoch(const unsigned* f, unsigned epoch) {
  while (ld_relaxed_u32(f) != epoch) __nanosleep(64);
  fence_acq_rel_gpu();
}

__device__ __forceinline__ Seg warp_seg_excl(Seg v, Seg* total) {
  const int l = threadIdx.x & 31;
  Seg inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Seg o = seg_shfl_up(inc, d);
    if (l >= d) inc = seg_cat(o, inc);
  }
  Seg ex = seg_shfl_up(inc, 1);
  if (l == 0) ex = Seg{0, mono_id()};
  if (total) {
    total->h = __shfl_sync(0xffffffffu, inc.h, 31);
    total->m.a0 = __shfl_sync(0xffffffffu, inc.m.a0, 31);
    total->m.a1 = __shfl_sync(0xffffffffu, inc.m.a1, 31);
  }
  return ex;
}

template <typename T>
__device__ __forceinline__ T warp_excl(T v, T* total) {
  const T inc = warp_incl_sum(v);
  if (total) *total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

template <typename Get>
__device__ double warp_grid_sum(const Get& get, long long nt, unsigned epoch, SliceLoc* loc, SliceSum* ps,
                                SliceDirect* pd, unsigned* sflag, WarpSumSmem& W, SliceDirect* sdir,
                                int* sslice, bool* fail, long long* tp = nullptr) {
  const unsigned FULL = 0xffffffffu;
#define WGS_STAMP(k) \
  if (tp && blockIdx.x == 0 && (threadIdx.x & 31) == 0) tp[k] = clock64();
  WGS_STAMP(0)
  const int lane = threadIdx.x & 31;
  const int cw = threadIdx.x >> 5;  // combine warp (warps 0..ceil(nbk/32)-1 call this)
  const int nbk = gridDim.x, b = blockIdx.x;
  constexpr int kR = kMaxSlices / 32;
  if (cw == 0) {
  // ---- A: summarize slice b (one per CTA), warp 0
  const long long per_slice = (nt + nbk - 1) / nbk;
  const long long s0 = min((long long)b * per_slice, nt), s1 = min(s0 + per_slice, nt);
  const long long n = s1 - s0;
  const long long per = (n + 31) / 32;
  const long long b0 = s0 + min((long long)lane * per, n), b1 = s0 + min((long long)(lane + 1) * per, n);
  double xv[kWarpCache];
  get.batch(b0, b1, xv);
  double cs = 0.0;
#pragma unroll
  for (int k = 0; k < kWarpCache; ++k) cs += xv[k];
  for (long long i = b0 + kWarpCache; i < b1; ++i) cs += get(i);
  WGS_STAMP(1)
  double T;
  const double ex = warp_excl<double>(cs, &T);
  if (lane == 0) {
    __stcg(&loc[b].s, T);
    st_release_u32(&loc[b].epoch, epoch);
  }
  // earlier slices' sums (approximate prefix; any order): polls together
  for (;;) {
    bool ready = true;
#pragma unroll
    for (int k = 0; k < kR; ++k) {
      const int c = lane + 32 * k;
      if (c < b) ready &= ld_relaxed_u32(&loc[c].epoch) == epoch;
    }
    if (__all_sync(FULL, ready)) break;
  }
  fence_acq_rel_gpu();  // relaxed polls + fence: acquire for the loads below
  double p0 = 0.0;
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    const int c = lane + 32 * k;
    if (c < b) p0 += __ldcg(&loc[c].s);
  }
  const double pre = warp_sum(p0) + ex;  // approximate prefix before my chunk
  WGS_STAMP(2)
  const double mg = seq_margin(nt);
  // classify the cached terms independently (their approximate prefixes
  // first: one add chain), so the branchy per-term work overlaps
  const int nc = (int)min((long long)kWarpCache, b1 - b0);
  // Slice 0 holds the head of the sum, where the small running value crosses
  // binades often (many directs, slow classification): lane 0 adds it
  // sequentially instead, and it enters the combine as one direct block.
  const bool head_slice = (b == 0) && (per <= kWarpCache);
  double hsum = 0.0;
  if (head_slice) {
    for (int l = 0; l < 32; ++l) {
      const int cl = __shfl_sync(FULL, nc, l);
#pragma unroll
      for (int k = 0; k < kWarpCache; ++k) {
        const double x = __shfl_sync(FULL, xv[k], l);
        if (k < cl) hsum = dadd(hsum, x);
      }
    }
    hsum = __shfl_sync(FULL, hsum, 0);
  }
  double Pv[kWarpCache + 1];
  Pv[0] = pre;
#pragma unroll
  for (int k = 0; k < kWarpCache; ++k) Pv[k + 1] = Pv[k] + xv[k];
  int cls[kWarpCache], ee[kWarpCache];
  Mono mm[kWarpCache];
#pragma unroll
  for (int k = 0; k < kWarpCache; ++k) {
    ee[k] = 0;
    mm[k] = mono_id();
    cls[k] = CLS_ZERO;
    if (k < nc && !head_slice) cls[k] = seq_classify_fp(b0 + k == 0, Pv[k], Pv[k + 1], xv[k], mg, &ee[k], &mm[k]);
  }
  Seg agg{0, mono_id()};
  int nd = 0;
  short le = (short)0x7fff;
  if (head_slice && nc > 0) {
    agg.h = 1;
    le = E_DIRECT;
  }
#pragma unroll
  for (int k = 0; k < kWarpCache; ++k) {
    if (k < nc && !head_slice) {
      if (cls[k] == CLS_REG) {
        agg.m = mono_cat(agg.m, mm[k]);
        le = (short)ee[k];
      } else {
        agg.h = 1;
        agg.m = mono_id();
        if (cls[k] == CLS_DIRECT) ++nd;
        le = (cls[k] == CLS_DIRECT) ? E_DIRECT : E_ZERO;
      }
    }
  }
  // terms beyond the register cache (large slices): sequential
  double P = Pv[kWarpCache];
  for (long long i = b0 + kWarpCache; i < b1; ++i) {
    const double x = get(i);
    const double Pc = P + x;
    int e = 0;
    Mono m;
    const int c = seq_classify_fp(i == 0, P, Pc, x, mg, &e, &m);
    if (c == CLS_REG) {
      agg.m = mono_cat(agg.m, m);
      le = (short)e;
    } else {
      agg.h = 1;
      agg.m = mono_id();
      if (c == CLS_DIRECT) ++nd;
      le = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
    }
    P = Pc;
  }
  const short le_chunk = (b0 < b1) ? le : (short)0x7fff;
  Seg tot;
  const Seg carry = warp_seg_excl(agg, &tot);
  int ntot;
  int dpos = warp_excl<int>(nd, &ntot);
  const bool over = ntot > kSliceDirects;
  // e of the element before my chunk: the previous lane's last (chunks fill
  // lanes in order), else the previous slice (resolved in the combine)
  const short prev_lane_e = (short)__shfl_up_sync(FULL, (int)le_chunk, 1);
  if (!over && nd > 0) {
    short prev_e = (lane > 0) ? prev_lane_e : (short)0x7ffe;
    Mono M = carry.m;
    int inh = carry.h ? 0 : 1;
    auto step = [&](int c, int e, const Mono& m, double x) {
      if (c == CLS_REG) {
        M = mono_cat(M, m);
        prev_e = (short)e;
      } else {
        if (c == CLS_DIRECT) {
          SliceDirect d;
          d.x = x;
          d.m = M;
          d.inh = inh;
          d.e = prev_e;
          pd[(long long)b * kSliceDirects + dpos] = d;
          ++dpos;
        }
        M = mono_id();
        inh = 0;
        prev_e = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
      }
    };
#pragma unroll
    for (int k = 0; k < kWarpCache; ++k)
      if (k < nc) step(cls[k], ee[k], mm[k], xv[k]);
    double P2 = Pv[kWarpCache];
    for (long long i = b0 + kWarpCache; i < b1; ++i) {
      const double x = get(i);
      const double Pc = P2 + x;
      int e = 0;
      Mono m;
      const int c = seq_classify(i == 0, P2, Pc, x, mg, &e, &m);
      step(c, e, m, x);
      P2 = Pc;
    }
  }
  WGS_STAMP(3)
  const long long tlast = n > 0 ? (n - 1) / per : 0;
  if (lane == tlast) {
    SliceSum s;
    s.agg = tot;
    s.nd = over ? -1 : ntot;
    s.last_e = (n > 0) ? le : (short)0x7fff;
    s.head = hsum;
    ps[b] = s;
  }
  __syncwarp();  // orders the other lanes' summary/direct writes before lane 0's release
  if (lane == 0) st_release_u32(&sflag[b * kFlagStride], epoch);
#ifdef CTD_WGS_GT
  if (lane == 0) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); CTD_WGS_GT[b] = g; }
#endif
  }  // warp 0: part A
  // ---- B: combine all slices (redundantly in every CTA).  Combine warp w
  // takes slices 32w..32w+31 (one warp scan each); the rounds' totals are
  // exchanged through shared memory and each warp applies its carry.
  const int R = (nbk + 31) / 32;
  const int c = 32 * cw + lane;
  SliceSum sv;
  sv.agg = Seg{0, mono_id()};
  sv.nd = 0;
  sv.last_e = (short)0x7fff;
  sv.head = 0.0;
  if (cw == 0) {
    // warp 0 alone polls every slice's flag (no polling traffic from the
    // other combine warps), then releases them
    for (;;) {
      bool ready = true;
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const int cc = lane + 32 * k;
        if (cc < nbk) ready &= ld_relaxed_u32(&sflag[cc * kFlagStride]) == epoch;
      }
      if (__all_sync(FULL, ready)) break;
    }
    fence_acq_rel_gpu();
  }
  asm volatile("bar.sync %0, %1;" ::"r"(kCombineBar), "r"(R * 32) : "memory");
  if (c < nbk) sv = ldcg_struct(ps + c);
#ifdef CTD_WGS_GT
  if (lane == 0 && cw == 0) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); CTD_WGS_GT[256 + b] = g; }
#endif
  WGS_STAMP(4)
  Seg rtot;
  const Seg ex = warp_seg_excl(sv.agg, &rtot);
  const int ndv = sv.nd < 0 ? 0 : sv.nd;
  int rnd;
  const int offl = warp_excl<int>(ndv, &rnd);
  int pl = sv.last_e;  // nearest non-empty slice before mine within the round
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(FULL, pl, d);
    if (lane >= d && pl == 0x7fff) pl = o;
  }
  int prevl = __shfl_up_sync(FULL, pl, 1);
  if (lane == 0) prevl = 0x7fff;
  const int rlast = __shfl_sync(FULL, pl, 31);
  const int rover = __any_sync(FULL, sv.nd < 0) ? 1 : 0;
  if (lane == 0) {
    W.rt_seg[cw] = rtot;
    W.rt_nd[cw] = rnd;
    W.rt_last[cw] = rlast;
    W.rt_over[cw] = rover;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(kCombineBar), "r"(R * 32) : "memory");
  Seg car{0, mono_id()};
  int doff0 = 0, last0 = 0x7fff, total_d = 0, last_all = 0x7fff, any_over = 0;
  for (int r = 0; r < R; ++r) {
    if (r < cw) {
      car = seg_cat(car, W.rt_seg[r]);
      doff0 += W.rt_nd[r];
      if (W.rt_last[r] != 0x7fff) last0 = W.rt_last[r];
    }
    total_d += W.rt_nd[r];
    any_over |= W.rt_over[r];
    if (W.rt_last[r] != 0x7fff) last_all = W.rt_last[r];
  }
  const bool over_all = any_over || total_d > kMaxDirectsTotal;
  if (c < nbk) {
    const Seg cin = seg_cat(car, ex);
    W.cin[c] = cin.m;
    W.doff[c] = doff0 + offl;
    W.nd[c] = ndv;
    W.sprev[c] = (short)(prevl != 0x7fff ? prevl : (last0 != 0x7fff ? last0 : E_ZERO));
    if (c == nbk - 1) W.finm = seg_cat(Seg{0, cin.m}, sv.agg).m;
    // this slice's directs into the ordered list, each with its run monoid
    // and preceding binade resolved against the carry
    if (!over_all) {
      const short pe = (short)(prevl != 0x7fff ? prevl : (last0 != 0x7fff ? last0 : E_ZERO));
      for (int k = 0; k < ndv; ++k) {
        SliceDirect d = ldcg_struct(pd + (long long)c * kSliceDirects + k);
        if (d.inh) d.m = mono_cat(cin.m, d.m);
        if (d.e == (short)0x7ffe) d.e = pe;  // "previous slice"
        sdir[doff0 + offl + k] = d;
      }
    }
  }
  asm volatile("bar.sync %0, %1;" ::"r"(kCombineBar), "r"(R * 32) : "memory");
  if (cw != 0) return 0.0;  // warp 0 finishes
  WGS_STAMP(5)
  WGS_STAMP(6)
  double acc = 0.0;
  int bad = 0;
  if (lane == 0) {
    bool ok = !over_all;
    double head = sv.head;  // slice 0's exact value (0 when it was classified)
    if (ok) {
      // only head -> run -> add is on the dependent path; the run checks are
      // accumulated into `ok` (seq_apply_run's conditions, evaluated lazily)
      for (int idx = 0; idx < total_d; ++idx) {
        const SliceDirect d = sdir[idx];
        const bool run = (d.e >= -1100) & (d.e <= 1100);
        const long long A = mono_apply(d.m, dsig(head));
        ok &= !run | ((head > 0.0) & (dexp(head) == d.e) & (A < (1LL << 53)) & (A >= (1LL << 52)));
        head = dadd(run ? dmake(A, d.e) : head, d.x);
      }
      acc = head;
      const short pl2 = (short)last_all;
      if (ok && pl2 >= -1100 && pl2 <= 1100) ok = seq_apply_run(head, pl2, W.finm, &acc);
    }
    if (!ok) {  // sequential fallback: always the reference order
      acc = 0.0;
      for (long long i = 0; i < nt; ++i) acc = dadd(acc, get(i));
    }
    bad = ok ? 0 : 1;
  }
  WGS_STAMP(7)
  if (tp && blockIdx.x == 0 && lane == 0) tp[9] = total_d;
#undef WGS_STAMP
  acc = __shfl_sync(FULL, acc, 0);
  bad = __shfl_sync(FULL, bad, 0);
  if (fail) *fail = bad != 0;
  (void)sslice;
  return acc;
}

}  // namespace ctdgpu
