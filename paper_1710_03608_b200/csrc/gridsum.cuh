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

}  // namespace ctdgpu
