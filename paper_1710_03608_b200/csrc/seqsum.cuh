// Exact reproduction of a *sequential* IEEE-double running sum of
// non-negative terms,  c_i = fl(c_{i-1} + x_i),  c_{-1} = 0,  in parallel.
//
// The reference accumulates several such sums in strict order: the sampling
// CDF (sampling.cpp:42-49), the normalizer (:26-27), fiber norms
// (tensor_ops.cpp:196-199), |x|^2 (sparse_matrix.cpp:10-14) and the residual
// (fiber_basis.cpp:66-77).  All terms are >= 0, so the running sum is
// monotone.  While c_{i-1} and c_i stay in one binade [2^e, 2^(e+1)), every
// representable value is a multiple of ulp_e = 2^(e-52) and
//     c_i / ulp_e = c_{i-1} / ulp_e + rne(x_i / ulp_e),
// an integer increment independent of c_{i-1} except on an exact half-ulp
// tie, where round-half-even depends on the parity of c_{i-1}/ulp_e.  Such a
// step is the map A -> A + a[A & 1]; these maps compose associatively
// (struct Mono), so a run of same-binade steps is one parallel scan.
//
// Which binade c_i lies in is decided from an approximate prefix P~ (any
// summation order; |P~ - c| <= 2 n u c for non-negative terms).  An element
// is "regular" when P~_{i-1} and P~_i are in the same binade and both lie
// farther than a 4nu relative margin from its edges; every other element is
// "direct" and is added with a real fl() add by a sequential walker (binade
// crossings, near-boundary values, subnormals: a few dozen per run).  The
// walker also verifies every run (start binade, no overflow of the binade);
// a failed check sets FLAG_SEQSUM and the caller falls back to a plain
// sequential loop, so the result is always the sequential one.
#pragma once

#include "common.cuh"

namespace ctdgpu {

struct Mono {
  long long a0, a1;  // A -> A + (A odd ? a1 : a0)
};
__device__ __forceinline__ Mono mono_id() { return Mono{0, 0}; }
__device__ __forceinline__ Mono mono_cat(const Mono& f, const Mono& g) {
  Mono h;
  h.a0 = f.a0 + ((f.a0 & 1) ? g.a1 : g.a0);
  h.a1 = f.a1 + (((f.a1 + 1) & 1) ? g.a1 : g.a0);
  return h;
}
__device__ __forceinline__ long long mono_apply(const Mono& f, long long A) {
  return A + ((A & 1) ? f.a1 : f.a0);
}

enum : int { CLS_ZERO = 0, CLS_DIRECT = 1, CLS_REG = 2 };
constexpr short E_DIRECT = -30000;
constexpr short E_ZERO = -30001;

__device__ __forceinline__ double seq_margin(long long n) {
  return 4.0 * (double)n * 1.1102230246251565e-16 + 2.8421709430404007e-14;
}

__device__ __forceinline__ bool near_binade_edge(double P, double mg) {
  const int e = dexp(P);
  if (e < -1021 || e > 1022) return true;
  const double lo = pow2(e);
  return (P - lo) <= mg * P || (2.0 * lo - P) <= mg * P;
}

// The grid increment of a regular element in binade ec: round(x / 2^(ec-52))
// with the tie flagged.  Pure integer work on the bit pattern (FRND/F2I are
// slow-pipe instructions on sm_100): x = mx * 2^(ex-52), so the scaled value
// is mx * 2^-d with d = ec - ex; floor = mx >> d and the fraction compares as
// the remainder against the half bit 2^(d-1).
__device__ __forceinline__ void seq_mono(double x, int ec, Mono* m_out) {
  const long long bits = __double_as_longlong(x);
  const int bexp = (int)((bits >> 52) & 0x7FF);
  long long mx = bits & 0xFFFFFFFFFFFFFLL;
  int ex = -1022;
  if (bexp != 0) {
    mx |= (1LL << 52);
    ex = bexp - 1023;
  }
  const int d = ec - ex;
  long long k0 = 0, rem = 0, half = 1;  // defaults: d > 55 -> 0, no tie
  if (d <= 0) {
    k0 = mx << (-d);
    rem = 0;
  } else if (d <= 55) {
    k0 = mx >> d;
    rem = mx & ((1LL << d) - 1);
    half = 1LL << (d - 1);
  } else {
    rem = 0;  // x / ulp < 2^-2: rounds to 0
    half = 1;
  }
  if (rem > half) {
    m_out->a0 = m_out->a1 = k0 + 1;
  } else if (rem < half) {
    m_out->a0 = m_out->a1 = k0;
  } else {  // exact tie: the result rounds to even
    m_out->a0 = k0 + (k0 & 1);
    m_out->a1 = k0 + ((k0 + 1) & 1);
  }
}

// Classify element i given approximate prefixes before (Pp) and after (Pc).
__device__ __forceinline__ int seq_classify(bool first, double Pp, double Pc, double x,
                                            double mg, int* e_out, Mono* m_out) {
  if (Pc == 0.0) return CLS_ZERO;
  if (first || !(Pp > 0.0) || !(Pc > 0.0) || !(x < 1.7976931348623157e308)) return CLS_DIRECT;
  const int ep = dexp(Pp), ec = dexp(Pc);
  if (ep != ec || ec < -960 || ec > 1020) return CLS_DIRECT;
  if (near_binade_edge(Pp, mg) || near_binade_edge(Pc, mg)) return CLS_DIRECT;
  seq_mono(x, ec, m_out);
  *e_out = ec;
  return CLS_REG;
}

// Branch-free seq_mono / seq_classify (same results): straight-line selects so
// the classifications of several terms interleave (block_exact_sum_ilp).
__device__ __forceinline__ Mono seq_mono_bf(double x, int ec) {
  const long long bits = __double_as_longlong(x);
  const int bexp = (int)((bits >> 52) & 0x7FF);
  const long long mx = (bits & 0xFFFFFFFFFFFFFLL) | (bexp != 0 ? (1LL << 52) : 0LL);
  const int ex = bexp != 0 ? bexp - 1023 : -1022;
  const int d = ec - ex;
  const int dl = min(max(-d, 0), 62);     // left shift when d <= 0
  const int dr = min(max(d, 1), 55);      // right shift when 0 < d <= 55
  const bool mid = (d > 0) & (d <= 55);
  const long long k0 = (d <= 0) ? (mx << dl) : (mid ? (mx >> dr) : 0LL);
  const long long rem = mid ? (mx & ((1LL << dr) - 1)) : 0LL;
  const long long half = mid ? (1LL << (dr - 1)) : 1LL;
  const bool tie = rem == half;
  const long long up = rem > half ? 1LL : 0LL;
  Mono m;
  m.a0 = tie ? k0 + (k0 & 1) : k0 + up;
  m.a1 = tie ? k0 + ((k0 + 1) & 1) : k0 + up;
  return m;
}

__device__ __forceinline__ int seq_classify_bf(bool first, double Pp, double Pc, double x, double mg, int* e_out,
                                               Mono* m_out) {
  const int ep = dexp(Pp), ec = dexp(Pc);
  bool direct = first | !(Pp > 0.0) | !(Pc > 0.0) | !(x < 1.7976931348623157e308) | (ep != ec) | (ec < -960) |
                (ec > 1020);
  const double lo = pow2(min(max(ec, -1020), 1020));
  direct |= ((Pp - lo) <= mg * Pp) | ((2.0 * lo - Pp) <= mg * Pp) | ((Pc - lo) <= mg * Pc) |
            ((2.0 * lo - Pc) <= mg * Pc);
  *m_out = seq_mono_bf(x, min(max(ec, -1022), 1023));
  *e_out = ec;
  return (Pc == 0.0) ? CLS_ZERO : (direct ? CLS_DIRECT : CLS_REG);
}

// seq_classify_bf with the grid increment taken in floating point: t =
// x 2^(52-e) is exact, (t + 2^52) - 2^52 rounds it to the nearest integer
// (ties to even) for t < 2^51, and without an exact half-ulp tie the
// increment does not depend on the parity of the running value.  Ties (or
// large t) take the integer monoid (seq_mono_bf).  Same results, fewer
// 64-bit integer instructions.
__device__ __forceinline__ int seq_classify_fp(bool first, double Pp, double Pc, double x, double mg, int* e_out,
                                               Mono* m_out) {
  const int ep = dexp(Pp), ec = dexp(Pc);
  bool direct = first | !(Pp > 0.0) | !(Pc > 0.0) | !(x < 1.7976931348623157e308) | (ep != ec) | (ec < -960) |
                (ec > 1020);
  const int ecc = min(max(ec, -960), 1020);
  const double lo = pow2(ecc);
  direct |= ((Pp - lo) <= mg * Pp) | ((2.0 * lo - Pp) <= mg * Pp) | ((Pc - lo) <= mg * Pc) |
            ((2.0 * lo - Pc) <= mg * Pc);
  const double t = __dmul_rn(x, pow2(52 - ecc));
  const double r = __dadd_rn(__dadd_rn(t, 4503599627370496.0), -4503599627370496.0);
  const double f = __dadd_rn(t, -r);
  const bool hard = !(t < 2251799813685248.0) | (f == 0.5) | (f == -0.5);
  if (hard && !direct) {
    *m_out = seq_mono_bf(x, ecc);
  } else {
    const long long ri = (long long)r;
    *m_out = Mono{ri, ri};
  }
  *e_out = ec;
  return (Pc == 0.0) ? CLS_ZERO : (direct ? CLS_DIRECT : CLS_REG);
}

// A whole chunk is regular in binade *e when the approximate prefix before it
// (pre) and after it (post) both lie strictly inside [2^e, 2^(e+1)) with the
// error margin to spare: the running sum is monotone, so every intermediate
// value (true or approximate) is inside too.
__device__ __forceinline__ bool seq_chunk_regular(double pre, double post, double mg, int* e) {
  if (!(pre > 0.0) || !(post > 0.0) || !(post < 1.7976931348623157e308)) return false;
  const int ep = dexp(pre);
  if (ep != dexp(post) || ep < -960 || ep > 1020) return false;
  const double lo = pow2(ep);
  if (!(pre - lo > 2.0 * mg * pre) || !(2.0 * lo - post > 4.0 * mg * post)) return false;
  *e = ep;
  return true;
}

// Applies a same-binade run summarized by M to the value `head` (the value of
// the run's leading direct element).  Returns false if the run's assumptions
// do not hold (caller falls back).
__device__ __forceinline__ bool seq_apply_run(double head, int e, const Mono& M, double* out) {
  if (!(head > 0.0) || dexp(head) != e) return false;
  const long long A = mono_apply(M, dsig(head));
  if (A >= (1LL << 53) || A < (1LL << 52)) return false;
  *out = dmake(A, e);
  return true;
}

// Segmented-scan element: (has_head, mono since the last head).
struct Seg {
  int h;
  Mono m;
};
__device__ __forceinline__ Seg seg_cat(const Seg& l, const Seg& r) {
  Seg o;
  o.h = l.h | r.h;
  o.m = r.h ? r.m : mono_cat(l.m, r.m);
  return o;
}
__device__ __forceinline__ Seg seg_shfl_up(const Seg& s, int d) {
  Seg o;
  o.h = __shfl_up_sync(0xffffffffu, s.h, d);
  o.m.a0 = __shfl_up_sync(0xffffffffu, s.m.a0, d);
  o.m.a1 = __shfl_up_sync(0xffffffffu, s.m.a1, d);
  return o;
}

// Exclusive segmented block scan of one Seg per thread.  sh: >= 32 Segs.
__device__ inline Seg block_seg_excl(Seg v, Seg* sh, Seg* total) {
  const unsigned w = warp_id(), l = lane_id(), nw = (blockDim.x + 31) >> 5;
  Seg inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Seg o = seg_shfl_up(inc, d);
    if ((int)l >= d) inc = seg_cat(o, inc);
  }
  if (l == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    Seg s = (l < nw) ? sh[l] : Seg{0, mono_id()};
    Seg si = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      Seg o = seg_shfl_up(si, d);
      if ((int)l >= d) si = seg_cat(o, si);
    }
    // exclusive = inclusive of previous lane
    Seg ex = seg_shfl_up(si, 1);
    if (l == 0) ex = Seg{0, mono_id()};
    if (l < nw) sh[l] = ex;
    if (l == nw - 1) sh[32] = si;
  }
  __syncthreads();
  // exclusive prefix for this thread: warp prefix (sh[w]) then lanes before me
  Seg lanes_ex = seg_shfl_up(inc, 1);
  Seg res;
  if (l == 0) res = sh[w];
  else res = seg_cat(sh[w], lanes_ex);
  if (total) *total = sh[32];
  __syncthreads();
  return res;
}

// --------------------------------------------------------------------------
// Block-level exact sequential total of n >= 0 terms produced by get(i).
// Deterministic; all threads return the same value.  `fail` set on self-check
// failure in which case the sequential fallback result is returned.
struct SeqSumSmem {
  double dsh[33];
  Seg ssh[33];
  int ish[33];
  int nd;
  int bad;
  double result;
  // direct list
  static constexpr int kCap = 512;
  double dx[kCap];
  Mono dm[kCap];
  short de[kCap];
  int di[kCap];
  // per-thread boundary info
  short last_e[1024];
  Mono fin_m;
  short fin_e;
};

template <typename Get>
__device__ double block_exact_sum(const Get& get, long long n, SeqSumSmem& S, bool* fail,
                                  long long* tp = nullptr) {
#define SEQ_STAMP(k) \
  if (tp && threadIdx.x == 0) tp[k] = clock64();
  SEQ_STAMP(0)
  const int T = blockDim.x, t = threadIdx.x;
  if (n <= 0) return 0.0;
  const long long per = (n + T - 1) / T;
  const long long b0 = min((long long)t * per, n), b1 = min(b0 + per, n);
  // Pass A: approximate chunk sums -> exclusive prefix.
  double cs = 0.0;
  for (long long i = b0; i < b1; ++i) cs += get(i);
  double tot;
  double pre = block_excl_sum<double>(cs, S.dsh, &tot);
  SEQ_STAMP(1)
  const double mg = seq_margin(n);
  // Pass B: thread aggregate + direct count.
  Seg agg{0, mono_id()};
  int nd = 0;
  short le = E_ZERO;
  int fe = 0;
  const bool fast = (b0 > 0) && (b0 < b1) && seq_chunk_regular(pre, pre + cs, mg, &fe);
  if (fast) {
    for (long long i = b0; i < b1; ++i) {
      Mono m;
      seq_mono(get(i), fe, &m);
      agg.m = mono_cat(agg.m, m);
    }
    le = (short)fe;
  } else {
    double P = pre;
    for (long long i = b0; i < b1; ++i) {
      const double x = get(i);
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
  if (t == 0) S.bad = 0;
  S.last_e[t] = (b0 < b1) ? le : (short)0x7fff;  // 0x7fff: empty chunk
  SEQ_STAMP(2)
  Seg carry = block_seg_excl(agg, S.ssh, nullptr);
  SEQ_STAMP(3)
  int ntot;
  int dpos = block_excl_sum<int>(nd, S.ish, &ntot);
  if (ntot > SeqSumSmem::kCap) {
    if (t == 0) S.bad = 1;
  } else if (fast) {
    // no heads in this chunk: only the final run summary may be needed
    if (b1 == n) {
      S.fin_m = mono_cat(carry.m, agg.m);
      S.fin_e = (short)fe;
    }
  } else {
    // Pass C: record each direct's preceding run summary.
    double P = pre;
    Mono M = carry.m;
    // e of the element before my chunk: chunks fill in thread order, so it is
    // the previous thread's last element.
    short prev_e = (t > 0) ? S.last_e[t - 1] : E_ZERO;
    for (long long i = b0; i < b1; ++i) {
      const double x = get(i);
      const double Pc = P + x;
      int e = 0;
      Mono m;
      const int c = seq_classify(i == 0, P, Pc, x, mg, &e, &m);
      if (c == CLS_REG) {
        M = mono_cat(M, m);
        prev_e = (short)e;
      } else {
        if (c == CLS_DIRECT) {
          S.dx[dpos] = x;
          S.dm[dpos] = M;
          S.de[dpos] = prev_e;  // e of the element before (REG) or a sentinel
          S.di[dpos] = (int)i;
          ++dpos;
        }
        M = mono_id();
        prev_e = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
      }
      P = Pc;
    }
    if (b1 == n && b0 < b1) {
      S.fin_m = M;
      S.fin_e = prev_e;
    }
  }
  SEQ_STAMP(4)
  __syncthreads();
  SEQ_STAMP(5)
  if (t == 0) {
    bool ok = !S.bad;
    double acc = 0.0, head = 0.0;
    if (ok) {
      for (int q = 0; q < ntot && ok; ++q) {
        if (S.de[q] >= -1100 && S.de[q] <= 1100) ok = seq_apply_run(head, S.de[q], S.dm[q], &acc);
        acc = dadd(acc, S.dx[q]);
        head = acc;
      }
      if (ok && S.fin_e >= -1100 && S.fin_e <= 1100) ok = seq_apply_run(head, S.fin_e, S.fin_m, &acc);
    }
    if (!ok) {  // sequential fallback: always the reference order
      acc = 0.0;
      for (long long i = 0; i < n; ++i) acc = dadd(acc, get(i));
    }
    S.result = acc;
    S.bad = ok ? 0 : 1;
  }
  __syncthreads();
  SEQ_STAMP(6)
#undef SEQ_STAMP
  const double r = S.result;
  if (fail) *fail = S.bad != 0;
  __syncthreads();
  return r;
}

// --------------------------------------------------------------------------
// block_exact_sum with the per-thread work restructured for instruction-level
// parallelism: each thread's chunk (cached in registers, kCache terms) is
// classified kGroup terms at a time with their approximate prefixes computed
// first.  Evaluated for the filter's residual (every CTA summing all terms
// redundantly, no cross-CTA exchange) and measured slower than the
// distributed warp_grid_sum (gridsum.cuh): the slowest chunk still costs ~1k
// cycles per term (tools/ubench_p3.cu keeps the comparison).  `get` provides
// operator()(i), batch(b0, b1, out[N]) and strided(i0, step, n, out[N]).
template <int kCache, int kGroup, typename Get, typename Overlap>
__device__ double block_exact_sum_ilp(const Get& get, long long n, SeqSumSmem& S, bool* fail,
                                      const Overlap& overlap, double* tbuf = nullptr, long long* tp = nullptr) {
#define BES_STAMP(k) \
  if (tp && threadIdx.x == 0) tp[k] = clock64();
  BES_STAMP(0)
  const int T = blockDim.x, t = threadIdx.x;
  if (n <= 0) {
    if (t >= 32) overlap();
    __syncthreads();
    if (fail) *fail = false;
    return 0.0;
  }
  const long long per = (n + T - 1) / T;
  const long long b0 = min((long long)t * per, n), b1 = min(b0 + per, n);
  double xv[kCache];
  if (tbuf && per <= kCache) {
    // coalesced: lane l loads the warp's elements l, l+32, ... then the warp
    // transposes them through shared memory into contiguous per-thread chunks
    // (row stride kCache+1: conflict-free)
    const int w = t >> 5, l = t & 31;
    double* wb = tbuf + w * 32 * (kCache + 1);
    const long long wb0 = min((long long)w * 32 * per, n);
    double lv[kCache];
    get.strided(wb0 + l, 32, n, lv);
    const unsigned p = (unsigned)per, inv = 65536u / p + 1u;  // e / p for e < 32 kCache
#pragma unroll
    for (int k = 0; k < kCache; ++k) {
      if (k < (int)p) {
        const unsigned e = (unsigned)(k * 32 + l), row = (e * inv) >> 16, col = e - row * p;
        wb[row * (kCache + 1) + col] = lv[k];
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kCache; ++k) xv[k] = (b0 + k < b1) ? wb[l * (kCache + 1) + k] : 0.0;
  } else {
    get.batch(b0, b1, xv);
  }
  double cs = 0.0;
#pragma unroll
  for (int k = 0; k < kCache; ++k) cs += xv[k];
  for (long long i = b0 + kCache; i < b1; ++i) cs += get(i);
  BES_STAMP(1)
  const double pre = block_excl_sum<double>(cs, S.dsh, nullptr);
  BES_STAMP(2)
  const double mg = seq_margin(n);
  const int nc = (int)min((long long)kCache, b1 - b0);
  // classify cached terms group by group; `step` folds one classified term
  Seg agg{0, mono_id()};
  int nd = 0;
  short le = E_ZERO;
  auto fold = [&](int c, int e, const Mono& m) {
    if (c == CLS_REG) {
      agg.m = mono_cat(agg.m, m);
      le = (short)e;
    } else {
      agg.h = 1;
      agg.m = mono_id();
      if (c == CLS_DIRECT) ++nd;
      le = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
    }
  };
  int fe = 0;
  const bool fast = (b0 > 0) && (b0 < b1) && seq_chunk_regular(pre, pre + cs, mg, &fe);
  double P = pre;
  if (fast) {
#pragma unroll
    for (int k = 0; k < kCache; ++k)
      if (k < nc) {
        Mono m;
        seq_mono(xv[k], fe, &m);
        agg.m = mono_cat(agg.m, m);
      }
    for (long long i = b0 + kCache; i < b1; ++i) {
      Mono m;
      seq_mono(get(i), fe, &m);
      agg.m = mono_cat(agg.m, m);
    }
    le = (short)fe;
  } else {
#pragma unroll
    for (int k0 = 0; k0 < kCache; k0 += kGroup) {
      if (k0 < nc) {
        double Pv[kGroup + 1];
        Pv[0] = P;
#pragma unroll
        for (int k = 0; k < kGroup; ++k) Pv[k + 1] = Pv[k] + ((k0 + k < nc) ? xv[k0 + k] : 0.0);
        int cl[kGroup], ee[kGroup];
        Mono mm[kGroup];
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
          ee[k] = 0;
          mm[k] = mono_id();
          cl[k] = (k0 + k < nc) ? seq_classify_bf(b0 + k0 + k == 0, Pv[k], Pv[k + 1], xv[k0 + k], mg, &ee[k], &mm[k])
                                : -1;
        }
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (cl[k] >= 0) fold(cl[k], ee[k], mm[k]);
        P = Pv[kGroup];
      }
    }
    for (long long i = b0 + kCache; i < b1; ++i) {
      const double x = get(i);
      const double Pc = P + x;
      int e = 0;
      Mono m;
      fold(seq_classify(i == 0, P, Pc, x, mg, &e, &m), e, m);
      P = Pc;
    }
  }
  if (t == 0) S.bad = 0;
  S.last_e[t] = (b0 < b1) ? le : (short)0x7fff;
  BES_STAMP(3)
  const Seg carry = block_seg_excl(agg, S.ssh, nullptr);
  BES_STAMP(4)
  int ntot;
  int dpos = block_excl_sum<int>(nd, S.ish, &ntot);
  BES_STAMP(5)
  if (ntot > SeqSumSmem::kCap) {
    if (t == 0) S.bad = 1;
  } else if (fast) {
    if (b1 == n) {
      S.fin_m = mono_cat(carry.m, agg.m);
      S.fin_e = (short)fe;
    }
  } else {
    // record each direct with the run monoid before it (re-classify, grouped)
    Mono M = carry.m;
    short prev_e = (t > 0) ? S.last_e[t - 1] : E_ZERO;
    auto step = [&](long long i, int c, int e, const Mono& m, double x) {
      if (c == CLS_REG) {
        M = mono_cat(M, m);
        prev_e = (short)e;
      } else {
        if (c == CLS_DIRECT) {
          S.dx[dpos] = x;
          S.dm[dpos] = M;
          S.de[dpos] = prev_e;
          S.di[dpos] = (int)i;
          ++dpos;
        }
        M = mono_id();
        prev_e = (c == CLS_DIRECT) ? E_DIRECT : E_ZERO;
      }
    };
    if (nd > 0) {
      double P2 = pre;
#pragma unroll
      for (int k0 = 0; k0 < kCache; k0 += kGroup) {
        if (k0 < nc) {
          double Pv[kGroup + 1];
          Pv[0] = P2;
#pragma unroll
          for (int k = 0; k < kGroup; ++k) Pv[k + 1] = Pv[k] + ((k0 + k < nc) ? xv[k0 + k] : 0.0);
          int cl[kGroup], ee[kGroup];
          Mono mm[kGroup];
#pragma unroll
          for (int k = 0; k < kGroup; ++k) {
            ee[k] = 0;
            mm[k] = mono_id();
            cl[k] = (k0 + k < nc)
                        ? seq_classify_bf(b0 + k0 + k == 0, Pv[k], Pv[k + 1], xv[k0 + k], mg, &ee[k], &mm[k])
                        : -1;
          }
#pragma unroll
          for (int k = 0; k < kGroup; ++k)
            if (cl[k] >= 0) step(b0 + k0 + k, cl[k], ee[k], mm[k], xv[k0 + k]);
          P2 = Pv[kGroup];
        }
      }
      for (long long i = b0 + kCache; i < b1; ++i) {
        const double x = get(i);
        const double Pc = P2 + x;
        int e = 0;
        Mono m;
        step(i, seq_classify(i == 0, P2, Pc, x, mg, &e, &m), e, m, x);
        P2 = Pc;
      }
    } else {
      // no directs here: only the run through my chunk matters
      M = agg.h ? agg.m : mono_cat(M, agg.m);
      if (b0 < b1) prev_e = le;
    }
    if (b1 == n && b0 < b1) {
      S.fin_m = M;
      S.fin_e = prev_e;
    }
  }
  BES_STAMP(6)
  __syncthreads();
  BES_STAMP(7)
  if (t == 0) {
    bool ok = !S.bad;
    double acc = 0.0, head = 0.0;
    if (ok) {
      for (int q = 0; q < ntot && ok; ++q) {
        if (S.de[q] >= -1100 && S.de[q] <= 1100) ok = seq_apply_run(head, S.de[q], S.dm[q], &acc);
        acc = dadd(acc, S.dx[q]);
        head = acc;
      }
      if (ok && S.fin_e >= -1100 && S.fin_e <= 1100) ok = seq_apply_run(head, S.fin_e, S.fin_m, &acc);
    }
    if (!ok) {  // sequential fallback: always the reference order
      acc = 0.0;
      for (long long i = 0; i < n; ++i) acc = dadd(acc, get(i));
    }
    S.result = acc;
    S.bad = ok ? 0 : 1;
    BES_STAMP(8)
  } else if (t >= 32) {
    overlap();  // independent work while thread 0 walks the directs
  }
  __syncthreads();
  BES_STAMP(9)
#undef BES_STAMP
  const double r = S.result;
  if (fail) *fail = S.bad != 0;
  __syncthreads();
  return r;
}

}  // namespace ctdgpu
