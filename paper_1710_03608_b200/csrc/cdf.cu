// Device-wide exact sequential cumulative sum (see seqsum.cuh for the
// algorithm) and the sampling law built from it:
//   T   = sequential sum of fiber norms            (sampling.cpp:26-27)
//   p_j = fl(n_j / T)                              (sampling.cpp:29)
//   cum = sequential running sum of p, tail clamped (sampling.cpp:42-54)
// All three are bit-identical to the reference.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cdf.cuh"
#include "seqsum.cuh"

namespace ctdgpu {

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 8;
constexpr int kBS = kThreads * kPerThread;  // elements per block
constexpr int kDMax = 128;                  // directs per block before the block is walked
constexpr int kOver = kDMax + 1;            // bnd[] of a walked block
constexpr short E_WALKED = -30002;          // element summed by the walker (walked block)

__global__ void k_chunk_sum(const double* __restrict__ x, long long n, double* bsum) {
  __shared__ double sh[33];
  const long long base = (long long)blockIdx.x * kBS + (long long)threadIdx.x * kPerThread;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k)
    if (base + k < n) s += x[base + k];
  double tot = block_sum<double>(s, sh);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// Exclusive scan (approximate, any association) of nb block sums; 1 block.
__global__ void k_scan_bsum(const double* bsum, long long nb, double* bpre) {
  __shared__ double sh[33];
  double carry = 0.0;
  for (long long b0 = 0; b0 < nb; b0 += (long long)blockDim.x * 4) {
    double v[4];
    double s = 0.0;
    const long long base = b0 + (long long)threadIdx.x * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = (base + k < nb) ? bsum[base + k] : 0.0;
      s += v[k];
    }
    double tot;
    double pre = block_excl_sum<double>(s, sh, &tot) + carry;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (base + k < nb) bpre[base + k] = pre;
      pre += v[k];
    }
    carry += tot;
  }
}

struct LocalOut {
  short* e;      // per element: REG binade, E_DIRECT or E_ZERO
  Mono* m;       // per element: run mono (in-block, from head or block start)
  int* slot;     // per element: head slot (>=0), -1 inherited, -2 zero
  double* dl_x;  // per block direct list
  Mono* dl_m;
  short* dl_e;
  int* dl_inh;
  int* bnd;      // directs per block
  Seg* bagg;     // block aggregate
  short* blast;  // e/cls of the block's last element
};

__global__ void k_seq_local(const double* __restrict__ x, long long n, const double* bpre,
                            LocalOut o, unsigned* flags) {
  __shared__ double dsh[33];
  __shared__ Seg ssh[33];
  __shared__ int ish[33];
  __shared__ short last_e[kThreads];
  const long long bb = (long long)blockIdx.x * kBS;
  const long long b0 = bb + (long long)threadIdx.x * kPerThread;
  const double mg = seq_margin(n);
  double xv[kPerThread];
  double cs = 0.0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    xv[k] = (b0 + k < n) ? x[b0 + k] : 0.0;
    cs += xv[k];
  }
  double pre = block_excl_sum<double>(cs, dsh, nullptr) + bpre[blockIdx.x];
  // Pass B.
  Seg agg{0, mono_id()};
  int nd = 0;
  short le = (short)0x7fff;
  {
    double P = pre;
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
      const long long i = b0 + k;
      if (i >= n) break;
      const double Pc = P + xv[k];
      int e = 0;
      Mono m;
      const int c = seq_classify(i == 0, P, Pc, xv[k], mg, &e, &m);
      if (c == CLS_REG) {
        agg.m = mono_cat(agg.m, m);
        le = (short)e;
      } else {
        agg.h = 1;
        agg.m = mono_id();
        if (c == CLS_DIRECT) ++nd;
        le = c == CLS_DIRECT ? E_DIRECT : E_ZERO;
      }
      P = Pc;
    }
  }
  last_e[threadIdx.x] = le;
  Seg tot_seg;
  Seg carry = block_seg_excl(agg, ssh, &tot_seg);
  int ntot;
  int dpos = block_excl_sum<int>(nd, ish, &ntot);
  // A block with more directs than its slots (e.g. a CDF creeping up to a
  // binade edge in tiny steps: every element near the edge is direct) is
  // "walked": the walker adds all its elements sequentially.  To the carry
  // scan it is one head at its end (slot b*kDMax) followed by nothing.
  const bool over = ntot > kDMax;
  if (threadIdx.x == 0) {
    o.bnd[blockIdx.x] = over ? kOver : ntot;
    o.bagg[blockIdx.x] = over ? Seg{1, mono_id()} : tot_seg;
  }
  // e of the element before this thread's chunk (within the block).
  short prev_e = (short)0x7ffe;  // 0x7ffe: "previous block"
  for (int q = (int)threadIdx.x - 1; q >= 0; --q)
    if (last_e[q] != (short)0x7fff) { prev_e = last_e[q]; break; }
  // Pass C.
  if (over) {
#pragma unroll
    for (int k = 0; k < kPerThread; ++k)
      if (b0 + k < n) o.e[b0 + k] = E_WALKED;
    const long long last = min(n, bb + kBS) - 1;
    if ((last - bb) / kPerThread == (long long)threadIdx.x) o.blast[blockIdx.x] = E_DIRECT;
    return;
  }
  {
    double P = pre;
    Mono M = carry.m;
    int head_slot = carry.h ? -3 : -1;  // -3: head earlier in block (slot set below)
    // The last head before this chunk within the block: its slot = dpos-1
    // if any direct precedes, unless that head was a ZERO element.
    if (carry.h) head_slot = (dpos > 0) ? (int)(blockIdx.x * kDMax + dpos - 1) : -2;
    int inh = carry.h ? 0 : 1;
#pragma unroll
    for (int k = 0; k < kPerThread; ++k) {
      const long long i = b0 + k;
      if (i >= n) break;
      const double Pc = P + xv[k];
      int e = 0;
      Mono m;
      const int c = seq_classify(i == 0, P, Pc, xv[k], mg, &e, &m);
      if (c == CLS_REG) {
        M = mono_cat(M, m);
        o.e[i] = (short)e;
        o.m[i] = M;
        o.slot[i] = head_slot;
        prev_e = (short)e;
      } else if (c == CLS_DIRECT) {
        const int slot = (int)(blockIdx.x * kDMax + dpos);
        if (!over) {
          o.dl_x[slot] = xv[k];
          o.dl_m[slot] = M;
          o.dl_e[slot] = prev_e;
          o.dl_inh[slot] = inh;
        }
        o.e[i] = E_DIRECT;
        o.slot[i] = slot;
        ++dpos;
        head_slot = slot;
        M = mono_id();
        inh = 0;
        prev_e = E_DIRECT;
      } else {
        o.e[i] = E_ZERO;
        o.slot[i] = -2;
        head_slot = -2;
        M = mono_id();
        inh = 0;
        prev_e = E_ZERO;
      }
      P = Pc;
    }
  }
  const long long last = min(n, bb + kBS) - 1;  // the block's last element
  if ((last - bb) / kPerThread == (long long)threadIdx.x) o.blast[blockIdx.x] = le;
}

struct WalkOut {
  double* head_val;  // per slot
  Mono* carry_in;    // per block
  int* inh_head;     // per block: slot of the last head before the block (-2 zero)
  double* total;
  Mono* final_m;     // run mono from the last head to the end
};

__device__ __forceinline__ bool is_reg_e(short e) { return e >= -1100 && e <= 1100; }

// Cross-block carries in parallel (one CTA): segmented exclusive scan of the
// block aggregates -> carry_in[b]; exclusive max-scan of each block's last
// direct slot -> inh_head[b]; ordered list of the blocks holding directs.
constexpr int kCarryThreads = 1024;
__global__ void __launch_bounds__(kCarryThreads) k_seq_carry(long long nb, LocalOut o, WalkOut w,
                                                             int* dblocks, int* n_dblocks) {
  __shared__ Seg ssh[33];
  __shared__ int ish[33];
  __shared__ int msh[kCarryThreads];
  const long long per = (nb + blockDim.x - 1) / blockDim.x;
  const long long b0 = min((long long)threadIdx.x * per, nb), b1 = min(b0 + per, nb);
  Seg agg{0, mono_id()};
  int last_slot = -2, nd = 0;
  for (long long b = b0; b < b1; ++b) {
    agg = seg_cat(agg, o.bagg[b]);
    if (o.bnd[b] > 0) {
      last_slot = (int)(b * kDMax + (o.bnd[b] == kOver ? 0 : o.bnd[b] - 1));
      ++nd;
    }
  }
  Seg carry = block_seg_excl(agg, ssh, nullptr);
  msh[threadIdx.x] = last_slot;
  __syncthreads();
  // exclusive max over earlier threads (slots increase with block index)
  int inh = -2;
  for (int q = (int)threadIdx.x - 1; q >= 0; --q)
    if (msh[q] != -2) { inh = msh[q]; break; }
  int pos = block_excl_sum<int>(nd, ish, n_dblocks);
  for (long long b = b0; b < b1; ++b) {
    w.carry_in[b] = carry.m;
    w.inh_head[b] = inh;
    carry = seg_cat(carry, o.bagg[b]);
    if (o.bnd[b] > 0) {
      inh = (int)(b * kDMax + (o.bnd[b] == kOver ? 0 : o.bnd[b] - 1));
      dblocks[pos++] = (int)b;
    }
  }
  if (threadIdx.x == blockDim.x - 1 || b1 == nb) {
    if (b1 == nb && b0 < b1) w.final_m[0] = carry.m;
  }
}

// Sequential walker over the (few) blocks that hold direct elements.
__global__ void k_seq_walk(const double* __restrict__ x, long long n, long long nb, LocalOut o,
                           WalkOut w, const int* dblocks, const int* n_dblocks, double* cum,
                           unsigned* flags, double* diag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*flags & FLAG_SEQSUM) return;
  double head = 0.0;
  bool ok = true;
  const int nbd = *n_dblocks;
  for (int q0 = 0; q0 < nbd && ok; ++q0) {
    const long long b = dblocks[q0];
    const Mono cin = w.carry_in[b];
    const short prev_last = b > 0 ? o.blast[b - 1] : E_ZERO;
    const int nd = o.bnd[b];
    if (nd == kOver) {  // walked block: the pending run, then every element in order
      double acc = head;
      if (is_reg_e(prev_last)) ok = seq_apply_run(head, prev_last, cin, &acc);
      if (!ok && diag) {
        diag[0] = (double)b; diag[1] = -1.0; diag[2] = (double)prev_last; diag[3] = head;
      }
      const long long i0 = b * kBS, i1 = min(n, i0 + kBS);
#pragma unroll 8
      for (long long i = i0; i < i1; ++i) {
        acc = dadd(acc, x[i]);
        if (cum) cum[i] = acc;
      }
      head = acc;
      w.head_val[b * kDMax] = acc;
      continue;
    }
    for (int q = 0; q < nd && ok; ++q) {
      const int slot = (int)(b * kDMax + q);
      const Mono M = o.dl_inh[slot] ? mono_cat(cin, o.dl_m[slot]) : o.dl_m[slot];
      const short eb = (o.dl_e[slot] == (short)0x7ffe) ? prev_last : o.dl_e[slot];
      double acc = head;
      if (is_reg_e(eb)) ok = seq_apply_run(head, eb, M, &acc);
      if (!ok && diag) {
        diag[0] = (double)b; diag[1] = (double)q; diag[2] = (double)eb; diag[3] = head;
        diag[4] = (double)M.a0; diag[5] = (double)M.a1; diag[6] = o.dl_x[slot]; diag[7] = (double)nd;
      }
      acc = dadd(acc, o.dl_x[slot]);
      head = acc;
      w.head_val[slot] = acc;
    }
  }
  double total = head;
  const short last_e = o.blast[nb - 1];
  if (ok && is_reg_e(last_e)) {
    ok = seq_apply_run(head, last_e, w.final_m[0], &total);
    if (!ok && diag) {
      diag[0] = -1.0; diag[2] = (double)last_e; diag[3] = head;
      diag[4] = (double)w.final_m[0].a0; diag[5] = (double)w.final_m[0].a1;
    }
  }
  if (!ok) atomicOr(flags, FLAG_SEQSUM);
  else *w.total = total;
}

__global__ void k_seq_final(long long n, LocalOut o, WalkOut w, double* cum,
                            const unsigned* flags) {
  if (*flags & FLAG_SEQSUM) return;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const short e = o.e[i];
  if (e == E_WALKED) return;  // written by the walker
  double c;
  if (e == E_ZERO) {
    c = 0.0;
  } else if (e == E_DIRECT) {
    c = w.head_val[o.slot[i]];
  } else {
    const long long b = i / kBS;
    const int s = o.slot[i];
    const int hs = s >= 0 ? s : w.inh_head[b];
    const Mono M = s >= 0 ? o.m[i] : mono_cat(w.carry_in[b], o.m[i]);
    c = dmake(mono_apply(M, dsig(w.head_val[hs])), e);
  }
  cum[i] = c;
}

// Plain sequential loop: taken only when a self-check failed.
__global__ void k_seq_fallback(const double* x, long long n, double* cum, double* total,
                               const unsigned* flags) {
  if (!(*flags & FLAG_SEQSUM)) return;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) {
    acc = dadd(acc, x[i]);
    if (cum) cum[i] = acc;
  }
  *total = acc;
}

}  // namespace

void seq_cumsum(Ctx* ctx, const double* x, int64_t n, double* cum, double* d_total) {
  if (n <= 0) {
    ctx->zero(d_total, sizeof(double));
    return;
  }
  const long long nb = (n + kBS - 1) / kBS;
  Buf<double> bsum(ctx, nb), bpre(ctx, nb);
  Buf<short> ge(ctx, n);
  Buf<Mono> gm(ctx, n);
  Buf<int> gslot(ctx, n);
  Buf<double> dlx(ctx, nb * kDMax);
  Buf<Mono> dlm(ctx, nb * kDMax);
  Buf<short> dle(ctx, nb * kDMax);
  Buf<int> dli(ctx, nb * kDMax);
  Buf<int> bnd(ctx, nb);
  Buf<Seg> bagg(ctx, nb);
  Buf<short> blast(ctx, nb);
  Buf<double> headv(ctx, nb * kDMax);
  Buf<Mono> cin(ctx, nb);
  Buf<int> inh(ctx, nb);
  Buf<unsigned> fl(ctx, 1);
  fl.zero();
  LocalOut o{ge.p, gm.p, gslot.p, dlx.p, dlm.p, dle.p, dli.p, bnd.p, bagg.p, blast.p};
  Buf<Mono> finm(ctx, 1);
  Buf<int> dblocks(ctx, nb), ndb(ctx, 1);
  WalkOut w{headv.p, cin.p, inh.p, d_total, finm.p};
  LAUNCH(ctx, k_chunk_sum, (unsigned)nb, kThreads, 0, x, (long long)n, bsum.p);
  LAUNCH(ctx, k_scan_bsum, 1, 1024, 0, bsum.p, nb, bpre.p);
  LAUNCH(ctx, k_seq_local, (unsigned)nb, kThreads, 0, x, (long long)n, bpre.p, o, fl.p);
  LAUNCH(ctx, k_seq_carry, 1, kCarryThreads, 0, nb, o, w, dblocks.p, ndb.p);
  static const bool trace = getenv("CTD_SEQ_TRACE") != nullptr;
  Buf<double> diag(ctx, 8);
  if (trace) diag.zero();
  LAUNCH(ctx, k_seq_walk, 1, 32, 0, x, (long long)n, nb, o, w, dblocks.p, ndb.p, cum, fl.p,
         trace ? diag.p : nullptr);
  if (cum) LAUNCH(ctx, k_seq_final, ceil_div(n, 256), 256, 0, (long long)n, o, w, cum, fl.p);
  LAUNCH(ctx, k_seq_fallback, 1, 32, 0, x, (long long)n, cum, d_total, fl.p);
  if (trace) {  // diagnostics: which self-check sent the sum to the fallback
    std::vector<int> hb(nb);
    ctx->to_host(hb.data(), bnd.p, nb);
    const unsigned f = ctx->read1(fl.p);
    const int nd = ctx->read1(ndb.p);
    long long tot = 0;
    int shown = 0;
    for (long long b = 0; b < nb; ++b) {
      if (hb[b] == kOver && shown < 6) {
        ++shown;
        double xs[8], pb;
        ctx->to_host(xs, x + b * kBS, std::min<long long>(8, n - b * kBS));
        ctx->to_host(&pb, bpre.p + b, 1);
        ctx->sync();
        fprintf(stderr, "[seq_cumsum] walked block %lld: prefix %.17g, x[0..3] %.17g %.17g %.17g %.17g\n",
                b, pb, xs[0], xs[1], xs[2], xs[3]);
      }
      tot += hb[b] == kOver ? 0 : hb[b];
    }
    double dg[8];
    ctx->to_host(dg, diag.p, 8);
    ctx->sync();
    fprintf(stderr, "[seq_cumsum] n=%lld blocks=%lld direct_blocks=%d directs=%lld fallback=%d\n",
            (long long)n, nb, nd, tot, (int)((f & FLAG_SEQSUM) != 0));
    if (f & FLAG_SEQSUM)
      fprintf(stderr, "[seq_cumsum] walk failed: block=%.0f q=%.0f e=%.0f head=%.17g a0=%.0f a1=%.0f x=%.17g nd=%.0f\n",
              dg[0], dg[1], dg[2], dg[3], dg[4], dg[5], dg[6], dg[7]);
  }
}

// ---------------------------------------------------------------------------
// Sampling law.
namespace {

// (grid-stride; the last positive position is reduced per thread and per warp,
// one atomicMax per warp at the end -- one per element serialises 8e7 atomics
// on a single address at C5)
__global__ void k_probs(const double* __restrict__ norms, long long F, const double* total,
                        double* probs, int* last_pos) {
  const double tot = *total;
  int lp = -1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < F;
       i += (long long)gridDim.x * blockDim.x) {
    const double p = ddiv(norms[i], tot);  // sampling.cpp:29
    probs[i] = p;
    if (p > 0.0) lp = (int)i;  // i ascends per thread
  }
  lp = __reduce_max_sync(0xffffffffu, lp);
  if ((threadIdx.x & 31) == 0 && lp >= 0) atomicMax(last_pos, lp);
}

__global__ void k_lastpos(const double* probs, long long n, int* last_pos) {
  int lp = -1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (probs[i] > 0.0) lp = (int)i;
  lp = __reduce_max_sync(0xffffffffu, lp);
  if ((threadIdx.x & 31) == 0 && lp >= 0) atomicMax(last_pos, lp);
}

__global__ void k_clamp(double* cum, long long F, const int* last_pos, unsigned* flags) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lp = *last_pos;
  if (lp < 0) {
    if (i == 0) atomicOr(flags, FLAG_EMPTY);  // all-zero law: EmptyInputError
    return;
  }
  if (i < F && i >= lp) cum[i] = 1.0;  // sampling.cpp:54
}

}  // namespace

void sampling_law(Ctx* ctx, const double* norms, int64_t F, double* d_total, double* probs,
                  double* cum, unsigned* d_law_flags) {
  Buf<double> scratch(ctx, F > 0 ? F : 1);
  seq_cumsum(ctx, norms, F, scratch.p, d_total);  // T: sequential over columns
  Buf<int> lp(ctx, 1);
  CUDA_OK(cudaMemsetAsync(lp.p, 0xff, sizeof(int), ctx->stream));
  if (F > 0) LAUNCH(ctx, k_probs, std::min<unsigned>(ceil_div(F, 256), (unsigned)ctx->sm_count * 16), 256, 0, norms, (long long)F, d_total, probs, lp.p);
  Buf<double> t2(ctx, 1);
  seq_cumsum(ctx, probs, F, cum, t2.p);
  LAUNCH(ctx, k_clamp, ceil_div(F > 0 ? F : 1, 256), 256, 0, cum, (long long)F, lp.p, d_law_flags);
}

void probs_from_norms(Ctx* ctx, const double* norms, int64_t F, const double* d_total, double* probs,
                      int* d_last_pos) {
  CUDA_OK(cudaMemsetAsync(d_last_pos, 0xff, sizeof(int), ctx->stream));
  if (F > 0) LAUNCH(ctx, k_probs, std::min<unsigned>(ceil_div(F, 256), (unsigned)ctx->sm_count * 16), 256, 0, norms, (long long)F, d_total, probs, d_last_pos);
}

void clamp_from(Ctx* ctx, double* cum, int64_t n, const int* d_last_pos) {
  Buf<unsigned> fl(ctx, 1);
  fl.zero();
  if (n > 0) LAUNCH(ctx, k_clamp, ceil_div(n, 256), 256, 0, cum, (long long)n, d_last_pos, fl.p);
}

void clamped_cdf(Ctx* ctx, const double* probs, int64_t n, double* cum, unsigned* d_flags) {
  Buf<int> lp(ctx, 1);
  CUDA_OK(cudaMemsetAsync(lp.p, 0xff, sizeof(int), ctx->stream));
  Buf<double> t(ctx, 1);
  seq_cumsum(ctx, probs, n, cum, t.p);
  if (n > 0) LAUNCH(ctx, k_lastpos, std::min<unsigned>(ceil_div(n, 256), (unsigned)ctx->sm_count * 16), 256, 0, probs, (long long)n, lp.p);
  LAUNCH(ctx, k_clamp, ceil_div(n > 0 ? n : 1, 256), 256, 0, cum, (long long)n, lp.p, d_flags);
}

}  // namespace ctdgpu
