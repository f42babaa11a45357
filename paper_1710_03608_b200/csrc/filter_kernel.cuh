// The persistent filter kernel (included inside filter.cu's anonymous
// namespace).  One CTA per SM, cooperative launch, software grid barrier.
//
// Per candidate n, with K kept columns:
//   P1  (all CTAs)  [if n-1 was accepted] the U block update fused into the
//       y pass: warp w owns row i of U; it reads U_old[i][:] once (coalesced),
//       forms U_new[i][j] = fl(U_old + fl(fl(y_i y_j)/d)) (fiber_basis.cpp:
//       97-98), the new column -y_i/d and corner 1/d (:102-105), writes them
//       back, and runs the sequential chain y'_i = sum_j fl(U_new[i][j] g_j)
//       (DenseMatrix::matvec, dense_matrix.cpp:42-47) on the same registers.
//       The previous accept is appended to R's CSC, its row index and the
//       first-appearance row order (consumed by P2 after the barrier).
//   P2  (all CTAs)  z_r = sum_k fl(y_k R[r,k]) per row of R in ascending k
//       (:56-65), one warp per row, y staged in shared memory.
//   P3  (every CTA, redundantly) stage the residual terms in the reference's
//       order in shared memory, exact sequential sum (seqsum.cuh), decision.
// Two grid barriers per candidate (P1|P2, P2|P3); P3 needs none after it
// because every CTA derives the same decision.

#include <type_traits>

constexpr int kFThreads = 512;
constexpr int kVec = 4096;  // doubles per staged vector (two buffers)

constexpr int kWin = 256;  // per-warp window doubles (sizes the shared window area)

// Producer/consumer ring (P1, P2 when the staged vector fits): warps
// 0..kProdWarps-1 compute the terms of up to 32 chains (one chain per row
// this CTA owns) for kRingW consecutive steps into ring slot q&1; the chain
// warp (the last warp) runs all 32 sequential add chains at once, one per
// lane.  Slots are handed over with named barriers: "full" 1+b, "empty"
// 1+kRingSlots+b.  (Measured with tools/ubench_ring.cu: fewer/smaller slots
// couple the chain to the producers' latency.)
#ifndef CTD_RING_W
#define CTD_RING_W 96
#endif
#ifndef CTD_RING_SLOTS
#define CTD_RING_SLOTS 3
#endif
constexpr int kRingW = CTD_RING_W;         // steps per ring chunk
// Slot layout: row-major, [32 rows][kRingLS] doubles: a producer warp (32
// consecutive steps of one row) stores 256 contiguous bytes; the chain lane
// reads its row two steps per 16-byte load (kRingLS = kRingW + 2: 49 16-byte
// units per row, odd, so the 8 lanes of a load phase hit distinct banks).
constexpr int kRingLS = CTD_RING_W + 2;
constexpr int kRingSlots = CTD_RING_SLOTS;
constexpr int kRingSlot = 32 * kRingLS;  // doubles per slot
constexpr int kRingDoubles = kRingSlots * kRingSlot;
// (Keeping producers off the chain warp's SM sub-partition measured slower:
// the producers, not issue-slot sharing, bound the ring.)
constexpr int kChainWarp = kFThreads / 32 - 1;
#ifdef CTD_RING_AVOID_SMSP
// producers only on the three SM sub-partitions the chain warp does not use
// (warp w runs on sub-partition w % 4)
constexpr int kProdWarps = (kFThreads / 32) / 4 * 3;
__device__ __forceinline__ bool is_producer(int warp) { return (warp & 3) != (kChainWarp & 3); }
__device__ __forceinline__ int producer_index(int warp, int lane) { return (warp - (warp >> 2)) * 32 + lane; }
#else
constexpr int kProdWarps = kFThreads / 32 - 1;
__device__ __forceinline__ bool is_producer(int warp) { return warp < kProdWarps; }
__device__ __forceinline__ int producer_index(int warp, int lane) { return warp * 32 + lane; }
#endif
constexpr int kProdThreads = kProdWarps * 32;
constexpr int kRingThreads = kProdThreads + 32;   // named-barrier participants
// Producer thread p owns step t = p % kRingW of every chunk and the rows
// r = p / kRingW + kRowPh * k (k < kRowSlots) of the 32-row group.
constexpr int kRowPh = kProdThreads / kRingW;
constexpr int kRowSlots = (32 + kRowPh - 1) / kRowPh;
static_assert(kRowPh * kRingW == kProdThreads && kRingW % 32 == 0, "ring mapping");
constexpr int kMeta = kFThreads;           // P2 rows per ring session (one group per warp)
constexpr int kQuadRank = 160;             // sessions up to this many rows ranked by counting
// L2 prefetch distance (ring chunks) of the producers' operand streams
#ifndef CTD_PF_DIST
#define CTD_PF_DIST 2
#endif
constexpr int kPfDist = CTD_PF_DIST;
constexpr int kWinArea = (kFThreads / 32) * kWin > kRingDoubles ? (kFThreads / 32) * kWin : kRingDoubles;

constexpr size_t kFilterSmem = (size_t)(2 * kVec + kWinArea) * 8;

__device__ __forceinline__ void nbar_sync(int id, int cnt) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int cnt) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}

// acc <- (((acc + s_0) + s_1) + ... + s_95), s_t = rb[lane * kRingLS + t]:
// 32 independent chains, one per lane, over a full chunk (producers write
// every step of a chunk; steps past a row's end hold +-0.0, which leave a
// chain that starts at +0.0 unchanged: it never becomes -0.0).  Two steps per
// 16-byte load, batches of 16 steps loaded one batch ahead, ping-pong
// registers (no copies: the chain warp shares its sub-partition's issue slots
// with producer warps, so its instruction count per step is what it pays).
__device__ __forceinline__ double lane_chain(const double* rb, int lane, double acc) {
  static_assert(kRingW % 32 == 0, "lane_chain: pairs of 16-step batches");
  const double2* p = reinterpret_cast<const double2*>(rb + lane * kRingLS);
  double2 u[8], w[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) u[q] = p[q];
#pragma unroll 1
  for (int h = 0; h < kRingW / 16; h += 2) {
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = p[(h + 1) * 8 + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc = dadd(acc, u[q].x);
      acc = dadd(acc, u[q].y);
    }
    if (h + 2 < kRingW / 16) {
#pragma unroll
      for (int q = 0; q < 8; ++q) u[q] = p[(h + 2) * 8 + q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc = dadd(acc, w[q].x);
      acc = dadd(acc, w[q].y);
    }
  }
  return acc;
}

// The first cnt steps only (short last chunks: a full chunk costs ~9 cycles
// per step, this loop ~4x that per step).
__device__ __forceinline__ double lane_chain_n(const double* rb, int lane, int cnt, double acc) {
  const double* p = rb + lane * kRingLS;
#pragma unroll 4
  for (int t = 0; t < cnt; ++t) acc = dadd(acc, p[t]);
  return acc;
}
constexpr int kShortChunk = 24;

// The residual terms of try_append_fiber in the reference's summation order
// (fiber_basis.cpp:66-77): x's rows ascending ((x_i - z_i)^2, :69-70), then
// R's rows in first-touch order (z_r^2, :74-75).
struct ResidualTerms {
  const double* xv;
  const int32_t* xr;
  const double* zd;
  long long m;
  const double* tsrc;
  double* wcol = nullptr;  // optional: the W panel's column for this candidate (x rows get x - z)
  long long wld = 0;
  __device__ double operator()(long long i) const {
    if (i < m) {
      const int r = xr[i];
      const double d = dsub(xv[i], __ldcg(&zd[r]));
      if (wcol) wcol[(long long)r * wld] = d;
      return dsqr(d);
    }
    return __ldcg(&tsrc[i - m]);
  }
  // terms b0, b0+1, ... (< b1) into out[], every load of a level issued together
  template <int N>
  __device__ void batch(long long b0, long long b1, double (&out)[N]) const {
    int r[N];
    double v[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const long long i = b0 + k;
      r[k] = 0;
      v[k] = 0.0;
      if (i < b1) {
        if (i < m) {
          r[k] = xr[i];
          v[k] = xv[i];
        } else {
          v[k] = __ldcg(&tsrc[i - m]);
        }
      }
    }
    double d[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const long long i = b0 + k;
      out[k] = v[k];
      d[k] = 0.0;
      if (i < b1 && i < m) {
        d[k] = dsub(v[k], __ldcg(&zd[r[k]]));
        out[k] = dsqr(d[k]);
      }
    }
    if (wcol) {  // stores after every load of the batch (they may alias)
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (b0 + k < b1 && b0 + k < m) wcol[(long long)r[k] * wld] = d[k];
    }
  }
};

__global__ void __launch_bounds__(kFThreads, 1) k_filter(FArgs a) {
  __shared__ uint32_t hist[(kFThreads / 32) * kRadix];
  __shared__ uint32_t sh32[33];
  __shared__ int shi[33];
  __shared__ int s_cnt;
  __shared__ WarpSumSmem WS;
  __shared__ double s_res;
  __shared__ int s_bad;
  // Per-warp product windows: lanes compute kWin products in parallel, lane 0
  // replays the sequential add chain from shared memory (128-bit loads).
  extern __shared__ __align__(16) double dyn[];  // 2*kVec + (warps)*kWin doubles
  double* vA = dyn;
  double* vB = dyn + kVec;
  const unsigned nb = gridDim.x;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gthreads = (long long)nb * blockDim.x;
  const int lane = threadIdx.x & 31;
  const long long LD = a.LD;
  const int nu = a.n_u;
  // A launch resumes at candidate n_begin with the basis state a previous
  // segment left (K, rnnz; the last exactly processed candidate prev_n0, a
  // rejection, whose rows in W's column K are cleared below) and, with
  // exit_run > 0, returns after exit_run consecutive rejections so the host
  // can certify the following candidates in a batch (spec.cu).
  int K = a.Kstart;
  long long rnnz = a.rnnz_start;
  bool prev_acc = false;
  double prev_delta = 0.0;
  int prev_n = a.prev_n0;
  int run = 0;
  int next = nu;
  bool pre = false;  // candidate n's setup (tags, z half, g and y staging) done during P3 of n-1
  for (int n = a.n_begin; n <= nu; ++n) {
    const bool last = (n == nu);
    if (!last) stamp(a.trace, n, 0);
    const bool upd = prev_acc;
    const int Ko = K;
    const int Kn = upd ? K + 1 : K;
    double* yprev = (n & 1) ? a.ybuf0 : a.ybuf1;
    double* ycur = (n & 1) ? a.ybuf1 : a.ybuf0;
    long long off = 0;
    int m = 0;
    uint32_t tg = 0;
    double* zdn = a.zd + (n & 1) * (a.dim + 1);
    if (!last) {
      off = a.c.off[n];
      m = a.c.len[n];
      tg = a.tag_base + (uint32_t)n + 1u;
      // x's rows: tag them, start z at 0 (rows outside R stay untouched).
      // zd is double-buffered by parity: CTAs still in P3 of n-1 read the other half.
      for (long long t = gtid; !pre && t < m; t += gthreads) {
        a.tag[a.c.row[off + t]] = tg;
        zdn[a.c.row[off + t]] = 0.0;
      }
    }
    // ---------------- P1: append previous accept; fused U update + y --------
    if (a.W && !upd && prev_n >= 0) {
      // n-1 was not kept: its x rows outside R hold x - z in W's column K,
      // which candidate n reuses (R's rows and n's own rows are rewritten)
      const long long poff = a.c.off[prev_n];
      const int pm = a.c.len[prev_n];
      for (long long t = gtid; t < pm; t += gthreads) a.W[(long long)a.c.row[poff + t] * a.Wld + K] = 0.0;
    }
    if (upd && blockIdx.x == nb - 1) {
      // Ordered append of x_{n-1}'s rows not yet in R (first-appearance
      // order).  The last CTA does it: U rows are dealt from CTA 0 upward, so
      // it usually owns none and this overlaps the y chains.
      const long long poff = a.c.off[prev_n];
      const int pm = a.c.len[prev_n];
      int srn = ldg_cg(a.sr_n);
      // 4 consecutive entries per thread per block scan (C5 fibers hold
      // 1e4-1e5 entries; this CTA's append is what the others wait for)
      for (int base = 0; base < pm; base += 4 * blockDim.x) {
        const int t0 = base + 4 * threadIdx.x;
        int rr[4], nw[4], cnt = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u;
          rr[u] = t < pm ? a.c.row[poff + t] : 0;
          nw[u] = (t < pm) && (ldg_cg(&a.sr_pos[rr[u]]) < 0);
          cnt += nw[u];
        }
        int tot2;
        int pos = block_excl_sum<int>(cnt, shi, &tot2);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (nw[u]) {
            CTD_CHECK(rr[u] >= 0 && rr[u] < a.dim && srn + pos < a.dim);
            a.sr_list[srn + pos] = rr[u];
            a.sr_pos[rr[u]] = srn + pos;
            ++pos;
          }
        srn += tot2;
      }
      if (threadIdx.x == 0) {
        *a.sr_n = srn;
        a.kept_cand[Ko - a.K0] = prev_n;
        a.rptr[Ko + 1] = rnnz + a.c.len[prev_n];
      }
    }
    if (!last) stamp(a.trace, n, 1);
    if (upd || !last) {
      // g (and y_{n-1}) in shared memory when they fit (sm); otherwise g in
      // this CTA's global scratch row and y read from the global y buffer
      // (both L2-resident; the producers prefetch them with U).
      const bool sm = Kn <= a.kvec;
      double* gsc = a.gscr + (long long)blockIdx.x * (LD + 1);
      auto stage = [&](int c0, int c1) {
        __syncthreads();
        for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
          if (!last) {
            const double gj = (j < a.K0) ? a.Gb[(long long)j * nu + n]
                            : (j < Ko)   ? a.Gc[(long long)ldg_cg(&a.kept_cand[j - a.K0]) * nu + n]
                                         : a.Gc[(long long)prev_n * nu + n];  // j == Ko: x_{n-1}
            if (sm) vA[j - c0] = gj;
            else gsc[j] = gj;
          }
          if (upd && sm) vB[j - c0] = (j < Ko) ? ldg_cg(&yprev[j]) : 0.0;
        }
        __syncthreads();
      };
      auto yval = [&](long long i) -> double { return sm ? vB[i] : ldg_cg(&yprev[i]); };
      if (sm && pre) {
        // g (j < Ko), y_{n-1} and x_{n-1}'s column (speculatively: used only
        // if n-1 was kept) were staged during P3 of n-1
      } else {
        stage(0, Kn);
      }
      if (!last) stamp(a.trace, n, 2);
      // U_new[i][j] (fiber_basis.cpp:97-105): fl(U + fl(fl(y_i y_j)/d)), the
      // new column/row -y/d and the corner 1/d.  The division uses the
      // divisor's correctly rounded reciprocal (few FP64 instructions: the
      // chain warp shares the SM's FP64 pipe), certified; __ddiv_rn when the
      // check fails.
      const double rdelta = upd ? __drcp_rn(prev_delta) : 0.0;
      auto unew = [&](long long i, int j, double uo) -> double {
        const double yi = i < Ko ? yval(i) : 0.0, yj = j < Ko ? yval(j) : 0.0;
        const double num = (i < Ko && j < Ko) ? dmul(yi, yj)
                         : (i == Ko && j == Ko) ? 1.0
                         : (i == Ko) ? -yj : -yi;
        bool ok;
        double qd = ddiv_rcp(num, prev_delta, rdelta, &ok);
        if (!ok) qd = ddiv_slow(num, prev_delta);
        return (i < Ko && j < Ko) ? dadd(uo, qd) : qd;
      };
      // This CTA owns rows i = blockIdx.x + unb * r (r < Rs); groups of 32.
      // While one group per CTA suffices, the last CTA owns none: it runs the
      // ordered append of x_{n-1} above, which the other CTAs' P2 waits for.
#ifdef CTD_NO_UNB
      const unsigned unb = nb;
#else
      const unsigned unb = (nb > 1 && Kn <= 32 * (int)(nb - 1)) ? nb - 1 : nb;
#endif
      const int Rs = ((int)blockIdx.x < Kn && blockIdx.x < unb) ? (Kn - 1 - (int)blockIdx.x) / (int)unb + 1 : 0;
      const int nch = (Kn + kRingW - 1) / kRingW;
      const int Q = ((Rs + 31) / 32) * nch;
      const int warp = threadIdx.x >> 5;
      double* ring = dyn + 2 * kVec;
      if (last) {
        for (long long e = threadIdx.x; e < (long long)Rs * Kn; e += blockDim.x) {
          const int r = (int)(e / Kn), j = (int)(e - (long long)r * Kn);
          const long long i = blockIdx.x + (long long)unb * r;
          double* up = a.U + i * LD + j;
          *up = unew(i, j, (i < Ko && j < Ko) ? ldg_cg(up) : 0.0);
        }
      } else if (is_producer(warp)) {
        // producers: U_new and the products U_new[i][j] g_j of 32 rows x
        // kRingW steps; the next chunk's U loads are in flight meanwhile.
        // The producers are issue-bound, so the row slots this thread owns
        // in a group (NA <= kRowSlots, warp-uniform) are a compile-time
        // count: no predicated-off work for absent rows.
        // (Bulk/TMA staging of the U segments measured slower: it inflates
        // the chain warp's latency, tools/ubench_ring.cu.)
        const int pi = producer_index(warp, lane);
        const int t = pi % kRingW, rq = pi / kRingW;  // rq is warp-uniform
        double* ring_t = ring + rq * kRingLS + t;  // + slot, + row phase k * kRowPh * kRingLS
        const bool ptr = a.trace && blockIdx.x == 0 && pi == 0;
        long long pwt = 0, pct = 0;
        int q = 0;
        auto group = [&](int g, auto na_c) {
          constexpr int NA = decltype(na_c)::value;
          double* up[NA];
          double yi[NA];
          unsigned inew = 0;
#pragma unroll
          for (int k = 0; k < NA; ++k) {
            const long long i = blockIdx.x + (long long)unb * (32 * g + rq + kRowPh * k);
            up[k] = a.U + i * LD;
            CTD_CHECK(32 * g + rq + kRowPh * k >= Rs || i < Kn);
            yi[k] = (upd && i < Ko) ? yval(i) : 0.0;
            inew |= (unsigned)(i == Ko) << k;
          }
          double uv[NA];
          double gn = 0.0, yn = 0.0;  // g_j, y_j of the prefetched chunk (global-operand mode)
          auto load = [&](int j) {
#pragma unroll
            for (int k = 0; k < NA; ++k) uv[k] = (j < Ko && !((inew >> k) & 1)) ? ldg_cg(up[k] + j) : 0.0;
            if (!sm) {
              gn = j < Kn ? ldg_cg(&gsc[j]) : 0.0;
              yn = (upd && j < Ko) ? ldg_cg(&yprev[j]) : 0.0;
            }
          };
          load(t);
          for (int j0 = 0; j0 < Kn; j0 += kRingW, ++q) {
            const int j = j0 + t;
            const int b = q % kRingSlots;
            double* rb = ring_t + b * kRingSlot;
            const long long pt0 = ptr ? clock64() : 0;
            if (q >= kRingSlots) nbar_sync(1 + kRingSlots + b, kRingThreads);
            const long long pt1 = ptr ? clock64() : 0;
            const bool jin = j < Kn;
            const double gj = sm ? (jin ? vA[j] : 0.0) : gn;
            double un[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) un[k] = uv[k];
            if (upd) {
              // fiber_basis.cpp:97-105: fl(U + fl(fl(y_i y_j)/d)); the new
              // row/column -y/d; the corner 1/d
              const double yj = sm ? ((j < Ko) ? vB[j] : 0.0) : yn;
              const bool jnew = j == Ko;
              unsigned bad = 0;
#pragma unroll
              for (int k = 0; k < NA; ++k) {
                const bool in = (inew >> k) & 1;
                const double num = in ? (jnew ? 1.0 : -yj) : (jnew ? -yi[k] : dmul(yi[k], yj));
                bool ok;
                const double qd = ddiv_rcp(num, prev_delta, rdelta, &ok);
                bad |= (unsigned)!ok << k;
                un[k] = (in || jnew) ? qd : dadd(uv[k], qd);
              }
              if (bad) {  // rare: quotients the fast path could not certify
#pragma unroll
                for (int k = 0; k < NA; ++k)
                  if ((bad >> k) & 1) {
                    const bool in = (inew >> k) & 1;
                    const double num = in ? (jnew ? 1.0 : -yj) : (jnew ? -yi[k] : dmul(yi[k], yj));
                    const double qd = ddiv_slow(num, prev_delta);
                    un[k] = (in || jnew) ? qd : dadd(uv[k], qd);
                  }
              }
              if (jin) {
#pragma unroll
                for (int k = 0; k < NA; ++k) up[k][j] = un[k];
              }
            }
#pragma unroll
            for (int k = 0; k < NA; ++k) rb[kRowPh * k * kRingLS] = dmul(un[k], gj);
            nbar_arrive(1 + b, kRingThreads);
            if (ptr) {
              pwt += pt1 - pt0;
              pct += clock64() - pt1;
            }
            if (j0 + kRingW < Kn) load(j + kRingW);
          }
        };
        for (int g = 0; g < (Rs + 31) / 32; ++g) {
          const int nr = min(32, Rs - 32 * g);
          const int nact = nr > rq ? (nr - rq + kRowPh - 1) / kRowPh : 0;  // row slots of this thread
          switch (nact) {
            case 0: {  // no rows: hand the slots over
              for (int j0 = 0; j0 < Kn; j0 += kRingW, ++q) {
                const int b = q % kRingSlots;
                if (q >= kRingSlots) nbar_sync(1 + kRingSlots + b, kRingThreads);
                nbar_arrive(1 + b, kRingThreads);
              }
              break;
            }
            case 1: group(g, std::integral_constant<int, 1>{}); break;
            case 2: group(g, std::integral_constant<int, 2>{}); break;
            case 3: group(g, std::integral_constant<int, 3>{}); break;
            case 4: group(g, std::integral_constant<int, 4>{}); break;
            case 5: group(g, std::integral_constant<int, 5>{}); break;
            case 6: group(g, std::integral_constant<int, 6>{}); break;
            default: group(g, std::integral_constant<int, kRowSlots>{}); break;
          }
        }
        if (ptr) {
          a.trace[(long long)n * kTraceW + 28] = pwt;
          a.trace[(long long)n * kTraceW + 29] = pct;
        }
      } else if (warp == kChainWarp) {
        // chain warp: y_i = sum_j fl(U_new[i][j] g_j) in j order (dense_matrix.cpp:42-47)
        double acc = 0.0;
        long long tw = 0, tcc = 0, tprobe = 0;
        for (int q = 0; q < Q; ++q) {
          const int g = q / nch, ch = q - g * nch;
          const int cnt = min(kRingW, Kn - ch * kRingW);
          const int b = q % kRingSlots;
          const long long tw0 = clock64();
          nbar_sync(1 + b, kRingThreads);
          tw += clock64() - tw0;
#ifdef CTD_EXP_DADD_PROBE
          {
            // in-situ latency probe: 96 dependent register DADDs
            const long long tp0 = clock64();
            double d = (double)lane;
#pragma unroll 1
            for (int s = 0; s < 6; ++s) {
#pragma unroll
              for (int u = 0; u < 16; ++u) d = dadd(d, 1e-300);
            }
            tprobe += clock64() - tp0;
            if (d == 12345.0) ring[lane] = d;
          }
#endif
          const long long tc0 = clock64();
#ifndef CTD_EXP_NOCHAIN
          // (steps >= Kn hold +-0.0)
          acc = cnt > kShortChunk ? lane_chain(ring + b * kRingSlot, lane, acc)
                                  : lane_chain_n(ring + b * kRingSlot, lane, cnt, acc);
#endif
          tcc += clock64() - tc0;
          if (q + kRingSlots < Q) nbar_arrive(1 + kRingSlots + b, kRingThreads);
          if (ch == nch - 1) {
            const int r = 32 * g + lane;
            if (r < Rs) ycur[blockIdx.x + (long long)unb * r] = acc;
            acc = 0.0;
          }
        }
        if (a.trace && blockIdx.x == 0 && lane == 0) {
          a.trace[(long long)n * kTraceW + 13] = tw;
          a.trace[(long long)n * kTraceW + 11] = tcc;
          a.trace[(long long)n * kTraceW + 27] = tprobe;
        }
      }
    }
    if (upd) {
      // x_{n-1}'s entries into R's CSC and row index (read by P2 after the
      // barrier, not by P1): the producer warps do it after their last ring
      // chunk, while the chain warp finishes (off the critical path)
      const long long poff = a.c.off[prev_n];
      const int pm = a.c.len[prev_n];
      const int warp = threadIdx.x >> 5;
      const bool doer = last || is_producer(warp);
      const long long per_cta = last ? blockDim.x : kProdThreads;
      const long long me = last ? threadIdx.x : (is_producer(warp) ? producer_index(warp, lane) : 0);
      for (long long t = (long long)blockIdx.x * per_cta + me; doer && t < pm; t += (long long)nb * per_cta) {
        const int r = a.c.row[poff + t];
        const double v = a.c.val[poff + t];
        a.rrow[rnnz + t] = r;
        a.rval[rnnz + t] = v;
        const int L = ldg_cg(&a.rowlen[r]);
        const long long p = a.rowbase[r] + L;
        CTD_CHECK(r >= 0 && r < a.dim && p < a.rowbase[r + 1]);  // the row's capacity (k_row_caps)
        a.rek[p] = Ko;
        a.rev[p] = v;
        a.rowlen[r] = L + 1;
      }
      rnnz += pm;
    }
    K = Kn;
    if (last) break;
    stamp(a.trace, n, 3);
    grid_barrier(a.bar, nb);
    stamp(a.trace, n, 4);
#ifdef CTD_CHECKED
    // every CTA took the same decisions: the basis size and R's entry count agree
    if (threadIdx.x == 0) {
      a.chk[blockIdx.x * 2] = K;
      a.chk[blockIdx.x * 2 + 1] = rnnz;
    }
#endif
    // ---------------- P2: z over R's rows, residual terms ---------------------
    const int srn = ldg_cg(a.sr_n);
    const bool y_fits = K <= a.kvec;
    auto stage_y = [&](int c0, int c1) {
      __syncthreads();
      for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) vA[j - c0] = ldg_cg(&ycur[j]);
      __syncthreads();
    };
    if (y_fits) stage_y(0, K);
    stamp(a.trace, n, 10);
    {
      // Ring sessions of up to kMeta rows of R owned by this CTA (positions
      // q = blockIdx.x + nb * r of the first-appearance list).  The rows of a
      // session are ranked by length (longest first) so the 32-row groups are
      // homogeneous: a group's chain runs for its longest row.
      int* s_row = reinterpret_cast<int*>(vB);
      int* s_len = s_row + kMeta;
      int* s_tf = s_len + kMeta;
      int* s_inx = s_tf + kMeta;
      int* s_pos = s_inx + kMeta;  // original session position of ranked row
      int* s_gch = s_pos + kMeta;  // [32] chunks per group
      int* s_gmx = s_gch + 32;     // [32] longest row per group
      long long* s_base = reinterpret_cast<long long*>(s_gmx + 32);
      int* s_key = reinterpret_cast<int*>(s_base + kMeta);  // ranking keys
      double* ring = dyn + 2 * kVec;
      const int warp = threadIdx.x >> 5;
      const int Rs2 = ((int)blockIdx.x < srn) ? (srn - 1 - (int)blockIdx.x) / (int)nb + 1 : 0;
      for (int sb0 = 0; sb0 < Rs2; sb0 += kMeta) {
        const int ns = min(kMeta, Rs2 - sb0);
        __syncthreads();
        {
          const int r = threadIdx.x;
          int row = 0, L = 0;
          if (r < ns) {
            const long long q = blockIdx.x + (long long)nb * (sb0 + r);
            row = ldg_cg(&a.sr_list[q]);
            L = ldg_cg(&a.rowlen[row]);
          }
          hist[r] = (uint32_t)row;  // by session position (hist is P3 scratch)
          // rank by length, longest first, ties by position: bitonic sort of
          // the keys (2^22 - 1 - L) << 10 | r, one per thread (L < 2^22: K is)
          // (small sessions, C2: each thread counts the keys below its own,
          // O(ns) per thread, cheaper than the 45 bitonic stages)
          uint32_t* kk = reinterpret_cast<uint32_t*>(s_key);
          static_assert(kMeta == kFThreads && kMeta == 512, "bitonic ranking: one key per thread");
          const uint32_t mykey = r < ns ? ((uint32_t)(0x3FFFFF - L) << 10) | (uint32_t)r : 0xFFFFFFFFu;
          kk[r] = mykey;
          const bool quad = ns <= kQuadRank;
          if (quad) {
            __syncthreads();
            int rank = 0;
            if (r < ns)
              for (int u = 0; u < ns; ++u) rank += kk[u] < mykey;
            __syncthreads();
            if (r < ns) kk[rank] = mykey;
          }
          for (int kb = 2; !quad && kb <= kMeta; kb <<= 1) {
            for (int j = kb >> 1; j > 0; j >>= 1) {
              __syncthreads();
              const int pj = r ^ j;
              if (pj > r) {
                const uint32_t x = kk[r], x2 = kk[pj];
                if ((x > x2) == ((r & kb) == 0)) {
                  kk[r] = x2;
                  kk[pj] = x;
                }
              }
            }
          }
          __syncthreads();
          if (r < ns) {
            const int rank = r;  // slot r of the sorted keys holds the row of rank r
            const uint32_t key = kk[r];
            const int src = (int)(key & 1023u);
            row = (int)hist[src];
            L = 0x3FFFFF - (int)(key >> 10);
            s_row[rank] = row;
            s_base[rank] = a.rowbase[row];
            s_len[rank] = L;
            s_inx[rank] = ldg_cg(&a.tag[row]) == tg;
            s_tf[rank] = 0x7fffffff;
            s_pos[rank] = src;
          }
          __syncthreads();
          const int Lr = r < ns ? s_len[r] : 0;
          const int mx = __reduce_max_sync(0xffffffffu, Lr);
          if (lane == 0) {
            s_gch[warp] = max(1, (mx + kRingW - 1) / kRingW);
            s_gmx[warp] = mx;
          }
        }
        __syncthreads();
        const int ngr = (ns + 31) / 32;
        int Q = 0;
        for (int g = 0; g < ngr; ++g) Q += s_gch[g];
        if (is_producer(warp)) {
          // the next chunk's entries (k, value) are in flight meanwhile;
          // thread: step t of each chunk, rows rq + kRowPh * k of the group
          // (NA active row slots, compile-time as in P1)
          const int pi = producer_index(warp, lane);
          const int t = pi % kRingW, rq = pi / kRingW;
          double* ring_t = ring + rq * kRingLS + t;
          int q = 0;
          auto group = [&](int g, auto na_c) {
            constexpr int NA = decltype(na_c)::value;
            const int nchk = s_gch[g];
            int slen[NA];
            long long sbase[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) {
              slen[k] = s_len[32 * g + rq + kRowPh * k];
              sbase[k] = s_base[32 * g + rq + kRowPh * k];
            }
            int kv[NA];
            double vv[NA];
            unsigned okm = 0;    // rows with an entry at this step (prefetched chunk)
            unsigned found = 0;  // rows whose first y != 0 entry is known (warp-uniform)
            const int t0 = t & ~31;  // first step of this warp's 32
            auto load = [&](int te) {
              okm = 0;
#pragma unroll
              for (int k = 0; k < NA; ++k) {
                const bool ok = te < slen[k];
#if defined(CTD_EXP_L2FAKE)
                kv[k] = ok ? ldg_cg(&a.rek[(sbase[k] & 0xFFFFFll) + te]) : 0;
                vv[k] = ok ? ldg_cg(&a.rev[(sbase[k] & 0xFFFFFll) + te]) : 0.0;
#elif defined(CTD_EXP_NOLOAD2)
                kv[k] = ok ? (te & 1023) : 0;
                vv[k] = ok ? 1.0 : 0.0;
#else
                kv[k] = ok ? ldg_cg(&a.rek[sbase[k] + te]) : 0;
                vv[k] = ok ? ldg_cg(&a.rev[sbase[k] + te]) : 0.0;
#endif
                okm |= (unsigned)ok << k;
              }
            };
            // R's row index does not fit L2 at C5 scale: per-line L2
            // prefetches kPfDist chunks ahead (thread pi < 288 takes line
            // pi / 32 of row pi % 32: 3 lines of k, 6 of values per chunk).
            // (Bulk cp.async.bulk.prefetch of whole row segments measured
            // slower; r2 experiments.)
            const int lr = 32 * g + (pi & 31), ll = pi >> 5;
            const bool lok = pi < 288 && (pi & 31) < min(32, ns - 32 * g);
            const int llen = lok ? s_len[lr] : 0;
            const long long lbase = lok ? s_base[lr] : 0;
            auto prefetch = [&](int c) {
              const int e = c * kRingW + (ll < 3 ? ll * 32 : (ll - 3) * 16);
              if (e >= llen) return;
              const void* pp = ll < 3 ? (const void*)(a.rek + lbase + e) : (const void*)(a.rev + lbase + e);
              asm volatile("prefetch.global.L2 [%0];" ::"l"(pp));
            };
#ifndef CTD_NO_PF_P2
            for (int c = 1; c <= kPfDist && c < nchk; ++c) prefetch(c);
#endif
            load(t);
            for (int ch = 0; ch < nchk; ++ch, ++q) {
              const int b = q % kRingSlots;
              double* rb = ring_t + b * kRingSlot;
              const int te = ch * kRingW + t;
#ifndef CTD_NO_PF_P2
              if (ch + 1 + kPfDist < nchk) prefetch(ch + 1 + kPfDist);
#endif
              if (q >= kRingSlots) nbar_sync(1 + kRingSlots + b, kRingThreads);
#ifdef CTD_EXP_NOPROD2
              if (okm != 0xFFFFFFFFu) {
                nbar_arrive(1 + b, kRingThreads);
                continue;
              }
#endif
#pragma unroll
              for (int k = 0; k < NA; ++k) {
                const int r = rq + kRowPh * k;
                // the warp's steps are te0 .. te0+31 (t0 is a multiple of 32):
                // past the row's end they only hold +0.0
                if (ch * kRingW + t0 >= slen[k]) {
                  rb[kRowPh * k * kRingLS] = 0.0;
                  continue;
                }
                const bool ok = (okm >> k) & 1;
                CTD_CHECK(!ok || (kv[k] >= 0 && kv[k] < K));
                const double yk = ok ? (y_fits ? vA[kv[k]] : ldg_cg(&ycur[kv[k]])) : 0.0;
                rb[kRowPh * k * kRingLS] = dmul(yk, vv[k]);
                if (!((found >> k) & 1)) {
                  // first kept column of the row with y != 0 (the touch order)
                  const unsigned nz = __ballot_sync(0xffffffffu, ok && yk != 0.0);
                  if (nz) {
                    if (lane == __ffs(nz) - 1) atomicMin(&s_tf[32 * g + r], te);
                    found |= 1u << k;
                  }
                }
              }
              nbar_arrive(1 + b, kRingThreads);
              if (ch + 1 < nchk) load(te + kRingW);
            }
          };
          for (int g = 0; g < ngr; ++g) {
            const int nr = min(32, ns - 32 * g);
            const int nact = nr > rq ? (nr - rq + kRowPh - 1) / kRowPh : 0;
            switch (nact) {
              case 0: {
                for (int ch = 0; ch < s_gch[g]; ++ch, ++q) {
                  const int b = q % kRingSlots;
                  if (q >= kRingSlots) nbar_sync(1 + kRingSlots + b, kRingThreads);
                  nbar_arrive(1 + b, kRingThreads);
                }
                break;
              }
              case 1: group(g, std::integral_constant<int, 1>{}); break;
              case 2: group(g, std::integral_constant<int, 2>{}); break;
              case 3: group(g, std::integral_constant<int, 3>{}); break;
              case 4: group(g, std::integral_constant<int, 4>{}); break;
              case 5: group(g, std::integral_constant<int, 5>{}); break;
              case 6: group(g, std::integral_constant<int, 6>{}); break;
              default: group(g, std::integral_constant<int, kRowSlots>{}); break;
            }
          }
        } else if (warp == kChainWarp) {
          // chain warp: z_r = sum_k fl(y_k R[r,k]) in ascending k (fiber_basis.cpp:56-65)
          int q = 0;
          long long p2w = 0, p2c = 0;  // trace: cycles waiting for full slots / chaining
          if (a.trace && blockIdx.x == 0 && lane == 0 && sb0 == 0) {
            a.trace[(long long)n * kTraceW + 14] = clock64();
            long long st = 0;
            for (int g = 0; g < ngr; ++g) st += s_gmx[g];
            a.trace[(long long)n * kTraceW + 31] = st * 1000 + ngr;
          }
          for (int g = 0; g < ngr; ++g) {
            const int nchk = s_gch[g], mx = s_gmx[g];
            double z = 0.0;
            for (int ch = 0; ch < nchk; ++ch, ++q) {
              const int b = q % kRingSlots;
              const long long tw0 = a.trace ? clock64() : 0;
              nbar_sync(1 + b, kRingThreads);
              const long long tw1 = a.trace ? clock64() : 0;
              // steps past a row's length hold +0.0, which leave z unchanged
#ifndef CTD_EXP_NOCHAIN2
              const int cnt = min(kRingW, mx - ch * kRingW);
              z = cnt > kShortChunk ? lane_chain(ring + b * kRingSlot, lane, z)
                                    : lane_chain_n(ring + b * kRingSlot, lane, cnt, z);
#endif
              if (a.trace) {
                p2w += tw1 - tw0;
                p2c += clock64() - tw1;
              }
              if (q + kRingSlots < Q) nbar_arrive(1 + kRingSlots + b, kRingThreads);
            }
            const int r = 32 * g + lane;
            if (r < ns) {
              const int row = s_row[r];
              const int L = s_len[r];
              const long long b0 = s_base[r];
              const int tf = s_tf[r];
              const int kfd = tf < L ? ldg_cg(&a.rek[b0 + tf]) : -1;
              const int kst = L > 0 ? ldg_cg(&a.rek[b0]) : -1;
              CTD_CHECK(row >= 0 && row < a.dim && K < a.Wld + (a.W ? 0 : K + 1));
              CTD_CHECK(blockIdx.x + (long long)nb * (sb0 + s_pos[r]) < srn);
              zdn[row] = z;
              if (a.W) a.W[(long long)row * a.Wld + K] = -z;  // W's column K on R's rows (relerr.cu)
              a.kf[row] = kfd;
              a.term[blockIdx.x + (long long)nb * (sb0 + s_pos[r])] = s_inx[r] ? 0.0 : dsqr(z);
              // touched order differs from first-appearance order only if
              // the row's first kept column has y == 0 while it is touched
              if (z != 0.0 && kfd != kst) atomicExch(&a.slow[n], 1);
            }
          }
          if (a.trace && blockIdx.x == 0 && lane == 0) {
            a.trace[(long long)n * kTraceW + 15] = clock64();
            a.trace[(long long)n * kTraceW + 26] += p2w;  // summed over sessions
            a.trace[(long long)n * kTraceW + 27] += p2c;
          }
        }
      }
    }
    stamp(a.trace, n, 5);
    grid_barrier(a.bar, nb);
    stamp(a.trace, n, 6);
#ifdef CTD_CHECKED
    if (threadIdx.x == 0) {
      const unsigned o = (blockIdx.x + 1) % nb;
      CTD_CHECK(__ldcg(&a.chk[o * 2]) == K && __ldcg(&a.chk[o * 2 + 1]) == rnnz);
    }
#endif
    // ---------------- P3: exact residual, decision (every CTA) ---------------
    const bool slow = ldg_cg(&a.slow[n]) != 0;
    long long nterm = srn;
    const double* tsrc = a.term;
    if (slow) {
      // Rebuild the touched list in the reference's order: rows r not in x
      // with kfd(r) >= 0, sorted by (kfd, position within column kfd) which is
      // (kfd, r).  Done by CTA 0, then shared through a barrier.
      if (blockIdx.x == 0) {
        uint32_t* ka = a.skey;
        uint32_t* kb = ka + a.dim;
        uint32_t* ia = kb + a.dim;
        uint32_t* ib = ia + a.dim;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int qq = threadIdx.x; qq < srn; qq += blockDim.x) {
          const int r = ldg_cg(&a.sr_list[qq]);
          if (ldg_cg(&a.kf[r]) >= 0 && ldg_cg(&a.tag[r]) != tg) {
            const int p = atomicAdd(&s_cnt, 1);
            ka[p] = (uint32_t)r;
            ia[p] = (uint32_t)r;
          }
        }
        __syncthreads();
        const int cnt = s_cnt;
        // sort by r, then stable by kfd
        bool inb = block_radix_sort<uint32_t>(ka, kb, ia, ib, cnt, 32, hist, sh32);
        uint32_t* K2 = inb ? kb : ka;
        uint32_t* I2 = inb ? ib : ia;
        uint32_t* K3 = inb ? ka : kb;
        uint32_t* I3 = inb ? ia : ib;
        for (int p = threadIdx.x; p < cnt; p += blockDim.x) {
          K3[p] = (uint32_t)ldg_cg(&a.kf[I2[p]]);
          I3[p] = I2[p];
        }
        __syncthreads();
        inb = block_radix_sort<uint32_t>(K3, K2, I3, I2, cnt, 32, hist, sh32);
        const uint32_t* IF = inb ? I2 : I3;
        for (int p = threadIdx.x; p < cnt; p += blockDim.x) a.term2[p] = dsqr(ldg_cg(&zdn[IF[p]]));
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          a.slow[n] = 2 + cnt;  // publish count
        }
      }
      grid_barrier(a.bar, nb);
      nterm = ldg_cg(&a.slow[n]) - 2;
      tsrc = a.term2;
    }
    const double* xv = a.c.val + off;
    const int32_t* xr = a.c.row + off;
    const long long nt = (long long)m + nterm;
    bool bad = false;
    // Terms in the reference's summation order (fiber_basis.cpp:66-77): x's
    // rows ascending, then R's rows in first-touch order.
    // (also writes the x rows of W's column K: x - z, see relerr.cu)
    const ResidualTerms get{xv, xr, zdn, (long long)m, tsrc, a.W ? a.W + K : nullptr, a.Wld};
    // exact sequential residual: warp 0 of every CTA (warp_grid_sum); the
    // other warps wait at the CTA barrier
    stamp(a.trace, n, 7);
    stamp(a.trace, n, 12);
    // the other warps set up candidate n+1 meanwhile (independent of n's
    // decision): tag its rows, zero its z half, stage g_{n+1} over the current
    // K columns and y_n.  Not when the slow touch-order path is active (it
    // reads the tags of n) or the vectors do not fit one staging chunk.
    const bool prestage = !slow && n + 1 < nu && K + 1 <= a.kvec;
    const int ncw = (int)(nb + 31) / 32;  // combine warps of warp_grid_sum
    if ((int)(threadIdx.x >> 5) < ncw) {
      SliceDirect* sd = reinterpret_cast<SliceDirect*>(dyn + 2 * kVec);  // ring area, idle in P3
      const double r = warp_grid_sum(get, nt, tg, a.sloc, a.ssum, a.sdir, a.sflag, WS, sd,
                                     reinterpret_cast<int*>(sd + kMaxDirectsTotal), &bad,
                                     a.trace ? a.trace + (long long)n * kTraceW + 16 : nullptr);
      if (threadIdx.x == 0) {
        s_res = r;
        s_bad = bad;
      }
    } else if (prestage) {
      const int n1 = n + 1;
      const int pw = blockDim.x - 32 * ncw;  // prestage threads per CTA
      const long long tw = (long long)nb * pw;
      const long long off1 = a.c.off[n1];
      const int m1 = a.c.len[n1];
      const uint32_t tg1 = a.tag_base + (uint32_t)n1 + 1u;
      double* zd1 = a.zd + (n1 & 1) * (a.dim + 1);
      for (long long t = (long long)blockIdx.x * pw + threadIdx.x - 32 * ncw; t < m1; t += tw) {
        const int r = a.c.row[off1 + t];
        a.tag[r] = tg1;
        zd1[r] = 0.0;
      }
      for (int j = threadIdx.x - 32 * ncw; j <= K; j += pw) {
        if (j == K) {  // column K if n is kept: g(x_n, x_{n+1})
          vA[K] = a.Gc[(long long)n * nu + n1];
          vB[K] = 0.0;
          continue;
        }
        vA[j] = (j < a.K0) ? a.Gb[(long long)j * nu + n1]
                           : a.Gc[(long long)ldg_cg(&a.kept_cand[j - a.K0]) * nu + n1];
        vB[j] = ldg_cg(&ycur[j]);
      }
    }
    __syncthreads();
    pre = prestage;
    const double res = s_res;
    bad = s_bad != 0;
    stamp(a.trace, n, 8);
    const double xs = a.xsq[n];
    const bool reject = __dsqrt_rn(res) <= dmul(a.eps, __dsqrt_rn(xs));  // :79
    bool acc = false, degen = false;
    if (!reject) {
      degen = !(res > 0.0) || isinf(res) || isnan(res) || isinf(ddiv(1.0, res));  // :84-85
      acc = !degen;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.accepted[n] = acc;
      a.degenerate[n] = degen;
      a.delta[n] = acc ? res : 0.0;
      a.res_out[n] = res;
      if (bad) {
        atomicOr(a.flags, FLAG_SEQSUM);
        atomicAdd(a.nfallback, 1);
      }
    }
    if (a.y_last && n == nu - 1 && blockIdx.x == 0)
      for (int i = threadIdx.x; i < K; i += blockDim.x) a.y_last[i] = ldg_cg(&ycur[i]);
    prev_acc = acc;
    prev_delta = res;
    prev_n = n;
    stamp(a.trace, n, 9);
    // every CTA took the same decision, so they all leave together
    run = reject ? run + 1 : 0;
    if (a.exit_run > 0 && run >= a.exit_run && n + 1 < nu) {
      next = n + 1;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.final_K = K;
    *a.final_rnnz = rnnz;
    if (a.next_out) *a.next_out = next;
  }
}
