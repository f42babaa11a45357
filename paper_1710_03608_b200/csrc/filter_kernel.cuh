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

constexpr int kFThreads = 512;
constexpr int kVec = 8192;  // doubles per staged vector (two buffers)

// acc <- (((acc + p_0) + p_1) + ... + p_{cnt-1}) where lane q holds p_q.
// Lanes stage their products in the warp's shared slot; lane 0 runs the
// dependent chain (the result is meaningful on lane 0 only).
__device__ __forceinline__ double warp_chain(double* wbuf, int lane, double p, int cnt, double acc) {
  wbuf[lane] = p;
  __syncwarp();
  if (lane == 0) {
    // all loads issued before the dependent chain starts
    const double2* w2 = reinterpret_cast<const double2*>(wbuf);
    double v[32];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double2 t = w2[q];
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
    if (cnt == 32) {
#pragma unroll
      for (int q = 0; q < 32; ++q) acc = dadd(acc, v[q]);
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < cnt) acc = dadd(acc, v[q]);
    }
  }
  __syncwarp();
  return acc;
}

constexpr int kWin = 256;  // products per warp window

// acc <- (((acc + w_0) + w_1) + ... + w_{cnt-1}) over the warp's window (lanes
// wrote it); lane 0 runs the chain, batches of 16 128-bit loads ahead of it.
__device__ __forceinline__ double window_chain(const double* wwin, int lane, int cnt, double acc) {
  __syncwarp();
  if (lane == 0) {
    const double2* w2 = reinterpret_cast<const double2*>(wwin);
    for (int b = 0; b < cnt; b += 32) {
      double v[32];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 t = w2[(b >> 1) + q];
        v[2 * q] = t.x;
        v[2 * q + 1] = t.y;
      }
      const int mm = min(32, cnt - b);
      if (mm == 32) {
#pragma unroll
        for (int q = 0; q < 32; ++q) acc = dadd(acc, v[q]);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < mm) acc = dadd(acc, v[q]);
      }
    }
  }
  __syncwarp();
  return acc;
}

__global__ void __launch_bounds__(kFThreads, 1) k_filter(FArgs a) {
  __shared__ SeqSumSmem S;
  __shared__ uint32_t hist[(kFThreads / 32) * kRadix];
  __shared__ uint32_t sh32[33];
  __shared__ int shi[33];
  __shared__ int s_cnt;
  // Per-warp product windows: lanes compute kWin products in parallel, lane 0
  // replays the sequential add chain from shared memory (128-bit loads).
  extern __shared__ __align__(16) double dyn[];  // 2*kVec + (warps)*kWin doubles
  double* vA = dyn;
  double* vB = dyn + kVec;
  double* wwin = dyn + 2 * kVec + (threadIdx.x >> 5) * kWin;
  double* wbuf = wwin;
  const unsigned nb = gridDim.x;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gthreads = (long long)nb * blockDim.x;
  const int lane = threadIdx.x & 31;
  // Rows are dealt round-robin over SMs first (warp-major), so a few hundred
  // dependent chains spread over all SMs instead of saturating the FP64 pipes
  // of the first few.
  const long long gwarp = (long long)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const long long gwarps = (long long)nb * (blockDim.x >> 5);
  const long long LD = a.LD;
  const int nu = a.n_u;
  int K = a.K0;
  long long rnnz = a.rnnz0;
  bool prev_acc = false;
  double prev_delta = 0.0;
  int prev_n = -1;
  for (int n = 0; n <= nu; ++n) {
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
      for (long long t = gtid; t < m; t += gthreads) {
        a.tag[a.c.row[off + t]] = tg;
        zdn[a.c.row[off + t]] = 0.0;
      }
    }
    // ---------------- P1: append previous accept; fused U update + y --------
    if (upd) {
      const long long poff = a.c.off[prev_n];
      const int pm = a.c.len[prev_n];
      for (long long t = gtid; t < pm; t += gthreads) {
        const int r = a.c.row[poff + t];
        const double v = a.c.val[poff + t];
        a.rrow[rnnz + t] = r;
        a.rval[rnnz + t] = v;
        const int L = ldg_cg(&a.rowlen[r]);
        const long long p = a.rowbase[r] + L;
        a.rek[p] = Ko;
        a.rev[p] = v;
        a.rowlen[r] = L + 1;
      }
      if (blockIdx.x == nb - 1) {
        // Ordered append of x's rows not yet in R (first-appearance order).
        // The last CTA does it: U rows are dealt from CTA 0 upward, so it
        // usually owns none and this overlaps the y chains.
        int srn = ldg_cg(a.sr_n);
        for (int base = 0; base < pm; base += blockDim.x) {
          const int t = base + threadIdx.x;
          const int r = t < pm ? a.c.row[poff + t] : 0;
          const int isnew = (t < pm) && (ldg_cg(&a.sr_pos[r]) < 0);
          int tot2;
          const int pos = block_excl_sum<int>(isnew, shi, &tot2);
          if (isnew) {
            a.sr_list[srn + pos] = r;
            a.sr_pos[r] = srn + pos;
          }
          srn += tot2;
        }
        if (threadIdx.x == 0) {
          *a.sr_n = srn;
          a.kept_cand[Ko - a.K0] = prev_n;
          a.rptr[Ko + 1] = rnnz + pm;
        }
      }
      rnnz += pm;
    }
    if (!last) stamp(a.trace, n, 1);
    if (upd || !last) {
      // Stage g (and y_{n-1}) in shared memory: once when it fits (rows then
      // proceed without CTA synchronization), else per chunk of kVec.
      const bool one_chunk = Kn <= kVec;
      auto stage = [&](int c0, int c1) {
        __syncthreads();
        for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
          if (!last)
            vA[j - c0] = (j < a.K0) ? a.Gb[(long long)j * nu + n]
                       : (j < Ko)   ? a.Gc[(long long)ldg_cg(&a.kept_cand[j - a.K0]) * nu + n]
                                    : a.Gc[(long long)prev_n * nu + n];  // j == Ko: x_{n-1}
          if (upd) vB[j - c0] = (j < Ko) ? ldg_cg(&yprev[j]) : 0.0;
        }
        __syncthreads();
      };
      if (one_chunk) stage(0, Kn);
      if (!last) stamp(a.trace, n, 2);
      for (long long rb = 0; rb < Kn; rb += gwarps) {
        const long long i = rb + gwarp;
        const bool active = i < Kn;
        const double yi = (upd && active && i < Ko) ? ldg_cg(&yprev[i]) : 0.0;
        double* urow = a.U + (active ? i : 0) * LD;
        double acc = 0.0;
        for (int c0 = 0; c0 < Kn; c0 += kVec) {
          const int c1 = min(Kn, c0 + kVec);
          if (!one_chunk) stage(c0, c1);
          if (!active) continue;
          // Windows of kWin elements: 8 loads in flight per lane, all U
          // updates and products computed lane-parallel into the warp's
          // window, then lane 0 runs the add chain over the window.
          double u[kWin / 32];
#pragma unroll
          for (int s = 0; s < kWin / 32; ++s) {
            const int j = c0 + 32 * s + lane;
            u[s] = (j < c1 && j < Ko && i < Ko) ? ldg_cg(&urow[j]) : 0.0;
          }
          for (int j0 = c0; j0 < c1; j0 += kWin) {
            double unv[kWin / 32];
            if (upd) {
              // U_new[i][j] = fl(U + fl(fl(y_i y_j)/d)): branch-free exact
              // divisions (overlapping), certified; a lane whose check fails
              // redoes its window with __ddiv_rn.
              bool wok = true;
#pragma unroll
              for (int s = 0; s < kWin / 32; ++s) {
                const int j = j0 + 32 * s + lane;
                const double num = (i < Ko && j < Ko) ? dmul(yi, vB[j - c0])
                                 : (i == Ko && j == Ko) ? 1.0
                                 : (i == Ko) ? -vB[j - c0] : -yi;
                bool ok;
                const double qd = ddiv_try(num, prev_delta, &ok);
                wok &= ok | (j >= c1);
                unv[s] = (i < Ko && j < Ko) ? dadd(u[s], qd) : qd;
              }
              if (__any_sync(0xffffffffu, !wok) && !wok) {
#pragma unroll
                for (int s = 0; s < kWin / 32; ++s) {
                  const int j = j0 + 32 * s + lane;
                  if (j >= c1) continue;
                  if (i < Ko && j < Ko) unv[s] = dadd(u[s], ddiv(dmul(yi, vB[j - c0]), prev_delta));
                  else if (i == Ko && j == Ko) unv[s] = ddiv(1.0, prev_delta);
                  else if (i == Ko) unv[s] = ddiv(-vB[j - c0], prev_delta);
                  else unv[s] = ddiv(-yi, prev_delta);
                }
              }
            } else {
#pragma unroll
              for (int s = 0; s < kWin / 32; ++s) unv[s] = u[s];
            }
#pragma unroll
            for (int s = 0; s < kWin / 32; ++s) {
              const int j = j0 + 32 * s + lane;
              double p = 0.0;
              if (j < c1) {
                if (upd) urow[j] = unv[s];
                if (!last) p = dmul(unv[s], vA[j - c0]);
              }
              wwin[32 * s + lane] = p;
            }
            const int jn = j0 + kWin;  // next window's U loads overlap this chain
            if (jn < c1) {
#pragma unroll
              for (int s = 0; s < kWin / 32; ++s) {
                const int j = jn + 32 * s + lane;
                u[s] = (j < c1 && j < Ko && i < Ko) ? ldg_cg(&urow[j]) : 0.0;
              }
            }
            if (!last) acc = window_chain(wwin, lane, min(kWin, c1 - j0), acc);
          }
        }
        if (!last && active && lane == 0) ycur[i] = acc;
      }
    }
    K = Kn;
    if (last) break;
    stamp(a.trace, n, 3);
    grid_barrier(a.bar, nb);
    stamp(a.trace, n, 4);
    // ---------------- P2: z over R's rows, residual terms ---------------------
    const int srn = ldg_cg(a.sr_n);
    const bool y_fits = K <= kVec;
    auto stage_y = [&](int c0, int c1) {
      __syncthreads();
      for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) vA[j - c0] = ldg_cg(&ycur[j]);
      __syncthreads();
    };
    if (y_fits) stage_y(0, K);
    stamp(a.trace, n, 10);
    if (y_fits) {
      // Warp w owns rows q = w + k*gwarps.  Metadata (row id, base, length,
      // tag) of 32 of them is fetched at once, one row per lane, so the rows
      // themselves only wait on their entry windows.
      for (long long k0 = 0; gwarp + k0 * gwarps < srn; k0 += 32) {
        const long long qk = gwarp + (k0 + lane) * gwarps;
        int rk = 0, Lk = 0;
        long long bk = 0;
        uint32_t tk = 0;
        if (qk < srn) rk = ldg_cg(&a.sr_list[qk]);
        if (qk < srn) {
          bk = a.rowbase[rk];
          Lk = ldg_cg(&a.rowlen[rk]);
          tk = ldg_cg(&a.tag[rk]);
        }
        for (int kq = 0; kq < 32; ++kq) {
          const long long q = gwarp + (k0 + kq) * gwarps;
          if (q >= srn) break;
          const int r = __shfl_sync(0xffffffffu, rk, kq);
          const long long b0 = __shfl_sync(0xffffffffu, bk, kq);
          const int L = __shfl_sync(0xffffffffu, Lk, kq);
          const bool inx = __shfl_sync(0xffffffffu, tk, kq) == tg;
          double z = 0.0;
          int kfd = -1;
          const int kst = L > 0 ? __shfl_sync(0xffffffffu, ldg_cg(&a.rek[b0 + (lane & 0)]), 0) : -1;
          // software pipeline: the next window's entries are in flight while
          // the current window's chain runs
          int kk[kWin / 32];
          double vv[kWin / 32];
#pragma unroll
          for (int s = 0; s < kWin / 32; ++s) {
            const int t = 32 * s + lane;
            kk[s] = t < L ? ldg_cg(&a.rek[b0 + t]) : 0;
            vv[s] = t < L ? ldg_cg(&a.rev[b0 + t]) : 0.0;
          }
          for (int e = 0; e < L; e += kWin) {
            unsigned nzm[kWin / 32];
#pragma unroll
            for (int s = 0; s < kWin / 32; ++s) {
              const int t = e + 32 * s + lane;
              const double yk = t < L ? vA[kk[s]] : 0.0;
              wwin[32 * s + lane] = dmul(yk, vv[s]);
              nzm[s] = __ballot_sync(0xffffffffu, t < L && yk != 0.0);
            }
            if (kfd < 0) {
#pragma unroll
              for (int s = kWin / 32 - 1; s >= 0; --s)
                if (nzm[s]) kfd = __shfl_sync(0xffffffffu, kk[s], __ffs(nzm[s]) - 1);
            }
            const int en = e + kWin;
            if (en < L) {
#pragma unroll
              for (int s = 0; s < kWin / 32; ++s) {
                const int t = en + 32 * s + lane;
                kk[s] = t < L ? ldg_cg(&a.rek[b0 + t]) : 0;
                vv[s] = t < L ? ldg_cg(&a.rev[b0 + t]) : 0.0;
              }
            }
            z = window_chain(wwin, lane, min(kWin, L - e), z);
          }
          if (lane == 0) {
            zdn[r] = z;
            a.kf[r] = kfd;
            a.term[q] = inx ? 0.0 : dsqr(z);
            if (z != 0.0 && kfd != kst) atomicExch(&a.slow[n], 1);
          }
        }
      }
    }
    for (long long rb = 0; !y_fits && rb < srn; rb += gwarps) {
      const long long q = rb + gwarp;
      int r = 0, L = 0, e = 0, kfd = -1, kst = -1;
      long long b0 = 0;
      double z = 0.0;
      if (q < srn) {
        r = ldg_cg(&a.sr_list[q]);
        b0 = a.rowbase[r];
        L = ldg_cg(&a.rowlen[r]);
      }
      for (int c0 = 0; c0 < K; c0 += kVec) {
        const int c1 = min(K, c0 + kVec);
        if (!y_fits) stage_y(c0, c1);
        if (q >= srn) continue;
        if (K <= kVec) {
          // whole row in one chunk: windows of kWin entries, all loads first
          for (; e < L; e += kWin) {
            int kk[kWin / 32];
            double vv[kWin / 32];
#pragma unroll
            for (int s = 0; s < kWin / 32; ++s) {
              const int t = e + 32 * s + lane;
              kk[s] = t < L ? ldg_cg(&a.rek[b0 + t]) : 0;
              vv[s] = t < L ? ldg_cg(&a.rev[b0 + t]) : 0.0;
            }
#pragma unroll
            for (int s = 0; s < kWin / 32; ++s) {
              const int t = e + 32 * s + lane;
              const double yk = t < L ? vA[kk[s]] : 0.0;
              wwin[32 * s + lane] = dmul(yk, vv[s]);
              if (kst < 0) kst = __shfl_sync(0xffffffffu, kk[s], 0);
              const unsigned nz = __ballot_sync(0xffffffffu, t < L && yk != 0.0);
              if (kfd < 0 && nz) kfd = __shfl_sync(0xffffffffu, kk[s], __ffs(nz) - 1);
            }
            z = window_chain(wwin, lane, min(kWin, L - e), z);
          }
        } else {
          while (e < L) {
            const int t = e + lane;
            const int k = (t < L) ? ldg_cg(&a.rek[b0 + t]) : 0x7fffffff;
            const bool in = k < c1;  // entries sorted by k: `in` is a lane prefix
            const unsigned inmask = __ballot_sync(0xffffffffu, in);
            if (!inmask) break;
            const double yk = in ? vA[k - c0] : 0.0;
            const double p = in ? dmul(yk, ldg_cg(&a.rev[b0 + t])) : 0.0;
            if (kst < 0) kst = __shfl_sync(0xffffffffu, k, 0);
            const unsigned nzmask = __ballot_sync(0xffffffffu, in && yk != 0.0);
            if (kfd < 0 && nzmask) kfd = __shfl_sync(0xffffffffu, k, __ffs(nzmask) - 1);
            const int cnt = __popc(inmask);
            z = warp_chain(wbuf, lane, p, cnt, z);
            e += cnt;
            if (cnt < 32) break;
          }
        }
      }
      if (rb == 0) stamp(a.trace, n, 11);
      if (q < srn && lane == 0) {
        zdn[r] = z;
        a.kf[r] = kfd;
        a.term[q] = (ldg_cg(&a.tag[r]) == tg) ? 0.0 : dsqr(z);
        // touched order differs from first-appearance order only if the row's
        // first kept column has y == 0 while the row is still touched.
        if (z != 0.0 && kfd != kst) atomicExch(&a.slow[n], 1);
      }
    }
    stamp(a.trace, n, 5);
    grid_barrier(a.bar, nb);
    stamp(a.trace, n, 6);
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
    const double* zd = zdn;
    auto get = [=](long long i) -> double {
      if (i < m) return dsqr(dsub(xv[i], ldg_cg(&zd[xr[i]])));  // fiber_basis.cpp:69-70
      return ldg_cg(&tsrc[i - m]);                              // fiber_basis.cpp:74-75
    };
    slice_summarize(get, nt, a.ssum, a.sdir, S);
    stamp(a.trace, n, 7);
    grid_barrier(a.bar, nb);
    stamp(a.trace, n, 12);
    const double res = slice_combine(get, nt, a.ssum, a.sdir, S, dyn, &bad);
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
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.final_K = K;
    *a.final_rnnz = rnnz;
  }
}
