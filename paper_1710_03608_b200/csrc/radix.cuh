// Stable LSD block radix sort on 32-bit keys with an index payload.
// One CTA sorts m elements; keys/indices may live in shared or global
// memory (generic pointers).  Per pass: per-warp digit histograms (warp
// `w` owns a contiguous chunk), a digit-major exclusive scan over
// (digit, warp), then an in-order scatter in which each lane's rank among
// equal-digit lanes comes from __match_any_sync — stable by construction.
#pragma once
#include "common.cuh"

namespace ctdgpu {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

// hist: (blockDim.x/32) * 256 uint32 in shared memory; sh: 33 uint32.
// Returns true if the sorted data ended in (kb, ib), false if in (ka, ia).
template <typename IdxT>
__device__ bool block_radix_sort(uint32_t* ka, uint32_t* kb, IdxT* ia, IdxT* ib, int m, int bits,
                                 uint32_t* hist, uint32_t* sh) {
  const int nw = blockDim.x >> 5, w = warp_id(), l = lane_id();
  const int chunk = (((m + nw - 1) / nw) + 31) & ~31;
  const int c0 = min(w * chunk, m), c1 = min(c0 + chunk, m);
  const unsigned lt_mask = (1u << l) - 1u;
  bool flip = false;
  for (int shift = 0; shift < bits; shift += kRadixBits) {
    uint32_t* src = flip ? kb : ka;
    uint32_t* dst = flip ? ka : kb;
    IdxT* isrc = flip ? ib : ia;
    IdxT* idst = flip ? ia : ib;
    for (int d = l; d < kRadix; d += 32) hist[w * kRadix + d] = 0;
    __syncwarp();
    for (int g = c0; g < c1; g += 32) {
      const int p = g + l;
      const bool act = p < c1;
      const unsigned amask = __ballot_sync(0xffffffffu, act);
      if (act) {
        const uint32_t d = (src[p] >> shift) & (kRadix - 1);
        const unsigned peers = __match_any_sync(amask, d);
        if (l == __ffs(peers) - 1) hist[w * kRadix + d] += __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    // Exclusive scan over counters in digit-major order (L = d * nw + w).
    const int tot = kRadix * nw;
    const int per = (tot + blockDim.x - 1) / blockDim.x;
    uint32_t s = 0;
    for (int k = 0; k < per; ++k) {
      const int L = threadIdx.x * per + k;
      if (L < tot) s += hist[(L % nw) * kRadix + L / nw];
    }
    uint32_t pre = block_excl_sum<uint32_t>(s, sh, nullptr);
    for (int k = 0; k < per; ++k) {
      const int L = threadIdx.x * per + k;
      if (L < tot) {
        uint32_t* h = &hist[(L % nw) * kRadix + L / nw];
        const uint32_t c = *h;
        *h = pre;
        pre += c;
      }
    }
    __syncthreads();
    for (int g = c0; g < c1; g += 32) {
      const int p = g + l;
      const bool act = p < c1;
      const unsigned amask = __ballot_sync(0xffffffffu, act);
      uint32_t d = 0;
      unsigned peers = 0;
      if (act) {
        const uint32_t key = src[p];
        d = (key >> shift) & (kRadix - 1);
        peers = __match_any_sync(amask, d);
        const uint32_t pos = hist[w * kRadix + d] + __popc(peers & lt_mask);
        dst[pos] = key;
        idst[pos] = isrc[p];
      }
      __syncwarp();
      if (act && l == __ffs(peers) - 1) hist[w * kRadix + d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    flip = !flip;
  }
  return flip;
}

}  // namespace ctdgpu
