// Micro-benchmark of the filter's producer/consumer ring (P1 shape):
// 15 producer warps fill kRingW x 32 products per chunk, one chain warp runs
// 32 lane-parallel add chains.  Variants isolate what slows the chain.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_ring tools/ubench_ring.cu
#include <cstdio>
#include <vector>

#include "../paper_1710_03608_b200/csrc/common.cuh"

using namespace ctdgpu;

constexpr int kT = 512, kW = 64, kS = 33, kStages = 3;
constexpr int kPerMax = (32 * kW + 383) / 384;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void nsync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void narv(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void mb_init(uint64_t* m) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(m)) : "memory"); }
__device__ __forceinline__ void mb_tx(uint64_t* m, unsigned b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(b) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* m, unsigned par) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(su32(m)),
               "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned b, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s),
               "r"(b), "r"(su32(m)) : "memory");
}

__device__ __forceinline__ double lane_chain(const double* rb, int lane, double acc) {
  const double* p = rb + lane;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = p[q * kS];
#pragma unroll
  for (int h = 0; h < kW / 16; ++h) {
    double w[16];
    if (h + 1 < kW / 16) {
#pragma unroll
      for (int q = 0; q < 16; ++q) w[q] = p[((h + 1) * 16 + q) * kS];
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = ctdgpu::dadd(acc, v[q]);
    if (h + 1 < kW / 16) {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = w[q];
    }
  }
  return acc;
}

// pair layout: step t of lane l at double (t >> 1) * kP + 2 l + (t & 1)
constexpr int kP = 66;
__device__ __forceinline__ void lds2(double& x, double& y, uint32_t a) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ double lane_chain2(const double* rb, int lane, double acc) {
  const uint32_t base = su32(rb + 2 * lane);
  double v[16], w[16];
#pragma unroll
  for (int q = 0; q < 8; ++q) lds2(v[2 * q], v[2 * q + 1], base + q * kP * 8);
#pragma unroll
  for (int h = 0; h < kW / 16; ++h) {
    if (h + 1 < kW / 16) {
#pragma unroll
      for (int q = 0; q < 8; ++q) lds2(w[2 * q], w[2 * q + 1], base + ((h + 1) * 8 + q) * kP * 8);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = ctdgpu::dadd(acc, v[q]);
    if (h + 1 < kW / 16) {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = w[q];
    }
  }
  return acc;
}

// mode 0: producers write products from registers (no memory reads)
// mode 1: producers read U from global (ld.cg), 1 chunk register prefetch
// mode 2: U rows staged by bulk copies (thread 0 issues), mbarrier waits
// mode 3: consumer alone (producers do nothing; ring prefilled)
// div: producers also run ddiv_try per element
__global__ void __launch_bounds__(kT, 1) k_ring(const double* U, long long LD, int rows, int Q, int mode, int div,
                                                 int avoid, int pair, int first, long long* cyc, double* out) {
  const int kProd = avoid ? 384 : 480, kAll = kProd + 32;
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;
  double* stg = sm + 2 * kW * kS;
  const int mode_ = mode;
  __shared__ __align__(8) uint64_t mbar[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mb_init(&mbar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 2 * kW * kS; i += kT) ring[i] = 1e-3 * (i & 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = first ? (15 - (int)(threadIdx.x >> 5)) : (int)(threadIdx.x >> 5);  // first: chain warp is hw warp 0
  const int nch = Q;
  const long long row0 = blockIdx.x;
  long long t0 = clock64();
  if (mode == 3) {
    if (warp == 15) {
      double acc = 0.0;
      for (int q = 0; q < Q; ++q) acc = lane_chain(ring + (q & 1) * kW * kS, lane, acc);
      out[blockIdx.x * 32 + lane] = acc;
    }
  } else if (warp < 15 && !(avoid == 1 && (warp & 3) == 3) && !(avoid == 2 && warp >= 12)) {
    const int pi = avoid == 1 ? ((warp >> 2) * 3 + (warp & 3)) * 32 + lane : warp * 32 + lane;
    double uv[kPerMax];
    auto load = [&](int q) {
#pragma unroll
      for (int s = 0; s < kPerMax; ++s) {
        const int e = pi + s * kProd, r = e / kW, j = q * kW + e % kW;
        uv[s] = (e < 32 * kW && r < rows) ? __ldcg(&U[(row0 + 148 * r) * LD + j]) : 0.0;
      }
    };
    const double rcp17 = __drcp_rn(1.7);
    auto issue = [&](int q) {
      const int s = q % kStages;
      mb_tx(&mbar[s], rows * kW * 8);
      for (int r = 0; r < rows; ++r)
        bulk(stg + s * 32 * kW + r * kW, U + (row0 + 148 * r) * LD + q * kW, kW * 8, &mbar[s]);
    };
    double uv2[kPerMax];
    if (mode == 1 || mode == 5) load(0);
    if ((mode == 2 || mode == 4) && pi == 0)
      for (int q = 0; q < kStages && q < Q; ++q) issue(q);
    for (int q = 0; q < Q; ++q) {
      const int b = q & 1;
      double* rb = ring + b * kW * kS;
      if (q >= 2) nsync(3 + b, kAll);
      if (mode == 5) {
#pragma unroll
        for (int s2 = 0; s2 < kPerMax; ++s2) uv2[s2] = uv[s2];
        if (q + 1 < Q) load(q + 1);
      }
      if (mode == 2) mb_wait(&mbar[q % kStages], (q / kStages) & 1);
      if (mode == 4) {
        if (pi == 0) mb_wait(&mbar[q % kStages], (q / kStages) & 1);
        nsync(6, kProd);
        if (pi == 0 && q + kStages - 1 < Q && q >= 1) issue(q + kStages - 1);
      }
#pragma unroll
      for (int s = 0; s < kPerMax; ++s) {
        const int e = pi + s * kProd, r = e / kW, t = e % kW;
        if (e < 32 * kW && r < rows) {
          double u = mode == 0 ? 1e-3 * t : mode == 1 ? uv[s] : mode == 5 ? uv2[s] : stg[(q % kStages) * 32 * kW + r * kW + t];
          if (div == 1) {
            bool ok;
            u = ctdgpu::dadd(u, ctdgpu::ddiv_try(ctdgpu::dmul(u, 0.37), 1.7, &ok));
          } else if (div == 2) {
            bool ok;
            u = ctdgpu::dadd(u, ctdgpu::ddiv_rcp(ctdgpu::dmul(u, 0.37), 1.7, rcp17, &ok));
          }
          if (pair) rb[(t >> 1) * kP + 2 * r + (t & 1)] = ctdgpu::dmul(u, 1.0000001);
          else rb[t * kS + r] = ctdgpu::dmul(u, 1.0000001);
        }
      }
      narv(1 + b, kAll);
      if (mode == 1 && q + 1 < Q) load(q + 1);
      if (mode == 2) {
        nsync(5, kProd);
        if (pi == 0 && q + kStages < Q) issue(q + kStages);
      }
    }
  } else if (warp == 15) {
    double acc = 0.0;
    long long tc = 0, t16 = 0;
    for (int q = 0; q < Q; ++q) {
      const int b = q & 1;
      nsync(1 + b, kAll);
      const long long c0 = clock64();
      if (pair == 2) {
        // split: first 16 steps, then the remaining 48
        const double* p = ring + b * kW * kS + lane;
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = p[k * kS];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = ctdgpu::dadd(acc, v[k]);
        const long long c1 = clock64();
        t16 += c1 - c0;
#pragma unroll
        for (int h = 1; h < 4; ++h) {
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = p[(h * 16 + k) * kS];
#pragma unroll
          for (int k = 0; k < 16; ++k) acc = ctdgpu::dadd(acc, v[k]);
        }
      } else
      acc = pair ? lane_chain2(ring + b * kW * kS, lane, acc) : lane_chain(ring + b * kW * kS, lane, acc);
      tc += clock64() - c0;
      if (q + 2 < Q) narv(3 + b, kAll);
    }
    out[blockIdx.x * 32 + lane] = acc;
    if (blockIdx.x == 0 && lane == 0) { cyc[1] = tc; cyc[2] = t16; }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

// Chain warp alone on a fixed ring while 15 "noise" warps run one kind of
// work until it finishes: which SM-shared resource slows the chain?
__global__ void __launch_bounds__(kT, 1) k_noise(const double* G, int Q, int noise, long long* cyc, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;
  double* scratch = sm + 2 * kW * kS;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  for (int i = threadIdx.x; i < 2 * kW * kS + 4096; i += kT) sm[i] = 1e-3 * (i & 7);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 15) {
    long long t0 = clock64();
    double acc = 0.0;
    for (int q = 0; q < Q; ++q) acc = lane_chain(ring + (q & 1) * kW * kS, lane, acc);
    long long t1 = clock64();
    if (lane == 0) done = 1;
    out[blockIdx.x * 32 + lane] = acc;
    if (blockIdx.x == 0 && lane == 0) cyc[0] = t1 - t0;
  } else if (noise) {
    double a0 = lane, a1 = 1, a2 = 2, a3 = 3;
    long long it = 0;
    const double* gp = G + ((long long)blockIdx.x * 15 + warp) * 4096;
    while (!done) {
#pragma unroll 4
      for (int k = 0; k < 64; ++k) {
        if (noise == 1) a0 += __ldcg(gp + ((k * 32 + lane + it) & 4095));
        else if (noise == 2) { scratch[(k * 32 + lane) & 4095] = a0; a0 += scratch[(k * 32 + lane + 7) & 4095]; }
        else if (noise == 3) { a0 = __fma_rn(a0, 1.0000001, 1e-9); a1 = __fma_rn(a1, 1.0000001, 1e-9); a2 = __fma_rn(a2, 1.0000001, 1e-9); a3 = __fma_rn(a3, 1.0000001, 1e-9); }
        else if (noise == 4) { a0 += (double)(it * k); }
        else if (noise == 5) { __nanosleep(100); }
        else if (noise == 6) { double v = __ldcg(gp + ((k * 32 + lane + it) & 4095)); ring[((k + it) & 63) * kS + (warp & 31)] = v; }
        else if (noise == 7) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a0)); a0 = r + 1.0; }
        else if (noise == 8) { ring[((k + it) & 63) * kS + (warp & 31)] = a0; }
        else if (noise == 9) { scratch[((k + it) & 63) * kS + (warp & 31)] = a0; }
      }
      ++it;
    }
    out[4736 + blockIdx.x * 512 + threadIdx.x] = a0 + a1 + a2 + a3;
  }
}

// Ring v2: NS slots of W steps; the chain warp copies a whole slot into
// registers and frees it before running its adds.
template <int W, int NS>
__global__ void __launch_bounds__(kT, 1) k_ring2(double* U, long long LD, int rows, int Q2, int ldg,
                                                  long long* cyc, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;  // [NS][W][kS]
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row0 = blockIdx.x;
  const double rcp17 = __drcp_rn(1.7);
  long long t0 = clock64();
  if (warp < 15) {
    const int pi = threadIdx.x;
    constexpr int kP2 = (32 * W + 479) / 480;
    double uv[kP2];
    auto load = [&](int q) {
#pragma unroll
      for (int s = 0; s < kP2; ++s) {
        const int e = pi + s * 480, r = e / W, j = q * W + e % W;
        uv[s] = (e < 32 * W && r < rows && ldg) ? __ldcg(&U[(row0 + 148 * r) * LD + j]) : 1e-3 * j;
      }
    };
    load(0);
    for (int q = 0; q < Q2; ++q) {
      const int sl = q % NS;
      double* rb = ring + sl * W * kS;
      if (q >= NS) nsync(1 + NS + sl, kT);
#pragma unroll
      for (int s = 0; s < kP2; ++s) {
        const int e = pi + s * 480, r = e / W, t = e % W;
        if (e < 32 * W && r < rows) {
          bool ok;
          double u = ctdgpu::dadd(uv[s], ctdgpu::ddiv_rcp(ctdgpu::dmul(uv[s], 0.37), 1.7, rcp17, &ok));
          if (ldg == 2) U[(row0 + 148 * r) * LD + q * W + t] = u;
          rb[t * kS + r] = ctdgpu::dmul(u, 1.0000001);
        }
      }
      narv(1 + sl, kT);
      if (q + 1 < Q2) load(q + 1);
    }
  } else {
    double acc = 0.0;
    for (int q = 0; q < Q2; ++q) {
      const int sl = q % NS;
      nsync(1 + sl, kT);
      const double* p = ring + sl * W * kS + lane;
#pragma unroll
      for (int k0 = 0; k0 < W; k0 += 16) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = p[(k0 + k) * kS];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = ctdgpu::dadd(acc, v[k]);
      }
      if (q + NS < Q2) narv(1 + NS + sl, kT);
    }
    out[blockIdx.x * 32 + lane] = acc;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

template <int W, int NS>
void run_ring2(double* U, long long LD, int rows, int K, long long* c, double* o) {
  const int smem = NS * W * kS * 8;
  cudaFuncSetAttribute(k_ring2<W, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ldg : {0, 1, 2}) {
    cudaMemset(c, 0, 24);
    k_ring2<W, NS><<<148, kT, smem>>>(U, LD, rows, K / W, ldg, c, o);
    cudaError_t e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("ring2 W=%d slots=%d ldg=%d: %.1f cycles/step %s\n", W, NS, ldg, (double)h / K, e ? cudaGetErrorString(e) : "");
  }
}

// Ring v3: producers stage U segments with cp.async.cg (16 B) DEPTH chunks
// ahead into a shared-memory stage ring, then compute from shared memory.
template <int W, int NS, int DEPTH>
__global__ void __launch_bounds__(kT, 1) k_ring3(double* U, long long LD, int rows, int Q2, long long* cyc, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;                   // [NS][W][kS]
  double* stage = sm + NS * W * kS;    // [DEPTH+1][32][W]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row0 = blockIdx.x;
  const double rcp17 = __drcp_rn(1.7);
  __syncthreads();
  long long t0 = clock64();
  if (warp < 15) {
    const int pi = threadIdx.x;
    // copy units: rows x (W/2) 16-byte pieces
    auto issue = [&](int q) {
      double* st = stage + (q % (DEPTH + 1)) * 32 * W;
      const int units = rows * (W / 2);
      for (int u = pi; u < units; u += 480) {
        const int r = u / (W / 2), c = (u % (W / 2)) * 2;
        const double* src = U + (row0 + 148 * r) * LD + q * W + c;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(st + r * W + c)), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int q = 0; q < DEPTH && q < Q2; ++q) issue(q);
    constexpr int kP2 = (32 * W + 479) / 480;
    for (int q = 0; q < Q2; ++q) {
      const int sl = q % NS;
      double* rb = ring + sl * W * kS;
      if (q + DEPTH < Q2) issue(q + DEPTH);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH) : "memory");
      nsync(9, 480);  // everyone's copies for chunk q landed
      const double* st = stage + (q % (DEPTH + 1)) * 32 * W;
      if (q >= NS) nsync(1 + NS + sl, kT);
#pragma unroll
      for (int s = 0; s < kP2; ++s) {
        const int e = pi + s * 480, r = e / W, t = e % W;
        if (e < 32 * W && r < rows) {
          bool ok;
          const double uv = st[r * W + t];
          double u = ctdgpu::dadd(uv, ctdgpu::ddiv_rcp(ctdgpu::dmul(uv, 0.37), 1.7, rcp17, &ok));
          rb[t * kS + r] = ctdgpu::dmul(u, 1.0000001);
        }
      }
      narv(1 + sl, kT);
      nsync(10, 480);  // stage slot free before it is refilled
    }
  } else {
    double acc = 0.0;
    for (int q = 0; q < Q2; ++q) {
      const int sl = q % NS;
      nsync(1 + sl, kT);
      const double* p = ring + sl * W * kS + lane;
#pragma unroll
      for (int k0 = 0; k0 < W; k0 += 16) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = p[(k0 + k) * kS];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = ctdgpu::dadd(acc, v[k]);
      }
      if (q + NS < Q2) narv(1 + NS + sl, kT);
    }
    out[blockIdx.x * 32 + lane] = acc;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = clock64() - t0;
}

template <int W, int NS, int DEPTH>
void run_ring3(double* U, long long LD, int rows, int K, long long* c, double* o) {
  const int smem = (NS * W * kS + (DEPTH + 1) * 32 * W) * 8;
  cudaFuncSetAttribute(k_ring3<W, NS, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(c, 0, 24);
  k_ring3<W, NS, DEPTH><<<148, kT, smem>>>(U, LD, rows, K / W, c, o);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("ring3 (cp.async) W=%d slots=%d depth=%d: %.1f cycles/step %s\n", W, NS, DEPTH, (double)h / K,
         e ? cudaGetErrorString(e) : "");
}

int main() {
  const int K = 1280, rows = 9;
  const long long LD = 1280;
  const int Q = K / kW;
  double *U, *o;
  long long* c;
  cudaMalloc(&U, (size_t)148 * rows * LD * 8 + 4096);
  cudaMemset(U, 0, (size_t)148 * rows * LD * 8);
  cudaMalloc(&o, 148 * 32 * 8);
  cudaMalloc(&c, 64);
  const int smem = (2 * kW * kS + kStages * 32 * kW) * 8;
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"regs", "ldcg", "bulk", "chain-only", "bulk-1wait", "ldcg-early"};
  {
    double* G;
    cudaMalloc(&G, (size_t)148 * 15 * 4096 * 8);
    cudaMemset(G, 0, (size_t)148 * 15 * 4096 * 8);
    double* o2;
    cudaMalloc(&o2, (4736 + 148 * 512) * 8);
    const char* nn[] = {"none", "LDG.cg", "LDS/STS", "DFMA", "I2F", "nanosleep", "LDG+STSring", "MUFU.rcp64", "STSring", "STS-conflict"};
    cudaFuncSetAttribute(k_noise, cudaFuncAttributeMaxDynamicSharedMemorySize, (2 * kW * kS + 4096) * 8);
    for (int noise = 0; noise < 10; ++noise) {
      k_noise<<<148, kT, (2 * kW * kS + 4096) * 8>>>(G, 64, noise, c, o2);
      cudaError_t e = cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("noise=%-9s chain %.2f cycles/step %s\n", nn[noise], (double)h / (64 * kW), e ? cudaGetErrorString(e) : "");
    }
  }
  run_ring2<64, 3>(U, LD, rows, K, c, o);
  run_ring2<128, 2>(U, LD, rows, K, c, o);
  run_ring3<64, 3, 2>(U, LD, rows, K, c, o);
  run_ring3<64, 3, 4>(U, LD, rows, K, c, o);
  run_ring3<128, 2, 2>(U, LD, rows, K, c, o);
  for (int first : {0})
  for (int pair : {2})
  for (int avoid : {0})
  for (int grid : {148})
    for (int mode : {0, 1, 5})
      for (int div : {0, 2}) {
        if (mode == 3 && div) continue;
        cudaMemset(c, 0, 24);
        k_ring<<<grid, kT, smem>>>(U, LD, rows, Q, mode, div, avoid, pair, first, c, o);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[3];
        cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
        printf("   first16: %.1f cycles/step, rest48: %.1f cycles/step\n", (double)h[2] / (Q * 16), (double)(h[1] - h[2]) / (Q * 48));
        printf("first=%d pair=%d avoid=%d grid=%3d mode=%-10s div=%d: %.1f cycles/step total, chain %.1f cycles/step  %s\n", first, pair, avoid, grid, names[mode], div,
               (double)h[0] / (Q * kW), (double)h[1] / (Q * kW), e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
