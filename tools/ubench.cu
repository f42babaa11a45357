// Micro-benchmarks for the filter's critical path on the B200:
//   dependent DADD latency, LDS->DADD chain, grid-barrier round trip.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_dadd(double* out, long long* cyc, int n) {
  double a = out[0], b = out[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  out[2] = a;
  cyc[0] = t1 - t0;
}

__global__ void k_dmul_dadd(double* out, long long* cyc, int n) {
  double a = out[0], b = out[1], c = out[3];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, __dmul_rn(b, c));
  long long t1 = clock64();
  out[2] = a;
  cyc[0] = t1 - t0;
}

#include "../paper_1710_03608_b200/csrc/common.cuh"

__global__ void k_barrier(unsigned* bar, long long* cyc, int iters) {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) ctdgpu::grid_barrier(bar, gridDim.x);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}

#include "../paper_1710_03608_b200/csrc/seqsum.cuh"

__global__ void __launch_bounds__(512) k_xsum(const double* x, int n, double* out, long long* cyc) {
  __shared__ ctdgpu::SeqSumSmem S;
  extern __shared__ double d[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = x[i];
  __syncthreads();
  long long t0 = clock64();
  bool bad = false;
  const double* dd = d;
  auto get = [dd](long long i) { return dd[i]; };
  double r = ctdgpu::block_exact_sum(get, n, S, &bad, cyc + 1);
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = r;
    out[1] = bad;
    cyc[0] = t1 - t0;
  }
}

__global__ void k_elem(const double* x, long long* cyc, double* out) {
  double a = x[0];
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) a = floor(a * 1.0000001 + 0.5);
  long long t1 = clock64();
  long long s = 0;
  double b = x[1];
  for (int i = 0; i < 1024; ++i) { s += (long long)b; b = b + (double)(s & 1); }
  long long t2 = clock64();
  ctdgpu::Mono agg = ctdgpu::mono_id();
  for (int i = 0; i < 1024; ++i) {
    ctdgpu::Mono m;
    ctdgpu::seq_mono(x[i & 7] * 1e-3, 10, &m);
    agg = ctdgpu::mono_cat(agg, m);
  }
  long long t3 = clock64();
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
  out[0] = a + b + s + agg.a0;
}

// Per-thread chunk loops of block_exact_sum in isolation (512 threads, n in smem).
__global__ void __launch_bounds__(512) k_paths(const double* x, int n, long long* cyc, double* out) {
  extern __shared__ double d[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = x[i];
  __syncthreads();
  const int per = (n + 511) / 512;
  const int b0 = min((int)threadIdx.x * per, n), b1 = min(b0 + per, n);
  __syncthreads();
  long long t0 = clock64();
  ctdgpu::Mono agg = ctdgpu::mono_id();
  for (int i = b0; i < b1; ++i) {
    ctdgpu::Mono m;
    ctdgpu::seq_mono(d[i], 12, &m);
    agg = ctdgpu::mono_cat(agg, m);
  }
  __syncthreads();
  long long t1 = clock64();
  double P = b0 * 0.5;
  int cls = 0;
  for (int i = b0; i < b1; ++i) {
    const double Pc = P + d[i];
    int e;
    ctdgpu::Mono m;
    cls += ctdgpu::seq_classify(i == 0, P, Pc, d[i], 1e-11, &e, &m);
    agg = ctdgpu::mono_cat(agg, m);
    P = Pc;
  }
  __syncthreads();
  long long t2 = clock64();
  double s = 0;
  for (int i = b0; i < b1; ++i) s += d[i];
  __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
  out[threadIdx.x] = agg.a0 + cls + s;
}

__global__ void __launch_bounds__(512) k_scans(long long* cyc) {
  __shared__ double dsh[33];
  __shared__ ctdgpu::Seg ssh[33];
  __shared__ int ish[33];
  double v = threadIdx.x * 0.5;
  long long t0 = clock64();
  double tot;
  double a = ctdgpu::block_excl_sum<double>(v, dsh, &tot);
  long long t1 = clock64();
  ctdgpu::Seg s{(int)(threadIdx.x % 7 == 0), {threadIdx.x, threadIdx.x + 1}};
  ctdgpu::Seg c = ctdgpu::block_seg_excl(s, ssh, nullptr);
  long long t2 = clock64();
  int nt;
  int b = ctdgpu::block_excl_sum<int>((int)threadIdx.x & 3, ish, &nt);
  long long t3 = clock64();
  __syncthreads();
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = (long long)(a + c.m.a0 + b);
  }
}

// window_chain as in the filter: lanes write 256 products, lane 0 chains.
constexpr int kWinB = 256;
__device__ __forceinline__ double window_chain_b(const double* wwin, int lane, int cnt, double acc) {
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
        for (int q = 0; q < 32; ++q) acc = __dadd_rn(acc, v[q]);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < mm) acc = __dadd_rn(acc, v[q]);
      }
    }
  }
  __syncwarp();
  return acc;
}

__global__ void k_wchain(const double* x, int reps, long long* cyc, double* out) {
  extern __shared__ __align__(16) double wsm[];
  double* wwin = wsm + (threadIdx.x >> 5) * kWinB;
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int s = 0; s < kWinB / 32; ++s) wwin[32 * s + lane] = x[(32 * s + lane + r) & 1023] * 1.0000001;
    acc = window_chain_b(wwin, lane, kWinB, acc);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// The filter's P1 row loop for one row (fused U update + products + chain).
__global__ void k_p1row(double* U, const double* g, const double* yv, int K, double delta, int upd,
                        long long* cyc, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* vA = sm;
  double* vB = sm + 4096;
  double* wwin = sm + 8192 + (threadIdx.x >> 5) * kWinB;
  const int lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    vA[j] = g[j];
    vB[j] = yv[j];
  }
  __syncthreads();
  const int i = threadIdx.x >> 5;  // row per warp
  double* urow = U + (long long)i * K;
  const double yi = yv[i];
  const int Ko = K;
  long long t0 = clock64();
  double acc = 0.0;
  double u[kWinB / 32];
#pragma unroll
  for (int s = 0; s < kWinB / 32; ++s) {
    const int j = 32 * s + lane;
    u[s] = j < K ? __ldcg(&urow[j]) : 0.0;
  }
  for (int j0 = 0; j0 < K; j0 += kWinB) {
    if (upd == 3) {
      double unv[kWinB / 32];
      bool wok = true;
#pragma unroll
      for (int s = 0; s < kWinB / 32; ++s) {
        const int j = j0 + 32 * s + lane;
        bool ok;
        const double qd = ctdgpu::ddiv_try(__dmul_rn(yi, vB[j]), delta, &ok);
        wok &= ok;
        unv[s] = __dadd_rn(u[s], qd);
      }
      if (__any_sync(0xffffffffu, !wok) && !wok) {
#pragma unroll
        for (int s = 0; s < kWinB / 32; ++s) {
          const int j = j0 + 32 * s + lane;
          unv[s] = __dadd_rn(u[s], __ddiv_rn(__dmul_rn(yi, vB[j]), delta));
        }
      }
#pragma unroll
      for (int s = 0; s < kWinB / 32; ++s) {
        const int j = j0 + 32 * s + lane;
        double p = 0.0;
        if (j < K) {
          urow[j] = unv[s];
          p = __dmul_rn(unv[s], vA[j]);
        }
        wwin[32 * s + lane] = p;
      }
    } else
#pragma unroll
    for (int s = 0; s < kWinB / 32; ++s) {
      const int j = j0 + 32 * s + lane;
      double p = 0.0;
      if (j < K) {
        double un = u[s];
        if (upd) {
          if (i < Ko && j < Ko)
            un = __dadd_rn(u[s], upd == 2 ? __ddiv_rn(__dmul_rn(yi, vB[j]), delta)
                                          : ctdgpu::ddiv_exact(__dmul_rn(yi, vB[j]), delta));
          urow[j] = un;
        }
        p = __dmul_rn(un, vA[j]);
      }
      wwin[32 * s + lane] = p;
    }
    const int jn = j0 + kWinB;
    if (jn < K) {
#pragma unroll
      for (int s = 0; s < kWinB / 32; ++s) {
        const int j = jn + 32 * s + lane;
        u[s] = j < K ? __ldcg(&urow[j]) : 0.0;
      }
    }
    acc = window_chain_b(wwin, lane, min(kWinB, K - j0), acc);
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[i] = acc;
    if (i == 0) cyc[0] = t1 - t0;
  }
}

// ddiv_exact vs __ddiv_rn on pseudo-random operands of several kinds.
__global__ void k_divcheck(unsigned long long seed, long long n, unsigned long long* bad, double* ex) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long nb = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned long long s = seed ^ (i * 0x9E3779B97F4A7C15ull);
    auto nx = [&]() {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      return s;
    };
    const int kind = (int)(i & 7);
    double a, b;
    if (kind < 3) {  // random mantissas, moderate exponents, random signs
      a = __longlong_as_double((long long)((nx() & 0x800FFFFFFFFFFFFFull) | ((unsigned long long)(1023 + (int)(nx() % 200) - 100) << 52)));
      b = __longlong_as_double((long long)((nx() & 0x800FFFFFFFFFFFFFull) | ((unsigned long long)(1023 + (int)(nx() % 200) - 100) << 52)));
    } else if (kind < 5) {  // products of small integers / integers: many exact & tie cases
      a = (double)(long long)(nx() % 2000001) - 1000000.0;
      b = (double)(long long)(nx() % 1999) + 1.0;
      a = a * (double)(1ll << (nx() % 40));
    } else if (kind == 5) {  // y_i*y_j / delta shapes from the filter
      const double y1 = ((double)(nx() >> 11) * 0x1.0p-53 - 0.5) * 1e-3, y2 = ((double)(nx() >> 11) * 0x1.0p-53 - 0.5) * 1e-2;
      a = __dmul_rn(y1, y2);
      b = (double)(nx() >> 11) * 0x1.0p-53 * 1e-4 + 1e-12;
    } else if (kind == 6) {  // quotients near powers of two
      b = (double)(nx() % 1000 + 1);
      a = b * (double)(1ll << (nx() % 30));
      a = __longlong_as_double(__double_as_longlong(a) + (long long)(nx() % 5) - 2);
    } else {  // extreme exponents (fallback paths)
      a = __longlong_as_double((long long)(nx() & 0xFFFFFFFFFFFFFFFull));
      b = __longlong_as_double((long long)(nx() & 0xFFFFFFFFFFFFFFFull));
      if (b == 0.0) b = 1.0;
    }
    const double q1 = ctdgpu::ddiv_exact(a, b), q2 = __ddiv_rn(a, b);
    bool ok;
    const double q3 = ctdgpu::ddiv_try(a, b, &ok);
    if (!ok) atomicAdd(bad + 1, 1ull);
    bool ok4;
    const double q4 = ctdgpu::ddiv_rcp(a, b, __drcp_rn(b), &ok4);
    if (!ok4) atomicAdd(bad + 2, 1ull);
    if (ok4 && __double_as_longlong(q4) != __double_as_longlong(q2)) atomicAdd(bad + 3, 1ull);
    if ((__double_as_longlong(q1) != __double_as_longlong(q2) && !(q1 != q1 && q2 != q2)) ||
        (ok && __double_as_longlong(q3) != __double_as_longlong(q2))) {
      ++nb;
      ex[0] = a;
      ex[1] = b;
    }
  }
  if (nb) atomicAdd(bad, nb);
}

// FP64 issue throughput: every thread runs 8 independent chains.
__global__ void k_fp64tp(double* out, long long* cyc, int n, int kind) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = out[k] + threadIdx.x;
  const double m = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = kind == 0 ? __fma_rn(a[k], m, c) : kind == 1 ? __dadd_rn(a[k], c) : __dmul_rn(a[k], m);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[16 + blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  unsigned* bar;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 64);
  cudaMalloc(&bar, 64);
  double h[4] = {1.0, 1e-9, 0, 3.0};
  cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
  long long cyc;
  const int n = 1 << 20;
  k_dadd<<<1, 1>>>(d, c, n);
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.2f cycles\n", (double)cyc / n);
  k_dmul_dadd<<<1, 1>>>(d, c, n);
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent DADD(DMUL): %.2f cycles\n", (double)cyc / n);
  {
    double* fo;
    cudaMalloc(&fo, (16 + 148 * 1024) * 8);
    cudaMemset(fo, 0, (16 + 148 * 1024) * 8);
    const char* kn[] = {"DFMA", "DADD", "DMUL"};
    for (int kind = 0; kind < 3; ++kind)
      for (int thr : {32, 128, 512, 1024}) {
        const int n = 4096;
        k_fp64tp<<<148, thr>>>(fo, c, n, kind);
        cudaDeviceSynchronize();
        long long st;
        cudaMemcpy(&st, c, 8, cudaMemcpyDeviceToHost);
        printf("%s throughput, %4d threads/SM: %.2f lane-ops/cycle/SM\n", kn[kind], thr, (double)thr * n * 8 / st);
      }
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {1, 16, 74, sms}) {
    cudaMemset(bar, 0, 64);
    const int it = 2000;
    void* args[] = {&bar, &c, (void*)&it};
    cudaLaunchCooperativeKernel((void*)k_barrier, g, 512, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("grid barrier (%d CTAs): %.0f cycles\n", g, (double)cyc / it);
  }
  {
    double* xx;
    double* oo;
    cudaMalloc(&xx, 1024 * 8);
    cudaMalloc(&oo, 148 * 512 * 8);
    cudaMemset(xx, 0, 1024 * 8);
    cudaFuncSetAttribute(k_wchain, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * kWinB * 8);
    for (int warps : {1, 4, 16}) {
      k_wchain<<<1, 32 * warps, warps * kWinB * 8>>>(xx, 64, c, oo);
      cudaDeviceSynchronize();
      long long st;
      cudaMemcpy(&st, c, 8, cudaMemcpyDeviceToHost);
      printf("window_chain: %d warps/SM: %.2f cycles/element\n", warps, (double)st / (64.0 * kWinB));
    }
  }
  {
    const int K = 1024;
    double *U, *g, *yv, *o;
    cudaMalloc(&U, (size_t)16 * K * 8);
    cudaMalloc(&g, K * 8);
    cudaMalloc(&yv, K * 8);
    cudaMalloc(&o, 64 * 8);
    {
      std::vector<double> h((size_t)16 * K);
      unsigned long long s = 99;
      for (auto& v : h) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        v = (double)(s >> 11) * 0x1.0p-53 - 0.5;
      }
      cudaMemcpy(U, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(g, h.data() + 7, K * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(yv, h.data() + 5000, K * 8, cudaMemcpyHostToDevice);
    }
    const int smem = (8192 + 16 * kWinB) * 8;
    cudaFuncSetAttribute(k_p1row, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int upd : {0, 1, 2, 3})
      for (int warps : {1, 4, 16}) {
        k_p1row<<<1, 32 * warps, smem>>>(U, g, yv, K, 0.37, upd, c, o);
        cudaDeviceSynchronize();
        long long st;
        cudaMemcpy(&st, c, 8, cudaMemcpyDeviceToHost);
        printf("P1 row (upd=%d, %d warps/SM): %.2f cycles/element\n", upd, warps, (double)st / K);
      }
  }
  {
    unsigned long long* nbad;
    double* ex;
    cudaMalloc(&nbad, 32);
    cudaMalloc(&ex, 16);
    cudaMemset(nbad, 0, 32);
    const long long N = 1ll << 30;
    k_divcheck<<<148 * 8, 256>>>(12345, N, nbad, ex);
    cudaDeviceSynchronize();
    unsigned long long hb2[4];
    double hex[2];
    cudaMemcpy(hb2, nbad, 32, cudaMemcpyDeviceToHost);
    cudaMemcpy(hex, ex, 16, cudaMemcpyDeviceToHost);
    const unsigned long long hb = hb2[0];
    printf("ddiv_exact/ddiv_try vs __ddiv_rn: %llu mismatches of %lld, try not-ok %llu (last a=%.17g b=%.17g)\n",
           hb, N, hb2[1], hb ? hex[0] : 0.0, hb ? hex[1] : 0.0);
    printf("ddiv_rcp vs __ddiv_rn: %llu mismatches among certified, not-ok %llu of %lld\n", hb2[3], hb2[2], N);
  }
  {
    k_elem<<<1, 1>>>(d, c, d + 4);
    cudaDeviceSynchronize();
    long long st[3];
    cudaMemcpy(st, c, 24, cudaMemcpyDeviceToHost);
    printf("per-element (1024 iters): floor-chain=%lld f2i-chain=%lld seq_mono+cat=%lld\n", st[0], st[1], st[2]);
  }
  {
    k_scans<<<1, 512>>>(c);
    cudaDeviceSynchronize();
    long long st[5];
    cudaMemcpy(st, c, 40, cudaMemcpyDeviceToHost);
    printf("scans: excl_sum<double>=%lld seg_excl=%lld excl_sum<int>=%lld syncthreads=%lld\n", st[0], st[1],
           st[2], st[3]);
  }
  {
    const int nmax = 16384;
    double* hx = new double[nmax];
    double* dx;
    double* dout;
    cudaMalloc(&dx, nmax * 8);
    cudaMalloc(&dout, 16);
    cudaFuncSetAttribute(k_xsum, cudaFuncAttributeMaxDynamicSharedMemorySize, nmax * 8);
    for (int kind = 0; kind < 3; ++kind) {
      unsigned long long s = 88172645463325252ull;
      for (int i = 0; i < nmax; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        const double u = (double)(s >> 11) * 0x1.0p-53;
        hx[i] = kind == 0 ? u : kind == 1 ? u * u * u * u * 1e6 : 1.0;
      }
      cudaMemcpy(dx, hx, nmax * 8, cudaMemcpyHostToDevice);
      if (kind == 0) {
        double* dout2;
        cudaMalloc(&dout2, 512 * 8);
        cudaFuncSetAttribute(k_paths, cudaFuncAttributeMaxDynamicSharedMemorySize, nmax * 8);
        for (int n : {900, 10000}) {
          k_paths<<<1, 512, nmax * 8>>>(dx, n, c, dout2);
          cudaDeviceSynchronize();
          long long st[3];
          cudaMemcpy(st, c, 24, cudaMemcpyDeviceToHost);
          printf("paths n=%d: fast-mono=%lld classify=%lld plain-sum=%lld\n", n, st[0], st[1], st[2]);
        }
      }
      for (int n : {900, 4000, 10000, 16000}) {
        k_xsum<<<1, 512, nmax * 8>>>(dx, n, dout, c);
        cudaDeviceSynchronize();
        double o[2];
        cudaMemcpy(o, dout, 16, cudaMemcpyDeviceToHost);
        long long st[8];
        cudaMemcpy(st, c, 64, cudaMemcpyDeviceToHost);
        cyc = st[0];
        printf("   stamps:");
        for (int k = 1; k < 7; ++k) printf(" %lld", st[k + 1] - st[k]);
        printf("\n");
        double ref = 0;
        for (int i = 0; i < n; ++i) ref += hx[i];
        printf("block_exact_sum kind=%d n=%d: %lld cycles exact=%d fallback=%d\n", kind, n, cyc,
               (int)(o[0] == ref), (int)o[1]);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
