// Micro-benchmarks for the filter's critical path on the B200:
//   dependent DADD latency, LDS->DADD chain, grid-barrier round trip.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cstdio>
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
