// Micro-benchmark of warp_grid_sum (the filter's exact residual sum) on a
// synthetic term vector: stage times from CTA 0, checked against the
// sequential sum.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_p3 tools/ubench_p3.cu
#include <cstdio>
#include <vector>

__device__ unsigned long long g_gt[512];
#define CTD_WGS_GT g_gt
#include "../paper_1710_03608_b200/csrc/gridsum.cuh"

using namespace ctdgpu;

struct Terms {
  const double* t;
  __device__ double operator()(long long i) const { return __ldcg(&t[i]); }
  template <int N>
  __device__ void strided(long long i0, long long step, long long n, double (&out)[N]) const {
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = (i0 + k * step < n) ? __ldcg(&t[i0 + k * step]) : 0.0;
  }
  template <int N>
  __device__ void batch(long long b0, long long b1, double (&out)[N]) const {
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = (b0 + k < b1) ? __ldcg(&t[b0 + k]) : 0.0;
  }
};

__global__ void __launch_bounds__(512, 1) k_p3(const double* t, long long nt, int reps, SliceLoc* loc, SliceSum* ps,
                                               SliceDirect* pd, unsigned* sflag, long long* tp, double* out, unsigned* bar) {
  __shared__ WarpSumSmem W;
  extern __shared__ __align__(16) double dyn[];
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 32) {
      bool bad = false;
      SliceDirect* sd = reinterpret_cast<SliceDirect*>(dyn);
      const double v = warp_grid_sum(Terms{t}, nt, (unsigned)(r + 1), loc, ps, pd, sflag, W, sd,
                                     reinterpret_cast<int*>(sd + kMaxDirectsTotal), &bad, tp + 16 * r);
      if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = v;
        out[1] = bad;
      }
    }
    grid_barrier(bar, gridDim.x);
  }
}

__global__ void k_pieces(const double* t, long long* cyc, double* out) {
  const int lane = threadIdx.x & 31;
  // 1) warp_seg_excl x100 (dependent through the carry)
  Seg v{lane % 7 == 0, {lane, lane + 1}};
  long long t0 = clock64();
  for (int r = 0; r < 100; ++r) {
    Seg tot;
    Seg e = warp_seg_excl(v, &tot);
    v.m.a0 = e.m.a0 ^ tot.m.a1;
  }
  long long t1 = clock64();
  // 2) warp_excl<int> x100
  int iv = lane;
  for (int r = 0; r < 100; ++r) {
    int tot;
    iv = warp_excl<int>(iv & 7, &tot) + (tot & 1);
  }
  long long t2 = clock64();
  // 3) classify 10 elements x10
  double P = 1.0;
  Mono agg = mono_id();
  const double mg = seq_margin(10000);
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const double x = t[(lane * 10 + k + r) & 1023];
      const double Pc = P + x;
      int e;
      Mono m;
      const int c = seq_classify(false, P, Pc, x, mg, &e, &m);
      if (c == CLS_REG) agg = mono_cat(agg, m);
      P = Pc;
    }
  }
  long long t3 = clock64();
  if (lane == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
  out[lane] = v.m.a0 + iv + agg.a0 + P;
}

template <int KC, int KG>
__global__ void __launch_bounds__(512, 1) k_block(const double* t, long long nt, long long* cyc, double* out) {
  __shared__ SeqSumSmem S;
  extern __shared__ __align__(16) double tb[];
  bool bad = false;
  __syncthreads();
  long long t0 = clock64();
  double v = 0;
  for (int r = 0; r < 4; ++r) v = block_exact_sum_ilp<KC, KG>(Terms{t}, nt, S, &bad, [] {}, tb, blockIdx.x == 0 ? cyc + 8 : nullptr);
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 4;
    out[0] = v;
    out[1] = bad;
  }
}

template <int KC, int KG>
void run_block(const double* t, long long nt, double ref, long long* c, double* o) {
  const int sm = 16 * 32 * (KC + 1) * 8;
  cudaFuncSetAttribute(k_block<KC, KG>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k_block<KC, KG><<<148, 512, sm>>>(t, nt, c, o);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  double ho[2];
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
  printf("block_exact_sum_ilp<%d,%d> n=%lld: %lld cycles exact=%d bad=%g %s\n", KC, KG, nt, h, ho[0] == ref, ho[1],
         e ? cudaGetErrorString(e) : "");
  long long st[10];
  cudaMemcpy(st, c + 8, 80, cudaMemcpyDeviceToHost);
  printf("   stages:");
  for (int k = 1; k < 10; ++k) printf(" %lld", st[k] - st[k - 1]);
  printf("\n");
}

int main() {
  const long long nt = 10000;
  std::vector<double> h(nt);
  unsigned long long s = 7;
  for (auto& v : h) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = (double)(s >> 11) * 0x1.0p-53 * 1e-3;
  }
  h[0] = 1.5;
  double ref = 0.0;
  for (double v : h) ref += v;
  double *t, *o;
  cudaMalloc(&t, nt * 8);
  cudaMemcpy(t, h.data(), nt * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 16);
  {
    long long* c;
    cudaMalloc(&c, 64);
    double* ob;
    cudaMalloc(&ob, 32 * 8);
    k_pieces<<<1, 32>>>(t, c, ob);
    cudaDeviceSynchronize();
    long long hc[3];
    cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
    printf("warp_seg_excl: %.0f cycles, warp_excl<int>: %.0f cycles, classify: %.0f cycles/element\n", hc[0] / 100.0,
           hc[1] / 100.0, hc[2] / 100.0);
  }
  {
    long long* c;
    cudaMalloc(&c, 256);
    run_block<24, 4>(t, nt, ref, c, o);
    run_block<24, 2>(t, nt, ref, c, o);
    run_block<12, 4>(t, nt, ref, c, o);
    run_block<8, 4>(t, nt, ref, c, o);
    run_block<24, 1>(t, nt, ref, c, o);
  }
  for (int grid : {148}) {
    SliceLoc* loc;
    SliceSum* ps;
    SliceDirect* pd;
    unsigned* sf;
    long long* tp;
    const int reps = 4;
    cudaMalloc(&loc, grid * sizeof(SliceLoc));
    cudaMemset(loc, 0, grid * sizeof(SliceLoc));
    cudaMalloc(&ps, grid * sizeof(SliceSum));
    cudaMalloc(&pd, (size_t)grid * kSliceDirects * sizeof(SliceDirect));
    cudaMalloc(&sf, (size_t)grid * kFlagStride * 4);
    cudaMemset(sf, 0, (size_t)grid * kFlagStride * 4);
    cudaMalloc(&tp, 16 * reps * 8);
    cudaMemset(tp, 0, 16 * reps * 8);
    const int smem = kMaxDirectsTotal * (sizeof(SliceDirect) + 4);
    cudaFuncSetAttribute(k_p3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned* bar;
    cudaMalloc(&bar, 64);
    cudaMemset(bar, 0, 64);
    void* args[] = {&t, (void*)&nt, (void*)&reps, &loc, &ps, &pd, &sf, &tp, &o, &bar};
    cudaLaunchCooperativeKernel((void*)k_p3, grid, 512, args, smem, 0);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[2];
    cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
    std::vector<long long> ht(16 * reps);
    cudaMemcpy(ht.data(), tp, ht.size() * 8, cudaMemcpyDeviceToHost);
    printf("grid=%d exact=%d bad=%g %s\n", grid, ho[0] == ref, ho[1], e ? cudaGetErrorString(e) : "");
    {
      unsigned long long g[512];
      cudaMemcpyFromSymbol(g, g_gt, sizeof(g));
      unsigned long long mn = ~0ull, mx = 0, mn2 = ~0ull, mx2 = 0;
      int amx = 0;
      for (int i = 0; i < grid; ++i) {
        if (g[i] < mn) mn = g[i];
        if (g[i] > mx) { mx = g[i]; amx = i; }
        if (g[256 + i] < mn2) mn2 = g[256 + i];
        if (g[256 + i] > mx2) mx2 = g[256 + i];
      }
      printf("  last rep: publish spread %llu ns (latest CTA %d), first poll done %llu ns after last publish, poll-done spread %llu ns\n",
             mx - mn, amx, mn2 - mx, mx2 - mn2);
    }
    for (int r = 0; r < reps; ++r) {
      printf("  rep %d:", r);
      for (int k = 1; k <= 7; ++k)
        if (ht[16 * r + k] && ht[16 * r + k - 1]) printf(" %lld", ht[16 * r + k] - ht[16 * r + k - 1]);
      printf(" directs=%lld\n", ht[16 * r + 9]);
    }
  }
  return 0;
}
