// Times device allocation growth: cudaMalloc vs cudaMallocAsync (default pool,
// release threshold max) for N chunks of S bytes, with a small interleaved
// temporary allocation like a CTD-D step's.
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
static double ms_since(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}
int main(int argc, char** argv) {
  const size_t S = (size_t)(argc > 1 ? atol(argv[1]) : 1024) << 20;
  const int N = argc > 2 ? atoi(argv[2]) : 40;
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  std::vector<void*> keep;
  double mx = 0, tot = 0;
  for (int i = 0; i < N; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    void* p;
    cudaMallocAsync(&p, S, st);
    cudaMemsetAsync(p, 0, 4096, st);
    cudaStreamSynchronize(st);
    double m = ms_since(t0);
    mx = m > mx ? m : mx; tot += m;
    keep.push_back(p);
  }
  printf("mallocAsync %zu MB x %d: mean %.2f ms max %.2f ms\n", S >> 20, N, tot / N, mx);
  for (void* p : keep) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  uint64_t zero = 0;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &zero);
  cudaMemPoolTrimTo(pool, 0);
  keep.clear(); mx = 0; tot = 0;
  for (int i = 0; i < N; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    void* p;
    cudaMalloc(&p, S);
    cudaMemset(p, 0, 4096);
    cudaDeviceSynchronize();
    double m = ms_since(t0);
    mx = m > mx ? m : mx; tot += m;
    keep.push_back(p);
  }
  printf("cudaMalloc %zu MB x %d: mean %.2f ms max %.2f ms\n", S >> 20, N, tot / N, mx);
  for (void* p : keep) cudaFree(p);
  return 0;
}
