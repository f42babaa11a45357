// cudaMalloc 1 GB chunks then a full-chunk memset: malloc vs first-touch time.
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 60;
  const size_t S = size_t(1) << 30;
  void* scratch;
  cudaMalloc(&scratch, S);
  std::vector<void*> keep;
  double mx_m = 0, mx_s = 0, mx_r = 0;
  for (int i = 0; i < N; ++i) {
    auto t0 = clk::now();
    void* p;
    cudaMalloc(&p, S);
    auto t1 = clk::now();
    cudaMemset(p, 1, S);
    cudaDeviceSynchronize();
    auto t2 = clk::now();
    cudaMemcpy(p, scratch, S / 4, cudaMemcpyDeviceToDevice);
    cudaDeviceSynchronize();
    auto t3 = clk::now();
    keep.push_back(p);
    printf("%d malloc %.2f memset %.2f reuse-copy %.2f ms\n", i, ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  return 0;
}
