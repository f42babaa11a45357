// Which SMs share a die: round-trip latency of a flag ping-pong between the
// CTA on SM 0 and the CTA on each other SM (one CTA per SM, 148 CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_die ubench_die.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k(unsigned* flags, int* smids, long long* rtt, int iters) {
  __shared__ int partner;
  unsigned sm;
  asm("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) smids[blockIdx.x] = sm;
  // CTA 0 pings CTA b (b = 1..grid-1) one after another; flags[2b] ping, flags[2b+1] pong
  if (threadIdx.x != 0) return;
  if (blockIdx.x == 0) {
    for (int b = 1; b < gridDim.x; ++b) {
      long long t0 = clock64();
      for (int i = 1; i <= iters; ++i) {
        st_rel(&flags[64 * b], i);
        while (ld_acq(&flags[64 * b + 32]) != (unsigned)i) {
        }
      }
      rtt[b] = (clock64() - t0) / iters;
    }
  } else {
    for (int i = 1; i <= iters; ++i) {
      while (ld_acq(&flags[64 * blockIdx.x]) != (unsigned)i) {
      }
      st_rel(&flags[64 * blockIdx.x + 32], i);
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* flags;
  int* smids;
  long long* rtt;
  cudaMalloc(&flags, 64 * sms * sizeof(unsigned) * 2);
  cudaMemset(flags, 0, 64 * sms * sizeof(unsigned) * 2);
  cudaMalloc(&smids, sms * sizeof(int));
  cudaMalloc(&rtt, sms * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  void* args[] = {&flags, &smids, &rtt, nullptr};
  int iters = 200;
  args[3] = &iters;
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k, sms, 512, args, 150 * 1024, 0);
  cudaDeviceSynchronize();
  printf("launch %s\n", cudaGetErrorString(e));
  int hs[256];
  long long hr[256];
  cudaMemcpy(hs, smids, sms * sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(hr, rtt, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("cta0 on sm %d\n", hs[0]);
  for (int b = 1; b < sms; ++b) printf("cta %3d sm %3d rtt %lld\n", b, hs[b], hr[b]);
  return 0;
}
