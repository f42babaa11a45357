// Feasibility + latency probe: cooperative launch with thread-block clusters
// (one CTA per SM, 512 threads, ~140 KB dynamic smem), cluster barrier and
// DSMEM round-trip latency.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k(long long* out, int iters) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  if (threadIdx.x == 0) sm[0] = (double)rank;
  cl.sync();
  // cluster barrier latency
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  // DSMEM dependent load latency (thread 0 of each CTA reads rank 0's smem)
  double* remote = cl.map_shared_rank(sm, 0);
  double acc = 0;
  long long t2 = clock64();
  if (threadIdx.x == 0)
    for (int i = 0; i < iters; ++i) acc += remote[(int)acc & 0];
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = (t1 - t0) / iters;
    out[blockIdx.x * 4 + 1] = (t3 - t2) / iters;
    out[blockIdx.x * 4 + 2] = (long long)acc;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x * 4 + 3] = smid;
  }
  cl.sync();
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = 140 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int cs : {2, 4, 8, 16}) {
    if (cs == 16) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    int grid = (sms / cs) * cs;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int nclusters = 0;
    cudaLaunchConfig_t q = cfg;
    q.numAttrs = 1;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclusters, k, &q);
    long long* d;
    cudaMalloc(&d, grid * 4 * sizeof(long long));
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, 1000);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("cluster %2d grid %3d maxActiveClusters %d (%s) launch=%s sync=%s\n", cs, grid, nclusters,
           cudaGetErrorString(oe), cudaGetErrorString(e), cudaGetErrorString(e2));
    if (e == cudaSuccess && e2 == cudaSuccess) {
      long long h[4 * 160];
      cudaMemcpy(h, d, grid * 4 * sizeof(long long), cudaMemcpyDeviceToHost);
      long long bmin = 1 << 30, bmax = 0, lmin = 1 << 30, lmax = 0;
      for (int b = 0; b < grid; ++b) {
        bmin = h[4 * b] < bmin ? h[4 * b] : bmin;
        bmax = h[4 * b] > bmax ? h[4 * b] : bmax;
        lmin = h[4 * b + 1] < lmin ? h[4 * b + 1] : lmin;
        lmax = h[4 * b + 1] > lmax ? h[4 * b + 1] : lmax;
      }
      printf("   cluster.sync %lld..%lld cycles, DSMEM load %lld..%lld cycles\n", bmin, bmax, lmin, lmax);
    }
    cudaGetLastError();
    cudaFree(d);
  }
  return 0;
}
