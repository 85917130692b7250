// Cost of cooperative_groups grid.sync() and cluster.sync() on the B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void gs(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
__global__ void __cluster_dims__(16, 1, 1) cs(int iters, int* out) {
  cg::cluster_group c = cg::this_cluster();
  for (int i = 0; i < iters; ++i) c.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
int main() {
  int* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {8, 14, 36, 71, 141, 148}) {
    int iters = 2000;
    void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)gs, grid, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)gs, grid, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  grid %3d: %.3f us per sync (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  {
    int iters = 2000;
    cs<<<16, 256>>>(iters, d); cudaDeviceSynchronize();
    cudaEventRecord(a); cs<<<16, 256>>>(iters, d); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cluster.sync 16 CTAs: %.3f us per sync (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
