#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(8, 1, 1) k(int* out) {
  cg::grid_group g = cg::this_grid();
  cg::cluster_group c = cg::this_cluster();
  if (threadIdx.x == 0) atomicAdd(out, 1);
  g.sync();
  __shared__ int v;
  if (threadIdx.x == 0) v = blockIdx.x;
  c.sync();
  int* rv = c.map_shared_rank(&v, (c.block_rank() + 1) % 8);
  if (threadIdx.x == 0) out[1 + blockIdx.x] = *rv;
  g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] += 1000;
}
int main() {
  int* d; cudaMalloc(&d, 4 * 200); cudaMemset(d, 0, 800);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = (sms / 8) * 8;
  void* args[] = {&d};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k, dim3(grid), dim3(256), args, 0, 0);
  printf("coop+__cluster_dims__ launch: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize(); printf("sync: %s\n", cudaGetErrorString(e));
  int h[200]; cudaMemcpy(h, d, 800, cudaMemcpyDeviceToHost);
  printf("count %d (expect %d+1000), blk1 saw %d (expect 2)\n", h[0], grid, h[2]);
  return 0;
}
