// Achievable bandwidth of the trailing-update access pattern (64 x 64 tiles of
// an n x n matrix, read A(li, lj) -> write A2(i, j)), 120 CTAs x 512 threads,
// variants: 0 = 8-byte cp.async double-buffered (as ldlt_bkq.cuh),
// 1 = 16-byte cp.async, 2 = plain 16-byte loads to registers, 3 = 8-byte
// loads to registers.  Prints GB/s (read + write).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kT = 64, kThreads = 512, kLdA = kT + 8;
__device__ __forceinline__ void cp8(void* d, const void* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void cp16(void* d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s) : "memory");
}
template <int V>
__global__ void __launch_bounds__(kThreads, 1) probe(const double* a, double* a2, int n) {
  extern __shared__ __align__(16) double sm[];
  const int tm = n / kT, tiles = tm * tm, tid = threadIdx.x;
  if (V <= 1) {
    auto issue = [&](int tile, int buf) {
      if (tile < tiles) {
        const int i0 = (tile / tm) * kT, j0 = (tile % tm) * kT;
        double* A_ = sm + buf * kT * kLdA;
        if (V == 0) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int x = tid + u * kThreads, r = x / kT, c = x % kT;
            cp8(A_ + r * kLdA + c, a + (size_t)(i0 + r) * n + j0 + c);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int x = tid + u * kThreads, r = x / 32, c = 2 * (x % 32);
            cp16(A_ + r * kLdA + c, a + (size_t)(i0 + r) * n + j0 + c);
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    issue(blockIdx.x, 0);
    int t = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, t ^= 1) {
      __syncthreads();
      issue(tile + gridDim.x, t ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      __syncthreads();
      const int i0 = (tile / tm) * kT, j0 = (tile % tm) * kT;
      const double* A_ = sm + t * kT * kLdA;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = tid + u * kThreads, r = x / 32, c = 2 * (x % 32);
        const double2 v = *reinterpret_cast<const double2*>(A_ + r * kLdA + c);
        __stcg(reinterpret_cast<double2*>(a2 + (size_t)(i0 + r) * n + j0 + c), v);
      }
    }
  } else {
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int i0 = (tile / tm) * kT, j0 = (tile % tm) * kT;
      if (V == 2) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int x = tid + u * kThreads, r = x / 32, c = 2 * (x % 32);
          v[u] = __ldcg(reinterpret_cast<const double2*>(a + (size_t)(i0 + r) * n + j0 + c));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int x = tid + u * kThreads, r = x / 32, c = 2 * (x % 32);
          __stcg(reinterpret_cast<double2*>(a2 + (size_t)(i0 + r) * n + j0 + c), v[u]);
        }
      } else {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int x = tid + u * kThreads, r = x / kT, c = x % kT;
          v[u] = __ldcg(a + (size_t)(i0 + r) * n + j0 + c);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int x = tid + u * kThreads, r = x / kT, c = x % kT;
          __stcg(a2 + (size_t)(i0 + r) * n + j0 + c, v[u]);
        }
      }
    }
  }
}
template <int V>
void run(const double* a, double* a2, int n, int grid) {
  const int smem = 2 * kT * kLdA * 8;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<V><<<grid, kThreads, smem>>>(a, a2, n);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) probe<V><<<grid, kThreads, smem>>>(a, a2, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 2.0 * 8.0 * n * (double)n;
  printf("variant %d n %d grid %d: %.3f ms  %.0f GB/s  (%s)\n", V, n, grid, ms / reps, bytes / (ms / reps * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int n : {4480, 11264}) {
    double *a, *a2;
    cudaMalloc(&a, 8ull * n * n);
    cudaMalloc(&a2, 8ull * n * n);
    cudaMemset(a, 0, 8ull * n * n);
    for (int grid : {120, 148, 296}) {
      run<0>(a, a2, n, grid);
      run<1>(a, a2, n, grid);
      run<2>(a, a2, n, grid);
      run<3>(a, a2, n, grid);
    }
    cudaFree(a);
    cudaFree(a2);
  }
}
