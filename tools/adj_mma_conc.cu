// adj_mma_kernel correctness under overlap: two W / gz / partial sets, solo
// launches and back-to-back launches on two streams, each checked against a
// CPU sum over two row chunks.  Prints mismatches.
// nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2509_22462_b200/csrc \
//   tools/adj_mma_conc.cu -lcuda -o tools/adj_mma_conc.bin ; ./tools/adj_mma_conc.bin [reps]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "kernels.cuh"

using namespace gbb;

// co-resident noise: small CTAs streaming through their own buffer
__global__ void noise_kernel(double* buf, size_t n, int iters) {
  for (int it = 0; it < iters; ++it)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      buf[i] = buf[i] * 0.5 + 1.0;
}

static CUtensorMap tmap(const double* base, int64_t cols, int64_t rows, int64_t pitch) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(pitch * 8)};
  const cuuint32_t box[2] = {16, 16};
  const cuuint32_t estr[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    printf("encode failed\n");
  return m;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  const int noise = argc > 2 ? atoi(argv[2]) : 0;  // 1: a co-resident noise kernel on a third stream
  const int rows = 5120, cols = 5120, nv = 10, crows = dev::kAmRows, chunks = rows / crows;
  const int64_t ld_part = cols;
  cudaFuncSetAttribute(dev::adj_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kAmSmem);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(-1, 1);
  double *W[2], *gz[2], *part[2];
  std::vector<double> hW[2], hG[2];
  CUtensorMap tm[2];
  const size_t N = (size_t)chunks * nv * ld_part;
  for (int i = 0; i < 2; ++i) {
    hW[i].resize((size_t)rows * cols);
    hG[i].resize((size_t)nv * rows);
    for (auto& x : hW[i]) x = u(g);
    for (auto& x : hG[i]) x = u(g);
    cudaMalloc(&W[i], sizeof(double) * hW[i].size());
    cudaMemcpy(W[i], hW[i].data(), sizeof(double) * hW[i].size(), cudaMemcpyHostToDevice);
    cudaMalloc(&gz[i], sizeof(double) * hG[i].size());
    cudaMemcpy(gz[i], hG[i].data(), sizeof(double) * hG[i].size(), cudaMemcpyHostToDevice);
    cudaMalloc(&part[i], sizeof(double) * N);
    tm[i] = tmap(W[i], cols, rows, cols);
  }
  // CPU sums for chunks 0 and 7
  std::vector<double> want[2];
  for (int i = 0; i < 2; ++i) {
    want[i].assign((size_t)2 * nv * cols, 0.0);
    int ci = 0;
    for (int c : {0, 7}) {
      for (int v = 0; v < nv; ++v)
        for (int r = c * crows; r < (c + 1) * crows; ++r) {
          const double gv = hG[i][(size_t)v * rows + r];
          const double* wr = &hW[i][(size_t)r * cols];
          double* o = &want[i][((size_t)ci * nv + v) * cols];
          for (int k = 0; k < cols; ++k) o[k] += gv * wr[k];
        }
      ++ci;
    }
  }
  std::vector<double> got(N);
  auto check = [&](int i, const char* what) {
    cudaMemcpy(got.data(), part[i], sizeof(double) * N, cudaMemcpyDeviceToHost);
    size_t nbad = 0;
    int ci = 0;
    for (int c : {0, 7}) {
      for (int v = 0; v < nv; ++v)
        for (int k = 0; k < cols; ++k)
          nbad += fabs(got[((size_t)c * nv + v) * ld_part + k] - want[i][((size_t)ci * nv + v) * cols + k]) > 1e-9;
      ++ci;
    }
    if (nbad) printf("%s set %d: %zu of %d partials wrong\n", what, i, nbad, 2 * nv * cols);
    return nbad;
  };
  cudaStream_t s[2];
  for (int i = 0; i < 2; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  const dim3 grid((cols + 127) / 128, chunks);
  size_t bad = 0;
  for (int i = 0; i < 2; ++i) {  // solo, cold
    dev::adj_mma_kernel<<<grid, 288, dev::kAmSmem, s[i]>>>(tm[i], rows, cols, gz[i], rows, nv, 0, part[i], ld_part,
                                                            crows);
    cudaStreamSynchronize(s[i]);
    bad += check(i, "solo");
  }
  double* nbuf = nullptr;
  cudaStream_t s3;
  cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
  const size_t nn = size_t(64) << 20;
  if (noise) cudaMalloc(&nbuf, sizeof(double) * nn);
  for (int r = 0; r < reps; ++r) {  // both sets at once, back to back
    if (noise) noise_kernel<<<148 * 4, 256, 0, s3>>>(nbuf, nn, 4);
    for (int k = 0; k < 4; ++k)
      for (int i = 0; i < 2; ++i)
        dev::adj_mma_kernel<<<grid, 288, dev::kAmSmem, s[i]>>>(tm[i], rows, cols, gz[i], rows, nv, 0, part[i],
                                                                ld_part, crows);
    cudaDeviceSynchronize();
    for (int i = 0; i < 2; ++i) bad += check(i, "overlap");
  }
  printf("wrong partials in total: %zu (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}
