// Standalone probe of single-point forward GEMV variants (z = W y, FP64,
// row-major W [rows][ldw]) on the B200: achieved GB/s of each variant on the
// c2 layer shapes.  Build + run:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gemv_probe.cu -o /tmp/gemv_probe && /tmp/gemv_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)

struct d4 {
  double x, y, z, w;
};
__device__ __forceinline__ d4 ld256_stream(const double* p) {
  d4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ d4 ld256(const double* p) {
  d4 r;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}

// V0: current fwd_row1 (one warp per row, 16 B loads, 8 in flight)
__global__ void __launch_bounds__(256) v0(const double* __restrict__ w, int ldw, int rows, int k,
                                          const double* __restrict__ y, double* __restrict__ z) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const double* wr = w + static_cast<long>(row) * ldw;
  double a0 = 0, a1 = 0;
  const int chunks = (k + 63) / 64;
  int c = 0;
  for (; c + 8 <= chunks; c += 8) {
    double2 wv[8], yv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int kk = (c + u) * 64 + 2 * lane;
      wv[u] = kk < k ? __ldcs(reinterpret_cast<const double2*>(wr + kk)) : make_double2(0, 0);
      yv[u] = kk < k ? __ldg(reinterpret_cast<const double2*>(y + kk)) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(wv[u].x, yv[u].x, a0);
      a1 = fma(wv[u].y, yv[u].y, a1);
    }
  }
  for (; c < chunks; ++c) {
    const int kk = c * 64 + 2 * lane;
    if (kk < k) {
      const double2 wv = __ldcs(reinterpret_cast<const double2*>(wr + kk));
      const double2 yv = __ldg(reinterpret_cast<const double2*>(y + kk));
      a0 = fma(wv.x, yv.x, a0);
      a1 = fma(wv.y, yv.y, a1);
    }
  }
  double v = a0 + a1;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if (lane == 0) z[row] = v;
}

// V1: 32 B loads (LDG.256), U chunks of 1 KB per warp in flight; y staged
// once per CTA in shared memory; WPR warps per row (split K, fixed-order
// reduction); grid-stride over row groups with a persistent grid.
template <int U, int WPR, bool NOALLOC>
__global__ void __launch_bounds__(256) v1(const double* __restrict__ w, int ldw, int rows, int k,
                                          const double* __restrict__ y, double* __restrict__ z) {
  extern __shared__ double ys[];
  __shared__ double part[8];
  for (int i = threadIdx.x * 4; i < k; i += 256 * 4) {
    for (int j = 0; j < 4; ++j) ys[i + j] = (i + j < k) ? y[i + j] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kRowsPerCta = 8 / WPR;
  const int chunks = (k + 127) / 128;  // 128 doubles = 1 KB per warp step
  const int part_idx = warp % WPR;
  const int c0 = (chunks * part_idx) / WPR, c1 = (chunks * (part_idx + 1)) / WPR;
  for (int rb = blockIdx.x * kRowsPerCta; rb < rows; rb += gridDim.x * kRowsPerCta) {
    const int row = rb + warp / WPR;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    if (row < rows) {
      const double* wr = w + static_cast<long>(row) * ldw;
      int c = c0;
      for (; c + U <= c1; c += U) {
        d4 wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = (c + u) * 128 + 4 * lane;
          wv[u] = kk < k ? (NOALLOC ? ld256_stream(wr + kk) : ld256(wr + kk)) : d4{0, 0, 0, 0};
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = (c + u) * 128 + 4 * lane;
          const double4 yv = *reinterpret_cast<const double4*>(&ys[kk]);
          a0 = fma(wv[u].x, yv.x, a0);
          a1 = fma(wv[u].y, yv.y, a1);
          a2 = fma(wv[u].z, yv.z, a2);
          a3 = fma(wv[u].w, yv.w, a3);
        }
      }
      for (; c < c1; ++c) {
        const int kk = c * 128 + 4 * lane;
        if (kk < k) {
          const d4 wv = NOALLOC ? ld256_stream(wr + kk) : ld256(wr + kk);
          const double4 yv = *reinterpret_cast<const double4*>(&ys[kk]);
          a0 = fma(wv.x, yv.x, a0);
          a1 = fma(wv.y, yv.y, a1);
          a2 = fma(wv.z, yv.z, a2);
          a3 = fma(wv.w, yv.w, a3);
        }
      }
    }
    double v = (a0 + a1) + (a2 + a3);
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    if (WPR > 1) {
      __syncthreads();
      if (lane == 0) part[warp] = v;
      __syncthreads();
      if (part_idx == 0 && lane == 0 && row < rows) {
        double s = 0;
        for (int i = 0; i < WPR; ++i) s += part[warp + i];
        z[row] = s;
      }
    } else if (lane == 0 && row < rows) {
      z[row] = v;
    }
  }
}

// V2: the v0 structure (one warp per row, no staging) with 32 B loads.
template <int U, bool NOALLOC>
__global__ void __launch_bounds__(256) v2(const double* __restrict__ w, int ldw, int rows, int k,
                                          const double* __restrict__ y, double* __restrict__ z) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const double* wr = w + static_cast<long>(row) * ldw;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  const int chunks = (k + 127) / 128;
  int c = 0;
  for (; c + U <= chunks; c += U) {
    d4 wv[U], yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = (c + u) * 128 + 4 * lane;
      wv[u] = kk < k ? (NOALLOC ? ld256_stream(wr + kk) : ld256(wr + kk)) : d4{0, 0, 0, 0};
      yv[u] = kk < k ? ld256(y + kk) : d4{0, 0, 0, 0};
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0 = fma(wv[u].x, yv[u].x, a0);
      a1 = fma(wv[u].y, yv[u].y, a1);
      a2 = fma(wv[u].z, yv[u].z, a2);
      a3 = fma(wv[u].w, yv[u].w, a3);
    }
  }
  for (; c < chunks; ++c) {
    const int kk = c * 128 + 4 * lane;
    if (kk < k) {
      const d4 wv = NOALLOC ? ld256_stream(wr + kk) : ld256(wr + kk);
      const d4 yv = ld256(y + kk);
      a0 = fma(wv.x, yv.x, a0);
      a1 = fma(wv.y, yv.y, a1);
      a2 = fma(wv.z, yv.z, a2);
      a3 = fma(wv.w, yv.w, a3);
    }
  }
  double v = (a0 + a1) + (a2 + a3);
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if (lane == 0) z[row] = v;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  struct Shape {
    int rows, k;
  } shapes[] = {{5120, 5120}, {5120, 784}, {10, 5120}, {1024, 1024}};
  for (auto sh : shapes) {
    const int ldw = (sh.k + 15) / 16 * 16;
    const size_t wn = static_cast<size_t>(sh.rows) * ldw;
    // rotate over enough copies that the working set exceeds L2 (126 MB)
    const int copies = static_cast<int>(std::max<size_t>(1, (600ull << 20) / (wn * 8)));
    double *w, *y, *z;
    CK(cudaMalloc(&w, wn * 8 * copies));
    CK(cudaMalloc(&y, ldw * 8));
    CK(cudaMalloc(&z, sh.rows * 8));
    std::vector<double> hw(wn);
    for (size_t i = 0; i < wn; ++i) hw[i] = ((i * 2654435761u) % 1000) * 1e-3;
    for (int c = 0; c < copies; ++c) CK(cudaMemcpy(w + wn * c, hw.data(), wn * 8, cudaMemcpyHostToDevice));
    std::vector<double> hy(ldw, 0.5);
    CK(cudaMemcpy(y, hy.data(), ldw * 8, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double bytes = static_cast<double>(sh.rows) * sh.k * 8;
    auto run = [&](const char* name, auto launch) {
      for (int i = 0; i < 3; ++i) launch(w + wn * (i % copies));
      CK(cudaDeviceSynchronize());
      const int reps = 60;
      CK(cudaEventRecord(e0));
      for (int i = 0; i < reps; ++i) launch(w + wn * (i % copies));
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = ms * 1e3 / reps;
      std::printf("  %-28s %8.2f us  %7.1f GB/s\n", name, us, bytes / us * 1e-3);
    };
    std::printf("rows %d k %d (%.1f MB, %d copies)\n", sh.rows, sh.k, bytes / 1e6, copies);
    run("v0 current", [&](const double* W) { v0<<<(sh.rows + 7) / 8, 256>>>(W, ldw, sh.rows, sh.k, y, z); });
    const size_t smem = static_cast<size_t>(ldw) * 8;
    auto v1run = [&](const char* name, auto kern, int wpr, int ctas_per_sm) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const int groups = (sh.rows + (8 / wpr) - 1) / (8 / wpr);
      const int grid = std::min(groups, sms * ctas_per_sm);
      run(name, [&](const double* W) { kern<<<grid, 256, smem>>>(W, ldw, sh.rows, sh.k, y, z); });
    };
    (void)v1run;
    run("v2 U4 na", [&](const double* W) { v2<4, true><<<(sh.rows + 7) / 8, 256>>>(W, ldw, sh.rows, sh.k, y, z); });
    run("v2 U8 na", [&](const double* W) { v2<8, true><<<(sh.rows + 7) / 8, 256>>>(W, ldw, sh.rows, sh.k, y, z); });
    run("v2 U4 nc", [&](const double* W) { v2<4, false><<<(sh.rows + 7) / 8, 256>>>(W, ldw, sh.rows, sh.k, y, z); });
    run("v2 U8 nc", [&](const double* W) { v2<8, false><<<(sh.rows + 7) / 8, 256>>>(W, ldw, sh.rows, sh.k, y, z); });
    run("v2 U2 na", [&](const double* W) { v2<2, true><<<(sh.rows + 7) / 8, 256>>>(W, ldw, sh.rows, sh.k, y, z); });
    CK(cudaFree(w));
    CK(cudaFree(y));
    CK(cudaFree(z));
  }
  return 0;
}
