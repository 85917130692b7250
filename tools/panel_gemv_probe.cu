// Micro-benchmark of the blocked factorisation's per-column step on ONE CTA
// (ldlt_bkp.cuh panel_column): z broadcast, in-panel GEMV over the rows
// (W[c][P] in shared memory), out[P] store, CTA-wide (max, index)
// reduction.  Cycles per column for thread counts / reduction variants.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/panel_gemv_probe.cu -o tools/panel_gemv_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void max_pair(double& v, int& i, double v2, int i2) {
  if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) { v = v2; i = i2; }
}
// the same order on the bit patterns of non-negative doubles (integer compares)
__device__ __forceinline__ void max_pair_u(unsigned long long& v, int& i, unsigned long long v2, int i2) {
  if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) { v = v2; i = i2; }
}

template <int T, int MODE>  // MODE 0: full; 1: no reduction; 2: no gemv; 3: reduction only with one sync
__global__ void __launch_bounds__(T, 1) probe(int n, int jj, int reps, long long* out_cycles, double* sink) {
  extern __shared__ double sm[];
  double* W = sm;                 // [jj][n]
  double* outv = W + jj * n;      // [n]
  __shared__ double zs[32];
  __shared__ double rv[32];
  __shared__ int ri[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int x = threadIdx.x; x < jj * n; x += T) W[x] = 1e-3 * (x % 97);
  __syncthreads();
  long long t0 = clock64();
  double acc_all = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    const int q = rep % n;
    if (threadIdx.x < jj) zs[threadIdx.x] = W[threadIdx.x * n + q] * 0.5;
    __syncthreads();
    double m = -1.0; int mi = -1;
    if (MODE == 4) {
      unsigned long long mu = 0; int mui = -1;
      for (int P = threadIdx.x; P < n; P += T) {
        double s0 = 0.0, s1 = 0.0;
        int c = 0;
        for (; c + 1 < jj; c += 2) { s0 = fma(W[c * n + P], zs[c], s0); s1 = fma(W[(c + 1) * n + P], zs[c + 1], s1); }
        if (c < jj) s0 = fma(W[c * n + P], zs[c], s0);
        const double v = 1.0 - (s0 + s1);
        outv[P] = v;
        if (P != q) max_pair_u(mu, mui, __double_as_longlong(fabs(v)), P);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v2 = __shfl_xor_sync(0xffffffffu, mu, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, mui, o);
        max_pair_u(mu, mui, v2, i2);
      }
      __shared__ unsigned long long ru[32];
      if (lane == 0) { ru[warp] = mu; ri[warp] = mui; }
      __syncthreads();
      mu = lane < T / 32 ? ru[lane] : 0; mui = lane < T / 32 ? ri[lane] : -1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v2 = __shfl_xor_sync(0xffffffffu, mu, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, mui, o);
        max_pair_u(mu, mui, v2, i2);
      }
      __syncthreads();
      acc_all += __longlong_as_double(mu) + mui;
      continue;
    }
    if (MODE == 7) {  // packed 64-bit (|v| truncated to 40 mantissa bits, ~index) keys
      unsigned long long key = 0;
      for (int P = threadIdx.x; P < n; P += T) {
        double s0 = 0.0, s1 = 0.0;
        int c = 0;
        for (; c + 1 < jj; c += 2) { s0 = fma(W[c * n + P], zs[c], s0); s1 = fma(W[(c + 1) * n + P], zs[c + 1], s1); }
        if (c < jj) s0 = fma(W[c * n + P], zs[c], s0);
        const double v = 1.0 - (s0 + s1);
        outv[P] = v;
        if (P != q) {
          const unsigned long long k2 = (static_cast<unsigned long long>(__double_as_longlong(fabs(v))) & ~0xFFFull) |
                                        static_cast<unsigned long long>(0xFFF - P);
          key = k2 > key ? k2 : key;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
        key = k2 > key ? k2 : key;
      }
      __shared__ unsigned long long kw[32];
      if (lane == 0) kw[warp] = key;
      __syncthreads();
      unsigned long long best = 0;
#pragma unroll
      for (int w = 0; w < T / 32; ++w) best = kw[w] > best ? kw[w] : best;
      __syncthreads();
      acc_all += static_cast<double>(best & 0xFFF);
      continue;
    }
    if (MODE == 5 || MODE == 6) {  // 5: rows loop, store only; 6: rows loop, max only
      for (int P = threadIdx.x; P < n; P += T) {
        const double v = 1.0 - 0.25 * P;
        if (MODE == 5) outv[P] = v;
        if (MODE == 6 && P != q) max_pair(m, mi, fabs(v), P);
      }
    } else if (MODE != 2) {
      for (int P = threadIdx.x; P < n; P += T) {
        double s0 = 0.0, s1 = 0.0;
        int c = 0;
        for (; c + 1 < jj; c += 2) { s0 = fma(W[c * n + P], zs[c], s0); s1 = fma(W[(c + 1) * n + P], zs[c + 1], s1); }
        if (c < jj) s0 = fma(W[c * n + P], zs[c], s0);
        const double v = 1.0 - (s0 + s1);
        outv[P] = v;
        if (P != q) max_pair(m, mi, fabs(v), P);
      }
    }
    if (MODE != 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, m, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, mi, o);
        max_pair(m, mi, v2, i2);
      }
      if (lane == 0) { rv[warp] = m; ri[warp] = mi; }
      __syncthreads();
      m = lane < T / 32 ? rv[lane] : -1.0; mi = lane < T / 32 ? ri[lane] : -1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, m, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, mi, o);
        max_pair(m, mi, v2, i2);
      }
      if (MODE != 3) __syncthreads();
    } else {
      __syncthreads();
    }
    acc_all += m + mi;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out_cycles[0] = (t1 - t0) / reps; sink[0] = acc_all; }
}

template <int T, int MODE>
void run(int n, int jj) {
  long long* dc; double* ds;
  cudaMalloc(&dc, 8); cudaMalloc(&ds, 8);
  const size_t smem = sizeof(double) * (jj * n + n);
  cudaFuncSetAttribute(probe<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<T, MODE><<<1, T, smem>>>(n, jj, 2000, dc, ds);
  long long c = 0; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("T=%4d mode=%d n=%d jj=%2d: %lld cycles/column %s\n", T, MODE, n, jj, c, e ? cudaGetErrorString(e) : "");
  cudaFree(dc); cudaFree(ds);
}

int main() {
  run<512, 7>(804, 0);
  run<512, 7>(804, 16);
  run<512, 7>(804, 31);
  run<1024, 7>(804, 16);
  for (int jj : {0, 8, 16, 31}) {
    run<512, 0>(804, jj);
  }
  run<512, 1>(804, 16);
  run<512, 2>(804, 16);
  run<512, 3>(804, 16);
  run<256, 0>(804, 16);
  run<1024, 0>(804, 16);
  run<1024, 1>(804, 16);
  run<1024, 2>(804, 16);
  return 0;
}
