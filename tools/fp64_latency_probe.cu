// Dependent-chain latency of FP64 DADD / DFMA / DSETP+select and of a
// shared-memory store->load round trip on sm_100a (one thread).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_latency_probe.cu -o tools/fp64_latency_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double seed, long long* out, double* sink) {
  __shared__ double sm[64];
  double a = seed, b = seed * 0.5;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { a = fma(a, b, b); a = fma(a, b, b); a = fma(a, b, b); a = fma(a, b, b); }
  long long t2 = clock64();
  int idx = 0;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    const double v = fabs(a - i);
    if (v > b || (v == b && i < idx)) { b = v; idx = i; }
    a = a + b * 1e-9;
  }
  long long t3 = clock64();
  sm[threadIdx.x] = a;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { sm[(i + 1) & 31] = sm[i & 31] + 1.0; }
  long long t4 = clock64();
  float f = (float)a, g = (float)b;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { f = f + g; f = f + g; f = f + g; f = f + g; }
  long long t5 = clock64();
  out[0] = (t1 - t0) / 4000; out[1] = (t2 - t1) / 4000; out[2] = (t3 - t2) / 1000; out[3] = (t4 - t3) / 1000;
  out[4] = (t5 - t4) / 4000;
  sink[0] = a + b + idx + sm[5] + f;
}

int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  lat<<<1, 1>>>(1.0, d, s);
  long long h[5]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("DADD %lld, DFMA %lld, max-step (DADD+DSETP+select) %lld, smem store->load %lld, FADD %lld cycles\n", h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
