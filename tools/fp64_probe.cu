// Throwaway microbenchmark: FP64 issue rates on sm_100a (DFMA vs DMMA.8x8x4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double s) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], b, s);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += acc[i];
  if (r == 12345.678) out[threadIdx.x] = r;
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[threadIdx.x] = r;
}

int main() {
  double* d; cudaMalloc(&d, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d  max clock %d MHz\n", sms, clk / 1000);
  const int iters = 20000;
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {128, 256}) {
      dim3 grid(sms * bpsm);
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_loop<8><<<grid, threads>>>(d, iters, 0.5);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * 8 * iters * (double)threads * grid.x;
      printf("DFMA  bpsm=%d thr=%d : %.2f TFLOP/s\n", bpsm, threads, flops / best / 1e9);
      best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dmma_loop<4><<<grid, threads>>>(d, iters / 4);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      flops = 2.0 * 256 * 4 * (iters / 4) * (double)(threads / 32) * grid.x;
      printf("DMMA  bpsm=%d thr=%d : %.2f TFLOP/s\n", bpsm, threads, flops / best / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
