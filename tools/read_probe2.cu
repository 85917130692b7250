// HBM read-stream probe for the forward GEMV (throwaway measurement tool).
// Streams one 5120 x 5120 FP64 matrix (210 MB) and the whole c2 weight set
// (5 such matrices + the 784-column one, 872 MB) with:
//   rows   - one warp per row, 8 x 16 B loads in flight per lane, dot with y
//            from L1 (the current fwd_row1_kernel)
//   flat   - persistent grid-stride sum, 4 x 16 B loads per thread per step
//   bulk   - persistent, one CTA per SM: a producer thread streams the CTA's
//            contiguous byte range with 1-D TMA bulk copies (cp.async.bulk)
//            into a 6-stage shared-memory ring; 8 consumer warps sum
// L2 flushed (256 MB write) before every timed run; best of 10 (CUDA events).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/read_probe2.bin tools/read_probe2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void rows_kernel(const double* __restrict__ w, int rows, int k_dim, const double* __restrict__ y,
                            double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const double* wr = w + static_cast<int64_t>(row) * k_dim;
  double a0 = 0, a1 = 0;
  const int chunks = k_dim / 64;
  int c = 0;
  for (; c + 8 <= chunks; c += 8) {
    double2 wv[8], yv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = (c + u) * 64 + 2 * lane;
      wv[u] = __ldcs(reinterpret_cast<const double2*>(wr + k));
      yv[u] = __ldg(reinterpret_cast<const double2*>(y + k));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(wv[u].x, yv[u].x, a0);
      a1 = fma(wv[u].y, yv[u].y, a1);
    }
  }
  for (; c < chunks; ++c) {
    const int k = c * 64 + 2 * lane;
    const double2 wv = __ldcs(reinterpret_cast<const double2*>(wr + k));
    const double2 yv = __ldg(reinterpret_cast<const double2*>(y + k));
    a0 = fma(wv.x, yv.x, a0);
    a1 = fma(wv.y, yv.y, a1);
  }
  double v = a0 + a1;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[row] = v;
}

__global__ void flat_kernel(const double2* __restrict__ w, int64_t n2, double* __restrict__ out) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
  double s = 0;
  int64_t i = tid;
  for (; i + 3 * nt < n2; i += 4 * nt) {
    const double2 a = __ldcs(w + i), b = __ldcs(w + i + nt), c = __ldcs(w + i + 2 * nt), d = __ldcs(w + i + 3 * nt);
    s += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
  }
  for (; i < n2; i += nt) {
    const double2 a = __ldcs(w + i);
    s += a.x + a.y;
  }
  if (s == 12345.0) out[0] = s;
}

constexpr int kStages = 6;
constexpr int kStageBytes = 32768;

__global__ void __launch_bounds__(288, 1) bulk_kernel(const char* __restrict__ w, int64_t bytes, double* out) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5;
  // this CTA's contiguous range, whole 4 KB pages
  const int64_t pages = bytes / 4096;
  const int64_t p0 = pages * blockIdx.x / gridDim.x, p1 = pages * (blockIdx.x + 1) / gridDim.x;
  const int64_t b0 = p0 * 4096, b1 = p1 * 4096;
  const int nchunks = static_cast<int>((b1 - b0 + kStageBytes - 1) / kStageBytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if ((threadIdx.x & 31) == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % kStages;
        if (c >= kStages) {
          const uint32_t par = ((c / kStages) - 1) & 1;
          asm volatile(
              "{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n}" ::"r"(
                  smem_u32(empty + s)),
              "r"(par)
              : "memory");
        }
        const int64_t off = b0 + static_cast<int64_t>(c) * kStageBytes;
        const uint32_t sz = static_cast<uint32_t>(b1 - off < kStageBytes ? b1 - off : kStageBytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(sz)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem + s * kStageBytes)),
            "l"(w + off), "r"(sz), "r"(smem_u32(full + s))
            : "memory");
      }
    }
    return;
  }
  double acc = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % kStages;
    const uint32_t par = (c / kStages) & 1;
    asm volatile(
        "{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n}" ::"r"(
            smem_u32(full + s)),
        "r"(par)
        : "memory");
    const int64_t off = b0 + static_cast<int64_t>(c) * kStageBytes;
    const int sz = static_cast<int>(b1 - off < kStageBytes ? b1 - off : kStageBytes);
    const double2* st = reinterpret_cast<const double2*>(smem + s * kStageBytes);
    for (int i = threadIdx.x; i < sz / 16; i += 256) {
      const double2 v = st[i];
      acc += v.x + v.y;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + s)) : "memory");
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const int64_t n = 5120;
  const int64_t big = 5 * n * n + n * 784;  // c2's weights (doubles), the 10-row layer left out
  double *w, *y, *out, *flush;
  CK(cudaMalloc(&w, big * 8));
  CK(cudaMemset(w, 0, big * 8));
  CK(cudaMalloc(&y, n * 8));
  CK(cudaMemset(y, 0, n * 8));
  CK(cudaMalloc(&out, 6 * n * 8));
  CK(cudaMalloc(&flush, 256 << 20));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int bulk_smem = kStages * kStageBytes + 2 * kStages * 8;
  CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bulk_smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, int64_t bytes, auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 10; ++rep) {
      cudaMemsetAsync(flush, rep, 256 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    std::printf("%-28s %8.1f MB  %8.2f us  %6.3f TB/s  (%s)\n", name, bytes / 1e6, best * 1e3, bytes / (best * 1e-3) / 1e12,
                cudaGetErrorString(cudaGetLastError()));
  };
  const int64_t m1 = n * n * 8;
  run("rows 5120x5120", m1, [&] { rows_kernel<<<n / 8, 256>>>(w, n, n, y, out); });
  run("rows c2 (5 layers)", 5 * m1, [&] {
    for (int l = 0; l < 5; ++l) rows_kernel<<<n / 8, 256>>>(w + l * n * n, n, n, y, out);
  });
  for (int g : {sms, 2 * sms, 4 * sms, 8 * sms}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "flat 5120^2 grid %d", g);
    run(nm, m1, [&] { flat_kernel<<<g, 256>>>(reinterpret_cast<const double2*>(w), m1 / 16, out); });
  }
  run("flat c2 (one launch)", big * 8,
      [&] { flat_kernel<<<4 * sms, 256>>>(reinterpret_cast<const double2*>(w), big * 8 / 16, out); });
  run("bulk 5120^2 (1 CTA/SM)", m1, [&] { bulk_kernel<<<sms, 288, bulk_smem>>>(reinterpret_cast<const char*>(w), m1, out); });
  run("bulk c2 (one launch)", big * 8,
      [&] { bulk_kernel<<<sms, 288, bulk_smem>>>(reinterpret_cast<const char*>(w), big * 8, out); });
  return 0;
}
