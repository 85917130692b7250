// Symmetric-indefinite LDL^T on the GPU for the KKT systems of the
// interior-point caller (reference
// proj/include/gbopt/linalg.hpp:24-78, proj/src/linalg.cpp:39-438).
//
// Same contract as the reference ldlt_factor / LdltFactorization:
//   * checks: finite entries (NumericError), symmetry to
//     1e-12 * max(1, max|A|) (StructuralError)            linalg.cpp:45-71
//   * symmetric Ruiz equilibration, <= 20 rounds, tol 0.01  linalg.cpp:72-99
//   * Bunch-Kaufman factorisation P S A S P^T = L D L^T of the equilibrated
//     matrix -- ldlt_bk.cuh: one cooperative launch, left-looking, the
//     reference's pivoting rule (alpha = (1 + sqrt 17) / 8); cuSOLVER's dsytrf
//     only beyond n = 20000 (shared-memory limit of the native kernel)
//   * inertia from the 1x1 / 2x2 pivot blocks with zero threshold
//     1e-11 * max|S A S|                                     linalg.cpp:101-120
//   * solve: refuses singular factorizations (SingularError); x = S y with
//     S A S y = S b, iterative refinement while the residual shrinks, at
//     most 10 rounds, returning the best iterate              linalg.cpp:393-438
// Everything O(n^2) per pass (checks, equilibration, residuals) runs on the
// device too; only the 2n pivot-block entries and vectors cross PCIe after
// the matrix upload.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "device_net.hpp"
#include "ldlt.hpp"
#include "ldlt_bk.cuh"
#include "ldlt_bkc.cuh"
#include "ldlt_bkp.cuh"
#include "ldlt_bkq.cuh"

namespace gbb {

namespace {

void cs_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS)
    throw DeviceError(std::string("cuSOLVER error in ") + what + ": " + std::to_string(static_cast<int>(s)));
}
#define CK(x) cuda_check((x), #x)
#define CS(x) cs_check((x), #x)
namespace cg = cooperative_groups;

__device__ inline void atomic_max_pos(double* addr, double v) {
  // v >= 0: ordering of non-negative doubles matches their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

// r = b - A x (one warp per row), also |r|_inf and |x|_inf into out[0..1]
// (grid-stride over rows: the launch is capped, n is not)
__global__ void ldlt_residual_kernel(const double* __restrict__ a, int64_t n, const double* __restrict__ x,
                                     const double* __restrict__ b, double* __restrict__ r, double* out) {
  const int64_t wpb = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * wpb + (threadIdx.x >> 5); row < n;
       row += static_cast<int64_t>(gridDim.x) * wpb) {
    double s = 0.0;
    for (int64_t k = lane; k < n; k += 32) s = fma(a[row * n + k], x[k], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double v = b[row] - s;
      r[row] = v;
      atomic_max_pos(out + 0, fabs(v));
      atomic_max_pos(out + 1, fabs(x[row]));
    }
  }
}

// Checks and Ruiz equilibration in ONE cooperative launch (linalg.cpp:45-99):
// the same quantities as ldlt_check_kernel / ldlt_colmax_kernel /
// ldlt_scale_kernel, with the round control on the device (a per-round
// maximum |cmax - 1| in scal[8 + round], read by every thread after the
// grid barrier) instead of a host round trip per round.
// scal: [0] max|A|, [1] max|A - A^T|, [2] #non-finite, [3] max cmax of the
// final matrix, [8 + r] round r's deviation; all zeroed by the caller.
__global__ void ldlt_prep_kernel(double* __restrict__ a, int64_t n, double* __restrict__ rs,
                                 double* __restrict__ scale, double* __restrict__ cmax, double* scal) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t gw = tid >> 5, nw = nt >> 5;
  {
    double amax = 0.0, asym = 0.0, bad = 0.0;
    for (int64_t e = tid; e < n * n; e += nt) {
      const int64_t i = e / n, j = e % n;
      const double v = a[e];
      if (!isfinite(v)) {
        bad += 1.0;
        continue;
      }
      amax = fmax(amax, fabs(v));
      if (j < i) asym = fmax(asym, fabs(v - a[j * n + i]));
    }
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
      bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
      atomic_max_pos(scal + 0, amax);
      if (asym == asym) atomic_max_pos(scal + 1, asym);
      if (bad > 0) atomicAdd(scal + 2, bad);
    }
  }
  grid.sync();
  if (__ldcg(scal + 2) > 0 || __ldcg(scal + 1) > 1e-12 * fmax(1.0, __ldcg(scal + 0))) return;  // the host throws
  for (int64_t i = tid; i < n; i += nt) scale[i] = 1.0;
  bool converged = false;
  for (int round = 0; round < 20; ++round) {
    // cmax of row i == column i (symmetric): one warp per row
    for (int64_t row = gw; row < n; row += nw) {
      double m = 0.0;
      for (int64_t k = lane; k < n; k += 32) m = fmax(m, fabs(a[row * n + k]));
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) {
        cmax[row] = m;
        rs[row] = m > 0.0 ? 1.0 / sqrt(m) : 1.0;
        if (m > 0.0) atomic_max_pos(scal + 8 + round, fabs(m - 1.0));
      }
    }
    grid.sync();
    if (__ldcg(scal + 8 + round) <= 0.01) {  // the same value in every thread
      converged = true;
      break;
    }
    for (int64_t e = tid; e < n * n; e += nt) a[e] *= __ldcg(rs + e / n) * __ldcg(rs + e % n);
    for (int64_t i = tid; i < n; i += nt) scale[i] *= __ldcg(rs + i);
    grid.sync();
  }
  if (!converged) {
    // all 20 rounds rescaled: the maxima measured before the last scaling
    // are stale; the zero threshold needs max|balanced| of the final matrix
    // (linalg.cpp:101)
    for (int64_t row = gw; row < n; row += nw) {
      double m = 0.0;
      for (int64_t k = lane; k < n; k += 32) m = fmax(m, fabs(a[row * n + k]));
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) cmax[row] = m;
    }
    grid.sync();
  }
  for (int64_t i = tid; i < n; i += nt) atomic_max_pos(scal + 3, __ldcg(cmax + i));  // cmax of the final matrix
}

// A(i, i) += delta_w for i < n_var; A(i, i) -= delta_c for i >= n_var
// (each only when non-zero)
__global__ void ldlt_shift_diag_kernel(double* __restrict__ a, int64_t n, int64_t n_var, double delta_w,
                                       double delta_c) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i < n_var) {
    if (delta_w != 0.0) a[i * n + i] += delta_w;
  } else if (delta_c != 0.0) {
    a[i * n + i] -= delta_c;
  }
}

// Device buffers of finished factorisations are kept for reuse (exact size
// match, per device, up to kPoolCap bytes): the IPM's inertia correction
// factors same-sized trial matrices back to back, and cudaMalloc / cudaFree
// of the multi-MB buffers cost more than a small factorisation's kernels.
struct BufPool {
  std::mutex m;
  std::multimap<std::pair<int, size_t>, void*> free;
  size_t cached = 0;
};
constexpr size_t kPoolCap = size_t(4) << 30;
BufPool& buf_pool() {
  static BufPool* pool = new BufPool;  // never destroyed: no teardown-order issues at exit
  return *pool;
}
void* pool_alloc(int dev, size_t bytes) {
  BufPool& pool = buf_pool();
  {
    std::lock_guard<std::mutex> lock(pool.m);
    auto it = pool.free.find({dev, bytes});
    if (it != pool.free.end()) {
      void* p = it->second;
      pool.free.erase(it);
      pool.cached -= bytes;
      return p;
    }
  }
  void* p = nullptr;
  CK(cudaMalloc(&p, bytes));
  return p;
}
void pool_release(int dev, size_t bytes, void* p) {
  BufPool& pool = buf_pool();
  std::lock_guard<std::mutex> lock(pool.m);
  if (pool.cached + bytes <= kPoolCap) {
    pool.free.emplace(std::make_pair(dev, bytes), p);
    pool.cached += bytes;
  } else {
    cudaFree(p);
  }
}

}  // namespace

template <class T>
void Ldlt::palloc(T** ptr, size_t bytes) {
  *ptr = static_cast<T*>(pool_alloc(dev_, bytes));
  pooled_.emplace_back(static_cast<void*>(*ptr), bytes);
}

namespace {

int blocks_for(int64_t work, int per) { return static_cast<int>(std::min<int64_t>((work + per - 1) / per, 4096)); }

}  // namespace

// Native Bunch-Kaufman for every size (round 2: the grid kernel's shared
// memory no longer grows with n); cuSOLVER dsytrf only past this bound,
// where int32 indexing of the factor kernels would overflow.
constexpr int64_t kNativeMaxN = 46340;
constexpr int kScal = 32;  // device scalars after the four n-vectors of d_vec_ (ldlt_prep_kernel)
constexpr int64_t kCtaSolveMaxN = 3000;  // one-CTA substitution below (n 804: 0.20 vs 0.44 ms; 4500: 3.08 vs 2.45)

// GBOPT_LDLT_TIMING=1: host wall time of the factorisation phases on stderr
struct PhaseTimer {
  bool on = std::getenv("GBOPT_LDLT_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "ldlt: %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

__global__ void bk_iota_kernel(int* perm, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) perm[i] = static_cast<int>(i);
}

Ldlt::~Ldlt() {
  if (dev_ >= 0) {
    DeviceGuard g(dev_);
    for (const auto& pb : pooled_) pool_release(dev_, pb.second, pb.first);
    if (handle_) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(handle_));
    if (stream_) cudaStreamDestroy(stream_);
  }
}

std::unique_ptr<Ldlt> Ldlt::factor(const double* a, int64_t n, bool keep_input, int device) {
  return factor_impl(a, false, n, n, 0.0, 0.0, keep_input, device, nullptr);
}

std::unique_ptr<Ldlt> Ldlt::factor_device(const double* d_a, int64_t n, int64_t n_var, double delta_w,
                                          double delta_c, bool keep_input, int device, cudaStream_t src) {
  return factor_impl(d_a, true, n, n_var, delta_w, delta_c, keep_input, device, src);
}

std::unique_ptr<Ldlt> Ldlt::factor_impl(const double* a, bool on_device, int64_t n, int64_t n_var, double delta_w,
                                        double delta_c, bool keep_input, int device, cudaStream_t src) {
  if (n < 0) throw StructuralError("ldlt_factor: negative dimension");
  auto f = std::unique_ptr<Ldlt>(new Ldlt());
  f->n_ = n;
  if (n == 0) return f;
  if (device < 0) {
    if (cudaGetDevice(&device) != cudaSuccess) {
      cudaGetLastError();
      throw DeviceError("no CUDA device available");
    }
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw DeviceError("no CUDA device available");
  }
  f->dev_ = device;
  DeviceGuard g(device);
  cudaStream_t st;
  PhaseTimer pt;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  f->stream_ = st;
  const size_t bytes = sizeof(double) * static_cast<size_t>(n) * n;
  f->palloc(&f->d_fact_, bytes);
  f->palloc(&f->d_vec_, sizeof(double) * (4 * n + kScal));  // rs | scale | cmax | x ... | scalars
  f->palloc(&f->d_rhs_, sizeof(double) * n);
  if (on_device) {
    // try_mat = A + delta_w I (head) - delta_c I (tail), ipm.cpp:529-536:
    // the shifts only when non-zero, one rounding each, as the reference
    if (src) CK(cudaStreamSynchronize(src));
    CK(cudaMemcpyAsync(f->d_fact_, a, bytes, cudaMemcpyDeviceToDevice, st));
    if (delta_w != 0.0 || delta_c != 0.0) {
      ldlt_shift_diag_kernel<<<blocks_for(n, 256), 256, 0, st>>>(f->d_fact_, n, n_var, delta_w, delta_c);
      CK(cudaGetLastError());
    }
  } else {
    CK(cudaMemcpyAsync(f->d_fact_, a, bytes, cudaMemcpyHostToDevice, st));
  }
  double* rs = f->d_vec_;
  double* scale = rs + n;
  double* cmax = scale + n;
  double* scal = f->d_vec_ + 4 * n;  // 8 scalars

  pt.mark("setup+upload", st);
  // checks (linalg.cpp:45-71) and Ruiz equilibration (linalg.cpp:72-99):
  // one cooperative launch, one host round trip
  CK(cudaMemsetAsync(scal, 0, sizeof(double) * kScal, st));
  {
    int sms_p = 0, per_p = 0;
    CK(cudaDeviceGetAttribute(&sms_p, cudaDevAttrMultiProcessorCount, device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_p, ldlt_prep_kernel, 256, 0));
    const int g = std::max(1, std::min(sms_p * std::max(per_p, 1), blocks_for(n * n, 256)));
    double* ap = f->d_fact_;
    int64_t nn = n;
    void* pargs[] = {&ap, &nn, &rs, &scale, &cmax, &scal};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ldlt_prep_kernel), dim3(g), dim3(256), pargs, 0, st));
  }
  double chk[kScal];
  f->scale_.assign(static_cast<size_t>(n), 1.0);
  CK(cudaMemcpyAsync(chk, scal, sizeof(chk), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(f->scale_.data(), scale, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (chk[2] > 0) throw NumericError("ldlt_factor: matrix contains NaN or Inf");
  if (chk[1] > 1e-12 * std::max(1.0, chk[0]))
    throw StructuralError("ldlt_factor: matrix is not symmetric (max deviation " + std::to_string(chk[1]) + ")");
  pt.mark("checks", st);
  f->zero_thresh_ = 1e-11 * chk[3];
  pt.mark("ruiz", st);
  if (keep_input) {
    f->palloc(&f->d_input_, bytes);
    CK(cudaMemcpyAsync(f->d_input_, f->d_fact_, bytes, cudaMemcpyDeviceToDevice, st));
  }

  auto classify = [&](double eig) {
    if (std::fabs(eig) <= f->zero_thresh_) ++f->n_zero_;
    else if (eig > 0.0) ++f->n_pos_;
    else ++f->n_neg_;
  };
  auto classify_2x2 = [&](double p, double q, double r) {
    const double mid = 0.5 * (p + r), rad = std::hypot(0.5 * (p - r), q);
    classify(mid + rad);
    classify(mid - rad);
  };
  pt.mark("keep-input", st);
  if (n <= kNativeMaxN) {
    // ---- native Bunch-Kaufman: one cooperative launch ----
    f->native_ = true;
    int sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    // blocked grid kernel: panel width (GBOPT_LDLT_GRID_NB; 0 = unblocked
    // left-looking, every column update spanning all previous columns)
    int grid_nb = 64;
    if (const char* e = std::getenv("GBOPT_LDLT_GRID_NB")) grid_nb = std::max(0, std::min(std::atoi(e), bk::kMaxGridNb));
    // the unblocked mode keeps an n-long vector in shared memory; blocked
    // panels need only the panel's columns (bk_factor_kernel)
    int smem_cap = 0;
    CK(cudaDeviceGetAttribute(&smem_cap, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    if (grid_nb == 0 && 8 * (n + 64) > smem_cap) grid_nb = 64;
    const int64_t v_doubles = grid_nb > 0 ? grid_nb + 4 : n;
    const size_t smem =
        sizeof(double) * static_cast<size_t>(std::max<int64_t>({v_doubles, bk::trailing_smem_doubles(grid_nb), 32 * 33}));
    CK(cudaFuncSetAttribute(bk::bk_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bk::bk_factor_kernel, bk::kThreads, smem));
    if (per_sm < 1) throw DeviceError("ldlt_factor: the Bunch-Kaufman kernel does not fit on an SM");
    // whole waves only (a partial second wave leaves SMs with twice the work):
    // one CTA per SM while that is at most 3 rows per warp, else every
    // co-resident CTA; at most one row per warp.  Barriers and the maxima
    // reduction grow with the CTA count (n = 2531: 148 CTAs 19.2 ms, 159 20.7;
    // 2812: 148 21.5, 176 23.3, 296 23.7; 5062: 159 50.3, 296 47.5; 10125:
    // 148 134, 296 123)
    const int64_t wave1 = n <= static_cast<int64_t>(sms) * bk::kWarps * 3 ? sms : static_cast<int64_t>(sms) * per_sm;
    int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(wave1, (n + bk::kWarps - 1) / bk::kWarps)));
    if (const char* e = std::getenv("GBOPT_LDLT_GRID_CTAS")) grid = std::max(1, std::min(grid, std::atoi(e)));
    f->ldl_ = (n + 1) / 2 * 2;  // 16-byte rows
    const size_t lbytes = sizeof(double) * static_cast<size_t>(n) * f->ldl_;
    f->palloc(&f->d_l_, 2 * lbytes);  // L | W = L D
    CK(cudaMemsetAsync(f->d_l_, 0, 2 * lbytes, st));
    int solve_per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&solve_per_sm, bk::bk_solve_kernel, bk::kThreads, 0));
    f->solve_grid_ = std::max(1, std::min(sms * std::max(solve_per_sm, 1), 32 * bk::kSlices / bk::kWarps));
    // d | e | w | wr | z (solve scratch) | w2 | maxima (part, part3, part2; the solve's partials)
    f->palloc(&f->d_bk_, sizeof(double) * (6 * static_cast<size_t>(n) +
                                                std::max<size_t>({6 * static_cast<size_t>(grid), 32 * bk::kSlices,
                                                                  32 * static_cast<size_t>(f->solve_grid_)})));
    f->palloc(&f->d_bki_, sizeof(int) * 2 * static_cast<size_t>(n));
    bk_iota_kernel<<<blocks_for(n, 256), 256, 0, st>>>(f->d_bki_ + n, n);
    CK(cudaGetLastError());
    bk::Factor F;
    F.a = f->d_fact_;
    F.l = f->d_l_;
    F.wd = f->d_l_ + static_cast<size_t>(n) * f->ldl_;
    F.d = f->d_bk_;
    F.e = F.d + n;
    F.w = F.e + n;
    F.wr = F.w + n;
    F.w2 = F.wr + 2 * n;  // (z at wr + n is the solve's scratch)
    F.part = F.w2 + n;
    F.part3 = F.part + 2 * grid;
    F.part2 = F.part3 + 2 * grid;
    F.piv = f->d_bki_;
    F.perm = f->d_bki_ + n;
    F.n = static_cast<int>(n);
    F.ldl = static_cast<int>(f->ldl_);
    F.nb = grid_nb;
    F.eps = f->zero_thresh_;
    F.trace = nullptr;
    CK(cudaMemsetAsync(F.e, 0, sizeof(double) * n, st));
    // Kernel choice (GBOPT_LDLT_KERNEL = panel | cpanel | cluster | grid forces one):
    //   panel   (ldlt_bkp.cuh): blocked; CTA 0 factors nb-column panels in
    //           shared memory, the grid applies rank-nb updates -- n <= 2048
    //           when a panel of nb >= 4 columns fits in shared memory;
    //   cpanel  (ldlt_bkq.cuh): blocked; an 8-CTA cluster factors each panel,
    //           a grid launch applies the update + the panel's permutation on
    //           the FP64 tensor pipe -- the default for 2048 < n <= 8500;
    //   cluster (ldlt_bkc.cuh): the lower triangle in one cluster's shared
    //           memory, one pivot per step;
    //   grid    (ldlt_bk.cuh):  left-looking, every SM, any n <= 20000.
    const char* env_k = std::getenv("GBOPT_LDLT_KERNEL");
    const std::string want = env_k ? env_k : "";
    int smem_optin_dev = 0;
    CK(cudaDeviceGetAttribute(&smem_optin_dev, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    int pnb = 0;
    {
      cudaFuncAttributes pa = {};
      CK(cudaFuncGetAttributes(&pa, bkp::bkp_factor_kernel));
      const int64_t avail = smem_optin_dev - static_cast<int64_t>(pa.sharedSizeBytes);
      for (int nb = bkp::kMaxNb; nb >= 4; --nb)
        if (bkp::smem_bytes(static_cast<int>(n), nb) <= avail) {
          pnb = nb;
          break;
        }
    }
    // cpanel (ldlt_bkq.cuh): per panel one 8-CTA cluster launch factors it
    // (rows spread over the cluster's shared memory), one grid launch applies
    // the rank-nb update and the panel's permutation on the FP64 tensor pipe
    // measured crossovers (tools/ldlt_split.py, profiles/r02_ldlt_kernels.md).
    // The cluster-panel kernel's per-pivot cost follows the box's DSMEM /
    // cluster-barrier latency (the same build: dim 4500 26.6 ms on one box,
    // 31.4 on another), the other kernels' does not; the range below wins on
    // both: the one-CTA panel up to its n = 2048 (1687: 8.9 ms vs cpanel
    // 7.8 / 9.5), cpanel up to 8500 (4500: 26.6 / 31.4 vs grid 40; 7987: 71 /
    // 79 vs 83; 9000: 94 / 102 vs 97)
    constexpr int64_t kCpanelMinN = 2048, kCpanelMaxN = 8500;
    const bool cpanel_default = want.empty() && n > kCpanelMinN && n <= kCpanelMaxN;
    int qnb = 0, qctas = 0;
    if ((want == "cpanel" || cpanel_default) && n <= bkq::kMaxN) {
      // panel width nb (<= 32) the cluster's shared memory allows, and whether
      // such a cluster can be resident; 8 CTAs unless GBOPT_LDLT_CPANEL_CTAS=16
      auto try_ctas = [&](auto kern, int ctas) -> int {
        cudaFuncAttributes qa = {};
        if (cudaFuncGetAttributes(&qa, kern) != cudaSuccess) return 0;
        const int64_t avail = smem_optin_dev - static_cast<int64_t>(qa.sharedSizeBytes);
        int nb = 0;
        for (int w = bkq::kMaxNb; w >= 4 && !nb; --w)
          if (bkq::smem_bytes(static_cast<int>(n), w, ctas) <= avail) nb = w;
        if (!nb || n > static_cast<int64_t>(ctas) * bkq::kThreads * bkq::kR) return 0;
        const int qsmem = static_cast<int>(bkq::smem_bytes(static_cast<int>(n), nb, ctas));
        if (ctas > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
          return 0;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, qsmem) != cudaSuccess) return 0;
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(ctas);
        q.blockDim = dim3(bkq::kThreads);
        q.dynamicSmemBytes = static_cast<size_t>(qsmem);
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kern, &q) != cudaSuccess) clusters = 0;
        return clusters >= 1 ? nb : 0;
      };
      const char* env_c = std::getenv("GBOPT_LDLT_CPANEL_CTAS");
      const int force_c = env_c ? std::atoi(env_c) : 0;
      if (force_c != 16) {
        qnb = try_ctas(bkq::bkq_panel_kernel<8>, 8);
        qctas = qnb ? 8 : 0;
      }
      // (16 CTAs measured slower where tried: the wider cluster barrier and
      // record reads cost more per pivot than nb = 32 saves in update traffic
      // -- dim 4500 42.0 vs 26.6 ms, 11250 165 vs 168; profiles/r02_ldlt_kernels.md)
      if (force_c == 16) {
        const int nb16 = try_ctas(bkq::bkq_panel_kernel<16>, 16);
        qnb = nb16;
        qctas = nb16 ? 16 : 0;
      }
      cudaGetLastError();
      if (qnb > 0)
        CK(cudaFuncSetAttribute(bkq::bkq_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                bkq::kUpdSmem));
    }
    const bool use_cpanel = qnb > 0;
    const bool use_panel = use_cpanel || (pnb > 0 && n <= bkp::kThreads * bkp::kMaxRowsPerThread &&
                                          ((want.empty() && !cpanel_default) || want == "panel"));
    f->panel_ = use_panel;
    if (use_cpanel) {
      const size_t qsmem = static_cast<size_t>(bkq::smem_bytes(static_cast<int>(n), qnb, qctas));
      // pan_w | pan_l | the second n x n buffer | orig_a, orig_b, locg, ctl
      const size_t nn = static_cast<size_t>(n);
      f->palloc(&f->d_pan_, sizeof(double) * (2 * bkq::kMaxNb * nn + nn * nn + 2 * nn + 8));
      bkq::Params P;
      P.a = f->d_fact_;
      P.lcols = f->d_l_ + static_cast<size_t>(n) * f->ldl_;
      P.l = f->d_l_;
      P.ldl = static_cast<int>(f->ldl_);
      P.d = F.d;
      P.e = F.e;
      P.piv = F.piv;
      P.perm = F.perm;
      P.pan_w = f->d_pan_;
      P.pan_l = P.pan_w + bkq::kMaxNb * nn;
      P.a2 = P.pan_l + bkq::kMaxNb * nn;
      P.orig_a = reinterpret_cast<int*>(P.a2 + nn * nn);
      P.orig_b = P.orig_a + nn;
      P.locg = P.orig_b + nn;
      P.ctl = P.locg + nn;
      P.n = static_cast<int>(n);
      P.nb = qnb;
      P.eps = f->zero_thresh_;
      P.trace = nullptr;
      cudaEvent_t c0 = nullptr, c1 = nullptr;
      const bool timing = std::getenv("GBOPT_LDLT_TIMING") != nullptr;
      if (timing) {
        CK(cudaMalloc(&P.trace, sizeof(long long) * 16));
        CK(cudaMemset(P.trace, 0, sizeof(long long) * 16));
        CK(cudaEventCreate(&c0));
        CK(cudaEventCreate(&c1));
        CK(cudaEventRecord(c0, st));
      }
      // each panel is >= nb - 1 columns wide (a 2x2 block that does not fit
      // opens the next one); surplus launches return at once (k0 >= n)
      const int64_t panels = (n + qnb - 2) / (qnb - 1);
      bkq::bkq_init_kernel<<<blocks_for(n, 256), 256, 0, st>>>(P);
      CK(cudaGetLastError());
      for (int64_t pi = 0; pi < panels; ++pi) {
        double* A = pi & 1 ? P.a2 : P.a;
        double* A2 = pi & 1 ? P.a : P.a2;
        const int* orig = pi & 1 ? P.orig_b : P.orig_a;
        int* orig2 = pi & 1 ? P.orig_a : P.orig_b;
        if (qctas == 16)
          bkq::bkq_panel_kernel<16><<<16, bkq::kThreads, qsmem, st>>>(P, A, orig, orig2);
        else
          bkq::bkq_panel_kernel<8><<<8, bkq::kThreads, qsmem, st>>>(P, A, orig, orig2);
        bkq::bkq_update_kernel<<<3 * sms, bkq::kUpdThreads, bkq::kUpdSmem, st>>>(P, A, A2);
      }
      bkq::bkq_gather_kernel<<<static_cast<int>(std::min<int64_t>(n, 4 * sms)), 256, 0, st>>>(P);
      CK(cudaGetLastError());
      if (timing) {
        CK(cudaEventRecord(c1, st));
        CK(cudaEventSynchronize(c1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c0, c1));
        long long tr[16];
        CK(cudaMemcpy(tr, P.trace, sizeof(tr), cudaMemcpyDeviceToHost));
        CK(cudaFree(P.trace));
        std::fprintf(stderr, "ldlt: cpanel update clocks: issue %lld, wait %lld, fma %lld, stores %lld\n", tr[10],
                     tr[11], tr[12], tr[13]);
        std::fprintf(stderr,
                     "ldlt: n %lld cpanel nb %d ctas %d, %lld panel launches %.3f ms; panel CTA-0 clocks: zs %lld, column %lld, "
                     "cluster sync %lld, decide %lld, column r %lld, pivot %lld, publish %lld\n",
                     static_cast<long long>(n), qnb, qctas, static_cast<long long>(panels), ms, tr[0], tr[1], tr[2], tr[3],
                     tr[4], tr[5], tr[6]);
        cudaEventDestroy(c0);
        cudaEventDestroy(c1);
      }
    }
    if (use_panel && !use_cpanel) {
      const size_t psmem = static_cast<size_t>(bkp::smem_bytes(static_cast<int>(n), pnb));
      CK(cudaFuncSetAttribute(bkp::bkp_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(psmem)));
      int pper = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pper, bkp::bkp_factor_kernel, bkp::kThreads, psmem));
      if (pper < 1) throw DeviceError("ldlt_factor: the blocked kernel does not fit on an SM");
      f->palloc(&f->d_pan_, sizeof(double) * (bkp::kMaxNb * static_cast<size_t>(n) + 3 * bkp::kMaxNb + 8));
      bkp::Params P;
      P.a = f->d_fact_;
      P.lcols = f->d_l_ + static_cast<size_t>(n) * f->ldl_;  // the W half of d_l_: n x n scratch
      P.l = f->d_l_;
      P.ldl = static_cast<int>(f->ldl_);
      P.d = F.d;
      P.e = F.e;
      P.piv = F.piv;
      P.perm = F.perm;
      P.pan_w = f->d_pan_;
      P.pan_g = f->d_pan_ + bkp::kMaxNb * static_cast<size_t>(n);
      P.ctl = reinterpret_cast<int*>(P.pan_g + 3 * bkp::kMaxNb);
      P.n = static_cast<int>(n);
      P.nb = pnb;
      P.eps = f->zero_thresh_;
      P.trace = nullptr;
      void* pargs[] = {&P};
      cudaEvent_t c0 = nullptr, c1 = nullptr;
      const bool timing = std::getenv("GBOPT_LDLT_TIMING") != nullptr;
      if (timing) {
        CK(cudaMalloc(&P.trace, sizeof(long long) * 8));
        CK(cudaEventCreate(&c0));
        CK(cudaEventCreate(&c1));
        CK(cudaEventRecord(c0, st));
      }
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bkp::bkp_factor_kernel), dim3(sms * std::min(pper, 1)),
                                     dim3(bkp::kThreads), pargs, psmem, st));
      if (timing) {
        CK(cudaEventRecord(c1, st));
        CK(cudaEventSynchronize(c1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c0, c1));
        long long tr[8];
        CK(cudaMemcpy(tr, P.trace, sizeof(tr), cudaMemcpyDeviceToHost));
        CK(cudaFree(P.trace));
        std::fprintf(stderr,
                     "ldlt: n %lld panel nb %d bkp_factor_kernel %.3f ms; CTA-0 clocks: column %lld, column r %lld, "
                     "pivot %lld, publish %lld, sync %lld, update %lld, sync %lld, loop %lld\n",
                     static_cast<long long>(n), pnb, ms, tr[0], tr[1], tr[2], tr[3], tr[4], tr[5], tr[6], tr[7]);
        cudaEventDestroy(c0);
        cudaEventDestroy(c1);
      }
    }
    // small n: the whole lower triangle in one cluster's shared memory
    // (ldlt_bkc.cuh), one cluster barrier per pivot
    const char* env_cl = std::getenv("GBOPT_LDLT_CLUSTER");
    bool use_cluster = !use_panel && (want.empty() || want == "cluster") &&
                       (env_cl == nullptr || std::atoi(env_cl) != 0);
    const int64_t cl_smem = bkc::smem_bytes(static_cast<int>(n));
    int smem_optin = 0;
    CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    cudaFuncAttributes fa = {};
    CK(cudaFuncGetAttributes(&fa, bkc::bkc_factor_kernel));
    smem_optin -= static_cast<int>(fa.sharedSizeBytes);  // dynamic part available beside the static arrays
    // measured crossover (tools/ldlt_split.py, GBOPT_LDLT_CLUSTER=0/1): the
    // cluster kernel wins below ~800 (n = 112: 0.37 vs 1.06 ms, 337: 1.57 vs
    // 2.35, 562: 3.41 vs 4.03) and ties at 804 (6.21 ms each)
    constexpr int64_t kClusterMaxN = 800;
    use_cluster = use_cluster && cl_smem <= smem_optin && (want == "cluster" || n <= kClusterMaxN);
    if (use_cluster) {
      // function attributes are per device: check (and set) once per device and thread
      static thread_local std::map<int, int> cluster_ok_by_dev;
      int& cluster_ok = cluster_ok_by_dev.try_emplace(device, -1).first->second;
      if (cluster_ok < 0) {
        cluster_ok = 0;
        if (cudaFuncSetAttribute(bkc::bkc_factor_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(bkc::bkc_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin) ==
                cudaSuccess) {
          cudaLaunchConfig_t q = {};
          q.gridDim = dim3(bkc::kCtas);
          q.blockDim = dim3(bkc::kThreads);
          q.dynamicSmemBytes = static_cast<size_t>(smem_optin);
          cudaLaunchAttribute qa[1];
          qa[0].id = cudaLaunchAttributeClusterDimension;
          qa[0].val.clusterDim.x = bkc::kCtas;
          qa[0].val.clusterDim.y = 1;
          qa[0].val.clusterDim.z = 1;
          q.attrs = qa;
          q.numAttrs = 1;
          int clusters = 0;
          const cudaError_t oe = cudaOccupancyMaxActiveClusters(&clusters, bkc::bkc_factor_kernel, &q);
          if (oe == cudaSuccess && clusters > 0) cluster_ok = 1;
          if (std::getenv("GBOPT_LDLT_TIMING"))
            std::fprintf(stderr, "ldlt: cluster occupancy query %s, %d clusters\n", cudaGetErrorString(oe), clusters);
        } else if (std::getenv("GBOPT_LDLT_TIMING")) {
          std::fprintf(stderr, "ldlt: cluster attributes rejected: %s\n", cudaGetErrorString(cudaGetLastError()));
        }
        cudaGetLastError();
      }
      use_cluster = cluster_ok == 1;
    }
    f->cluster_ = use_cluster;
    if (use_cluster) {
      bkc::Params P;
      P.a = f->d_fact_;
      P.l = f->d_l_;
      P.ldl = static_cast<int>(f->ldl_);
      P.d = F.d;
      P.e = F.e;
      P.piv = F.piv;
      P.perm = F.perm;
      P.n = static_cast<int>(n);
      P.eps = f->zero_thresh_;
      P.trace = nullptr;
      const bool timing = std::getenv("GBOPT_LDLT_TIMING") != nullptr;
      if (timing) {
        CK(cudaMalloc(&P.trace, sizeof(long long) * 6 * n));
        CK(cudaMemsetAsync(P.trace, 0, sizeof(long long) * 6 * n, st));
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(bkc::kCtas);
      cfg.blockDim = dim3(bkc::kThreads);
      cfg.dynamicSmemBytes = static_cast<size_t>(cl_smem);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = bkc::kCtas;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaEvent_t c0 = nullptr, c1 = nullptr;
      if (timing) {
        CK(cudaEventCreate(&c0));
        CK(cudaEventCreate(&c1));
        CK(cudaEventRecord(c0, st));
      }
      CK(cudaLaunchKernelEx(&cfg, bkc::bkc_factor_kernel, P));
      if (timing) {
        CK(cudaEventRecord(c1, st));
        CK(cudaEventSynchronize(c1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c0, c1));
        std::fprintf(stderr, "ldlt: n %lld cluster bkc_factor_kernel %.3f ms (smem %lld B)\n",
                     static_cast<long long>(n), ms, static_cast<long long>(cl_smem));
        cudaEventDestroy(c0);
        cudaEventDestroy(c1);
        std::vector<long long> tr(6 * static_cast<size_t>(n));
        CK(cudaMemcpy(tr.data(), P.trace, sizeof(long long) * tr.size(), cudaMemcpyDeviceToHost));
        CK(cudaFree(P.trace));
        double ph[5] = {0, 0, 0, 0, 0};
        int steps = 0;
        for (int64_t k = 0; k < n; ++k) {
          const long long* t = tr.data() + 6 * k;
          if (t[0] == 0 || t[5] == 0) continue;
          for (int i = 0; i < 5; ++i) ph[i] += static_cast<double>(t[i + 1] - t[i]);
          ++steps;
        }
        if (steps)
          std::fprintf(stderr, "ldlt: cluster per-step clocks (%d steps): decide %.0f swap %.0f update %.0f bcast %.0f "
                       "barrier %.0f\n", steps, ph[0] / steps, ph[1] / steps, ph[2] / steps, ph[3] / steps,
                       ph[4] / steps);
      }
    }
    void* args[] = {&F};
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    const bool timing = std::getenv("GBOPT_LDLT_TIMING") != nullptr;
    if (timing) {
      CK(cudaEventCreate(&t0));
      CK(cudaEventCreate(&t1));
      CK(cudaEventRecord(t0, st));
      CK(cudaMalloc(&F.trace, sizeof(long long) * 16));
      CK(cudaMemsetAsync(F.trace, 0, sizeof(long long) * 16, st));
    }
    if (!use_cluster && !use_panel)
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bk::bk_factor_kernel), dim3(grid), dim3(bk::kThreads),
                                     args, smem, st));
    if (timing) {
      CK(cudaEventRecord(t1, st));
      CK(cudaEventSynchronize(t1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, t0, t1));
      long long tr[16] = {};
      if (!use_cluster && !use_panel) CK(cudaMemcpy(tr, F.trace, sizeof(tr), cudaMemcpyDeviceToHost));
      CK(cudaFree(F.trace));
      std::fprintf(stderr, "ldlt: n %lld grid %d per_sm %d nb %d bk_factor_kernel %.3f ms; CTA-0 clocks: trailing "
                   "updates %lld of %lld; phases (clocks / count): column k %lld/%lld, decide %lld/%lld, column r "
                   "%lld/%lld, look-ahead %lld/%lld, interchange+L %lld/%lld\n",
                   static_cast<long long>(n), grid, per_sm, grid_nb, ms, tr[0], tr[1], tr[2], tr[7], tr[3], tr[8],
                   tr[4], tr[9], tr[5], tr[10], tr[6], tr[11]);
      cudaEventDestroy(t0);
      cudaEventDestroy(t1);
    }
    pt.mark("factor", st);
    std::vector<double> dd(static_cast<size_t>(n)), ee(static_cast<size_t>(n));
    std::vector<int> pv(static_cast<size_t>(n));
    CK(cudaMemcpyAsync(dd.data(), F.d, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ee.data(), F.e, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pv.data(), F.piv, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t k = 0; k < n;) {
      if (pv[static_cast<size_t>(k)] == 1) {
        classify(dd[k]);
        k += 1;
      } else {
        classify_2x2(dd[k], ee[k], dd[k + 1]);
        k += 2;
      }
    }
    return f;
  }

  // Bunch-Kaufman on the device (lower; row-major == column-major here)
  cusolverDnHandle_t h = nullptr;
  CS(cusolverDnCreate(&h));
  f->handle_ = h;
  CS(cusolverDnSetStream(h, st));
  f->palloc(&f->d_ipiv_, sizeof(int) * n);
  f->palloc(&f->d_ipiv64_, sizeof(int64_t) * n);
  f->palloc(&f->d_info_, sizeof(int));
  int lwork = 0;
  CS(cusolverDnDsytrf_bufferSize(h, static_cast<int>(n), f->d_fact_, static_cast<int>(n), &lwork));
  f->palloc(&f->d_work_, sizeof(double) * std::max(lwork, 1));
  CS(cusolverDnDsytrf(h, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), f->d_fact_, static_cast<int>(n), f->d_ipiv_,
                      f->d_work_, lwork, f->d_info_));
  // only the pivot blocks come back: diagonal and first subdiagonal
  std::vector<double> diag(static_cast<size_t>(n)), sub(static_cast<size_t>(n), 0.0);
  f->ipiv_.assign(static_cast<size_t>(n), 0);
  int info = 0;
  CK(cudaMemcpy2DAsync(diag.data(), sizeof(double), f->d_fact_, sizeof(double) * (n + 1), sizeof(double), n,
                       cudaMemcpyDeviceToHost, st));
  if (n > 1)
    CK(cudaMemcpy2DAsync(sub.data(), sizeof(double), f->d_fact_ + 1, sizeof(double) * (n + 1), sizeof(double), n - 1,
                         cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(f->ipiv_.data(), f->d_ipiv_, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&info, f->d_info_, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (info < 0) throw DeviceError("ldlt_factor: dsytrf rejected argument " + std::to_string(-info));
  std::vector<int64_t> ipiv64(f->ipiv_.begin(), f->ipiv_.end());
  CK(cudaMemcpyAsync(f->d_ipiv64_, ipiv64.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  for (int64_t k = 0; k < n;) {
    if (f->ipiv_[static_cast<size_t>(k)] > 0) {  // 1x1 block (LAPACK lower convention)
      classify(diag[k]);
      k += 1;
    } else {  // 2x2 block D(k:k+1, k:k+1), D(k+1,k) in the subdiagonal
      classify_2x2(diag[k], sub[k], diag[k + 1]);
      k += 2;
    }
  }
  size_t dws = 0, hws = 0;
  CS(cusolverDnXsytrs_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, 1, CUDA_R_64F, f->d_fact_, n, f->d_ipiv64_, CUDA_R_64F,
                                 f->d_rhs_, n, &dws, &hws));
  f->sws_dev_ = std::max<size_t>(dws, 8);
  f->sws_host_ = std::max<size_t>(hws, 8);
  f->palloc(&f->d_sbuf_, f->sws_dev_);
  CK(cudaStreamSynchronize(st));
  return f;
}

// in place on the device vector v: v <- (S A S)^{-1} v
void Ldlt::solve_factored(double* d_v) const {
  if (native_) {
    const double* d = d_bk_;
    double* z = d_bk_ + 4 * n_;
    double* part = d_bk_ + 6 * n_;  // the factor's maxima slots, >= 32 * max(kSlices, solve grid) doubles
    const double* l = d_l_;
    int ldl = static_cast<int>(ldl_), n = static_cast<int>(n_);
    const double* e = d + n_;
    const int* piv = d_bki_;
    const int* perm = d_bki_ + n_;
    const double* bb = d_v;
    double* x = d_v;
    // one CTA up to kCtaSolveMaxN (measured: tools/ldlt_solve_probe.py),
    // the grid-wide version beyond; GBOPT_LDLT_SOLVE = cta | grid forces one
    const char* env_s = std::getenv("GBOPT_LDLT_SOLVE");
    const bool cta = env_s ? std::string(env_s) == "cta" : n_ <= kCtaSolveMaxN;
    if (cta) {
      bk::bk_solve_cta_kernel<<<1, bk::kCtaThreads, 0, stream_>>>(l, ldl, d, e, piv, perm, n, bb, z, x);
      CK(cudaGetLastError());
      return;
    }
    void* args[] = {&l, &ldl, &d, &e, &piv, &perm, &n, &bb, &z, &x, &part};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bk::bk_solve_kernel), dim3(solve_grid_),
                                   dim3(bk::kThreads), args, 0, stream_));
    return;
  }
  auto h = static_cast<cusolverDnHandle_t>(handle_);
  std::vector<char> hbuf(sws_host_);
  CS(cusolverDnXsytrs(h, CUBLAS_FILL_MODE_LOWER, n_, 1, CUDA_R_64F, d_fact_, n_, d_ipiv64_, CUDA_R_64F, d_v, n_,
                      d_sbuf_, sws_dev_, hbuf.data(), sws_host_, d_info_));
}

std::vector<double> Ldlt::solve(const double* b, int64_t len) const {
  if (len != n_)
    throw StructuralError("ldlt_solve: right-hand side has size " + std::to_string(len) + ", expected " +
                          std::to_string(n_));
  if (n_zero_ > 0)
    throw SingularError("ldlt_solve: matrix is singular (" + std::to_string(n_zero_) + " zero pivots)");
  std::vector<double> bs(static_cast<size_t>(n_));
  for (int64_t i = 0; i < n_; ++i) bs[i] = scale_[i] * b[i];
  return solve_scaled(std::move(bs));
}

std::vector<double> Ldlt::solve_device(const double* d_b, int64_t len, cudaStream_t src) const {
  if (len != n_)
    throw StructuralError("ldlt_solve: right-hand side has size " + std::to_string(len) + ", expected " +
                          std::to_string(n_));
  if (n_zero_ > 0)
    throw SingularError("ldlt_solve: matrix is singular (" + std::to_string(n_zero_) + " zero pivots)");
  std::vector<double> b(static_cast<size_t>(n_));
  if (n_ > 0) {
    DeviceGuard g(dev_);
    CK(cudaMemcpyAsync(b.data(), d_b, sizeof(double) * n_, cudaMemcpyDeviceToHost, src));
    CK(cudaStreamSynchronize(src));
  }
  return solve(b.data(), len);
}

// x = S (S A S)^{-1} bs for bs = S b (host), refined as the reference
std::vector<double> Ldlt::solve_scaled(std::vector<double> bs) const {
  const int64_t n = n_;
  std::vector<double> x(static_cast<size_t>(n));
  if (n == 0) return x;
  DeviceGuard g(dev_);
  cudaStream_t st = stream_;
  double b_norm = 0.0;
  for (double v : bs) b_norm = std::max(b_norm, std::fabs(v));
  double* d_bs = d_vec_;            // reuse: rs slot
  double* d_x = d_vec_ + 2 * n;     // cmax slot
  double* d_r = d_vec_ + 3 * n;
  double* scal = d_vec_ + 4 * n;
  CK(cudaMemcpyAsync(d_bs, bs.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_x, d_bs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  solve_factored(d_x);
  if (d_input_) {
    // refinement (linalg.cpp:403-435): residuals on the device, round
    // control on the host from two scalars per round
    const double a_max = zero_thresh_ / 1e-11;
    const double eps = std::numeric_limits<double>::epsilon();
    double* d_best = d_rhs_;
    double best_res = std::numeric_limits<double>::infinity();
    CK(cudaMemcpyAsync(d_best, d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    for (int round = 0; round < 10; ++round) {
      CK(cudaMemsetAsync(scal, 0, sizeof(double) * 2, st));
      ldlt_residual_kernel<<<blocks_for(n, 8), 256, 0, st>>>(d_input_, n, d_x, d_bs, d_r, scal);
      CK(cudaGetLastError());
      double rr[2];
      CK(cudaMemcpyAsync(rr, scal, sizeof(rr), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (!(rr[0] < best_res)) break;
      best_res = rr[0];
      CK(cudaMemcpyAsync(d_best, d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      if (rr[0] <= eps * (b_norm + a_max * rr[1])) break;
      solve_factored(d_r);
      refine_add_kernel_launch(d_x, d_r, n, st);
    }
    CK(cudaMemcpyAsync(x.data(), d_best, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(x.data(), d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) x[i] *= scale_[i];
  return x;
}

namespace {
__global__ void ldlt_axpy_kernel(double* __restrict__ x, const double* __restrict__ r, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] += r[i];
}
}  // namespace

void Ldlt::refine_add_kernel_launch(double* d_x, const double* d_r, int64_t n, cudaStream_t st) const {
  ldlt_axpy_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, st>>>(d_x, d_r, n);
  CK(cudaGetLastError());
}

}  // namespace gbb
