// Symmetric-indefinite LDL^T on the GPU for the KKT systems of the
// interior-point caller (reference
// proj/include/gbopt/linalg.hpp:24-78, proj/src/linalg.cpp:39-438).
//
// Same contract as the reference ldlt_factor / LdltFactorization:
//   * checks: finite entries (NumericError), symmetry to
//     1e-12 * max(1, max|A|) (StructuralError)            linalg.cpp:45-71
//   * symmetric Ruiz equilibration, <= 20 rounds, tol 0.01  linalg.cpp:72-99
//   * Bunch-Kaufman factorisation P S A S P^T = L D L^T of the equilibrated
//     matrix -- here cuSOLVER's dsytrf on the device (a plain library
//     factorisation: this row is outside the oracle's hot path)
//   * inertia from the 1x1 / 2x2 pivot blocks with zero threshold
//     1e-11 * max|S A S|                                     linalg.cpp:101-120
//   * solve: refuses singular factorizations (SingularError); x = S y with
//     S A S y = S b, iterative refinement while the residual shrinks, at
//     most 10 rounds, returning the best iterate              linalg.cpp:393-438
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "device_net.hpp"
#include "ldlt.hpp"

namespace gbb {

namespace {

void cs_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS)
    throw DeviceError(std::string("cuSOLVER error in ") + what + ": " + std::to_string(static_cast<int>(s)));
}
#define CK(x) cuda_check((x), #x)
#define CS(x) cs_check((x), #x)

}  // namespace

Ldlt::~Ldlt() {
  if (dev_ >= 0) {
    DeviceGuard g(dev_);
    if (d_fact_) cudaFree(d_fact_);
    if (d_ipiv_) cudaFree(d_ipiv_);
    if (d_work_) cudaFree(d_work_);
    if (d_info_) cudaFree(d_info_);
    if (d_rhs_) cudaFree(d_rhs_);
    if (handle_) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(handle_));
    if (stream_) cudaStreamDestroy(stream_);
  }
}

std::unique_ptr<Ldlt> Ldlt::factor(const double* a, int64_t n, bool keep_input, int device) {
  if (n < 0) throw StructuralError("ldlt_factor: negative dimension");
  for (int64_t i = 0; i < n * n; ++i)
    if (!std::isfinite(a[i])) throw NumericError("ldlt_factor: matrix contains NaN or Inf");
  double amax = 0.0;
  for (int64_t i = 0; i < n * n; ++i) amax = std::max(amax, std::fabs(a[i]));
  const double sym_tol = 1e-12 * std::max(1.0, amax);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < i; ++j) {
      const double dev = std::fabs(a[i * n + j] - a[j * n + i]);
      if (dev > sym_tol)
        throw StructuralError("ldlt_factor: matrix is not symmetric (max deviation " + std::to_string(dev) + ")");
    }

  auto f = std::unique_ptr<Ldlt>(new Ldlt());
  f->n_ = n;
  // Symmetric Ruiz equilibration (linalg.cpp:72-99).
  std::vector<double> bal(a, a + n * n);
  f->scale_.assign(static_cast<size_t>(n), 1.0);
  {
    constexpr int kRuizMaxRounds = 20;
    constexpr double kRuizTol = 0.01;
    std::vector<double> rs(static_cast<size_t>(n));
    for (int round = 0; round < kRuizMaxRounds; ++round) {
      double dev = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        double cmax = 0.0;
        for (int64_t k = 0; k < n; ++k) cmax = std::max(cmax, std::fabs(bal[k * n + i]));
        rs[i] = cmax > 0.0 ? 1.0 / std::sqrt(cmax) : 1.0;
        if (cmax > 0.0) dev = std::max(dev, std::fabs(cmax - 1.0));
      }
      if (dev <= kRuizTol) break;
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) bal[i * n + j] *= rs[i] * rs[j];
      for (int64_t i = 0; i < n; ++i) f->scale_[i] *= rs[i];
    }
  }
  double bmax = 0.0;
  for (double v : bal) bmax = std::max(bmax, std::fabs(v));
  f->zero_thresh_ = 1e-11 * (n > 0 ? bmax : 0.0);
  if (keep_input) f->input_ = bal;
  if (n == 0) return f;

  // Device factorisation (lower triangle; row-major == column-major for a
  // symmetric matrix).
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
  CK(cudaStreamCreateWithFlags(&f->stream_, cudaStreamNonBlocking));
  cusolverDnHandle_t h = nullptr;
  CS(cusolverDnCreate(&h));
  f->handle_ = h;
  CS(cusolverDnSetStream(h, f->stream_));
  const size_t bytes = sizeof(double) * static_cast<size_t>(n) * n;
  CK(cudaMalloc(&f->d_fact_, bytes));
  CK(cudaMalloc(&f->d_ipiv_, sizeof(int) * n));
  CK(cudaMalloc(&f->d_info_, sizeof(int)));
  CK(cudaMalloc(&f->d_rhs_, sizeof(double) * n));
  CK(cudaMemcpyAsync(f->d_fact_, bal.data(), bytes, cudaMemcpyHostToDevice, f->stream_));
  int lwork = 0;
  CS(cusolverDnDsytrf_bufferSize(h, static_cast<int>(n), f->d_fact_, static_cast<int>(n), &lwork));
  CK(cudaMalloc(&f->d_work_, sizeof(double) * std::max(lwork, 1)));
  CS(cusolverDnDsytrf(h, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), f->d_fact_, static_cast<int>(n), f->d_ipiv_,
                      f->d_work_, lwork, f->d_info_));
  // D blocks and pivots back to the host for the inertia.
  std::vector<double> fact(static_cast<size_t>(n) * n);
  f->ipiv_.assign(static_cast<size_t>(n), 0);
  int info = 0;
  CK(cudaMemcpyAsync(fact.data(), f->d_fact_, bytes, cudaMemcpyDeviceToHost, f->stream_));
  CK(cudaMemcpyAsync(f->ipiv_.data(), f->d_ipiv_, sizeof(int) * n, cudaMemcpyDeviceToHost, f->stream_));
  CK(cudaMemcpyAsync(&info, f->d_info_, sizeof(int), cudaMemcpyDeviceToHost, f->stream_));
  CK(cudaStreamSynchronize(f->stream_));
  if (info < 0) throw DeviceError("ldlt_factor: dsytrf rejected argument " + std::to_string(-info));
  // column-major element (i, j) of the factor: fact[j * n + i]
  auto D = [&](int64_t i, int64_t j) { return fact[static_cast<size_t>(j * n + i)]; };
  auto classify = [&](double eig) {
    if (std::fabs(eig) <= f->zero_thresh_) ++f->n_zero_;
    else if (eig > 0.0) ++f->n_pos_;
    else ++f->n_neg_;
  };
  for (int64_t k = 0; k < n;) {
    if (f->ipiv_[static_cast<size_t>(k)] > 0) {  // 1x1 block (LAPACK lower convention)
      classify(D(k, k));
      k += 1;
    } else {  // 2x2 block in rows/cols k, k+1
      const double p = D(k, k), q = D(k + 1, k), r = D(k + 1, k + 1);
      const double mid = 0.5 * (p + r), rad = std::hypot(0.5 * (p - r), q);
      classify(mid + rad);
      classify(mid - rad);
      k += 2;
    }
  }
  return f;
}

void Ldlt::solve_factored(std::vector<double>& x) const {
  DeviceGuard g(dev_);
  auto h = static_cast<cusolverDnHandle_t>(handle_);
  const int64_t n = n_;
  std::vector<int64_t> ipiv64(ipiv_.begin(), ipiv_.end());
  int64_t* d_ipiv64 = nullptr;
  CK(cudaMalloc(&d_ipiv64, sizeof(int64_t) * n));
  CK(cudaMemcpyAsync(d_ipiv64, ipiv64.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, stream_));
  CK(cudaMemcpyAsync(d_rhs_, x.data(), sizeof(double) * n, cudaMemcpyHostToDevice, stream_));
  size_t dws = 0, hws = 0;
  CS(cusolverDnXsytrs_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, 1, CUDA_R_64F, d_fact_, n, d_ipiv64, CUDA_R_64F, d_rhs_,
                                 n, &dws, &hws));
  void* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, std::max<size_t>(dws, 8)));
  std::vector<char> hbuf(std::max<size_t>(hws, 8));
  int* d_info = nullptr;
  CK(cudaMalloc(&d_info, sizeof(int)));
  CS(cusolverDnXsytrs(h, CUBLAS_FILL_MODE_LOWER, n, 1, CUDA_R_64F, d_fact_, n, d_ipiv64, CUDA_R_64F, d_rhs_, n, dbuf,
                      dws, hbuf.data(), hws, d_info));
  CK(cudaMemcpyAsync(x.data(), d_rhs_, sizeof(double) * n, cudaMemcpyDeviceToHost, stream_));
  CK(cudaStreamSynchronize(stream_));
  cudaFree(dbuf);
  cudaFree(d_info);
  cudaFree(d_ipiv64);
}

std::vector<double> Ldlt::solve(const double* b, int64_t len) const {
  if (len != n_)
    throw StructuralError("ldlt_solve: right-hand side has size " + std::to_string(len) + ", expected " +
                          std::to_string(n_));
  if (n_zero_ > 0)
    throw SingularError("ldlt_solve: matrix is singular (" + std::to_string(n_zero_) + " zero pivots)");
  const int64_t n = n_;
  std::vector<double> bs(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) bs[i] = scale_[i] * b[i];
  std::vector<double> x = bs;
  if (n > 0) solve_factored(x);
  if (!input_.empty() && n > 0) {
    double a_max = 0.0, b_norm = 0.0;
    for (double v : input_) a_max = std::max(a_max, std::fabs(v));
    for (double v : bs) b_norm = std::max(b_norm, std::fabs(v));
    constexpr int kMaxRounds = 10;
    const double eps = std::numeric_limits<double>::epsilon();
    std::vector<double> best_x = x, r(static_cast<size_t>(n));
    double best_res = std::numeric_limits<double>::infinity();
    for (int round = 0; round < kMaxRounds; ++round) {
      double res = 0.0, xn = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        double s = bs[i];
        const double* row = input_.data() + i * n;
        for (int64_t k = 0; k < n; ++k) s -= row[k] * x[k];
        r[i] = s;
        res = std::max(res, std::fabs(s));
        xn = std::max(xn, std::fabs(x[i]));
      }
      if (!(res < best_res)) break;  // stalled at this factorization's accuracy
      best_res = res;
      best_x = x;
      if (res <= eps * (b_norm + a_max * xn)) break;
      solve_factored(r);
      for (int64_t i = 0; i < n; ++i) x[i] += r[i];
    }
    x = best_x;
  }
  for (int64_t i = 0; i < n; ++i) x[i] *= scale_[i];
  return x;
}

}  // namespace gbb
