// Dense KKT assembly and inertia correction on the device (SURVEY §8f row
// f3; reference proj/src/ipm.cpp:466-557, declared at
// proj/include/gbopt/ipm.hpp:80-118).
//
// assemble_kkt (ipm.cpp:466-518) builds, per IPM iteration,
//   mat = [[H + Sigma + dw I, J^T], [J, -dc I]],  Sigma_ii = z_i / (x_i - lower_i)
//   rhs = [-grad_f - J^T lambda + mu / (x - lower); -g]
// from triplets (Hessian lower triangle mirrored on the fly, duplicates
// summed).  Here the pattern is analysed once on the host: every matrix
// element that receives triplet values gets the ordered list of its
// contributions, so one device thread per element sums them in the
// reference's triplet order starting from 0 -- the same additions in the
// same order, bit-identical -- and the diagonal terms follow in the
// reference's order (Hessian, then Sigma, then dw; the (2,2) block's 0 - dc).
// J^T lambda (ipm.cpp:33-42) likewise sums per column in triplet order with
// separately rounded products.  The matrix never leaves the device:
// inertia_correct (ipm.cpp:520-557) factors shifted copies of it with the
// native Bunch-Kaufman LDL^T (ldlt.cu) until the inertia is (n, m, 0).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "device_net.hpp"
#include "kkt.hpp"

namespace gbb {

namespace {

#define CK(x) cuda_check((x), #x)

constexpr double kDeltaC = 1e-8;     // ipm.cpp:23
constexpr double kDeltaCMax = 1e-2;  // ipm.cpp:24

// mat[target[t]] = sum of vals[src[p]] for p in [seg[t], seg[t+1]), in order
__global__ void kkt_scatter_kernel(const int64_t* __restrict__ target, const int32_t* __restrict__ seg,
                                   const int32_t* __restrict__ src, int64_t n_targets, const double* __restrict__ vals,
                                   double* __restrict__ mat) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_targets) return;
  double v = 0.0;
  for (int32_t p = seg[t]; p < seg[t + 1]; ++p) v = __dadd_rn(v, vals[src[p]]);
  mat[target[t]] = v;
}

// Diagonal terms and the right-hand side, one thread per row of the system.
// in = x | lower | z | grad_f | lambda | g | hess values | jac values
__global__ void kkt_diag_rhs_kernel(const double* __restrict__ in, int64_t n, int64_t m, size_t nnz_h,
                                    const int32_t* __restrict__ jt_seg, const int32_t* __restrict__ jt_src,
                                    const int32_t* __restrict__ jrow, double mu, double delta_w, double delta_c,
                                    double* __restrict__ mat, double* __restrict__ rhs) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t dim = n + m;
  if (i >= dim) return;
  const double* x = in;
  const double* lower = x + n;
  const double* z = lower + n;
  const double* grad = z + n;
  const double* lam = grad + n;
  const double* g = lam + m;
  const double* jv = g + m + nnz_h;
  if (i < n) {
    const bool bounded = isfinite(lower[i]);
    double d = mat[i * dim + i];
    if (bounded) d = __dadd_rn(d, __ddiv_rn(z[i], __dsub_rn(x[i], lower[i])));
    if (delta_w != 0.0) d = __dadd_rn(d, delta_w);
    mat[i * dim + i] = d;
    // jac_t_lambda: out[cols[k]] += values[k] * lambda[rows[k]], triplet order
    double jt = 0.0;
    for (int32_t p = jt_seg[i]; p < jt_seg[i + 1]; ++p) {
      const int32_t k = jt_src[p];
      jt = __dadd_rn(jt, __dmul_rn(jv[k], lam[jrow[k]]));
    }
    double r = __dsub_rn(-grad[i], jt);
    if (bounded) r = __dadd_rn(r, __ddiv_rn(mu, __dsub_rn(x[i], lower[i])));
    rhs[i] = r;
  } else {
    if (delta_c != 0.0) mat[i * dim + i] = __dsub_rn(mat[i * dim + i], delta_c);
    rhs[i] = -g[i - n];
  }
}

void check_index(int64_t v, int64_t hi, const char* what) {
  if (v < 0 || v >= hi)
    throw StructuralError(std::string("kkt: ") + what + " index " + std::to_string(v) + " out of range [0, " +
                          std::to_string(hi) + ")");
}

}  // namespace

Kkt::Kkt(int64_t n, int64_t m, const int64_t* hr, const int64_t* hc, size_t nnz_h, const int64_t* jr,
         const int64_t* jc, size_t nnz_j, int device)
    : n_(n), m_(m), nnz_h_(nnz_h), nnz_j_(nnz_j) {
  if (n < 0 || m < 0) throw StructuralError("kkt: negative dimension");
  if (nnz_h + nnz_j > static_cast<size_t>(std::numeric_limits<int32_t>::max()))
    throw StructuralError("kkt: too many triplets");
  const int64_t dim = n + m;
  // ---- pattern analysis: contributions per element, in triplet order ----
  // (element, source) pairs in the reference's scatter order, then a
  // stable sort by element keeps each element's order
  std::vector<std::pair<int64_t, int32_t>> contrib;
  contrib.reserve(2 * (nnz_h + nnz_j));
  for (size_t k = 0; k < nnz_h; ++k) {
    check_index(hr[k], n, "Hessian row");
    check_index(hc[k], n, "Hessian column");
    contrib.emplace_back(hr[k] * dim + hc[k], static_cast<int32_t>(k));
    if (hr[k] != hc[k]) contrib.emplace_back(hc[k] * dim + hr[k], static_cast<int32_t>(k));
  }
  for (size_t k = 0; k < nnz_j; ++k) {
    check_index(jr[k], m, "Jacobian row");
    check_index(jc[k], n, "Jacobian column");
    const int32_t s = static_cast<int32_t>(nnz_h + k);
    contrib.emplace_back((n + jr[k]) * dim + jc[k], s);
    contrib.emplace_back(jc[k] * dim + n + jr[k], s);
  }
  std::stable_sort(contrib.begin(), contrib.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<int64_t> target;
  std::vector<int32_t> seg, src;
  src.reserve(contrib.size());
  for (size_t p = 0; p < contrib.size(); ++p) {
    if (p == 0 || contrib[p].first != contrib[p - 1].first) {
      target.push_back(contrib[p].first);
      seg.push_back(static_cast<int32_t>(p));
    }
    src.push_back(contrib[p].second);
  }
  seg.push_back(static_cast<int32_t>(contrib.size()));
  n_targets_ = static_cast<int64_t>(target.size());
  // J^T lambda per column
  std::vector<int32_t> jt_seg(static_cast<size_t>(n) + 1, 0), jt_src(nnz_j), jrow(nnz_j);
  for (size_t k = 0; k < nnz_j; ++k) ++jt_seg[static_cast<size_t>(jc[k]) + 1];
  for (int64_t c = 0; c < n; ++c) jt_seg[c + 1] += jt_seg[c];
  {
    std::vector<int32_t> fill(jt_seg.begin(), jt_seg.end() - 1);
    for (size_t k = 0; k < nnz_j; ++k) {
      jt_src[fill[jc[k]]++] = static_cast<int32_t>(k);
      jrow[k] = static_cast<int32_t>(jr[k]);
    }
  }
  // ---- device state ----
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
  dev_ = device;
  DeviceGuard guard(device);
  CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  auto upload = [&](auto** dptr, const auto& v) {
    using T = std::remove_reference_t<decltype(v[0])>;
    const size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
    CK(cudaMalloc(reinterpret_cast<void**>(dptr), bytes));
    if (!v.empty()) CK(cudaMemcpy(*dptr, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  };
  upload(&d_target_, target);
  upload(&d_seg_, seg);
  upload(&d_src_, src);
  upload(&d_jt_seg_, jt_seg);
  upload(&d_jt_src_, jt_src);
  upload(&d_jrow_, jrow);
  CK(cudaMalloc(&d_mat_, sizeof(double) * std::max<int64_t>(dim * dim, 1)));
  CK(cudaMalloc(&d_rhs_, sizeof(double) * std::max<int64_t>(dim, 1)));
  in_len_ = static_cast<size_t>(4 * n + 2 * m) + nnz_h + nnz_j;
  CK(cudaMalloc(&d_in_, sizeof(double) * std::max<size_t>(in_len_, 1)));
  CK(cudaMallocHost(&h_in_, sizeof(double) * std::max<size_t>(in_len_, 1)));
}

Kkt::~Kkt() {
  if (dev_ < 0) return;
  DeviceGuard guard(dev_);
  for (void* p : {static_cast<void*>(d_target_), static_cast<void*>(d_seg_), static_cast<void*>(d_src_),
                  static_cast<void*>(d_jt_seg_), static_cast<void*>(d_jt_src_), static_cast<void*>(d_jrow_),
                  static_cast<void*>(d_mat_), static_cast<void*>(d_rhs_), static_cast<void*>(d_in_)})
    if (p) cudaFree(p);
  if (h_in_) cudaFreeHost(h_in_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Kkt::assemble(const double* x, const double* lower, const double* z, const double* lambda, const double* grad_f,
                   const double* g, const double* jac_values, const double* hess_values, double mu, double delta_w,
                   double delta_c) {
  DeviceGuard guard(dev_);
  const int64_t n = n_, m = m_, dim = n + m;
  double* p = h_in_;
  auto put = [&](const double* v, size_t len) {
    if (len) std::memcpy(p, v, sizeof(double) * len);
    p += len;
  };
  put(x, n);
  put(lower, n);
  put(z, n);
  put(grad_f, n);
  put(lambda, m);
  put(g, m);
  put(hess_values, nnz_h_);
  put(jac_values, nnz_j_);
  if (in_len_) CK(cudaMemcpyAsync(d_in_, h_in_, sizeof(double) * in_len_, cudaMemcpyHostToDevice, stream_));
  if (dim > 0) {
    CK(cudaMemsetAsync(d_mat_, 0, sizeof(double) * dim * dim, stream_));
    if (n_targets_ > 0) {
      kkt_scatter_kernel<<<static_cast<unsigned>((n_targets_ + 255) / 256), 256, 0, stream_>>>(
          d_target_, d_seg_, d_src_, n_targets_, d_in_ + 4 * n + 2 * m, d_mat_);
      CK(cudaGetLastError());
    }
    kkt_diag_rhs_kernel<<<static_cast<unsigned>((dim + 255) / 256), 256, 0, stream_>>>(
        d_in_, n, m, nnz_h_, d_jt_seg_, d_jt_src_, d_jrow_, mu, delta_w, delta_c, d_mat_, d_rhs_);
    CK(cudaGetLastError());
  }
  // the staging buffer is reused by the next call
  CK(cudaStreamSynchronize(stream_));
  assembled_ = true;
}

void Kkt::matrix(double* out) const {
  if (!assembled_) throw StructuralError("kkt: matrix requested before assemble");
  DeviceGuard guard(dev_);
  const int64_t dim = n_ + m_;
  if (dim == 0) return;
  CK(cudaMemcpyAsync(out, d_mat_, sizeof(double) * dim * dim, cudaMemcpyDeviceToHost, stream_));
  CK(cudaStreamSynchronize(stream_));
}

void Kkt::rhs(double* out) const {
  if (!assembled_) throw StructuralError("kkt: rhs requested before assemble");
  DeviceGuard guard(dev_);
  const int64_t dim = n_ + m_;
  if (dim == 0) return;
  CK(cudaMemcpyAsync(out, d_rhs_, sizeof(double) * dim, cudaMemcpyDeviceToHost, stream_));
  CK(cudaStreamSynchronize(stream_));
}

// ipm.cpp:520-557: delta_w starts at delta_w_start (0: no shift first),
// then delta0, then *= growth; zero pivots with constraints present switch
// on delta_c = 1e-8, escalated x100 up to 1e-2, before delta_w grows.
Kkt::Corrected Kkt::inertia_correct(double delta0, double delta_growth, double delta_max,
                                    double delta_w_start) const {
  if (!assembled_) throw StructuralError("kkt: inertia_correct before assemble");
  const int64_t n = n_, m = m_;
  double delta_w = delta_w_start, delta_c = 0.0;
  while (true) {
    auto fact = Ldlt::factor_device(d_mat_, n + m, n, delta_w, delta_c, /*keep_input=*/true, dev_, stream_);
    if (fact->n_pos() == n && fact->n_neg() == m && fact->n_zero() == 0) return {std::move(fact), delta_w, delta_c};
    if (fact->n_zero() > 0 && m > 0 && delta_c < kDeltaCMax) {
      delta_c = delta_c == 0.0 ? kDeltaC : delta_c * 1e2;
      continue;
    }
    delta_w = delta_w == 0.0 ? delta0 : delta_w * delta_growth;
    if (delta_w > delta_max)
      throw SingularError(
          "inertia correction: regularization exceeded the configured maximum without reaching the target inertia");
  }
}

std::vector<double> Kkt::solve(const Ldlt& fact) const {
  if (!assembled_) throw StructuralError("kkt: solve before assemble");
  return fact.solve_device(d_rhs_, n_ + m_, stream_);
}

}  // namespace gbb
