// Dense symmetric-indefinite factorisation for the IPM's KKT systems
// (reference proj/include/gbopt/linalg.hpp:24-78); see ldlt.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "errors.hpp"

namespace gbb {

class Ldlt {
 public:
  // Factors the symmetric n x n matrix `a` (row-major, host) on CUDA device
  // `device` (-1: current).  keep_input retains the equilibrated matrix on
  // the device for iterative refinement in solve().
  static std::unique_ptr<Ldlt> factor(const double* a, int64_t n, bool keep_input, int device = -1);
  // The same from a device-resident row-major matrix `d_a` (left unchanged),
  // factoring d_a + delta_w I (first n_var rows) - delta_c I (the rest): the
  // reference's inertia-correction trial matrix (ipm.cpp:529-536).  `src`
  // is the stream that produced d_a; the factorisation waits for it.
  static std::unique_ptr<Ldlt> factor_device(const double* d_a, int64_t n, int64_t n_var, double delta_w,
                                             double delta_c, bool keep_input, int device, cudaStream_t src);
  ~Ldlt();
  Ldlt(const Ldlt&) = delete;
  Ldlt& operator=(const Ldlt&) = delete;

  int64_t dim() const { return n_; }
  int64_t n_pos() const { return n_pos_; }
  int64_t n_neg() const { return n_neg_; }
  int64_t n_zero() const { return n_zero_; }
  std::vector<double> solve(const double* b, int64_t len) const;
  // solve with a device-resident right-hand side (len == dim(); `src` is
  // the stream that produced it), the result in host memory
  std::vector<double> solve_device(const double* d_b, int64_t len, cudaStream_t src) const;

 private:
  Ldlt() = default;
  static std::unique_ptr<Ldlt> factor_impl(const double* a, bool on_device, int64_t n, int64_t n_var, double delta_w,
                                           double delta_c, bool keep_input, int device, cudaStream_t src);
  std::vector<double> solve_scaled(std::vector<double> bs) const;
  void solve_factored(double* d_v) const;
  // device buffer from the reuse pool (ldlt.cu), returned to it by ~Ldlt
  template <class T>
  void palloc(T** ptr, size_t bytes);
  std::vector<std::pair<void*, size_t>> pooled_;
  void refine_add_kernel_launch(double* d_x, const double* d_r, int64_t n, cudaStream_t st) const;

  int64_t n_ = 0, n_pos_ = 0, n_neg_ = 0, n_zero_ = 0;
  double zero_thresh_ = 0.0;
  std::vector<double> scale_;
  std::vector<int> ipiv_;
  int dev_ = -1;
  cudaStream_t stream_ = nullptr;
  void* handle_ = nullptr;  // cusolverDnHandle_t
  double* d_fact_ = nullptr;
  double* d_input_ = nullptr;  // equilibrated copy (keep_input)
  int* d_ipiv_ = nullptr;
  int64_t* d_ipiv64_ = nullptr;
  double* d_work_ = nullptr;
  int* d_info_ = nullptr;
  double* d_rhs_ = nullptr;
  double* d_vec_ = nullptr;
  void* d_sbuf_ = nullptr;
  size_t sws_dev_ = 0, sws_host_ = 0;
  // native Bunch-Kaufman (ldlt_bk.cuh): n <= kNativeMaxN
  bool native_ = false;
  bool cluster_ = false;
  bool panel_ = false;  // factored by the blocked kernel (ldlt_bkp.cuh)  // factored by the one-cluster kernel (ldlt_bkc.cuh)
  double* d_pan_ = nullptr;  // blocked kernel (ldlt_bkp.cuh): panel L / W columns, control, inverse permutation
  double* d_l_ = nullptr;   // [n][ldl_] unit lower factor
  int64_t ldl_ = 0;
  int solve_grid_ = 1;
  double* d_bk_ = nullptr;  // d[n] | e[n] | w[n] | wr[n] | z[n] | part[4 * grid]
  int* d_bki_ = nullptr;    // piv[n] | perm[n]
};

}  // namespace gbb
