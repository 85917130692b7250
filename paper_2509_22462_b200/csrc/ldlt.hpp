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
  ~Ldlt();
  Ldlt(const Ldlt&) = delete;
  Ldlt& operator=(const Ldlt&) = delete;

  int64_t dim() const { return n_; }
  int64_t n_pos() const { return n_pos_; }
  int64_t n_neg() const { return n_neg_; }
  int64_t n_zero() const { return n_zero_; }
  std::vector<double> solve(const double* b, int64_t len) const;

 private:
  Ldlt() = default;
  void solve_factored(double* d_v) const;
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
  double* d_l_ = nullptr;   // [n][ldl_] unit lower factor
  int64_t ldl_ = 0;
  int solve_grid_ = 1;
  double* d_bk_ = nullptr;  // d[n] | e[n] | w[n] | wr[n] | z[n] | part[4 * grid]
  int* d_bki_ = nullptr;    // piv[n] | perm[n]
};

}  // namespace gbb
