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
  // Factors the symmetric n x n matrix `a` (row-major) on CUDA device
  // `device` (-1: current).  keep_input retains the equilibrated matrix for
  // iterative refinement in solve().
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
  void solve_factored(std::vector<double>& x) const;

  int64_t n_ = 0, n_pos_ = 0, n_neg_ = 0, n_zero_ = 0;
  double zero_thresh_ = 0.0;
  std::vector<double> scale_, input_;
  std::vector<int> ipiv_;
  int dev_ = -1;
  cudaStream_t stream_ = nullptr;
  void* handle_ = nullptr;  // cusolverDnHandle_t
  double* d_fact_ = nullptr;
  int* d_ipiv_ = nullptr;
  double* d_work_ = nullptr;
  int* d_info_ = nullptr;
  double* d_rhs_ = nullptr;
};

}  // namespace gbb
