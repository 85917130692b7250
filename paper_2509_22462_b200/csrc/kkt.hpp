// Dense KKT assembly and inertia correction on the device for the IPM's
// Newton systems (reference proj/include/gbopt/ipm.hpp:80-118,
// proj/src/ipm.cpp:466-557).  See kkt.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "ldlt.hpp"

namespace gbb {

// The sparsity pattern of one NLP (Hessian lower triplets, Jacobian
// triplets) is analysed once; every assemble() then scatters that IPM
// iteration's values into the device-resident dense matrix
//   [[H + Sigma + dw I, J^T], [J, -dc I]]   ((n + m) x (n + m), row-major)
// and the right-hand side [-grad_f - J^T lambda + mu / (x - lower); -g].
class Kkt {
 public:
  Kkt(int64_t n, int64_t m, const int64_t* hess_rows, const int64_t* hess_cols, size_t nnz_h,
      const int64_t* jac_rows, const int64_t* jac_cols, size_t nnz_j, int device = -1);
  ~Kkt();
  Kkt(const Kkt&) = delete;
  Kkt& operator=(const Kkt&) = delete;

  int64_t n_var() const { return n_; }
  int64_t n_con() const { return m_; }
  int64_t dim() const { return n_ + m_; }
  size_t nnz_h() const { return nnz_h_; }
  size_t nnz_j() const { return nnz_j_; }

  // assemble_kkt (ipm.cpp:466-518): x, lower, z, grad_f have n entries
  // (lower may be -inf: unbounded), lambda and g m, the values the pattern's
  // counts.  Host inputs; the system stays on the device.
  void assemble(const double* x, const double* lower, const double* z, const double* lambda, const double* grad_f,
                const double* g, const double* jac_values, const double* hess_values, double mu, double delta_w,
                double delta_c);
  void matrix(double* out) const;  // (n + m)^2, row-major
  void rhs(double* out) const;     // n + m

  struct Corrected {
    std::unique_ptr<Ldlt> fact;
    double delta_w = 0.0;
    double delta_c = 0.0;
  };
  // inertia_correct (ipm.cpp:520-557) on the assembled matrix
  Corrected inertia_correct(double delta0, double delta_growth, double delta_max, double delta_w_start) const;
  // fact.solve(rhs) with the device-resident right-hand side
  std::vector<double> solve(const Ldlt& fact) const;

 private:
  int64_t n_ = 0, m_ = 0;
  size_t nnz_h_ = 0, nnz_j_ = 0;
  int dev_ = -1;
  cudaStream_t stream_ = nullptr;
  bool assembled_ = false;
  // matrix scatter: unique target elements, each summing its contributions
  // (indices into [hess_values | jac_values]) in triplet order
  int64_t n_targets_ = 0;
  int64_t* d_target_ = nullptr;   // [n_targets] element offset r * (n + m) + c
  int32_t* d_seg_ = nullptr;      // [n_targets + 1]
  int32_t* d_src_ = nullptr;      // [contributions]
  // J^T lambda: per column c < n, the Jacobian triplets with cols[k] == c
  int32_t* d_jt_seg_ = nullptr;   // [n + 1]
  int32_t* d_jt_src_ = nullptr;   // [nnz_j] triplet index k
  int32_t* d_jrow_ = nullptr;     // [nnz_j] rows[k]
  double* d_mat_ = nullptr;       // [(n + m)^2]
  double* d_rhs_ = nullptr;       // [n + m]
  double* d_in_ = nullptr;        // x | lower | z | grad_f (n each) | lambda | g (m each) | hess | jac values
  double* h_in_ = nullptr;        // pinned staging for d_in_
  size_t in_len_ = 0;
};

}  // namespace gbb
