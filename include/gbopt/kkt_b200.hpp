// gbopt_b200 C++ drop-in for the reference's KKT linear algebra: ldlt_factor /
// LdltFactorization (proj/include/gbopt/linalg.hpp:24-78) and assemble_kkt /
// inertia_correct (proj/include/gbopt/ipm.hpp:80-118), header-only over the
// C ABI in gbopt_b200.h.  Same names, argument meaning and exceptions; the
// factorisation and the assembled system live on the B200.
//
// KktSystem here is a handle to the device-resident system (mat() / rhs()
// copy it out) rather than two Eigen members, so the IPM's
//     kkt = assemble_kkt(...); cf = inertia_correct(kkt, opts); sol = cf.fact.solve(kkt.rhs)
// never moves the (n+m)^2 matrix across PCIe; KktSystem::solve(fact) is the
// last step with the device-resident right-hand side.  For repeated IPM
// iterations on one NLP, KktPattern analyses the triplet pattern once.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "gbopt/nn_b200.hpp"

namespace gbopt {
namespace b200 {

struct Inertia {
  int64_t n_pos = 0, n_neg = 0, n_zero = 0;
  bool operator==(const Inertia& o) const { return n_pos == o.n_pos && n_neg == o.n_neg && n_zero == o.n_zero; }
};

class KktSystem;
struct IpmOptions;
struct CorrectedFactorization;

class LdltFactorization {
 public:
  LdltFactorization() = default;
  explicit LdltFactorization(gbopt_ldlt* h) : h_(h, &gbopt_ldlt_free) {}
  Inertia inertia() const {
    Inertia i;
    check(gbopt_ldlt_inertia(h_.get(), &i.n_pos, &i.n_neg, &i.n_zero));
    return i;
  }
  RealVec solve(const RealVec& b) const {
    RealVec x(b.size());
    check(gbopt_ldlt_solve(h_.get(), b.data(), b.size(), x.data()));
    return x;
  }
  int64_t dim() const { return dim_; }
  const gbopt_ldlt* handle() const { return h_.get(); }

 private:
  friend LdltFactorization ldlt_factor(const DenseMat&, bool);
  friend struct CorrectedFactorization;
  friend CorrectedFactorization inertia_correct(const KktSystem&, const IpmOptions&, double);
  std::shared_ptr<gbopt_ldlt> h_;
  int64_t dim_ = 0;
};

// linalg.hpp:77-78
inline RealVec ldlt_solve(const LdltFactorization& f, const RealVec& b) { return f.solve(b); }

// linalg.hpp:66-75: a square symmetric row-major matrix
inline LdltFactorization ldlt_factor(const DenseMat& a, bool keep_input = true) {
  if (a.rows != a.cols) throw StructuralError("ldlt_factor: matrix is not square");
  gbopt_ldlt* h = nullptr;
  check(gbopt_ldlt_factor(a.data.data(), static_cast<size_t>(a.rows), keep_input ? 1 : 0, &h));
  LdltFactorization f(h);
  f.dim_ = a.rows;
  return f;
}

// ipm.hpp:21-23 (the regularisation fields)
struct IpmOptions {
  double delta0 = 1e-4;
  double delta_growth = 10.0;
  double delta_max = 1e40;
};

using IndexVec = std::vector<int64_t>;

class KktPattern {
 public:
  KktPattern(int64_t n, int64_t m, const IndexVec& hess_rows, const IndexVec& hess_cols, const IndexVec& jac_rows,
             const IndexVec& jac_cols)
      : n_(n), m_(m), nnz_h_(hess_rows.size()), nnz_j_(jac_rows.size()) {
    if (hess_rows.size() != hess_cols.size() || jac_rows.size() != jac_cols.size())
      throw StructuralError("kkt: row and column triplet lists differ in length");
    gbopt_kkt* h = nullptr;
    check(gbopt_kkt_create(static_cast<size_t>(n), static_cast<size_t>(m), hess_rows.data(), hess_cols.data(),
                           nnz_h_, jac_rows.data(), jac_cols.data(), nnz_j_, &h));
    h_.reset(h, &gbopt_kkt_free);
  }
  inline KktSystem assemble(const RealVec& x, const RealVec& lower, const RealVec& z, const RealVec& lambda,
                            const RealVec& grad_f, const RealVec& g, const RealVec& jac_values,
                            const RealVec& hess_values, double mu, double delta_w = 0.0, double delta_c = 0.0);
  int64_t n_var() const { return n_; }
  int64_t n_con() const { return m_; }

 private:
  friend class KktSystem;
  int64_t n_, m_;
  size_t nnz_h_, nnz_j_;
  std::shared_ptr<gbopt_kkt> h_;
};

class KktSystem {
 public:
  int64_t n_var = 0;
  int64_t n_con = 0;
  DenseMat mat() const {
    DenseMat out(n_var + n_con, n_var + n_con);
    check(gbopt_kkt_matrix(h_.get(), out.data.data(), out.data.size()));
    return out;
  }
  RealVec rhs() const {
    RealVec out(static_cast<size_t>(n_var + n_con));
    check(gbopt_kkt_rhs(h_.get(), out.data(), out.size()));
    return out;
  }
  // fact.solve(rhs) with the device-resident right-hand side
  RealVec solve(const LdltFactorization& fact) const {
    RealVec out(static_cast<size_t>(n_var + n_con));
    check(gbopt_kkt_solve(h_.get(), fact.handle(), out.data(), out.size()));
    return out;
  }
  const gbopt_kkt* handle() const { return h_.get(); }

 private:
  friend class KktPattern;
  std::shared_ptr<gbopt_kkt> h_;
};

inline KktSystem KktPattern::assemble(const RealVec& x, const RealVec& lower, const RealVec& z, const RealVec& lambda,
                                      const RealVec& grad_f, const RealVec& g, const RealVec& jac_values,
                                      const RealVec& hess_values, double mu, double delta_w, double delta_c) {
  const auto want = [](const RealVec& v, size_t len, const char* what) {
    if (v.size() != len) throw StructuralError(std::string("assemble_kkt: ") + what + " has the wrong size");
  };
  const size_t n = static_cast<size_t>(n_), m = static_cast<size_t>(m_);
  want(x, n, "x");
  want(lower, n, "lower");
  want(z, n, "z");
  want(grad_f, n, "grad_f");
  want(lambda, m, "lambda");
  want(g, m, "g");
  want(jac_values, nnz_j_, "jac_values");
  want(hess_values, nnz_h_, "hess_values");
  check(gbopt_kkt_assemble(h_.get(), x.data(), lower.data(), z.data(), lambda.data(), grad_f.data(), g.data(),
                           jac_values.data(), hess_values.data(), mu, delta_w, delta_c));
  KktSystem s;
  s.n_var = n_;
  s.n_con = m_;
  s.h_ = h_;
  return s;
}

// ipm.hpp:89-102, same argument order (the pattern is analysed per call)
inline KktSystem assemble_kkt(const RealVec& x, const RealVec& lower, const RealVec& z, const RealVec& lambda,
                              const RealVec& grad_f, const RealVec& g, const IndexVec& jac_rows,
                              const IndexVec& jac_cols, const RealVec& jac_values, const IndexVec& hess_rows,
                              const IndexVec& hess_cols, const RealVec& hess_values, double mu, double delta_w = 0.0,
                              double delta_c = 0.0) {
  KktPattern p(static_cast<int64_t>(x.size()), static_cast<int64_t>(g.size()), hess_rows, hess_cols, jac_rows,
               jac_cols);
  return p.assemble(x, lower, z, lambda, grad_f, g, jac_values, hess_values, mu, delta_w, delta_c);
}

struct CorrectedFactorization {
  LdltFactorization fact;
  double delta_w = 0.0;
  double delta_c = 0.0;
};

// ipm.hpp:104-118
inline CorrectedFactorization inertia_correct(const KktSystem& kkt, const IpmOptions& opts = {},
                                              double delta_w_start = 0.0) {
  gbopt_ldlt* h = nullptr;
  CorrectedFactorization cf;
  check(gbopt_kkt_inertia_correct(kkt.handle(), opts.delta0, opts.delta_growth, opts.delta_max, delta_w_start, &h,
                                  &cf.delta_w, &cf.delta_c));
  cf.fact = LdltFactorization(h);
  cf.fact.dim_ = kkt.n_var + kkt.n_con;
  return cf;
}

}  // namespace b200
}  // namespace gbopt
