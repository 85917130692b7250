// gbopt_b200 C++ drop-in for gbopt::NeuralNet (reference
// proj/include/gbopt/nn.hpp:40-110), header-only over the C ABI in
// gbopt_b200.h.  Same method names, argument meaning and exception classes
// (reference proj/include/gbopt/errors.hpp); results come from the B200.
//
// Vectors are std::vector<double>; matrices are DenseMat (row-major, with
// operator()(i, j)), because Eigen is not required.  When <Eigen/Dense> is
// available an Eigen overload set is provided as well (GBOPT_B200_EIGEN).
//
// The reduced-space embedding (reference src/formulations.cpp:267-349) is
// supported by ReducedSpaceOracle below: one fused y/J/H evaluation per
// distinct x feeds the residual, Jacobian and Lagrangian-Hessian callbacks,
// instead of three separate forward passes.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gbopt_b200.h"

namespace gbopt {
namespace b200 {

// ---- errors (reference errors.hpp:10-71) ---------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class StructuralError : public Error { public: using Error::Error; };
class NumericError : public Error { public: using Error::Error; };
class SingularError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class FormatError : public IoError { public: using IoError::IoError; };
class DimensionError : public IoError { public: using IoError::IoError; };
class TruncatedError : public IoError { public: using IoError::IoError; };
class RangeError : public Error { public: using Error::Error; };
class ArgumentError : public StructuralError { public: using StructuralError::StructuralError; };
class DeviceError : public Error { public: using Error::Error; };

inline void check(gbopt_status s) {
  if (s == GBOPT_OK) return;
  const std::string msg = gbopt_last_error();
  switch (s) {
    case GBOPT_ERR_STRUCTURAL: throw StructuralError(msg);
    case GBOPT_ERR_NUMERIC: throw NumericError(msg);
    case GBOPT_ERR_SINGULAR: throw SingularError(msg);
    case GBOPT_ERR_IO: throw IoError(msg);
    case GBOPT_ERR_FORMAT: throw FormatError(msg);
    case GBOPT_ERR_DIMENSION: throw DimensionError(msg);
    case GBOPT_ERR_TRUNCATED: throw TruncatedError(msg);
    case GBOPT_ERR_RANGE: throw RangeError(msg);
    case GBOPT_ERR_ARGUMENT: throw ArgumentError(msg);
    case GBOPT_ERR_DEVICE: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

using RealVec = std::vector<double>;

// Row-major dense matrix.
struct DenseMat {
  int64_t rows = 0, cols = 0;
  std::vector<double> data;
  DenseMat() = default;
  DenseMat(int64_t r, int64_t c) : rows(r), cols(c), data(static_cast<size_t>(r * c)) {}
  double& operator()(int64_t i, int64_t j) { return data[static_cast<size_t>(i * cols + j)]; }
  double operator()(int64_t i, int64_t j) const { return data[static_cast<size_t>(i * cols + j)]; }
};

// Per-layer values of one forward pass (reference nn.hpp:31-36):
// z[l] = W_l y[l-1] + b_l (y[-1] = x), y[l] = sigma_l(z[l]).
struct ForwardTrace {
  std::vector<std::vector<double>> z;
  std::vector<std::vector<double>> y;
};

enum class ActivationKind : int32_t { Linear = 0, Tanh = 1, Sigmoid = 2, Softmax = 3, Softplus = 4 };

struct Layer {
  DenseMat weight;  // out x in
  RealVec bias;     // out
  ActivationKind activation = ActivationKind::Linear;
};

class NeuralNet {
 public:
  // "Load MLP weights and activations" (validates like nn.cpp:74-103).
  explicit NeuralNet(const std::vector<Layer>& layers) {
    std::vector<int64_t> widths;
    std::vector<int32_t> acts;
    std::vector<const double*> w, b;
    if (!layers.empty()) widths.push_back(layers.front().weight.cols);
    for (const Layer& l : layers) {
      widths.push_back(l.weight.rows);
      acts.push_back(static_cast<int32_t>(l.activation));
      w.push_back(l.weight.data.data());
      b.push_back(l.bias.data());
      if (static_cast<int64_t>(l.bias.size()) != l.weight.rows)
        throw StructuralError("NeuralNet: weight rows != bias length");
    }
    for (size_t l = 1; l < layers.size(); ++l)
      if (layers[l].weight.cols != layers[l - 1].weight.rows)
        throw StructuralError("NeuralNet: layer " + std::to_string(l) + " input width does not chain");
    gbopt_net* h = nullptr;
    check(gbopt_net_from_layers(layers.size(), widths.data(), acts.data(), w.data(), b.data(), &h));
    h_.reset(h, gbopt_net_free);
  }

  static NeuralNet adopt(gbopt_net* h) { return NeuralNet(h); }

  int64_t input_dim() const { return gbopt_net_input_dim(h_.get()); }
  int64_t output_dim() const { return gbopt_net_output_dim(h_.get()); }
  int64_t layer_count() const { return gbopt_net_layer_count(h_.get()); }
  int64_t param_count() const { return gbopt_net_param_count(h_.get()); }

  Layer layer(int64_t l) const {
    int64_t rows = 0, cols = 0;
    int32_t act = 0;
    check(gbopt_net_layer_info(h_.get(), l, &rows, &cols, &act));
    Layer out;
    out.weight = DenseMat(rows, cols);
    out.bias.resize(static_cast<size_t>(rows));
    out.activation = static_cast<ActivationKind>(act);
    check(gbopt_net_layer_copy(h_.get(), l, out.weight.data.data(), out.weight.data.size(), out.bias.data(),
                               out.bias.size()));
    return out;
  }

  // Binds to a CUDA device (weights uploaded to HBM once).
  const NeuralNet& bind_device(int ordinal) const {
    check(gbopt_net_bind_device(h_.get(), ordinal));
    return *this;
  }

  RealVec forward(const RealVec& x) const {
    RealVec y(static_cast<size_t>(output_dim()));
    check_len(x, input_dim(), "forward");
    check(gbopt_net_forward(h_.get(), x.data(), x.size(), y.data(), y.size()));
    return y;
  }

  // m x n, J(i, j) = d y_i / d x_j
  DenseMat jacobian(const RealVec& x) const {
    check_len(x, input_dim(), "jacobian");
    DenseMat j(output_dim(), input_dim());
    check(gbopt_net_jacobian(h_.get(), x.data(), x.size(), j.data.data(), j.data.size()));
    return j;
  }

  RealVec lagrangian_gradient(const RealVec& x, const RealVec& lambda) const {
    check_len(x, input_dim(), "lagrangian_gradient");
    check_len(lambda, output_dim(), "lagrangian_gradient");
    RealVec g(x.size());
    check(gbopt_net_lagrangian_gradient(h_.get(), x.data(), x.size(), lambda.data(), lambda.size(), g.data(),
                                        g.size()));
    return g;
  }

  // n x n, symmetric: sum_i lambda_i Hess NN_i(x)
  DenseMat lagrangian_hessian(const RealVec& x, const RealVec& lambda) const {
    check_len(x, input_dim(), "lagrangian_hessian");
    check_len(lambda, output_dim(), "lagrangian_hessian");
    DenseMat h(input_dim(), input_dim());
    check(gbopt_net_lagrangian_hessian(h_.get(), x.data(), x.size(), lambda.data(), lambda.size(), h.data.data(),
                                       h.data.size()));
    return h;
  }

  // Fused evaluation (new in this build): one forward pass for y, J and H.
  void oracle(const RealVec& x, const RealVec& lambda, RealVec* y, DenseMat* jac, DenseMat* hess) const {
    check_len(x, input_dim(), "oracle");
    check_len(lambda, output_dim(), "oracle");
    const int64_t n = input_dim(), m = output_dim();
    if (y) y->assign(static_cast<size_t>(m), 0.0);
    if (jac) *jac = DenseMat(m, n);
    if (hess) *hess = DenseMat(n, n);
    check(gbopt_net_oracle(h_.get(), x.data(), x.size(), lambda.data(), lambda.size(), y ? y->data() : nullptr,
                           jac ? jac->data.data() : nullptr, hess ? hess->data.data() : nullptr));
  }

  // Fused evaluation with the Hessian as its packed lower triangle in row
  // order (hess_lower[a (a + 1) / 2 + c] = H(a, c), c <= a), packed on the
  // device: the value order of the reduced-space Hessian callback.
  void oracle_lower(const RealVec& x, const RealVec& lambda, RealVec* y, DenseMat* jac, RealVec* hess_lower) const {
    check_len(x, input_dim(), "oracle_lower");
    check_len(lambda, output_dim(), "oracle_lower");
    const int64_t n = input_dim(), m = output_dim();
    if (y) y->assign(static_cast<size_t>(m), 0.0);
    if (jac) *jac = DenseMat(m, n);
    hess_lower->assign(static_cast<size_t>(n * (n + 1) / 2), 0.0);
    check(gbopt_net_oracle_lower(h_.get(), 1, x.data(), x.size(), lambda.data(), lambda.size(), y ? y->data() : nullptr,
                                 jac ? jac->data.data() : nullptr, hess_lower->data(), hess_lower->size()));
  }

  // Batched (y, J, H) of `batch` points (X: batch x n, Lambda: batch x m,
  // row-major; Y, J, H likewise, any may be null) split over `devices`:
  // one weight replica and one host thread per entry, each device writing
  // its rows straight into the outputs (gbopt_net_oracle_batched_multi).
  void oracle_batched_multi(const std::vector<int>& devices, int64_t batch, const double* X, const double* Lambda,
                            double* Y, double* J, double* H) const {
    check(gbopt_net_oracle_batched_multi(h_.get(), devices.data(), devices.size(), static_cast<size_t>(batch), X,
                                         static_cast<size_t>(input_dim()), Lambda,
                                         static_cast<size_t>(output_dim()), Y, J, H));
  }

  // nn.hpp:31-36, nn.cpp:127-146
  ForwardTrace forward_trace(const RealVec& x) const {
    check_len(x, input_dim(), "forward_trace");
    std::vector<int64_t> rows;
    int64_t total = 0;
    for (int64_t l = 0; l < layer_count(); ++l) {
      int64_t r = 0, c = 0;
      int32_t act = 0;
      check(gbopt_net_layer_info(h_.get(), l, &r, &c, &act));
      rows.push_back(r);
      total += r;
    }
    RealVec z(static_cast<size_t>(total)), y(static_cast<size_t>(total));
    check(gbopt_net_forward_trace(h_.get(), x.data(), x.size(), z.data(), y.data(), z.size()));
    ForwardTrace t;
    int64_t off = 0;
    for (int64_t r : rows) {
      t.z.emplace_back(z.begin() + off, z.begin() + off + r);
      t.y.emplace_back(y.begin() + off, y.begin() + off + r);
      off += r;
    }
    return t;
  }

  const gbopt_net* handle() const { return h_.get(); }

 private:
  explicit NeuralNet(gbopt_net* h) : h_(h, gbopt_net_free) {}
  // The reference raises StructuralError for wrong x / lambda lengths
  // (nn.cpp:105-111, 174-178, 200-204).
  static void check_len(const RealVec& v, int64_t want, const char* who) {
    if (static_cast<int64_t>(v.size()) != want)
      throw StructuralError(std::string(who) + ": input has length " + std::to_string(v.size()) + ", expected " +
                            std::to_string(want));
  }
  std::shared_ptr<gbopt_net> h_;
};

inline NeuralNet load_weights(const std::string& path) {
  gbopt_net* h = nullptr;
  check(gbopt_net_load(path.c_str(), &h));
  return NeuralNet::adopt(h);
}

inline void save_weights(const NeuralNet& nn, const std::string& path) {
  check(gbopt_net_save(nn.handle(), path.c_str()));
}

inline NeuralNet random_net(const std::vector<int64_t>& widths, const std::string& hidden,
                            const std::string& final_act, uint64_t seed) {
  gbopt_net* h = nullptr;
  check(gbopt_net_random(widths.data(), widths.size(), hidden.c_str(), final_act.c_str(), seed, &h));
  return NeuralNet::adopt(h);
}

// ---- reduced-space embedding callbacks (formulations.cpp:267-349) ---------
//
// Block variables are [x (n inputs); y (m outputs)], constraint
// r = y - NN(x).  Each callback does the least work that answers it and
// caches per x: residual -> forward pass; Jacobian -> reverse mode (m
// weight sweeps, like nn.cpp:148-170); Lagrangian Hessian -> the fused
// evaluation with the Hessian only.  Every quantity has one producer, so a
// callback's value at x is the same whatever ran before it (the reference
// is a pure function of x).  The IPM calls residual, Jacobian and Hessian at
// the same iterate (ipm.cpp:256, 278, 420), so no quantity is computed
// twice per x.
class ReducedSpaceOracle {
 public:
  explicit ReducedSpaceOracle(NeuralNet net) : net_(std::move(net)) {
    n_ = net_.input_dim();
    m_ = net_.output_dim();
  }

  // r = y - NN(x)   (formulations.cpp:317-319); xb = [x; y]
  void residual(const RealVec& xb, RealVec& r) {
    if (!same_x(xb, y_x_)) {
      y_ = net_.forward(head(xb));
      y_x_ = head(xb);
      ++evals_;
    }
    r.resize(static_cast<size_t>(m_));
    for (int64_t i = 0; i < m_; ++i) r[i] = xb[n_ + i] - y_[i];
  }

  // values in the pattern order of formulations.cpp:320-331: -J row-major
  // over the inputs, then +1 for each output's identity entry.
  void jacobian(const RealVec& xb, RealVec& values) {
    if (!same_x(xb, j_x_)) {
      jac_ = net_.jacobian(head(xb));
      j_x_ = head(xb);
      ++evals_;
    }
    values.resize(static_cast<size_t>(m_ * n_ + m_));
    size_t k = 0;
    for (int64_t i = 0; i < m_; ++i)
      for (int64_t j = 0; j < n_; ++j) values[k++] = -jac_(i, j);
    for (int64_t i = 0; i < m_; ++i) values[k++] = 1.0;
  }

  // Lower-triangle values for the pattern (a >= b) in row order; the oracle
  // sees -lambda (formulations.cpp:332-340).  Input indices are assumed
  // ascending (the reference flips (r, c) otherwise; H is symmetric).
  void lag_hessian(const RealVec& xb, const RealVec& lam, RealVec& values) {
    RealVec neg(lam.size());
    for (size_t i = 0; i < lam.size(); ++i) neg[i] = -lam[i];
    if (!same_x(xb, h_x_) || neg != h_lam_) {
      const RealVec x = head(xb);
      // packed on the device in the pattern's value order
      net_.oracle_lower(x, neg, nullptr, nullptr, &hess_lower_);
      h_x_ = x;
      h_lam_ = neg;
      ++evals_;
    }
    values = hess_lower_;
  }

  // Number of device evaluations issued so far.
  int64_t evaluations() const { return evals_; }

 private:
  RealVec head(const RealVec& xb) const { return RealVec(xb.begin(), xb.begin() + n_); }
  bool same_x(const RealVec& xb, const RealVec& cached) const {
    return !cached.empty() && std::memcmp(xb.data(), cached.data(), sizeof(double) * static_cast<size_t>(n_)) == 0;
  }

  NeuralNet net_;
  int64_t n_ = 0, m_ = 0, evals_ = 0;
  RealVec y_x_, j_x_, h_x_, h_lam_, y_, hess_lower_;
  DenseMat jac_;
};

}  // namespace b200
}  // namespace gbopt

#if defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#define GBOPT_B200_EIGEN 1
namespace gbopt {
namespace b200 {
// Eigen adapters matching the reference signatures (RealVec = VectorXd,
// RealMat = MatrixXd, linalg.hpp:10-11).
inline Eigen::VectorXd to_eigen(const RealVec& v) { return Eigen::Map<const Eigen::VectorXd>(v.data(), v.size()); }
inline Eigen::MatrixXd to_eigen(const DenseMat& m) {
  return Eigen::Map<const Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>>(m.data.data(),
                                                                                                   m.rows, m.cols);
}
inline RealVec from_eigen(const Eigen::VectorXd& v) { return RealVec(v.data(), v.data() + v.size()); }
}  // namespace b200
}  // namespace gbopt
#endif
#endif
