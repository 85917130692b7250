// C entry points around the reference's OWN sources, compiled unmodified
// (/root/reference/proj/src/nn.cpp, nn_io.cpp, linalg.cpp) against the
// Eigen subset in eigen_subset/.  Output: oracle/_ref/libgbopt_ref.so.
//
// TEST INFRASTRUCTURE ONLY.  Loaded by tests/ (parity pins), smoke() and
// the CPU legs of bench.py (cpu_baseline, --impl reference).  The product
// (paper_2509_22462_b200/) never loads it.
//
// Layouts: weights and J are row-major (the GBNN / gbopt_b200.h order), H
// is the full n x n matrix; matrices handed to the LDL^T entry points are
// symmetric, so their storage order does not matter.  Status codes are the
// reference's gbopt_status values (proj/include/gbopt.h:19-31); the
// exception mapping follows proj/src/capi.cpp:33-60.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "gbopt/errors.hpp"
#include "gbopt/linalg.hpp"
#include "gbopt/nn.hpp"
#include "gbopt/prng.hpp"

#ifdef GBOPT_REF_BLAS
extern "C" void scipy_openblas_set_num_threads64_(int);
extern "C" int scipy_openblas_get_num_threads64_(void);
#endif

namespace {

thread_local std::string t_err;

int status_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const gbopt::FormatError&) {
    return 5;
  } catch (const gbopt::DimensionError&) {
    return 6;
  } catch (const gbopt::TruncatedError&) {
    return 7;
  } catch (const gbopt::IoError&) {
    return 4;
  } catch (const gbopt::RangeError&) {
    return 8;
  } catch (const gbopt::NumericError&) {
    return 2;
  } catch (const gbopt::SingularError&) {
    return 3;
  } catch (const gbopt::StructuralError&) {
    return 1;
  } catch (...) {
    return 10;
  }
}

template <class F>
int guarded(F&& f) {
  try {
    t_err.clear();
    f();
    return 0;
  } catch (const std::exception& e) {
    t_err = e.what();
    return status_of(std::current_exception());
  } catch (...) {
    t_err = "unknown failure";
    return 10;
  }
}

gbopt::RealVec vec(const double* p, std::int64_t n) {
  gbopt::RealVec v(n);
  for (std::int64_t i = 0; i < n; ++i) v(i) = p[i];
  return v;
}

void put_rowmajor(const gbopt::RealMat& m, double* out) {
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) out[i * m.cols() + j] = m(i, j);
}

void put_vec(const gbopt::RealVec& v, double* out) {
  for (Eigen::Index i = 0; i < v.size(); ++i) out[i] = v(i);
}

struct Net {
  std::shared_ptr<const gbopt::NeuralNet> nn;
};

const gbopt::NeuralNet& N(void* h) { return *static_cast<Net*>(h)->nn; }

}  // namespace

extern "C" {

const char* gbref_last_error(void) { return t_err.c_str(); }

int gbref_set_threads(int n) {
#ifdef GBOPT_REF_BLAS
  scipy_openblas_set_num_threads64_(n);
  return scipy_openblas_get_num_threads64_();
#else
  (void)n;
  return 1;
#endif
}

int gbref_has_blas(void) {
#ifdef GBOPT_REF_BLAS
  return 1;
#else
  return 0;
#endif
}

// widths[0..L], acts[0..L-1]; params = per layer W (rows x cols, row-major)
// then b (rows), concatenated.  Construction runs NeuralNet's own
// validation (nn.cpp:74-103).
int gbref_net_create(int layers, const std::int64_t* widths, const std::uint8_t* acts,
                     const double* params, void** out) {
  return guarded([&] {
    std::vector<gbopt::Layer> ls(static_cast<size_t>(layers));
    const double* p = params;
    for (int l = 0; l < layers; ++l) {
      const std::int64_t rows = widths[l + 1], cols = widths[l];
      gbopt::Layer& lay = ls[static_cast<size_t>(l)];
      lay.weight.resize(rows, cols);
      for (std::int64_t r = 0; r < rows; ++r)
        for (std::int64_t c = 0; c < cols; ++c) lay.weight(r, c) = *p++;
      lay.bias.resize(rows);
      for (std::int64_t r = 0; r < rows; ++r) lay.bias(r) = *p++;
      lay.activation = static_cast<gbopt::ActivationKind>(acts[l]);
    }
    auto* h = new Net{std::make_shared<const gbopt::NeuralNet>(std::move(ls))};
    *out = h;
  });
}

int gbref_net_random(int nw, const std::int64_t* widths, int hidden, int final_act,
                     std::uint64_t seed, void** out) {
  return guarded([&] {
    std::vector<Eigen::Index> w(widths, widths + nw);
    auto* h = new Net{std::make_shared<const gbopt::NeuralNet>(gbopt::random_net(
        w, static_cast<gbopt::ActivationKind>(hidden), static_cast<gbopt::ActivationKind>(final_act),
        seed))};
    *out = h;
  });
}

int gbref_net_load(const char* path, void** out) {
  return guarded([&] {
    auto* h = new Net{std::make_shared<const gbopt::NeuralNet>(gbopt::load_weights(path))};
    *out = h;
  });
}

int gbref_net_save(void* h, const char* path) {
  return guarded([&] { gbopt::save_weights(N(h), path); });
}

void gbref_net_free(void* h) { delete static_cast<Net*>(h); }

// dims = {input_dim, output_dim, layer_count, param_count}
void gbref_net_dims(void* h, std::int64_t* dims) {
  const auto& nn = N(h);
  dims[0] = nn.input_dim();
  dims[1] = nn.output_dim();
  dims[2] = nn.layer_count();
  dims[3] = nn.param_count();
}

int gbref_net_layer(void* h, int l, std::int64_t* rows, std::int64_t* cols, int* act,
                    double* w, double* b) {
  return guarded([&] {
    const auto& lay = N(h).layer(l);
    *rows = lay.out_dim();
    *cols = lay.in_dim();
    *act = static_cast<int>(lay.activation);
    if (w) put_rowmajor(lay.weight, w);
    if (b) put_vec(lay.bias, b);
  });
}

int gbref_forward(void* h, const double* x, std::int64_t n, double* y) {
  return guarded([&] { put_vec(N(h).forward(vec(x, n)), y); });
}

// z and y of every layer, concatenated in layer order.
int gbref_forward_trace(void* h, const double* x, std::int64_t n, double* z, double* y) {
  return guarded([&] {
    const gbopt::ForwardTrace t = N(h).forward_trace(vec(x, n));
    for (size_t l = 0; l < t.z.size(); ++l) {
      put_vec(t.z[l], z);
      put_vec(t.y[l], y);
      z += t.z[l].size();
      y += t.y[l].size();
    }
  });
}

int gbref_jacobian(void* h, const double* x, std::int64_t n, double* jac) {
  return guarded([&] { put_rowmajor(N(h).jacobian(vec(x, n)), jac); });
}

int gbref_lagrangian_gradient(void* h, const double* x, std::int64_t n, const double* lam,
                              std::int64_t m, double* g) {
  return guarded([&] { put_vec(N(h).lagrangian_gradient(vec(x, n), vec(lam, m)), g); });
}

int gbref_lagrangian_hessian(void* h, const double* x, std::int64_t n, const double* lam,
                             std::int64_t m, double* hess) {
  return guarded([&] { put_rowmajor(N(h).lagrangian_hessian(vec(x, n), vec(lam, m)), hess); });
}

// One oracle evaluation the way the reduced-space callbacks consume it
// (formulations.cpp:317-340): forward, jacobian and lagrangian_hessian at
// the same x, for B points (row-major X: B x n, L: B x m; Y: B x m,
// J: B x m x n, H: B x n x n).  Points are spread over `threads` host
// threads (each point single-threaded inside), or run one after another
// with threads <= 1.
int gbref_oracle_batched(void* h, std::int64_t B, const double* X, const double* L,
                         double* Y, double* J, double* H, int threads) {
  return guarded([&] {
    const auto& nn = N(h);
    const std::int64_t n = nn.input_dim(), m = nn.output_dim();
    auto one = [&](std::int64_t b) {
      const gbopt::RealVec x = vec(X + b * n, n);
      const gbopt::RealVec lam = vec(L + b * m, m);
      if (Y) put_vec(nn.forward(x), Y + b * m);
      if (J) put_rowmajor(nn.jacobian(x), J + b * m * n);
      if (H) put_rowmajor(nn.lagrangian_hessian(x, lam), H + b * n * n);
    };
    if (threads <= 1 || B <= 1) {
      for (std::int64_t b = 0; b < B; ++b) one(b);
      return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(threads));
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          for (std::int64_t b = t; b < B; b += threads) one(b);
        } catch (...) {
          errs[static_cast<size_t>(t)] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

int gbref_activation_elementwise(int kind, const double* z, std::int64_t n, double* y,
                                 double* d1, double* d2) {
  return guarded([&] {
    gbopt::RealVec vy, v1, v2;
    gbopt::activation_elementwise(static_cast<gbopt::ActivationKind>(kind), vec(z, n), &vy, &v1,
                                  &v2);
    put_vec(vy, y);
    put_vec(v1, d1);
    put_vec(v2, d2);
  });
}

// ---- dense symmetric indefinite LDL^T (linalg.hpp:24-78, linalg.cpp)
struct Fact {
  gbopt::LdltFactorization f;
};

int gbref_ldlt_factor(const double* a, std::int64_t n, int keep_input, void** out,
                      int* inertia) {
  return guarded([&] {
    gbopt::RealMat A(n, n);
    std::memcpy(A.data(), a, sizeof(double) * static_cast<size_t>(n * n));
    auto* f = new Fact{gbopt::ldlt_factor(A, keep_input != 0)};
    inertia[0] = f->f.inertia().n_pos;
    inertia[1] = f->f.inertia().n_neg;
    inertia[2] = f->f.inertia().n_zero;
    *out = f;
  });
}

int gbref_ldlt_solve(void* f, const double* b, std::int64_t n, double* x) {
  return guarded([&] { put_vec(static_cast<Fact*>(f)->f.solve(vec(b, n)), x); });
}

int gbref_ldlt_reconstruct(void* f, double* a) {
  return guarded([&] { put_rowmajor(static_cast<Fact*>(f)->f.reconstruct(), a); });
}

void gbref_ldlt_free(void* f) { delete static_cast<Fact*>(f); }

// ---- seeded synthetic workloads without the product library.  The uniform
// draws are the reference's own Prng (prng.hpp:11-23); normals are
// Box-Muller on two uniform01 draws with u1 mapped to (0, 1], both values of
// a pair used in order (r cos, r sin) -- the SURVEY Appendix A contract the
// product's generator also implements (tests/test_ref_pin.py checks that
// the two agree bit for bit).
struct Gen {
  gbopt::Prng rng;
  bool has_spare = false;
  double spare = 0.0;
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = 1.0 - rng.uniform01();
    const double u2 = rng.uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
};

void* gbref_prng_new(std::uint64_t seed) { return new Gen{gbopt::Prng(seed)}; }
void gbref_prng_free(void* g) { delete static_cast<Gen*>(g); }
void gbref_prng_uniform(void* g, double lo, double hi, std::int64_t n, double* out) {
  auto* G = static_cast<Gen*>(g);
  for (std::int64_t i = 0; i < n; ++i) out[i] = G->rng.uniform(lo, hi);
}
void gbref_prng_normal(void* g, double mean, double sd, std::int64_t n, double* out) {
  auto* G = static_cast<Gen*>(g);
  for (std::int64_t i = 0; i < n; ++i) out[i] = mean + sd * G->normal();
}

}  // extern "C"
