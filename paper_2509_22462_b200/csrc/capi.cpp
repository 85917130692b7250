// C ABI of gbopt_b200 (include/gbopt_b200.h).
//
// Conventions restated from the reference C interface (proj/src/capi.cpp):
// status mapping most-derived-first (capi.cpp:37-59), `guarded` so no
// exception crosses the ABI and the thread-local message is set or cleared
// (capi.cpp:61-74), argument checks before any work (capi.cpp:163-172).
#include "gbopt_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "device_net.hpp"
#include "kkt.hpp"
#include "multi.hpp"
#include "ldlt.hpp"
#include "net.hpp"

struct gbopt_net {
  std::unique_ptr<gbb::Net> net;
};

struct gbopt_prng {
  gbb::Prng rng;
};

struct gbopt_ldlt {
  std::unique_ptr<gbb::Ldlt> f;
};

struct gbopt_kkt {
  std::unique_ptr<gbb::Kkt> k;
};

namespace {

thread_local std::string t_last_error;

gbopt_status to_status(const std::exception_ptr& ep) noexcept {
  try {
    std::rethrow_exception(ep);
  } catch (const gbb::FormatError&) {
    return GBOPT_ERR_FORMAT;
  } catch (const gbb::DimensionError&) {
    return GBOPT_ERR_DIMENSION;
  } catch (const gbb::TruncatedError&) {
    return GBOPT_ERR_TRUNCATED;
  } catch (const gbb::IoError&) {
    return GBOPT_ERR_IO;
  } catch (const gbb::RangeError&) {
    return GBOPT_ERR_RANGE;
  } catch (const gbb::NumericError&) {
    return GBOPT_ERR_NUMERIC;
  } catch (const gbb::SingularError&) {
    return GBOPT_ERR_SINGULAR;
  } catch (const gbb::StructuralError&) {
    return GBOPT_ERR_STRUCTURAL;
  } catch (const gbb::DeviceError&) {
    return GBOPT_ERR_DEVICE;
  } catch (const std::bad_alloc&) {
    return GBOPT_ERR_INTERNAL;
  } catch (...) {
    return GBOPT_ERR_INTERNAL;
  }
}

template <typename F>
gbopt_status guarded(F&& body) noexcept {
  try {
    body();
    t_last_error.clear();
    return GBOPT_OK;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return to_status(std::current_exception());
  } catch (...) {
    t_last_error = "unknown failure";
    return GBOPT_ERR_INTERNAL;
  }
}

gbopt_status fail_argument(const char* msg) noexcept {
  t_last_error = msg;
  return GBOPT_ERR_ARGUMENT;
}

bool dims_ok(const gbopt_net* net, size_t n, size_t m) {
  return static_cast<int64_t>(n) == net->net->input_dim() && static_cast<int64_t>(m) == net->net->output_dim();
}

}  // namespace

extern "C" {

const char* gbopt_last_error(void) { return t_last_error.c_str(); }

const char* gbopt_version(void) { return "gbopt_b200 1.0 sm_100a"; }

int gbopt_device_count(void) { return gbb::device_count(); }

/* ---- prng --------------------------------------------------------------- */

gbopt_status gbopt_prng_new(uint64_t seed, gbopt_prng** out) {
  if (!out) return fail_argument("gbopt_prng_new: out must be non-null");
  return guarded([&] { *out = new gbopt_prng{gbb::Prng(seed)}; });
}

void gbopt_prng_free(gbopt_prng* rng) { delete rng; }

gbopt_status gbopt_prng_raw(gbopt_prng* rng, uint64_t* buf, size_t n) {
  if (!rng || (!buf && n)) return fail_argument("gbopt_prng_raw: null argument");
  return guarded([&] {
    for (size_t i = 0; i < n; ++i) buf[i] = rng->rng.raw();
  });
}

gbopt_status gbopt_prng_uniform(gbopt_prng* rng, double lo, double hi, double* buf, size_t n) {
  if (!rng || (!buf && n)) return fail_argument("gbopt_prng_uniform: null argument");
  return guarded([&] {
    for (size_t i = 0; i < n; ++i) buf[i] = rng->rng.uniform(lo, hi);
  });
}

gbopt_status gbopt_prng_normal(gbopt_prng* rng, double mean, double stddev, double* buf, size_t n) {
  if (!rng || (!buf && n)) return fail_argument("gbopt_prng_normal: null argument");
  return guarded([&] {
    for (size_t i = 0; i < n; ++i) buf[i] = rng->rng.normal(mean, stddev);
  });
}

/* ---- networks ----------------------------------------------------------- */

gbopt_status gbopt_net_load(const char* path, gbopt_net** out) {
  if (path == nullptr || out == nullptr) return fail_argument("gbopt_net_load: path and out must be non-null");
  return guarded([&] {
    auto h = std::make_unique<gbopt_net>();
    h->net = gbb::load_weights(path);
    *out = h.release();
  });
}

gbopt_status gbopt_net_save(const gbopt_net* net, const char* path) {
  if (net == nullptr || path == nullptr) return fail_argument("gbopt_net_save: net and path must be non-null");
  return guarded([&] { gbb::save_weights(*net->net, path); });
}

gbopt_status gbopt_net_random(const int64_t* widths, size_t n_widths, const char* hidden_activation,
                              const char* final_activation, uint64_t seed, gbopt_net** out) {
  if (widths == nullptr || out == nullptr || hidden_activation == nullptr || final_activation == nullptr)
    return fail_argument("gbopt_net_random: pointer arguments must be non-null");
  return guarded([&] {
    std::vector<int64_t> w(widths, widths + n_widths);
    auto h = std::make_unique<gbopt_net>();
    h->net = gbb::random_net(w, gbb::act_from_name(hidden_activation), gbb::act_from_name(final_activation), seed);
    *out = h.release();
  });
}

gbopt_status gbopt_net_random_ex(gbopt_prng* rng, const int64_t* widths, size_t n_widths, int hidden_activation,
                                 int final_activation, int init, double bias_lo, double bias_hi, gbopt_net** out) {
  if (rng == nullptr || widths == nullptr || out == nullptr)
    return fail_argument("gbopt_net_random_ex: pointer arguments must be non-null");
  if (hidden_activation < 0 || hidden_activation > gbb::kMaxActCode || final_activation < 0 ||
      final_activation > gbb::kMaxActCode)
    return fail_argument("gbopt_net_random_ex: invalid activation code");
  return guarded([&] {
    std::vector<int64_t> w(widths, widths + n_widths);
    auto h = std::make_unique<gbopt_net>();
    h->net = gbb::random_net_ex(rng->rng, w, hidden_activation, final_activation, init, bias_lo, bias_hi);
    *out = h.release();
  });
}

gbopt_status gbopt_net_from_layers(size_t n_layers, const int64_t* widths, const int32_t* activations,
                                   const double* const* weights, const double* const* biases, gbopt_net** out) {
  if (out == nullptr || (n_layers > 0 && (widths == nullptr || activations == nullptr || weights == nullptr ||
                                          biases == nullptr)))
    return fail_argument("gbopt_net_from_layers: pointer arguments must be non-null");
  for (size_t l = 0; l < n_layers; ++l)
    if (weights[l] == nullptr || biases[l] == nullptr)
      return fail_argument("gbopt_net_from_layers: null layer buffer");
  return guarded([&] {
    std::vector<gbb::HostLayer> layers(n_layers);
    for (size_t l = 0; l < n_layers; ++l) {
      gbb::HostLayer& lay = layers[l];
      lay.rows = widths[l + 1];
      lay.cols = widths[l];
      lay.act = activations[l];
      if (lay.rows <= 0 || lay.cols <= 0)
        throw gbb::StructuralError("NeuralNet: layer " + std::to_string(l) + " has an empty weight matrix");
      lay.w.assign(weights[l], weights[l] + lay.rows * lay.cols);
      lay.b.assign(biases[l], biases[l] + lay.rows);
    }
    auto h = std::make_unique<gbopt_net>();
    h->net = std::make_unique<gbb::Net>(std::move(layers));
    *out = h.release();
  });
}

void gbopt_net_free(gbopt_net* net) {
  if (!net) return;
  try {
    delete net;
  } catch (...) {
  }
}

int64_t gbopt_net_input_dim(const gbopt_net* net) { return net == nullptr ? 0 : net->net->input_dim(); }
int64_t gbopt_net_output_dim(const gbopt_net* net) { return net == nullptr ? 0 : net->net->output_dim(); }
int64_t gbopt_net_param_count(const gbopt_net* net) { return net == nullptr ? 0 : net->net->param_count(); }
int64_t gbopt_net_layer_count(const gbopt_net* net) { return net == nullptr ? 0 : net->net->layer_count(); }

gbopt_status gbopt_net_layer_info(const gbopt_net* net, int64_t l, int64_t* rows, int64_t* cols,
                                  int32_t* activation) {
  if (net == nullptr) return fail_argument("gbopt_net_layer_info: net must be non-null");
  if (l < 0 || l >= net->net->layer_count()) return fail_argument("gbopt_net_layer_info: layer index out of range");
  return guarded([&] {
    const auto& lay = net->net->layer(l);
    if (rows) *rows = lay.rows;
    if (cols) *cols = lay.cols;
    if (activation) *activation = lay.act;
  });
}

gbopt_status gbopt_net_layer_copy(const gbopt_net* net, int64_t l, double* w, size_t w_len, double* b,
                                  size_t b_len) {
  if (net == nullptr) return fail_argument("gbopt_net_layer_copy: net must be non-null");
  if (l < 0 || l >= net->net->layer_count()) return fail_argument("gbopt_net_layer_copy: layer index out of range");
  const auto& lay = net->net->layer(l);
  if ((w && static_cast<int64_t>(w_len) != lay.rows * lay.cols) || (b && static_cast<int64_t>(b_len) != lay.rows))
    return fail_argument("gbopt_net_layer_copy: buffer lengths do not match the layer shape");
  return guarded([&] {
    if (w) std::memcpy(w, lay.w.data(), sizeof(double) * lay.w.size());
    if (b) std::memcpy(b, lay.b.data(), sizeof(double) * lay.b.size());
  });
}

gbopt_status gbopt_net_bind_device(gbopt_net* net, int ordinal) {
  if (net == nullptr) return fail_argument("gbopt_net_bind_device: net must be non-null");
  if (ordinal < 0) return fail_argument("gbopt_net_bind_device: ordinal must be >= 0");
  return guarded([&] { net->net->device(ordinal); });
}

int gbopt_net_device(const gbopt_net* net) { return net == nullptr ? -1 : net->net->bound_ordinal(); }

gbopt_status gbopt_net_set_graphs(gbopt_net* net, int enabled) {
  if (net == nullptr) return fail_argument("gbopt_net_set_graphs: net must be non-null");
  return guarded([&] { net->net->use_graphs = enabled != 0; });
}

gbopt_status gbopt_net_set_schedule(gbopt_net* net, int schedule) {
  if (net == nullptr) return fail_argument("gbopt_net_set_schedule: net must be non-null");
  if (schedule < -2 || schedule > 1)
    return fail_argument("gbopt_net_set_schedule: schedule must be -2, -1, 0 or 1");
  return guarded([&] { net->net->schedule = schedule; });
}

gbopt_status gbopt_net_dataflow_trace(const gbopt_net* net, size_t batch, const double* dX, const double* dLambda,
                                      double* out, size_t cap, size_t* n_items) {
  if (net == nullptr || dX == nullptr || dLambda == nullptr || n_items == nullptr)
    return fail_argument("gbopt_net_dataflow_trace: null argument");
  if (batch == 0) return fail_argument("gbopt_net_dataflow_trace: batch must be positive");
  return guarded([&] {
    const std::vector<double> t = net->net->device().dataflow_trace(static_cast<int>(batch), dX, dLambda);
    *n_items = t.size() / 12;
    if (out != nullptr) std::copy(t.begin(), t.begin() + static_cast<std::ptrdiff_t>(std::min(t.size(), cap)), out);
  });
}

int gbopt_net_last_schedule(const gbopt_net* net) {
  if (net == nullptr || net->net->device_if_bound() == nullptr) return -1;
  return net->net->device_if_bound()->last_dataflow() ? 1 : 0;
}

int64_t gbopt_net_last_launch_count(const gbopt_net* net) {
  if (net == nullptr || net->net->device_if_bound() == nullptr) return 0;
  return net->net->device_if_bound()->last_launches();
}

/* ---- oracle calls ------------------------------------------------------- */

gbopt_status gbopt_net_forward(const gbopt_net* net, const double* x, size_t n, double* y, size_t m) {
  if (net == nullptr || x == nullptr || y == nullptr)
    return fail_argument("gbopt_net_forward: pointer arguments must be non-null");
  if (!dims_ok(net, n, m))
    return fail_argument("gbopt_net_forward: buffer lengths do not match the network dimensions");
  return guarded([&] {
    net->net->device().evaluate_host(1, x, nullptr, y, nullptr, nullptr, nullptr);
  });
}

gbopt_status gbopt_net_forward_trace(const gbopt_net* net, const double* x, size_t n, double* z, double* y,
                                     size_t len) {
  if (net == nullptr || x == nullptr || z == nullptr || y == nullptr)
    return fail_argument("gbopt_net_forward_trace: pointer arguments must be non-null");
  const gbb::Net& nn = *net->net;
  int64_t total = 0;
  for (int64_t l = 0; l < nn.layer_count(); ++l) total += nn.layer(l).rows;
  if (static_cast<int64_t>(n) != nn.input_dim() || static_cast<int64_t>(len) != total)
    return fail_argument("gbopt_net_forward_trace: buffer lengths do not match the network dimensions");
  return guarded([&] {
    gbb::DeviceNet& d = net->net->device();
    const int64_t L = nn.layer_count();
    const int64_t last = nn.layer(L - 1).rows;
    // one forward pass; the final y (softmax applied) is the output, the
    // rest are the forward chain's per-layer buffers
    d.evaluate_host(1, x, nullptr, y + (total - last), nullptr, nullptr, nullptr);
    int64_t off = 0;
    for (int64_t l = 0; l < L; ++l) {
      d.copy_intermediate("z", static_cast<int>(l), 1, z + off);
      if (l + 1 < L) d.copy_intermediate("y", static_cast<int>(l), 1, y + off);
      off += nn.layer(l).rows;
    }
  });
}

gbopt_status gbopt_net_jacobian(const gbopt_net* net, const double* x, size_t n, double* jac, size_t jac_len) {
  if (net == nullptr || x == nullptr || jac == nullptr)
    return fail_argument("gbopt_net_jacobian: pointer arguments must be non-null");
  const int64_t m = net->net->output_dim();
  if (static_cast<int64_t>(n) != net->net->input_dim() || static_cast<int64_t>(jac_len) != m * static_cast<int64_t>(n))
    return fail_argument("gbopt_net_jacobian: buffer lengths do not match the network dimensions");
  return guarded([&] {
    net->net->device().evaluate_host(1, x, nullptr, nullptr, jac, nullptr, nullptr);
  });
}

gbopt_status gbopt_net_lagrangian_gradient(const gbopt_net* net, const double* x, size_t n, const double* lambda,
                                           size_t m, double* g, size_t g_len) {
  if (net == nullptr || x == nullptr || lambda == nullptr || g == nullptr)
    return fail_argument("gbopt_net_lagrangian_gradient: pointer arguments must be non-null");
  if (!dims_ok(net, n, m) || g_len != n)
    return fail_argument("gbopt_net_lagrangian_gradient: buffer lengths do not match the network dimensions");
  return guarded([&] {
    net->net->device().evaluate_host(1, x, lambda, nullptr, nullptr, nullptr, g);
  });
}

gbopt_status gbopt_net_lagrangian_hessian(const gbopt_net* net, const double* x, size_t n, const double* lambda,
                                          size_t m, double* hess, size_t hess_len) {
  if (net == nullptr || x == nullptr || lambda == nullptr || hess == nullptr)
    return fail_argument("gbopt_net_lagrangian_hessian: pointer arguments must be non-null");
  if (!dims_ok(net, n, m) || hess_len != n * n)
    return fail_argument("gbopt_net_lagrangian_hessian: buffer lengths do not match the network dimensions");
  return guarded([&] {
    net->net->device().evaluate_host(1, x, lambda, nullptr, nullptr, hess, nullptr);
  });
}

gbopt_status gbopt_net_oracle(const gbopt_net* net, const double* x, size_t n, const double* lambda, size_t m,
                              double* y, double* jac, double* hess) {
  return gbopt_net_oracle_batched(net, 1, x, n, lambda, m, y, jac, hess);
}

gbopt_status gbopt_net_oracle_batched(const gbopt_net* net, size_t batch, const double* X, size_t n,
                                      const double* Lambda, size_t m, double* Y, double* J, double* H) {
  if (net == nullptr || X == nullptr) return fail_argument("gbopt_net_oracle: net and x must be non-null");
  if (H != nullptr && Lambda == nullptr) return fail_argument("gbopt_net_oracle: lambda is required for the Hessian");
  if (!dims_ok(net, n, m)) return fail_argument("gbopt_net_oracle: lengths do not match the network dimensions");
  if (batch == 0) return fail_argument("gbopt_net_oracle: batch must be positive");
  if (batch > (1u << 30)) return fail_argument("gbopt_net_oracle: batch too large");
  return guarded([&] {
    net->net->device().evaluate_host(static_cast<int>(batch), X, Lambda, Y, J, H, nullptr);
  });
}

static gbopt_status multi_args(const gbopt_net* net, const int* devices, size_t n_devices, size_t batch,
                               const double* X, size_t n, const double* Lambda, size_t m, const double* H,
                               const char* who) {
  if (net == nullptr || X == nullptr || devices == nullptr)
    return fail_argument((std::string(who) + ": net, devices and X must be non-null").c_str());
  if (n_devices == 0 || n_devices > 1024) return fail_argument((std::string(who) + ": n_devices out of range").c_str());
  if (H != nullptr && Lambda == nullptr) return fail_argument((std::string(who) + ": lambda is required for the Hessian").c_str());
  if (!dims_ok(net, n, m)) return fail_argument((std::string(who) + ": lengths do not match the network dimensions").c_str());
  if (batch == 0 || batch > (1u << 30)) return fail_argument((std::string(who) + ": batch out of range").c_str());
  return GBOPT_OK;
}

gbopt_status gbopt_net_oracle_batched_multi(const gbopt_net* net, const int* devices, size_t n_devices, size_t batch,
                                            const double* X, size_t n, const double* Lambda, size_t m, double* Y,
                                            double* J, double* H) {
  const gbopt_status a = multi_args(net, devices, n_devices, batch, X, n, Lambda, m, H,
                                    "gbopt_net_oracle_batched_multi");
  if (a != GBOPT_OK) return a;
  return guarded([&] {
    net->net->multi().evaluate_host(std::vector<int>(devices, devices + n_devices), static_cast<int>(batch), X,
                                    Lambda, Y, J, H);
  });
}

gbopt_status gbopt_net_oracle_batched_multi_gather(const gbopt_net* net, const int* devices, size_t n_devices,
                                                   size_t batch, const double* dX, size_t n, const double* dLambda,
                                                   size_t m, double* dY, double* dJ, double* dH) {
  const gbopt_status a = multi_args(net, devices, n_devices, batch, dX, n, dLambda, m, dH,
                                    "gbopt_net_oracle_batched_multi_gather");
  if (a != GBOPT_OK) return a;
  return guarded([&] {
    net->net->multi().evaluate_gather(std::vector<int>(devices, devices + n_devices), static_cast<int>(batch), dX,
                                      dLambda, dY, dJ, dH);
  });
}

gbopt_status gbopt_net_oracle_lower(const gbopt_net* net, size_t batch, const double* X, size_t n,
                                    const double* Lambda, size_t m, double* Y, double* J, double* Hl,
                                    size_t hl_len) {
  if (net == nullptr || X == nullptr || Lambda == nullptr || Hl == nullptr)
    return fail_argument("gbopt_net_oracle_lower: net, X, Lambda and Hl must be non-null");
  if (!dims_ok(net, n, m)) return fail_argument("gbopt_net_oracle_lower: lengths do not match the network dimensions");
  if (batch == 0 || batch > (1u << 30)) return fail_argument("gbopt_net_oracle_lower: batch out of range");
  if (hl_len != batch * n * (n + 1) / 2)
    return fail_argument("gbopt_net_oracle_lower: Hl must hold batch * n * (n + 1) / 2 values");
  return guarded([&] {
    net->net->device().evaluate_host(static_cast<int>(batch), X, Lambda, Y, J, Hl, nullptr, true);
  });
}

gbopt_status gbopt_net_oracle_batched_device(const gbopt_net* net, size_t batch, const double* dX, size_t n,
                                             const double* dLambda, size_t m, double* dY, double* dJ, double* dH,
                                             void* stream) {
  if (net == nullptr || dX == nullptr) return fail_argument("gbopt_net_oracle_batched_device: null argument");
  if (dH != nullptr && dLambda == nullptr)
    return fail_argument("gbopt_net_oracle_batched_device: lambda is required for the Hessian");
  if (!dims_ok(net, n, m))
    return fail_argument("gbopt_net_oracle_batched_device: lengths do not match the network dimensions");
  if (batch == 0) return fail_argument("gbopt_net_oracle_batched_device: batch must be positive");
  return guarded([&] {
    net->net->device().evaluate_device(static_cast<int>(batch), dX, dLambda, dY, dJ, dH,
                                       static_cast<cudaStream_t>(stream));
  });
}

gbopt_status gbopt_net_profile(const gbopt_net* net, size_t batch, const double* dX, const double* dLambda,
                               int32_t* tags, float* ms, double* flops, double* bytes, size_t cap, size_t* count) {
  if (net == nullptr || dX == nullptr || dLambda == nullptr || count == nullptr)
    return fail_argument("gbopt_net_profile: null argument");
  if (batch == 0) return fail_argument("gbopt_net_profile: batch must be positive");
  return guarded([&] {
    std::vector<gbb::ProfResult> res;
    net->net->device().profile(static_cast<int>(batch), dX, dLambda, &res);
    *count = res.size();
    for (size_t i = 0; i < res.size() && i < cap; ++i) {
      if (tags) tags[i] = res[i].tag;
      if (ms) ms[i] = res[i].ms;
      if (flops) flops[i] = res[i].flops;
      if (bytes) bytes[i] = res[i].bytes;
    }
  });
}

const char* gbopt_kernel_tag_name(int tag) { return gbb::kernel_tag_name(tag); }

gbopt_status gbopt_net_profile_timeline(const gbopt_net* net, size_t batch, const double* dX, const double* dLambda,
                                        int32_t* tags, int32_t* streams, float* t_start, float* t_end, size_t cap,
                                        size_t* count) {
  if (net == nullptr || dX == nullptr || dLambda == nullptr || count == nullptr)
    return fail_argument("gbopt_net_profile_timeline: null argument");
  if (batch == 0) return fail_argument("gbopt_net_profile_timeline: batch must be positive");
  return guarded([&] {
    std::vector<gbb::ProfResult> res;
    net->net->device().profile(static_cast<int>(batch), dX, dLambda, &res, true);
    *count = res.size();
    for (size_t i = 0; i < res.size() && i < cap; ++i) {
      if (tags) tags[i] = res[i].tag;
      if (streams) streams[i] = res[i].stream;
      if (t_start) t_start[i] = res[i].t0;
      if (t_end) t_end[i] = res[i].t1;
    }
  });
}

gbopt_status gbopt_net_debug_intermediate(const gbopt_net* net, const char* name, int64_t layer, size_t batch,
                                          double* out, size_t len) {
  if (net == nullptr || name == nullptr || out == nullptr)
    return fail_argument("gbopt_net_debug_intermediate: null argument");
  if (layer < 0 || layer >= net->net->layer_count())
    return fail_argument("gbopt_net_debug_intermediate: layer out of range");
  if (len != batch * static_cast<size_t>(net->net->layer(layer).rows))
    return fail_argument("gbopt_net_debug_intermediate: len must be batch * rows(layer)");
  return guarded([&] {
    gbb::DeviceNet* d = net->net->device_if_bound();
    if (!d) throw gbb::StructuralError("gbopt_net_debug_intermediate: no evaluation has run");
    d->copy_intermediate(name, static_cast<int>(layer), static_cast<int>(batch), out);
  });
}

/* ---- KKT factorisation ---------------------------------------------------- */

gbopt_status gbopt_ldlt_factor(const double* A, size_t n, int keep_input, gbopt_ldlt** out) {
  if (out == nullptr || (A == nullptr && n > 0)) return fail_argument("gbopt_ldlt_factor: null argument");
  return guarded([&] {
    auto h = std::make_unique<gbopt_ldlt>();
    h->f = gbb::Ldlt::factor(A, static_cast<int64_t>(n), keep_input != 0);
    *out = h.release();
  });
}

gbopt_status gbopt_ldlt_inertia(const gbopt_ldlt* f, int64_t* n_pos, int64_t* n_neg, int64_t* n_zero) {
  if (f == nullptr) return fail_argument("gbopt_ldlt_inertia: null factorization");
  return guarded([&] {
    if (n_pos) *n_pos = f->f->n_pos();
    if (n_neg) *n_neg = f->f->n_neg();
    if (n_zero) *n_zero = f->f->n_zero();
  });
}

gbopt_status gbopt_ldlt_solve(const gbopt_ldlt* f, const double* b, size_t n, double* x) {
  if (f == nullptr || ((b == nullptr || x == nullptr) && n > 0)) return fail_argument("gbopt_ldlt_solve: null argument");
  return guarded([&] {
    const std::vector<double> r = f->f->solve(b, static_cast<int64_t>(n));
    std::copy(r.begin(), r.end(), x);
  });
}

void gbopt_ldlt_free(gbopt_ldlt* f) { delete f; }

/* ---- KKT assembly and inertia correction ---------------------------------- */

gbopt_status gbopt_kkt_create(size_t n, size_t m, const int64_t* hess_rows, const int64_t* hess_cols, size_t nnz_h,
                              const int64_t* jac_rows, const int64_t* jac_cols, size_t nnz_j, gbopt_kkt** out) {
  if (out == nullptr || ((hess_rows == nullptr || hess_cols == nullptr) && nnz_h > 0) ||
      ((jac_rows == nullptr || jac_cols == nullptr) && nnz_j > 0))
    return fail_argument("gbopt_kkt_create: null argument");
  return guarded([&] {
    auto h = std::make_unique<gbopt_kkt>();
    h->k = std::make_unique<gbb::Kkt>(static_cast<int64_t>(n), static_cast<int64_t>(m), hess_rows, hess_cols, nnz_h,
                                      jac_rows, jac_cols, nnz_j);
    *out = h.release();
  });
}

gbopt_status gbopt_kkt_assemble(gbopt_kkt* kkt, const double* x, const double* lower, const double* z,
                                const double* lambda, const double* grad_f, const double* g, const double* jac_values,
                                const double* hess_values, double mu, double delta_w, double delta_c) {
  if (kkt == nullptr) return fail_argument("gbopt_kkt_assemble: null system");
  const auto& k = *kkt->k;
  const bool nv = k.n_var() > 0, mv = k.n_con() > 0;
  if ((nv && (!x || !lower || !z || !grad_f)) || (mv && (!lambda || !g)) || (k.nnz_h() > 0 && !hess_values) ||
      (k.nnz_j() > 0 && !jac_values))
    return fail_argument("gbopt_kkt_assemble: null argument");
  return guarded([&] {
    kkt->k->assemble(x, lower, z, lambda, grad_f, g, jac_values, hess_values, mu, delta_w, delta_c);
  });
}

gbopt_status gbopt_kkt_matrix(const gbopt_kkt* kkt, double* out, size_t len) {
  if (kkt == nullptr) return fail_argument("gbopt_kkt_matrix: null system");
  const size_t dim = static_cast<size_t>(kkt->k->dim());
  if (len != dim * dim || (out == nullptr && len > 0)) return fail_argument("gbopt_kkt_matrix: out must hold (n+m)^2");
  return guarded([&] { kkt->k->matrix(out); });
}

gbopt_status gbopt_kkt_rhs(const gbopt_kkt* kkt, double* out, size_t len) {
  if (kkt == nullptr) return fail_argument("gbopt_kkt_rhs: null system");
  if (len != static_cast<size_t>(kkt->k->dim()) || (out == nullptr && len > 0))
    return fail_argument("gbopt_kkt_rhs: out must hold n+m");
  return guarded([&] { kkt->k->rhs(out); });
}

gbopt_status gbopt_kkt_inertia_correct(const gbopt_kkt* kkt, double delta0, double delta_growth, double delta_max,
                                       double delta_w_start, gbopt_ldlt** fact, double* delta_w, double* delta_c) {
  if (kkt == nullptr || fact == nullptr) return fail_argument("gbopt_kkt_inertia_correct: null argument");
  if (!(delta_growth > 1.0)) return fail_argument("gbopt_kkt_inertia_correct: delta_growth must be > 1");
  return guarded([&] {
    auto c = kkt->k->inertia_correct(delta0, delta_growth, delta_max, delta_w_start);
    auto h = std::make_unique<gbopt_ldlt>();
    h->f = std::move(c.fact);
    if (delta_w) *delta_w = c.delta_w;
    if (delta_c) *delta_c = c.delta_c;
    *fact = h.release();
  });
}

gbopt_status gbopt_kkt_solve(const gbopt_kkt* kkt, const gbopt_ldlt* fact, double* sol, size_t len) {
  if (kkt == nullptr || fact == nullptr) return fail_argument("gbopt_kkt_solve: null argument");
  if (len != static_cast<size_t>(kkt->k->dim()) || (sol == nullptr && len > 0))
    return fail_argument("gbopt_kkt_solve: sol must hold n+m");
  if (fact->f->dim() != kkt->k->dim()) return fail_argument("gbopt_kkt_solve: factorization of another size");
  return guarded([&] {
    const std::vector<double> r = kkt->k->solve(*fact->f);
    std::copy(r.begin(), r.end(), sol);
  });
}

void gbopt_kkt_free(gbopt_kkt* kkt) { delete kkt; }

}  // extern "C"
