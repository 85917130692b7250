// Host network construction, validation and seeded generation.
// Follows reference src/nn.cpp:21-41 (names), 74-103 (validation) and
// 336-367 (random_net).
#include "net.hpp"
#include "multi.hpp"

#include "device_net.hpp"
#include "parallel_host.hpp"

#include <atomic>
#include <cmath>
#include <utility>

namespace gbb {

const char* act_name(int act) {
  switch (act) {
    case kLinear: return "linear";
    case kTanh: return "tanh";
    case kSigmoid: return "sigmoid";
    case kSoftmax: return "softmax";
    case kSoftplus: return "softplus";
  }
  return "unknown";
}

int act_from_name(const std::string& name) {
  if (name == "linear") return kLinear;
  if (name == "tanh") return kTanh;
  if (name == "sigmoid") return kSigmoid;
  if (name == "softmax") return kSoftmax;
  if (name == "softplus") return kSoftplus;
  throw StructuralError("unknown activation name: " + name);
}

Net::Net(std::vector<HostLayer> layers) : layers_(std::move(layers)) {
  if (layers_.empty()) throw StructuralError("NeuralNet: at least one layer required");
  for (size_t l = 0; l < layers_.size(); ++l) {
    const HostLayer& lay = layers_[l];
    const std::string tag = "NeuralNet: layer " + std::to_string(l);
    if (lay.rows <= 0 || lay.cols <= 0) throw StructuralError(tag + " has an empty weight matrix");
    if (static_cast<std::int64_t>(lay.w.size()) != lay.rows * lay.cols)
      throw StructuralError(tag + " weight buffer does not match its shape");
    if (static_cast<std::int64_t>(lay.b.size()) != lay.rows)
      throw StructuralError(tag + " weight rows != bias length");
    if (l > 0 && lay.cols != layers_[l - 1].rows)
      throw StructuralError(tag + " input width does not chain");
    if (lay.act < 0 || lay.act > kMaxActCode) throw StructuralError(tag + " bad activation kind");
    std::atomic<bool> finite{true};
    parallel_slices(static_cast<int64_t>(lay.w.size()), int64_t(1) << 20, [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i)
        if (!std::isfinite(lay.w[static_cast<size_t>(i)])) {
          finite = false;
          return;
        }
    });
    if (!finite) throw NumericError(tag + " has non-finite entries");
    for (double v : lay.b)
      if (!std::isfinite(v)) throw NumericError(tag + " has non-finite entries");
    if (lay.act == kSoftmax && l + 1 != layers_.size())
      throw StructuralError("NeuralNet: softmax is only supported on the final layer");
    param_count_ += lay.rows * lay.cols + lay.rows;
  }
}

std::unique_ptr<Net> random_net(const std::vector<std::int64_t>& widths, int hidden,
                                int final_act, std::uint64_t seed) {
  Prng rng(seed);
  return random_net_ex(rng, widths, hidden, final_act, kUniformFanin, 0.0, 0.0);
}

std::unique_ptr<Net> random_net_ex(Prng& rng, const std::vector<std::int64_t>& widths,
                                   int hidden, int final_act, int init, double bias_lo,
                                   double bias_hi) {
  if (widths.size() < 2) throw StructuralError("random_net: need at least input and output width");
  if (init < kUniformFanin || init > kNormalFanin) throw StructuralError("random_net: bad init kind");
  std::vector<HostLayer> layers;
  layers.reserve(widths.size() - 1);
  for (size_t l = 1; l < widths.size(); ++l) {
    const std::int64_t rows = widths[l], cols = widths[l - 1];
    if (rows <= 0 || cols <= 0) throw StructuralError("random_net: widths must be positive");
    HostLayer lay;
    lay.rows = rows;
    lay.cols = cols;
    lay.w.resize(static_cast<size_t>(rows * cols));
    lay.b.resize(static_cast<size_t>(rows));
    const double fi = static_cast<double>(cols), fo = static_cast<double>(rows);
    // Row-major draw order, then the layer's biases (nn.cpp:354-362).
    switch (init) {
      case kUniformFanin: {
        const double bound = 1.0 / std::sqrt(fi);
        for (auto& v : lay.w) v = rng.uniform(-bound, bound);
        for (auto& v : lay.b) v = rng.uniform(-bound, bound);
        break;
      }
      case kXavierUniform: {
        const double bound = std::sqrt(6.0 / (fi + fo));
        for (auto& v : lay.w) v = rng.uniform(-bound, bound);
        break;
      }
      case kXavierNormal: {
        const double sd = std::sqrt(2.0 / (fi + fo));
        for (auto& v : lay.w) v = rng.normal(0.0, sd);
        break;
      }
      case kNormalFanin: {
        const double sd = 1.0 / std::sqrt(fi);
        for (auto& v : lay.w) v = rng.normal(0.0, sd);
        break;
      }
    }
    if (init != kUniformFanin) {
      if (bias_lo == bias_hi) {
        for (auto& v : lay.b) v = bias_lo;
      } else {
        for (auto& v : lay.b) v = rng.uniform(bias_lo, bias_hi);
      }
    }
    lay.act = (l + 1 == widths.size()) ? final_act : hidden;
    layers.push_back(std::move(lay));
  }
  return std::make_unique<Net>(std::move(layers));
}

}  // namespace gbb
