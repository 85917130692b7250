// Host-side network: the immutable parameter set of gbopt::NeuralNet
// (reference include/gbopt/nn.hpp:22-81) plus the device-resident copy the
// oracle kernels read.  Weights are kept row-major (GBNN order) on the host.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "errors.hpp"
#include "prng.hpp"

namespace gbb {

enum Act : int { kLinear = 0, kTanh = 1, kSigmoid = 2, kSoftmax = 3, kSoftplus = 4 };
constexpr int kMaxActCode = 4;

const char* act_name(int act);
int act_from_name(const std::string& name);  // throws StructuralError

struct HostLayer {
  std::int64_t rows = 0, cols = 0;  // out x in
  int act = kLinear;
  std::vector<double> w;  // rows*cols, row-major
  std::vector<double> b;  // rows
};

struct DeviceNet;  // oracle.cu
class MultiPool;   // multi.cpp

class Net {
 public:
  // Validates like the reference constructor (nn.cpp:74-103).
  explicit Net(std::vector<HostLayer> layers);
  ~Net();
  Net(const Net&) = delete;
  Net& operator=(const Net&) = delete;

  std::int64_t input_dim() const { return layers_.front().cols; }
  std::int64_t output_dim() const { return layers_.back().rows; }
  std::int64_t layer_count() const { return static_cast<std::int64_t>(layers_.size()); }
  std::int64_t param_count() const { return param_count_; }
  const HostLayer& layer(std::int64_t l) const { return layers_[static_cast<size_t>(l)]; }
  const std::vector<HostLayer>& layers() const { return layers_; }

  // Device side (oracle.cu).
  DeviceNet& device(int ordinal = -1);  // binds (uploads) on first use
  DeviceNet* device_if_bound() const { return dev_.get(); }
  int bound_ordinal() const;
  // Replicas on several devices for multi-device calls (multi.hpp).
  MultiPool& multi();
  bool use_graphs = true;
  int schedule = -1;  // oracle schedule: -1 auto, 0 layer-by-layer launches, 1 dataflow where the shape allows

 private:
  std::vector<HostLayer> layers_;
  std::int64_t param_count_ = 0;
  std::unique_ptr<DeviceNet> dev_;
  std::unique_ptr<MultiPool> multi_;  // declared after dev_: its slots may point at *dev_
};

// reference random_net (nn.cpp:336-367)
std::unique_ptr<Net> random_net(const std::vector<std::int64_t>& widths, int hidden,
                                int final_act, std::uint64_t seed);

enum Init : int { kUniformFanin = 0, kXavierUniform = 1, kXavierNormal = 2, kNormalFanin = 3 };
std::unique_ptr<Net> random_net_ex(Prng& rng, const std::vector<std::int64_t>& widths,
                                   int hidden, int final_act, int init, double bias_lo,
                                   double bias_hi);

// GBNN v1 (nn_io.cpp:144-247); ".json" paths use the JSON mirror.
std::unique_ptr<Net> load_weights(const std::string& path);
void save_weights(const Net& net, const std::string& path);

}  // namespace gbb
