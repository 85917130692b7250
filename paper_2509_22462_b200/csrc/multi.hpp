// Multi-device evaluation inside one process, for C++ callers that hold one
// network handle (the drop-in target: the reduced-space embedding keeps one
// shared_ptr<const NeuralNet>, reference formulations.cpp:276).
//
// The weights are replicated: one DeviceNet per slot, uploaded from the
// shared host copy; slot i runs on devices[i] (a device may appear more than
// once -- independent workspaces and streams on the same GPU).  B points are
// split into contiguous shards (the first B % S slots take one extra point,
// the rule of paper_2509_22462_b200/parallel.py), one host thread per slot.
// There is no reduction between devices:
//   * evaluate_host: each slot copies its shard of x / lambda from the
//     caller's host buffers and writes its (y, J, H) rows straight back into
//     the caller's host buffers (D2H per device, in parallel);
//   * evaluate_gather: inputs and outputs live on devices[0]; each remote
//     slot pulls its shard of x / lambda over NVLink (cudaMemcpyPeerAsync,
//     peer access enabled where the topology allows), evaluates, and pushes
//     its rows into the output buffers on devices[0] -- the result gather,
//     done by the copy engines, so device 0 can assemble the KKT system
//     (f3) from device-resident blocks.  Slots on devices[0] itself read and
//     write the caller's buffers directly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace gbb {

class Net;
class DeviceNet;

struct MultiSlot {
  int ordinal = 0;
  DeviceNet* dn = nullptr;           // the net's bound DeviceNet or `own`
  std::unique_ptr<DeviceNet> own;
  cudaStream_t st = nullptr;
  double *x = nullptr, *lam = nullptr, *y = nullptr, *j = nullptr, *h = nullptr;  // remote-slot staging
  int cap = 0;
  MultiSlot();
  ~MultiSlot();
  MultiSlot(MultiSlot&&) noexcept;
  MultiSlot& operator=(MultiSlot&&) noexcept;
};

class MultiPool {
 public:
  explicit MultiPool(Net& net);
  ~MultiPool();
  MultiPool(const MultiPool&) = delete;
  MultiPool& operator=(const MultiPool&) = delete;

  void evaluate_host(const std::vector<int>& devices, int nb, const double* X, const double* Lam, double* Y,
                     double* J, double* H);
  void evaluate_gather(const std::vector<int>& devices, int nb, const double* dX, const double* dLam, double* dY,
                       double* dJ, double* dH);
  // Contiguous shard [start, start + count) of `points` for slot r of s.
  static void shard(int points, int s, int r, int* start, int* count);

 private:
  void configure(const std::vector<int>& devices);
  void ensure_staging(MultiSlot& s, int nb);

  Net& net_;
  std::vector<int> devices_;
  std::vector<MultiSlot> slots_;
  std::mutex mu_;
};

}  // namespace gbb
