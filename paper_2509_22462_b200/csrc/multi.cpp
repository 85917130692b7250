// Multi-device evaluation inside one process; see multi.hpp.
#include "multi.hpp"

#include <cstdlib>
#include <exception>
#include <string>
#include <thread>
#include <utility>

#include "device_net.hpp"
#include "errors.hpp"
#include "net.hpp"

namespace gbb {

namespace {

void ck(cudaError_t e, const char* what) { cuda_check(e, what); }

// Direct NVLink reads/writes between the two devices when the topology
// allows; cudaMemcpyPeerAsync falls back to a staged copy otherwise.
void enable_peer(int a, int b) {
  if (a == b) return;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) {
    cudaGetLastError();
    return;
  }
  DeviceGuard g(a);
  const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
  cudaGetLastError();
}

template <class F>
void run_slots(int n, F&& f) {
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    th.emplace_back([&, i] {
      try {
        f(i);
      } catch (...) {
        err[static_cast<size_t>(i)] = std::current_exception();
      }
    });
  }
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

}  // namespace

MultiSlot::MultiSlot() = default;
// Moves hand over the raw CUDA handles: the moved-from slot must not free
// the stream and buffers the new owner keeps using.
MultiSlot::MultiSlot(MultiSlot&& o) noexcept { *this = std::move(o); }
MultiSlot& MultiSlot::operator=(MultiSlot&& o) noexcept {
  if (this == &o) return *this;
  ordinal = o.ordinal;
  own = std::move(o.own);
  dn = std::exchange(o.dn, nullptr);
  st = std::exchange(o.st, nullptr);
  x = std::exchange(o.x, nullptr);
  lam = std::exchange(o.lam, nullptr);
  y = std::exchange(o.y, nullptr);
  j = std::exchange(o.j, nullptr);
  h = std::exchange(o.h, nullptr);
  cap = std::exchange(o.cap, 0);
  return *this;
}
MultiSlot::~MultiSlot() {
  if (st == nullptr && x == nullptr && lam == nullptr && y == nullptr && j == nullptr && h == nullptr) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ordinal);
  for (double* p : {x, lam, y, j, h})
    if (p) cudaFree(p);
  if (st) cudaStreamDestroy(st);
  if (prev >= 0) cudaSetDevice(prev);
  cudaGetLastError();
}

MultiPool::MultiPool(Net& net) : net_(net) {}
MultiPool::~MultiPool() = default;

void MultiPool::shard(int points, int s, int r, int* start, int* count) {
  const int base = points / s, extra = points % s;
  *count = base + (r < extra ? 1 : 0);
  *start = r * base + (r < extra ? r : extra);
}

void MultiPool::configure(const std::vector<int>& devices) {
  if (devices.empty()) throw StructuralError("oracle_batched_multi: at least one device required");
  const int have = device_count();
  for (int d : devices)
    if (d < 0 || d >= have)
      throw DeviceError("oracle_batched_multi: CUDA device " + std::to_string(d) + " not available (" +
                        std::to_string(have) + " visible)");
  if (devices == devices_) return;
  slots_.clear();
  // The net's bound DeviceNet serves the first slot on its device; every
  // other slot owns a replica uploaded from the shared host copy.
  DeviceNet* bound = net_.device_if_bound();
  bool bound_used = false;
  for (int d : devices) {
    MultiSlot s;
    s.ordinal = d;
    if (bound && !bound_used && bound->ordinal() == d) {
      s.dn = bound;
      bound_used = true;
    } else {
      s.own = std::make_unique<DeviceNet>(net_, d);
      s.dn = s.own.get();
    }
    DeviceGuard g(d);
    ck(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking), "cudaStreamCreate");
    slots_.push_back(std::move(s));
  }
  for (size_t i = 1; i < devices.size(); ++i) {
    enable_peer(devices[0], devices[i]);
    enable_peer(devices[i], devices[0]);
  }
  devices_ = devices;
}

void MultiPool::ensure_staging(MultiSlot& s, int nb) {
  if (nb <= s.cap) return;
  DeviceGuard g(s.ordinal);
  for (double** p : {&s.x, &s.lam, &s.y, &s.j, &s.h}) {
    if (*p) ck(cudaFree(*p), "cudaFree");
    *p = nullptr;
  }
  const size_t n = static_cast<size_t>(net_.input_dim()), m = static_cast<size_t>(net_.output_dim());
  const size_t b = static_cast<size_t>(nb);
  ck(cudaMalloc(&s.x, sizeof(double) * b * n), "cudaMalloc");
  ck(cudaMalloc(&s.lam, sizeof(double) * b * m), "cudaMalloc");
  ck(cudaMalloc(&s.y, sizeof(double) * b * m), "cudaMalloc");
  ck(cudaMalloc(&s.j, sizeof(double) * b * m * n), "cudaMalloc");
  ck(cudaMalloc(&s.h, sizeof(double) * b * n * n), "cudaMalloc");
  s.cap = nb;
}

void MultiPool::evaluate_host(const std::vector<int>& devices, int nb, const double* X, const double* Lam, double* Y,
                              double* J, double* H) {
  std::lock_guard<std::mutex> lock(mu_);
  configure(devices);
  const int S = static_cast<int>(slots_.size());
  const size_t n = static_cast<size_t>(net_.input_dim()), m = static_cast<size_t>(net_.output_dim());
  run_slots(S, [&](int i) {
    int start = 0, count = 0;
    shard(nb, S, i, &start, &count);
    if (count == 0) return;
    const size_t s0 = static_cast<size_t>(start);
    slots_[static_cast<size_t>(i)].dn->evaluate_host(count, X + s0 * n, Lam ? Lam + s0 * m : nullptr,
                                                     Y ? Y + s0 * m : nullptr, J ? J + s0 * m * n : nullptr,
                                                     H ? H + s0 * n * n : nullptr, nullptr);
  });
}

void MultiPool::evaluate_gather(const std::vector<int>& devices, int nb, const double* dX, const double* dLam,
                                double* dY, double* dJ, double* dH) {
  std::lock_guard<std::mutex> lock(mu_);
  configure(devices);
  const int S = static_cast<int>(slots_.size());
  const int home = devices_[0];
  const size_t n = static_cast<size_t>(net_.input_dim()), m = static_cast<size_t>(net_.output_dim());
  run_slots(S, [&](int i) {
    MultiSlot& s = slots_[static_cast<size_t>(i)];
    int start = 0, count = 0;
    shard(nb, S, i, &start, &count);
    if (count == 0) return;
    const size_t s0 = static_cast<size_t>(start), c = static_cast<size_t>(count);
    DeviceGuard g(s.ordinal);
    // GBOPT_MULTI_STAGE=1 sends slots other than the first through the
    // staging + copy path even on the home device (tests on one GPU).
    const char* fs = std::getenv("GBOPT_MULTI_STAGE");
    const bool force_stage = fs && fs[0] == '1';
    if (s.ordinal == home && !(force_stage && i > 0)) {
      s.dn->evaluate_device(count, dX + s0 * n, dLam ? dLam + s0 * m : nullptr, dY ? dY + s0 * m : nullptr,
                            dJ ? dJ + s0 * m * n : nullptr, dH ? dH + s0 * n * n : nullptr, s.st);
    } else {
      ensure_staging(s, count);
      ck(cudaMemcpyPeerAsync(s.x, s.ordinal, dX + s0 * n, home, sizeof(double) * c * n, s.st), "peer copy x");
      if (dLam)
        ck(cudaMemcpyPeerAsync(s.lam, s.ordinal, dLam + s0 * m, home, sizeof(double) * c * m, s.st),
           "peer copy lambda");
      s.dn->evaluate_device(count, s.x, dLam ? s.lam : nullptr, dY ? s.y : nullptr, dJ ? s.j : nullptr,
                            dH ? s.h : nullptr, s.st);
      if (dY) ck(cudaMemcpyPeerAsync(dY + s0 * m, home, s.y, s.ordinal, sizeof(double) * c * m, s.st), "gather y");
      if (dJ)
        ck(cudaMemcpyPeerAsync(dJ + s0 * m * n, home, s.j, s.ordinal, sizeof(double) * c * m * n, s.st),
           "gather J");
      if (dH)
        ck(cudaMemcpyPeerAsync(dH + s0 * n * n, home, s.h, s.ordinal, sizeof(double) * c * n * n, s.st),
           "gather H");
    }
    ck(cudaStreamSynchronize(s.st), "multi-device evaluation");
  });
}

}  // namespace gbb
