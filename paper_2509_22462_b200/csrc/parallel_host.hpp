// Host-side data parallelism for the one-time bulk work around the
// device: reading GBNN payloads, validating weights, staging uploads
// (~872 MB for the 109M-parameter net).
#pragma once

#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace gbb {

// Calls fn(begin, end) on up to `max_threads` contiguous slices of
// [0, n); slices below `grain` elements are not split further.  fn must not
// throw (report failures through captured state, as the callers do).
template <class Fn>
void parallel_slices(int64_t n, int64_t grain, Fn&& fn, int max_threads = 8) {
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t parts = std::max<int64_t>(1, std::min<int64_t>({static_cast<int64_t>(max_threads), hw, n / std::max<int64_t>(grain, 1)}));
  if (parts <= 1) {
    fn(int64_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(static_cast<size_t>(parts - 1));
  for (int64_t p = 1; p < parts; ++p)
    pool.emplace_back([&fn, n, parts, p] { fn(n * p / parts, n * (p + 1) / parts); });
  fn(int64_t(0), n / parts);
  for (auto& t : pool) t.join();
}

}  // namespace gbb
