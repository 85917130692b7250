// Seeded generator: the reference Prng (include/gbopt/prng.hpp:11-23) --
// std::mt19937_64 with uniform01 = (raw >> 11) * 2^-53 -- plus a Box-Muller
// normal (builder-defined; the reference has no normal generator, SURVEY
// Appendix A).  Both values of every Box-Muller pair are used, in order
// (r cos, r sin); u1 is mapped to (0, 1] so log(u1) is finite.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

namespace gbb {

class Prng {
 public:
  explicit Prng(std::uint64_t seed) : eng_(seed) {}

  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  std::uint64_t raw() { return eng_(); }

  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform01();  // (0, 1]
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(a);
    has_spare_ = true;
    return r * std::cos(a);
  }
  double normal(double mean, double stddev) { return mean + stddev * normal(); }

 private:
  std::mt19937_64 eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

}  // namespace gbb
