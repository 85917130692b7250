// C++ drop-in checks for include/gbopt/kkt_b200.hpp (reference linalg.hpp /
// ipm.hpp KKT API) over libgbopt_b200.so; cases restated from
// proj/tests/test_ipm.cpp:313-470 and proj/tests/test_linalg.cpp:42-76.
//   ./test_kkt_b200        host-side checks (no GPU needed)
//   ./test_kkt_b200 gpu    + device checks
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>

#include "gbopt/kkt_b200.hpp"

using namespace gbopt::b200;

static int g_fail = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);       \
      ++g_fail;                                                      \
    }                                                                \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  const double inf = std::numeric_limits<double>::infinity();
  // ---- host side: argument and pattern checks come before any device work ----
  CHECK(throws<StructuralError>([] { KktPattern(3, 1, {0, 3}, {0, 0}, {}, {}); }));
  CHECK(throws<StructuralError>([] { KktPattern(3, 1, {0}, {0, 1}, {}, {}); }));
  CHECK(throws<StructuralError>([] { ldlt_factor(DenseMat(2, 3)); }));
  if (!gpu) {
    if (gbopt_device_count() == 0) CHECK(throws<DeviceError>([] { KktPattern(1, 0, {0}, {0}, {}, {}); }));
    std::printf(g_fail ? "FAILED %d\n" : "ok\n", g_fail);
    return g_fail ? 1 : 0;
  }
  // ---- device ----
  {  // test_ipm.cpp:313-326: bounded variable folds z/x into the (1,1) block
    KktSystem s = assemble_kkt({1.0}, {0.0}, {0.1}, {}, {0.3}, {}, {}, {}, {}, {0}, {0}, {2.0}, 0.1);
    CHECK(s.mat().rows == 1);
    CHECK(std::fabs(s.mat()(0, 0) - 2.1) < 1e-15);
    CHECK(std::fabs(s.rhs()[0] + 0.2) < 1e-15);
  }
  {  // test_ipm.cpp:328-344: one variable, one linear constraint, exact
    KktSystem s = assemble_kkt({0.4}, {-inf}, {0.0}, {0.0}, {0.0}, {0.4}, {0}, {0}, {1.0}, {0}, {0}, {3.0}, 0.1);
    const DenseMat a = s.mat();
    CHECK(a(0, 0) == 3.0 && a(0, 1) == 1.0 && a(1, 0) == 1.0 && a(1, 1) == 0.0);
    CHECK(std::fabs(s.rhs()[1] + 0.4) < 1e-15);
  }
  {  // test_ipm.cpp:430-446: negative-definite block needs delta_w = 10
    KktSystem s = assemble_kkt({0.0, 0.0}, {-inf, -inf}, {0.0, 0.0}, {}, {0.0, 0.0}, {}, {}, {}, {}, {0, 1}, {0, 1},
                               {-1.0, -1.0}, 0.0);
    CorrectedFactorization cf = inertia_correct(s, {});
    CHECK(std::fabs(cf.delta_w - 10.0) < 1e-12);
    CHECK((cf.fact.inertia() == Inertia{2, 0, 0}));
    CHECK(cf.fact.dim() == 2);
    IpmOptions tight;
    tight.delta_max = 1.0;
    CHECK(throws<SingularError>([&] { inertia_correct(s, tight); }));
  }
  {  // convex QP KKT (test_ipm.cpp:409-428): no regularisation; solve through the device rhs
    // q = [[4, 1], [1, 3]], a = [1, 1]; rhs from grad_f = (1, 2), g = (0.5)
    KktSystem s = assemble_kkt({0.0, 0.0}, {-inf, -inf}, {0.0, 0.0}, {0.0}, {1.0, 2.0}, {0.5}, {0, 0}, {0, 1},
                               {1.0, 1.0}, {0, 1, 1}, {0, 0, 1}, {4.0, 1.0, 3.0}, 0.0);
    CorrectedFactorization cf = inertia_correct(s);
    CHECK(cf.delta_w == 0.0 && cf.delta_c == 0.0);
    CHECK((cf.fact.inertia() == Inertia{2, 1, 0}));
    const RealVec x = s.solve(cf.fact), x2 = cf.fact.solve(s.rhs());
    CHECK(x == x2);
    const DenseMat a = s.mat();
    const RealVec b = s.rhs();
    for (int i = 0; i < 3; ++i) {
      double r = -b[i];
      for (int j = 0; j < 3; ++j) r += a(i, j) * x[j];
      CHECK(std::fabs(r) < 1e-12);
    }
  }
  {  // test_linalg.cpp:42-76: known inertias through ldlt_factor
    DenseMat d(2, 2);
    d(0, 0) = 2.0;
    d(1, 1) = -5.0;
    CHECK((ldlt_factor(d).inertia() == Inertia{1, 1, 0}));
    DenseMat z(2, 2);
    z(0, 1) = z(1, 0) = 1.0;
    CHECK((ldlt_factor(z).inertia() == Inertia{1, 1, 0}));
    const RealVec x = ldlt_solve(ldlt_factor(d), {2.0, 5.0});
    CHECK(std::fabs(x[0] - 1.0) < 1e-14 && std::fabs(x[1] + 1.0) < 1e-14);
  }
  std::printf(g_fail ? "FAILED %d\n" : "ok\n", g_fail);
  return g_fail ? 1 : 0;
}
