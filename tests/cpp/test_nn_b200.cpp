// C++ drop-in checks: include/gbopt/nn_b200.hpp over libgbopt_b200.so.
// Mirrors the network cases of proj/tests/test_capi.cpp and the reduced-space
// cases of proj/tests/test_formulations.cpp:215-274.
//   ./test_nn_b200        host-side checks (no GPU needed)
//   ./test_nn_b200 gpu    + device checks (oracle, reduced-space callbacks)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "gbopt/nn_b200.hpp"

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
  // ---- host side ----
  NeuralNet net = random_net({4, 6, 3}, "tanh", "softmax", 11);
  CHECK(net.input_dim() == 4 && net.output_dim() == 3);
  CHECK(net.param_count() == 4 * 6 + 6 + 6 * 3 + 3);
  const std::string path = "/tmp/gbopt_b200_cpp_test.gbnn";
  save_weights(net, path);
  NeuralNet back = load_weights(path);
  for (int64_t l = 0; l < net.layer_count(); ++l) {
    Layer a = net.layer(l), b = back.layer(l);
    CHECK(a.weight.data == b.weight.data && a.bias == b.bias && a.activation == b.activation);
  }
  std::remove(path.c_str());
  CHECK(throws<IoError>([] { load_weights("/nonexistent/net.gbnn"); }));
  CHECK(throws<StructuralError>([] { random_net({4, 3}, "tanh", "sideways", 1); }));
  CHECK(throws<StructuralError>([&] { net.forward(RealVec(5, 0.0)); }));
  {
    Layer l0;
    l0.weight = DenseMat(3, 2);
    l0.bias = RealVec(2, 0.0);  // wrong length
    CHECK(throws<StructuralError>([&] { NeuralNet bad({l0}); }));
  }
  if (!gpu) {
    if (gbopt_device_count() == 0) CHECK(throws<DeviceError>([&] { net.forward(RealVec(4, 0.1)); }));
    std::printf("%s host checks\n", g_fail ? "FAILED" : "passed");
    return g_fail ? 1 : 0;
  }
  // ---- device ----
  const RealVec x = {0.1, 0.7, 0.3, 0.9};
  RealVec y = net.forward(x);
  CHECK(std::fabs(y[0] + y[1] + y[2] - 1.0) <= 1e-12);  // softmax simplex (test_capi.cpp:42-43)
  RealVec y2 = back.forward(x);
  CHECK(y == y2);
  {  // forward_trace (nn.cpp:127-146): the last y is the forward output, z_L its pre-softmax values
    ForwardTrace tr = net.forward_trace(x);
    CHECK(tr.z.size() == 2 && tr.y.size() == 2 && tr.z[0].size() == 6 && tr.y[1].size() == 3);
    CHECK(tr.y[1] == y);
    double zs = 0.0, mx = tr.z[1][0];
    for (double v : tr.z[1]) mx = std::max(mx, v);
    for (double v : tr.z[1]) zs += std::exp(v - mx);
    CHECK(std::fabs(std::exp(tr.z[1][0] - mx) / zs - y[0]) <= 1e-14);
    CHECK(throws<StructuralError>([&] { net.forward_trace(RealVec(3, 0.0)); }));  // nn.cpp:105-111
  }
  // J vs central differences (test_nn.cpp:96-108 style)
  NeuralNet t = random_net({5, 7, 4}, "tanh", "tanh", 1234);
  const RealVec xt = {0.3, -0.2, 0.5, 1.1, -0.7};
  DenseMat j = t.jacobian(xt);
  for (int c = 0; c < 5; ++c) {
    RealVec xp = xt, xm = xt;
    xp[c] += 1e-5;
    xm[c] -= 1e-5;
    RealVec fp = t.forward(xp), fm = t.forward(xm);
    for (int r = 0; r < 4; ++r) CHECK(std::fabs(j(r, c) - (fp[r] - fm[r]) / 2e-5) <= 1e-6);
  }
  // reduced-space callbacks: residual 0 at the forward image, -J layout,
  // Hessian sees -lambda (test_formulations.cpp:215-274)
  ReducedSpaceOracle rs(t);
  RealVec xb = xt;
  RealVec fy = t.forward(xt);
  xb.insert(xb.end(), fy.begin(), fy.end());
  RealVec r;
  rs.residual(xb, r);
  for (double v : r) CHECK(v == 0.0);
  RealVec jv;
  rs.jacobian(xb, jv);
  CHECK(jv.size() == 4 * 5 + 4);
  for (int i = 0; i < 4; ++i)
    for (int c = 0; c < 5; ++c) CHECK(jv[static_cast<size_t>(i * 5 + c)] == -j(i, c));
  for (int i = 0; i < 4; ++i) CHECK(jv[20 + static_cast<size_t>(i)] == 1.0);
  const RealVec lam = {0.5, -1.0, 0.25, 2.0};
  RealVec hv;
  rs.lag_hessian(xb, lam, hv);
  RealVec neg = lam;
  for (double& v : neg) v = -v;
  DenseMat h = t.lagrangian_hessian(xt, neg);
  size_t k = 0;
  for (int a = 0; a < 5; ++a)
    for (int b = 0; b <= a; ++b) CHECK(std::fabs(hv[k++] - h(a, b)) <= 1e-14);
  const int64_t evals = rs.evaluations();
  rs.residual(xb, r);
  rs.jacobian(xb, jv);
  rs.lag_hessian(xb, lam, hv);
  CHECK(rs.evaluations() == evals);  // cached: no new device work at the same iterate
  {  // multi-device call (two and three replicas on device 0): each shard is
     // bit-identical to evaluating that shard alone on one device
    NeuralNet mn = random_net({9, 33, 17, 3}, "sigmoid", "tanh", 21);
    const int64_t B = 7, n = 9, m = 3;
    std::vector<double> X(B * n), Lm(B * m);
    for (size_t i = 0; i < X.size(); ++i) X[i] = std::sin(0.37 * static_cast<double>(i));
    for (size_t i = 0; i < Lm.size(); ++i) Lm[i] = std::cos(0.11 * static_cast<double>(i));
    for (int S : {2, 3}) {
      std::vector<int> devs(static_cast<size_t>(S), 0);
      std::vector<double> Y(B * m), J(B * m * n), H(B * n * n);
      mn.oracle_batched_multi(devs, B, X.data(), Lm.data(), Y.data(), J.data(), H.data());
      for (int r = 0; r < S; ++r) {
        const int64_t cnt = B / S + (r < B % S ? 1 : 0);
        const int64_t st = r * (B / S) + std::min<int64_t>(r, B % S);
        std::vector<double> y1(cnt * m), j1(cnt * m * n), h1(cnt * n * n);
        check(gbopt_net_oracle_batched(mn.handle(), cnt, X.data() + st * n, n, Lm.data() + st * m, m, y1.data(),
                                       j1.data(), h1.data()));
        CHECK(std::equal(y1.begin(), y1.end(), Y.begin() + st * m));
        CHECK(std::equal(j1.begin(), j1.end(), J.begin() + st * m * n));
        CHECK(std::equal(h1.begin(), h1.end(), H.begin() + st * n * n));
      }
    }
  }
  std::printf("%s host+device checks\n", g_fail ? "FAILED" : "passed");
  return g_fail ? 1 : 0;
}
