// TEST INFRASTRUCTURE: the C++ adapter (include/bertopt_b200_adapter.hpp)
// driven with the reference's own types, next to the reference's own
// functions on the same inputs. Built against the reference sources by
// oracle/ref/Makefile (target adapter_test); run by tests/test_gpu_adapter.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>

#include "bertopt/half.hpp"
#include "bertopt/lamb.hpp"
#include "bertopt/tensor.hpp"
#include "bertopt_b200_adapter.hpp"

using namespace bertopt;

static int failures = 0;
#define EXPECT(cond)                                              \
  do {                                                            \
    if (!(cond)) {                                                \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);  \
      ++failures;                                                 \
    }                                                             \
  } while (0)

static std::vector<Tensor> randn_list(const std::vector<int64_t>& sizes, uint64_t seed, float sd) {
  std::vector<Tensor> out;
  for (size_t i = 0; i < sizes.size(); ++i) out.push_back(Tensor::randn({sizes[i]}, seed + i, sd));
  return out;
}

static bool bits_equal(const Tensor& a, const Tensor& b) {
  return a.data.size() == b.data.size() &&
         std::memcmp(a.data.data(), b.data.data(), a.data.size() * 4) == 0;
}

static double max_rel(const Tensor& a, const Tensor& b) {
  double m = 0;
  for (size_t i = 0; i < a.data.size(); ++i) {
    const double d = std::fabs(double(a.data[i]) - b.data[i]) / std::max(1e-6, std::fabs(double(b.data[i])));
    m = std::max(m, d);
  }
  return m;
}

int main() {
  const std::vector<int64_t> sizes = {4097, 1, 300, 65536, 7};
  // --- lamb_step: 4 steps, reference on the host vs adapter on the device
  {
    std::vector<Tensor> pr = randn_list(sizes, 10, 0.02f), pd = pr;
    LambState sr, sd;
    LambConfig cfg;
    cfg.lr = 1e-2f;
    for (int s = 0; s < 4; ++s) {
      std::vector<Tensor> g = randn_list(sizes, 100 + 10 * s, 1e-3f);
      lamb_step(pr, g, sr, cfg);
      b200::lamb_step(pd, g, sd, cfg);
    }
    EXPECT(sr.step == 4 && sd.step == 4);
    for (size_t i = 0; i < sizes.size(); ++i) {
      EXPECT(bits_equal(sr.m[i], sd.m[i]));
      EXPECT(bits_equal(sr.v[i], sd.v[i]));
      EXPECT(max_rel(pd[i], pr[i]) <= 1e-6);
    }
  }
  // --- NonFiniteGradient with the reference's partial update
  {
    std::vector<Tensor> pr = randn_list(sizes, 20, 0.02f), pd = pr;
    LambState sr, sd;
    std::vector<Tensor> g = randn_list(sizes, 30, 1e-3f);
    g[3].data[1234] = std::numeric_limits<float>::infinity();
    bool er = false, ed = false;
    try { lamb_step(pr, g, sr, LambConfig{}); } catch (const NonFiniteGradient&) { er = true; }
    try { b200::lamb_step(pd, g, sd, LambConfig{}); } catch (const NonFiniteGradient&) { ed = true; }
    EXPECT(er && ed && sr.step == 1 && sd.step == 1);
    for (size_t i = 0; i < sizes.size(); ++i) {
      EXPECT(bits_equal(sr.m[i], sd.m[i]));
      EXPECT(bits_equal(sr.v[i], sd.v[i]));
      EXPECT(max_rel(pd[i], pr[i]) <= 1e-6);
    }
  }
  // --- ShapeMismatch cases (test_model.cpp:437-450)
  {
    std::vector<Tensor> p = {Tensor::randn({4}, 1)};
    LambState st;
    bool thrown = false;
    try { b200::lamb_step(p, {}, st, LambConfig{}); } catch (const ShapeMismatch&) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    try { b200::lamb_step(p, {Tensor::zeros({5})}, st, LambConfig{}); } catch (const ShapeMismatch&) { thrown = true; }
    EXPECT(thrown);
  }
  // --- unscale_gradients (test_half.cpp:108-141)
  {
    std::vector<float> g = {2048.0f};
    b200::unscale_gradients(g, LossScaler(4096.0f));
    EXPECT(g[0] == 0.5f);
    std::vector<float> bad = {1.0f, std::numeric_limits<float>::infinity()};
    bool thrown = false;
    try { b200::unscale_gradients(bad, LossScaler(4096.0f)); } catch (const OverflowDetected&) { thrown = true; }
    EXPECT(thrown && bad[0] == 1.0f);
  }
  std::printf(failures ? "ADAPTER FAILED %d\n" : "ADAPTER OK\n", failures);
  return failures ? 1 : 0;
}
