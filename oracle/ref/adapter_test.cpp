// TEST INFRASTRUCTURE: the C++ adapter (include/bertopt_b200_adapter.hpp)
// driven with the reference's own types, next to the reference's own
// functions on the same inputs. Built against the reference sources by
// oracle/ref/Makefile (target adapter_test); run by tests/test_gpu_adapter.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <thread>
#include <memory>

#include "bertopt/half.hpp"
#include "bertopt/lamb.hpp"
#include "bertopt/model.hpp"
#include "bertopt/tensor.hpp"
#include "bertopt/trainer.hpp"
#include "bertopt/transport.hpp"
#include "bertopt/collective.hpp"
#include "bertopt_b200_adapter.hpp"
#include "ref_shim.hpp"

extern "C" {
#include "../synth_grad.h"
}

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
  // --- GradPipeline::train_step against the REAL DistributedTrainer::train_step
  // (trainer.cpp:217-373, world 1, static loss scale, the synthetic-forward
  // shim making each micro's gradient exactly widen(h) / S): K = 3 micros,
  // ragged tensors, 4 KiB buckets, 3 steps. Moments bit-exact, parameters
  // within 1e-6 relative (fp64 norms summed in another order).
  {
    refshim::ModelSpec spec;
    const std::vector<std::vector<int64_t>> shapes = {{64, 65}, {1}, {300}, {4096}, {7}, {33, 17}};
    for (size_t i = 0; i < shapes.size(); ++i) {
      spec.names.push_back("p" + std::to_string(i));
      spec.shapes.push_back(shapes[i]);
      spec.init.push_back(i == 1 ? 2 : (i == 2 ? 1 : 0));
    }
    const std::vector<int> first_use = {2, 0, 5, 1, 4, 3};
    const int K = 3, steps = 3;
    const float S = 1024.0f;
    Model mr = refshim::build_model_from_spec(spec, 5);
    Model md = refshim::build_model_from_spec(spec, 5);
    TrainerConfig tc;
    tc.accumulation = K;
    tc.bucket_bytes = 4096;
    tc.loss_scale = S;
    tc.overlap = false;
    tc.lamb.lr = 1e-2f;
    WorkerGroup g;
    g.rank = 0;
    g.world = 1;
    DistributedTrainer trainer(g, mr, tc);
    const size_t T = shapes.size();
    std::vector<refshim::SynthMicro> micros(static_cast<size_t>(K));
    std::vector<std::vector<std::vector<uint16_t>>> h(static_cast<size_t>(K), std::vector<std::vector<uint16_t>>(T));
    auto fill = [&](int step) {
      int64_t flat = 0;
      for (size_t t = 0; t < T; ++t) {
        const int64_t n = mr.params[t].numel();
        for (int k = 0; k < K; ++k) {
          refshim::SynthMicro& sm = micros[static_cast<size_t>(k)];
          sm.first_use_order = first_use;
          sm.G.resize(T);
          sm.G[t].resize(static_cast<size_t>(n));
          h[static_cast<size_t>(k)][t].resize(static_cast<size_t>(n));
          const uint64_t base = bo_synth_base(3, 0, static_cast<uint64_t>(step), static_cast<uint64_t>(k));
          for (int64_t i = 0; i < n; ++i) {
            const float gt = bo_synth_true_grad(base, static_cast<uint64_t>(flat + i), 0, 1);
            const Binary16 b = f32_to_f16(gt * S);
            h[static_cast<size_t>(k)][t][static_cast<size_t>(i)] = b.bits;
            sm.G[t][static_cast<size_t>(i)] = f16_to_f32(b) / S;
          }
        }
        flat += n;
      }
    };
    // first consumers exactly as ensure_layout derives them (trainer.cpp:161-168)
    fill(0);
    refshim::register_micro(1, &micros[0]);
    std::vector<int> firsts(T);
    {
      Model probe = refshim::build_model_from_spec(spec, 5);
      Tape tape;
      Batch b;
      b.ids = {1};
      (void)forward(probe, tape, b, ForwardOptions{});
      const std::vector<int> all = tape.first_consumers();
      for (size_t p = 0; p < T; ++p) firsts[p] = all[static_cast<size_t>(probe.params[p].node)];
    }
    refshim::unregister_micro(1);
    const bo_scaler_config sc{S, 2.0f, 0.5f, 1.0f, 16777216.0f, 1 << 30, 0};  // static S
    b200::GradPipeline pipe(md, firsts, tc, sc, 0, 0, 1);
    std::vector<b200::DeviceBuffer> dev;
    for (int step = 0; step < steps; ++step) {
      fill(step);
      std::vector<Batch> batches(static_cast<size_t>(K));
      std::vector<std::vector<const uint16_t*>> ptrs(static_cast<size_t>(K));
      dev.clear();
      for (int k = 0; k < K; ++k) {
        refshim::register_micro(100 + k, &micros[static_cast<size_t>(k)]);
        batches[static_cast<size_t>(k)].ids = {100 + k};
        for (size_t t = 0; t < T; ++t) {
          const std::vector<uint16_t>& src = h[static_cast<size_t>(k)][t];
          dev.emplace_back(src.size() * 2);
          dev.back().upload(src.data(), src.size() * 2);
          ptrs[static_cast<size_t>(k)].push_back(dev.back().as<uint16_t>());
        }
      }
      (void)trainer.train_step(batches);
      pipe.train_step(ptrs);
      (void)pipe.status();  // stream sync before the inputs are freed
      for (int k = 0; k < K; ++k) refshim::unregister_micro(100 + k);
    }
    Model out = refshim::build_model_from_spec(spec, 5);
    pipe.read_params(out);
    LambState sd;
    pipe.read_moments(sd, out);
    const LambState& sr = trainer.state();
    EXPECT(sr.step == steps && sd.step == steps);
    for (size_t t = 0; t < T; ++t) {
      EXPECT(bits_equal(sr.m[t], sd.m[t]));
      EXPECT(bits_equal(sr.v[t], sd.v[t]));
      EXPECT(max_rel(out.params[t], mr.params[t]) <= 1e-6);
    }
    // the step API's own error: exactly K micros (trainer.cpp:219-221)
    bool thrown = false;
    try { pipe.train_step({}); } catch (const InvalidConfig&) { thrown = true; }
    EXPECT(thrown);
  }
  // --- ring_allreduce<float> / ring_allreduce_f16_wire through the adapter
  // (b200::ring_allreduce_f32 / _f16_wire: host data in, the library's NVLink
  // ring on the device) against the REAL reference collectives over InProcHub
  // (collective.hpp:53-99, collective.cpp:37-86) on the same inputs: N
  // contexts on this GPU in lockstep (bo_world_init_local), one host thread
  // per rank, as run_data_parallel (trainer.cpp:397-470). Bits equal on every
  // rank; sizes of test_collective.cpp:403-436 plus a ragged large one.
  {
    refshim::ModelSpec spec;
    spec.names = {"a", "b"};
    spec.shapes = {{4096}, {777}};
    spec.init = {0, 0};
    TrainerConfig tc;
    tc.accumulation = 1;
    tc.bucket_bytes = 4096;
    tc.f16_exchange = true;
    bo_trainer_config dc;
    bo_default_config(&dc);
    const bo_scaler_config sc = dc.scaler;
    for (int world : {2, 3, 4}) {
      std::vector<std::unique_ptr<b200::GradPipeline>> pipes;
      std::vector<bo_ctx*> ctxs;
      for (int r = 0; r < world; ++r) {
        Model m = refshim::build_model_from_spec(spec, 1);
        pipes.push_back(std::make_unique<b200::GradPipeline>(m, std::vector<int>{1, 0}, tc, sc, 0, r, world));
        ctxs.push_back(pipes.back()->handle());
      }
      b200::check(bo_world_init_local(ctxs.data(), world));
      // identical replicas: equal device hashes; the adapter's param_hash is
      // the reference's own model_param_hash of the same parameters
      {
        Model ref_model = refshim::build_model_from_spec(spec, 1), scratch = refshim::build_model_from_spec(spec, 1);
        for (int r = 0; r < world; ++r) {
          EXPECT(pipes[static_cast<size_t>(r)]->replica_hash() == pipes[0]->replica_hash());
          EXPECT(pipes[static_cast<size_t>(r)]->param_hash(scratch) == model_param_hash(ref_model));
        }
      }
      for (size_t n : {size_t{1}, size_t{5}, size_t{64}, size_t{1537}, size_t{100003}}) {
        for (int f16 = 0; f16 < 2; ++f16) {
          std::vector<std::vector<float>> ref(static_cast<size_t>(world)), dev;
          std::mt19937 gen(static_cast<unsigned>(world * 1000 + n + f16));
          std::normal_distribution<float> nd(0.0f, f16 ? 0.25f : 1.0f);
          for (auto& x : ref) {
            x.resize(n);
            for (float& y : x) y = nd(gen);
          }
          dev = ref;
          auto hub = std::make_shared<InProcHub>(world);
          std::vector<std::thread> th;
          std::vector<int> errs(static_cast<size_t>(world), 0);
          for (int r = 0; r < world; ++r) {
            th.emplace_back([&, r] {
              try {
                InProcTransport tr(hub, r);
                WorkerGroup g{r, world, 0, r, &tr};
                if (f16) ring_allreduce_f16_wire(g, ref[static_cast<size_t>(r)].data(), n, 7);
                else ring_allreduce<float>(g, ref[static_cast<size_t>(r)].data(), n, 7);
                if (f16) b200::ring_allreduce_f16_wire(ctxs[static_cast<size_t>(r)], dev[static_cast<size_t>(r)].data(), n);
                else b200::ring_allreduce_f32(ctxs[static_cast<size_t>(r)], dev[static_cast<size_t>(r)].data(), n);
              } catch (...) {
                errs[static_cast<size_t>(r)] = 1;
              }
            });
          }
          for (auto& t : th) t.join();
          for (int r = 0; r < world; ++r) {
            EXPECT(errs[static_cast<size_t>(r)] == 0);
            EXPECT(std::memcmp(ref[static_cast<size_t>(r)].data(), dev[static_cast<size_t>(r)].data(), n * 4) == 0);
          }
        }
      }
    }
  }
  std::printf(failures ? "ADAPTER FAILED %d\n" : "ADAPTER OK\n", failures);
  return failures ? 1 : 0;
}
