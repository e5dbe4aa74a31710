// TEST INFRASTRUCTURE (oracle only; never linked into the product).
//
// Link shims that let the reference's own hot-path sources
//   proj/core/src/{half,tensor,lamb,collective,transport,trainer,data}.cpp
// compile and link from /root/reference WITHOUT Eigen, CLI11, doctest or the
// BERT forward pass ("Shims needed"). Every function here is
// a restatement of the reference semantics it replaces, not a copy:
//
//   (1) widen_f16_block / narrow_f16_block  — graph.cpp:176-199 (F16C RNE with
//       a scalar tail; identical bits to half.cpp:23-77 except NaN payloads)
//   (2) Tape::{add, mul, scalar_mul, sum}   — ops.cpp:101-155, 522-534, equal
//       shapes only (all the synthetic forward needs)
//   (3) forward()                            — synthetic: loss = Σ_p sum(p ⊙ G_p)
//       with parameters consumed in the BERT first-use order, so that
//       ∂loss/∂p = G_p exactly and BucketLayout sees the real ready order
//   (4) build_model()                        — model.cpp:124-176 semantics for an
//       explicit parameter list (per-tensor seeds from mt19937_64, randn σ=0.02)
//   (5) make_batch / save_checkpoint         — unused by the harness; throw.
#include <immintrin.h>

#include <map>
#include <mutex>
#include <random>
#include <stdexcept>

#include "bertopt/model.hpp"
#include "bertopt/graph.hpp"
#include "ref_shim.hpp"

namespace bertopt {

// ---- (1) f16 block conversion -------------------------------------------
void widen_f16_block(const uint16_t* src, float* dst, size_t n) {
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    _mm256_storeu_ps(dst + i, _mm256_cvtph_ps(h));
  }
  for (; i < n; ++i) dst[i] = f16_to_f32(Binary16{src[i]});
}

void narrow_f16_block(const float* src, uint16_t* dst, size_t n) {
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    __m256 v = _mm256_loadu_ps(src + i);
    __m128i h = _mm256_cvtps_ph(v, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), h);
  }
  for (; i < n; ++i) dst[i] = f32_to_f16(src[i]).bits;
}

// ---- (2) the four tape ops the synthetic forward uses --------------------
static void require_same_shape(const Tensor& a, const Tensor& b, const char* op) {
  if (a.shape != b.shape || a.dtype != b.dtype) {
    throw ShapeMismatch(std::string("ref shim ") + op + ": operands must match");
  }
}

Tensor Tape::add(const Tensor& a, const Tensor& b) {
  require_same_shape(a, b, "add");
  Tensor out = Tensor::zeros(a.shape, a.dtype);
  for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = a.data[i] + b.data[i];
  quantize_inplace(out);
  if (a.node < 0 && b.node < 0) return out;
  const int an = a.node, bn = b.node;
  const std::vector<int64_t> shp = a.shape;
  out.node = record(out, {an, bn}, [an, bn, shp](const Tensor& g, std::vector<Tensor>& acc) {
    if (an >= 0) accumulate_grad(acc, an, shp, g);
    if (bn >= 0) accumulate_grad(acc, bn, shp, g);
  });
  return out;
}

Tensor Tape::mul(const Tensor& a, const Tensor& b) {
  require_same_shape(a, b, "mul");
  Tensor out = Tensor::zeros(a.shape, a.dtype);
  for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = a.data[i] * b.data[i];
  quantize_inplace(out);
  if (a.node < 0 && b.node < 0) return out;
  const int an = a.node, bn = b.node;
  const Tensor av = a, bv = b;
  out.node = record(out, {an, bn}, [an, bn, av, bv](const Tensor& g, std::vector<Tensor>& acc) {
    if (an >= 0) {
      Tensor ga = Tensor::zeros(g.shape);
      for (size_t i = 0; i < ga.data.size(); ++i) ga.data[i] = g.data[i] * bv.data[i];
      accumulate_grad(acc, an, av.shape, ga);
    }
    if (bn >= 0) {
      Tensor gb = Tensor::zeros(g.shape);
      for (size_t i = 0; i < gb.data.size(); ++i) gb.data[i] = g.data[i] * av.data[i];
      accumulate_grad(acc, bn, bv.shape, gb);
    }
  });
  return out;
}

Tensor Tape::scalar_mul(const Tensor& a, float c) {
  Tensor out = Tensor::zeros(a.shape, a.dtype);
  for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = c * a.data[i];
  quantize_inplace(out);
  if (a.node < 0) return out;
  const int an = a.node;
  const std::vector<int64_t> shp = a.shape;
  out.node = record(out, {an}, [an, shp, c](const Tensor& g, std::vector<Tensor>& acc) {
    Tensor ga = Tensor::zeros(g.shape);
    for (size_t i = 0; i < ga.data.size(); ++i) ga.data[i] = c * g.data[i];
    accumulate_grad(acc, an, shp, ga);
  });
  return out;
}

Tensor Tape::sum(const Tensor& a) {
  double s = 0.0;
  for (float v : a.data) s += v;
  Tensor out = Tensor::from({}, {static_cast<float>(s)});
  if (a.node < 0) return out;
  const int an = a.node;
  const std::vector<int64_t> shp = a.shape;
  out.node = record(out, {an}, [an, shp](const Tensor& g, std::vector<Tensor>& acc) {
    accumulate_grad(acc, an, shp, Tensor::full(shp, g.data[0]));
  });
  return out;
}

// ---- (3) synthetic forward -------------------------------------------------
namespace {
std::mutex g_reg_mu;
std::map<int64_t, const refshim::SynthMicro*> g_registry;
}  // namespace

ForwardResult forward(Model& m, Tape& tape, const Batch& batch, const ForwardOptions&) {
  for (Tensor& p : m.params) tape.watch(p);  // model.cpp:217: watch in model order
  const refshim::SynthMicro* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_registry.find(batch.ids.at(0));
    if (it == g_registry.end()) throw InvalidConfig("ref shim: unknown synthetic micro");
    s = it->second;
  }
  if (s->G.size() != m.params.size()) throw ShapeMismatch("ref shim: gradient set size");
  ForwardResult r;
  bool first = true;
  for (int p : s->first_use_order) {
    const Tensor& w = m.params[static_cast<size_t>(p)];
    Tensor G = Tensor::from(w.shape, s->G[static_cast<size_t>(p)]);
    Tensor term = tape.sum(tape.mul(w, G));
    r.loss = first ? term : tape.add(r.loss, term);
    first = false;
  }
  return r;
}

ForwardResult forward(Model& m, Tape& tape, const Batch& batch, uint64_t) {
  return forward(m, tape, batch, ForwardOptions{});
}

// ---- (4)/(5) ------------------------------------------------------------------
Model build_model(const ModelConfig&, uint64_t) {
  throw InvalidConfig("ref shim: use refshim::build_model_from_spec");
}
Batch make_batch(const std::vector<TrainingExample>&) {
  throw InvalidConfig("ref shim: make_batch is not part of the hot path");
}
void save_checkpoint(const Model&, const std::string&) {
  throw InvalidConfig("ref shim: save_checkpoint is not part of the hot path");
}

}  // namespace bertopt

namespace refshim {

using namespace bertopt;

void register_micro(int64_t handle, const SynthMicro* s) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_registry[handle] = s;
}

void unregister_micro(int64_t handle) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_registry.erase(handle);
}

Model build_model_from_spec(const ModelSpec& spec, uint64_t seed) {
  Model m;
  std::mt19937_64 seeds(seed);
  for (size_t t = 0; t < spec.names.size(); ++t) {
    Tensor x;
    switch (spec.init[t]) {
      case 0: x = Tensor::randn(spec.shapes[t], seeds(), 0.02f); break;  // kInitStddev
      case 1: x = Tensor::full(spec.shapes[t], 1.0f); break;
      default: x = Tensor::zeros(spec.shapes[t]); break;
    }
    m.index[spec.names[t]] = static_cast<int>(m.params.size());
    m.names.push_back(spec.names[t]);
    m.params.push_back(std::move(x));
  }
  return m;
}

}  // namespace refshim
