// bertopt_b200_adapter.hpp — header-only C++ adapter that puts the B200 C ABI
// (bertopt_b200.h) behind the reference's own operator API and types
// (proj/core/include/bertopt). A maintainer includes it from the reference
// tree; nothing in the reference changes. Every bo_status becomes the typed
// bertopt::Error subclass it mirrors (errors.hpp:35-48).
//
//   bertopt::b200::lamb_step          == bertopt::lamb_step      (lamb.hpp:47-48)
//   bertopt::b200::unscale_gradients  == unscale_gradients       (half.hpp:77)
//   bertopt::b200::ring_allreduce_f32 / _f16_wire over a device communicator
//                                     == ring_allreduce / ring_allreduce_f16_wire
//                                        (collective.hpp:104-114) on host data
//   bertopt::b200::GradPipeline       the DistributedTrainer gradient-to-update
//                                     seam (trainer.cpp:186-215, 356-366);
//                                     train_step == DistributedTrainer::train_step
//                                     (trainer.cpp:217-373) from the K micros'
//                                     binary16 gradients (the backward's output)
#ifndef BERTOPT_B200_ADAPTER_HPP_
#define BERTOPT_B200_ADAPTER_HPP_

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "bertopt/errors.hpp"
#include "bertopt/half.hpp"
#include "bertopt/lamb.hpp"
#include "bertopt/model.hpp"
#include "bertopt/tensor.hpp"
#include "bertopt/trainer.hpp"
#include "bertopt_b200.h"

namespace bertopt::b200 {

[[noreturn]] inline void raise(bo_status s) {
  const std::string msg = bo_last_error();
  switch (s) {
    case BO_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case BO_ERR_NON_FINITE_GRADIENT: throw NonFiniteGradient(msg);
    case BO_ERR_OVERFLOW_DETECTED: throw OverflowDetected(msg);
    case BO_ERR_LENGTH_MISMATCH: throw LengthMismatch(msg);
    case BO_ERR_INVALID_CONFIG: throw InvalidConfig(msg);
    case BO_ERR_BUCKET_LAYOUT_MISMATCH: throw BucketLayoutMismatch(msg);
    case BO_ERR_PEER_DISCONNECTED: throw PeerDisconnected(msg);
    case BO_ERR_WATCHDOG_TIMEOUT: throw WatchdogTimeout(msg);
    case BO_ERR_PROTOCOL: throw ProtocolError(msg);
    case BO_ERR_IO_FAILURE: throw IoFailure(msg);
    default: throw Error(std::string(bo_status_name(s)) + ": " + msg);
  }
}

inline void check(bo_status s) {
  if (s != BO_OK) raise(s);
}

// Device allocation owned by the adapter (no CUDA headers needed).
class DeviceBuffer {
 public:
  explicit DeviceBuffer(size_t bytes, int device = 0) { check(bo_malloc(&p_, bytes, device)); }
  ~DeviceBuffer() { bo_free(p_); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }
  void upload(const void* src, size_t bytes) { check(bo_memcpy(p_, src, bytes, 0)); }
  void download(void* dst, size_t bytes) const { check(bo_memcpy(dst, p_, bytes, 1)); }

 private:
  void* p_ = nullptr;
};

inline bo_lamb_config to_c(const LambConfig& c) {
  return bo_lamb_config{c.lr, c.beta1, c.beta2, c.eps, c.weight_decay, c.trust_clip};
}

// lamb_step with the reference's argument meaning and error behaviour
// (lamb.cpp:23-84): lazy zero moments, step incremented first, tensors
// before a failing one updated, then ShapeMismatch / NonFiniteGradient.
inline void lamb_step(std::vector<Tensor>& params, const std::vector<Tensor>& grads,
                      LambState& state, const LambConfig& cfg, int device = 0) {
  if (grads.size() != params.size()) {
    throw ShapeMismatch("lamb_step: " + std::to_string(grads.size()) + " gradients for " +
                        std::to_string(params.size()) + " parameters");
  }
  if (state.m.empty()) {
    for (const Tensor& p : params) {
      state.m.push_back(Tensor::zeros(p.shape));
      state.v.push_back(Tensor::zeros(p.shape));
    }
  }
  if (state.m.size() != params.size() || state.v.size() != params.size()) {
    throw ShapeMismatch("lamb_step: optimizer state layout mismatch");
  }
  size_t ok = 0;  // tensors before the first shape mismatch take the step
  while (ok < params.size() && grads[ok].shape == params[ok].shape) ++ok;
  // w, g, m, v of all tensors packed into four device arrays: four uploads
  // and three downloads per call, not four of each per tensor
  std::vector<int64_t> numels;
  std::vector<size_t> off;
  size_t total = 0;
  for (size_t i = 0; i < ok; ++i) {
    numels.push_back(static_cast<int64_t>(params[i].data.size()));
    off.push_back(total);
    total += params[i].data.size();
  }
  std::vector<float> host(total);
  DeviceBuffer dev[4] = {DeviceBuffer(total * sizeof(float) + 16, device), DeviceBuffer(total * sizeof(float) + 16, device),
                         DeviceBuffer(total * sizeof(float) + 16, device), DeviceBuffer(total * sizeof(float) + 16, device)};
  auto pack = [&](int a, auto&& get) {
    for (size_t i = 0; i < ok; ++i) {
      const std::vector<float>& src = get(i);
      std::copy(src.begin(), src.end(), host.begin() + static_cast<std::ptrdiff_t>(off[i]));
    }
    dev[a].upload(host.data(), total * sizeof(float));
  };
  pack(0, [&](size_t i) -> const std::vector<float>& { return params[i].data; });
  pack(1, [&](size_t i) -> const std::vector<float>& { return grads[i].data; });
  pack(2, [&](size_t i) -> const std::vector<float>& { return state.m[i].data; });
  pack(3, [&](size_t i) -> const std::vector<float>& { return state.v[i].data; });
  std::vector<float*> w, m, v;
  std::vector<const float*> g;
  for (size_t i = 0; i < ok; ++i) {
    w.push_back(dev[0].as<float>() + off[i]);
    g.push_back(dev[1].as<float>() + off[i]);
    m.push_back(dev[2].as<float>() + off[i]);
    v.push_back(dev[3].as<float>() + off[i]);
  }
  const bo_lamb_config c = to_c(cfg);
  const bo_status s = bo_lamb_step(static_cast<int32_t>(ok), numels.data(), w.data(), g.data(),
                                   m.data(), v.data(), &state.step, &c, nullptr);
  auto unpack = [&](int a, auto&& get) {
    dev[a].download(host.data(), total * sizeof(float));
    for (size_t i = 0; i < ok; ++i) {
      std::vector<float>& dst = get(i);
      std::copy_n(host.begin() + static_cast<std::ptrdiff_t>(off[i]), dst.size(), dst.begin());
    }
  };
  unpack(0, [&](size_t i) -> std::vector<float>& { return params[i].data; });
  unpack(2, [&](size_t i) -> std::vector<float>& { return state.m[i].data; });
  unpack(3, [&](size_t i) -> std::vector<float>& { return state.v[i].data; });
  for (size_t i = 0; i < ok; ++i) quantize_inplace(params[i]);  // lamb.cpp:82
  if (s != BO_OK) raise(s);
  if (ok < params.size()) {
    throw ShapeMismatch("lamb_step: gradient shape mismatch at tensor " + std::to_string(ok));
  }
}

// unscale_gradients (half.cpp:105-115): OverflowDetected before any change.
inline void unscale_gradients(std::span<float> grads, const LossScaler& s, int device = 0) {
  DeviceBuffer d(grads.size_bytes(), device);
  d.upload(grads.data(), grads.size_bytes());
  check(bo_unscale_gradients(d.as<float>(), grads.size(), s.scale(), s.enabled(), nullptr));
  d.download(grads.data(), grads.size_bytes());
}

// ring_allreduce<float> / ring_allreduce_f16_wire over ctx's communicator on
// host data (the reference's in-place, identical-bits-on-every-rank contract).
inline void ring_allreduce_f32(bo_ctx* ctx, float* data, size_t n, int device = 0) {
  DeviceBuffer d(n * sizeof(float), device);
  d.upload(data, n * sizeof(float));
  check(bo_ring_allreduce_f32(ctx, d.as<float>(), n));
  d.download(data, n * sizeof(float));
}

inline void ring_allreduce_f16_wire(bo_ctx* ctx, float* data, size_t n, int device = 0) {
  DeviceBuffer d(n * sizeof(float), device);
  d.upload(data, n * sizeof(float));
  check(bo_ring_allreduce_f16_wire(ctx, d.as<float>(), n));
  d.download(data, n * sizeof(float));
}

// The DistributedTrainer seam: a model's parameters resident on the device,
// fed one micro-batch of binary16 gradients at a time.
class GradPipeline {
 public:
  GradPipeline(const Model& model, const std::vector<int>& first_consumers,
               const TrainerConfig& tc, const bo_scaler_config& scaler, int device, int rank,
               int world) {
    bo_trainer_config cfg;
    bo_default_config(&cfg);
    cfg.lamb = to_c(tc.lamb);
    cfg.accumulation = tc.accumulation;
    cfg.bucket_bytes = tc.bucket_bytes;
    cfg.f16_exchange = tc.f16_exchange;
    cfg.scaler = scaler;
    std::vector<int64_t> numels, dims;
    std::vector<int32_t> ndims;
    std::vector<const char*> names;
    for (size_t p = 0; p < model.params.size(); ++p) {
      numels.push_back(model.params[p].numel());
      names.push_back(model.names[p].c_str());
      ndims.push_back(static_cast<int32_t>(model.params[p].shape.size()));
      for (int64_t d : model.params[p].shape) dims.push_back(d);
    }
    std::vector<int32_t> firsts(first_consumers.begin(), first_consumers.end());
    check(bo_create(&cfg, static_cast<int32_t>(numels.size()), numels.data(), firsts.data(),
                    names.data(), ndims.data(), dims.data(), device, rank, world, &ctx_));
    k_ = tc.accumulation;
    n_params_ = numels.size();
    std::vector<float> flat;
    for (const Tensor& t : model.params) flat.insert(flat.end(), t.data.begin(), t.data.end());
    check(bo_load_params(ctx_, flat.data(), 1));
  }
  ~GradPipeline() { bo_destroy(ctx_); }
  GradPipeline(const GradPipeline&) = delete;
  GradPipeline& operator=(const GradPipeline&) = delete;

  // NCCL communicator + peer mappings (bo_comm_init), or the NCCL-free pair:
  // comm_record() from every rank, all-gathered by the caller's transport,
  // then comm_import(records in rank order).
  void comm_init(const uint8_t* id128) { check(bo_comm_init(ctx_, id128)); }
  std::vector<uint8_t> comm_record() {
    uint64_t n = 0;
    check(bo_comm_export(ctx_, nullptr, &n));
    std::vector<uint8_t> r(n);
    check(bo_comm_export(ctx_, r.data(), &n));
    return r;
  }
  void comm_import(const std::vector<std::vector<uint8_t>>& records) {
    std::vector<uint8_t> all;
    for (const auto& r : records) {
      if (r.size() != records[0].size()) throw LengthMismatch("comm_import: record sizes differ");
      all.insert(all.end(), r.begin(), r.end());
    }
    check(bo_comm_import(ctx_, all.data(), records.empty() ? 0 : records[0].size()));
  }
  void set_watchdog(double seconds) { check(bo_set_watchdog(ctx_, seconds)); }
  void accumulate(int micro, const std::vector<const uint16_t*>& device_grads) {
    check(bo_accumulate(ctx_, micro, device_grads.data()));
  }
  // DistributedTrainer::train_step (trainer.cpp:217-373) from the K micros'
  // gradients: micros[k][p] is a device pointer to micro k's binary16
  // gradient of parameter p (loss-scaled by status().loss_scale), all resident
  // until the step has run. Throws InvalidConfig unless exactly K micros are
  // given (trainer.cpp:219-221). A non-finite reduced gradient does not throw
  // here: the step is skipped and the dynamic loss scaler backs off.
  void train_step(const std::vector<std::vector<const uint16_t*>>& micros) {
    if (static_cast<int>(micros.size()) != k_) {
      throw InvalidConfig("train_step expects exactly K micro batches");
    }
    std::vector<const uint16_t*> flat;
    for (const auto& m : micros) {
      if (m.size() != n_params_) throw ShapeMismatch("train_step: gradient count differs from the model");
      flat.insert(flat.end(), m.begin(), m.end());
    }
    check(bo_train_step(ctx_, flat.data()));
  }
  // TrainerConfig::overlap: the sync micro's gradients as they become final
  // (call from Tape::backward's progress hook, in ready order).
  void sync_ready(const std::vector<int32_t>& params, const std::vector<const uint16_t*>& device_grads) {
    if (params.size() != device_grads.size()) throw ShapeMismatch("sync_ready: sizes differ");
    check(bo_sync_ready(ctx_, static_cast<int32_t>(params.size()), params.data(), device_grads.data()));
  }
  void read_params(Model& model) {
    std::vector<float> flat(count(model));
    check(bo_read_params(ctx_, flat.data(), 1));
    size_t off = 0;
    for (Tensor& t : model.params) {
      std::copy_n(flat.data() + off, t.data.size(), t.data.data());
      off += t.data.size();
    }
  }
  // LambState m, v of the elements this rank owns (world 1: all), model order.
  void read_moments(LambState& state, const Model& model) {
    const size_t P = count(model);
    std::vector<float> m(P, 0.0f), v(P, 0.0f);
    check(bo_read_moments(ctx_, m.data(), v.data(), 1));
    state.m.clear();
    state.v.clear();
    size_t off = 0;
    for (const Tensor& t : model.params) {
      state.m.push_back(Tensor::zeros(t.shape));
      state.v.push_back(Tensor::zeros(t.shape));
      std::copy_n(m.data() + off, t.data.size(), state.m.back().data.data());
      std::copy_n(v.data() + off, t.data.size(), state.v.back().data.data());
      off += t.data.size();
    }
    state.step = status().lamb_step;
  }
  // DistributedTrainer::param_hash (trainer.cpp:375-377): the reference's
  // FNV-1a over the parameters in model order, from a host copy into
  // `scratch` (a model of the same shapes) — the value trainer.param_hash()
  // gives for the same parameters.
  uint64_t param_hash(Model& scratch) {
    read_params(scratch);
    return model_param_hash(scratch);
  }
  // The device-side replica hash (bo_replica_hash): one pass over the
  // replica, equal on every rank with bit-identical parameters — the cheap
  // per-step divergence check of trainer.cpp:442-453.
  uint64_t replica_hash() {
    uint64_t h = 0;
    check(bo_replica_hash(ctx_, &h));
    return h;
  }
  bo_step_status status() {
    bo_step_status s;
    check(bo_get_status(ctx_, &s));
    return s;
  }
  bo_ctx* handle() const { return ctx_; }

 private:
  static size_t count(const Model& model) {
    size_t n = 0;
    for (const Tensor& t : model.params) n += t.data.size();
    return n;
  }
  bo_ctx* ctx_ = nullptr;
  int k_ = 1;
  size_t n_params_ = 0;
};

}  // namespace bertopt::b200

#endif  // BERTOPT_B200_ADAPTER_HPP_
