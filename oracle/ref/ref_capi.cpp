// TEST INFRASTRUCTURE (oracle only; never linked into the product).
//
// extern "C" entry points over the REAL reference implementation compiled
// from /root/reference/proj/core/src (see oracle/ref/Makefile). Tests and the
// bench's CPU arm call these through ctypes to (a) pin the restated oracle
// (oracle/bo_oracle.cpp) and (b) produce golden fixtures under tests/golden/.
//
// Every entry point calls the reference function it is named after:
//   ref_f32_to_f16 / ref_f16_to_f32      half.cpp:23-77
//   ref_unscale_gradients                half.cpp:105-115
//   ref_lamb_step                        lamb.cpp:23-84
//   ref_ring_allreduce                   collective.hpp:53-99 / collective.cpp:37-86
//   ref_bucket_layout                    trainer.cpp:73-134
//   ref_train                            trainer.cpp:217-373 (DistributedTrainer::train_step)
//                                        + the dynamic loss-scaler extension
#include <algorithm>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "bertopt/collective.hpp"
#include "bertopt/graph.hpp"
#include "bertopt/half.hpp"
#include "bertopt/lamb.hpp"
#include "bertopt/trainer.hpp"
#include "bertopt/transport.hpp"
#include "ref_shim.hpp"

extern "C" {
#include "../synth_grad.h"
}

using namespace bertopt;

namespace {

// Status codes mirror include/bertopt_b200.h (bo_status).
enum {
  kOk = 0, kShapeMismatch = 1, kNonFinite = 2, kOverflow = 3, kLength = 4,
  kInvalidConfig = 5, kLayoutMismatch = 6, kPeerDisc = 7, kWatchdog = 8,
  kProtocol = 9, kOther = 99
};

int map_exception(std::exception_ptr e, char* err, int errlen) {
  int code = kOther;
  std::string msg = "unknown";
  try {
    std::rethrow_exception(e);
  } catch (const ShapeMismatch& x) { code = kShapeMismatch; msg = x.what();
  } catch (const NonFiniteGradient& x) { code = kNonFinite; msg = x.what();
  } catch (const OverflowDetected& x) { code = kOverflow; msg = x.what();
  } catch (const LengthMismatch& x) { code = kLength; msg = x.what();
  } catch (const InvalidConfig& x) { code = kInvalidConfig; msg = x.what();
  } catch (const BucketLayoutMismatch& x) { code = kLayoutMismatch; msg = x.what();
  } catch (const PeerDisconnected& x) { code = kPeerDisc; msg = x.what();
  } catch (const WatchdogTimeout& x) { code = kWatchdog; msg = x.what();
  } catch (const ProtocolError& x) { code = kProtocol; msg = x.what();
  } catch (const std::exception& x) { code = kOther; msg = x.what(); }
  if (err && errlen > 0) {
    std::snprintf(err, static_cast<size_t>(errlen), "%s", msg.c_str());
  }
  return code;
}

// Root-cause preference, as trainer.cpp:473-487.
std::exception_ptr preferred(const std::vector<std::exception_ptr>& errs) {
  std::exception_ptr first;
  for (const auto& e : errs) {
    if (!e) continue;
    if (!first) first = e;
    try {
      std::rethrow_exception(e);
    } catch (const PeerDisconnected&) {
    } catch (const WatchdogTimeout&) {
    } catch (...) {
      return e;
    }
  }
  return first;
}

}  // namespace

extern "C" {

struct bo_spec_c {
  int n_tensors;
  const char* const* names;
  const int* ndims;
  const int64_t* dims;      // flattened shapes
  const int* init;          // 0 randn, 1 ones, 2 zeros
  const int* first_use;     // permutation: tensor ids in forward first-use order
};

struct bo_scaler_c {
  float init_scale, growth_factor, backoff_factor, min_scale, max_scale;
  int growth_interval;
  int dynamic;
};

}  // extern "C"

namespace {

refshim::ModelSpec to_spec(const bo_spec_c* s) {
  refshim::ModelSpec out;
  size_t k = 0;
  for (int t = 0; t < s->n_tensors; ++t) {
    out.names.emplace_back(s->names[t]);
    std::vector<int64_t> shp;
    for (int d = 0; d < s->ndims[t]; ++d) shp.push_back(s->dims[k++]);
    out.shapes.push_back(shp);
    out.init.push_back(s->init[t]);
  }
  return out;
}

LambConfig to_lamb(const float* c) {
  LambConfig l;
  l.lr = c[0]; l.beta1 = c[1]; l.beta2 = c[2];
  l.eps = c[3]; l.weight_decay = c[4]; l.trust_clip = c[5];
  return l;
}

}  // namespace

extern "C" {

void ref_f32_to_f16(const float* x, uint16_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = f32_to_f16(x[i]).bits;
}

void ref_f16_to_f32(const uint16_t* h, float* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = f16_to_f32(Binary16{h[i]});
}

void ref_narrow_block(const float* x, uint16_t* out, size_t n) { narrow_f16_block(x, out, n); }
void ref_widen_block(const uint16_t* h, float* out, size_t n) { widen_f16_block(h, out, n); }

uint64_t ref_fnv1a(const void* data, size_t len, uint64_t seed) { return fnv1a(data, len, seed); }
size_t ref_ring_chunk_elems(size_t n, int world) { return ring_chunk_elems(n, world); }
uint64_t ref_ring_allreduce_bytes(size_t n, int world, size_t e) {
  return ring_allreduce_bytes(n, world, e);
}

int ref_unscale_gradients(float* g, size_t n, float scale, int enabled, char* err, int errlen) {
  try {
    LossScaler s(scale, enabled != 0);
    unscale_gradients(std::span<float>(g, n), s);
    return kOk;
  } catch (...) {
    return map_exception(std::current_exception(), err, errlen);
  }
}

// Real lamb_step over n_tensors tensors stored flat (model order).
// m/v are taken as the incoming LambState (zeros on a fresh state).
int ref_lamb_step(int n_tensors, const int64_t* numels, float* w, const float* g,
                  float* m, float* v, int64_t* step, const float* lamb6,
                  char* err, int errlen) {
  try {
    std::vector<Tensor> params, grads;
    LambState st;
    size_t off = 0;
    for (int t = 0; t < n_tensors; ++t) {
      const size_t n = static_cast<size_t>(numels[t]);
      params.push_back(Tensor::from({numels[t]}, std::vector<float>(w + off, w + off + n)));
      grads.push_back(Tensor::from({numels[t]}, std::vector<float>(g + off, g + off + n)));
      st.m.push_back(Tensor::from({numels[t]}, std::vector<float>(m + off, m + off + n)));
      st.v.push_back(Tensor::from({numels[t]}, std::vector<float>(v + off, v + off + n)));
      off += n;
    }
    st.step = *step;
    int rc = kOk;
    try {
      lamb_step(params, grads, st, to_lamb(lamb6));
    } catch (...) {
      rc = map_exception(std::current_exception(), err, errlen);
    }
    // Copy back whatever the reference left behind (including the partial
    // update that precedes a NonFiniteGradient throw).
    off = 0;
    for (int t = 0; t < n_tensors; ++t) {
      const size_t n = static_cast<size_t>(numels[t]);
      std::memcpy(w + off, params[static_cast<size_t>(t)].data.data(), n * 4);
      std::memcpy(m + off, st.m[static_cast<size_t>(t)].data.data(), n * 4);
      std::memcpy(v + off, st.v[static_cast<size_t>(t)].data.data(), n * 4);
      off += n;
    }
    *step = st.step;
    return rc;
  } catch (...) {
    return map_exception(std::current_exception(), err, errlen);
  }
}

// Real ring all-reduce over `world` InProcHub threads. data is [world][n].
// kind: 0 float, 1 float with f16 wire, 2 int64 (data reinterpreted).
int ref_ring_allreduce(int world, size_t n, void* data, int kind, uint64_t* payload_sent,
                       char* err, int errlen) {
  auto hub = std::make_shared<InProcHub>(world);
  std::vector<std::exception_ptr> errs(static_cast<size_t>(world));
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r) {
    th.emplace_back([&, r] {
      try {
        InProcTransport tr(hub, r);
        tr.set_watchdog(60.0);
        WorkerGroup g{r, world, 0, r, &tr};
        if (kind == 2) {
          int64_t* d = static_cast<int64_t*>(data) + static_cast<size_t>(r) * n;
          ring_allreduce<int64_t>(g, d, n, 7);
        } else {
          float* d = static_cast<float*>(data) + static_cast<size_t>(r) * n;
          if (kind == 1) ring_allreduce_f16_wire(g, d, n, 7);
          else ring_allreduce<float>(g, d, n, 7);
        }
        if (payload_sent) payload_sent[r] = tr.payload_bytes_sent();
      } catch (...) {
        errs[static_cast<size_t>(r)] = std::current_exception();
      }
    });
  }
  for (auto& t : th) t.join();
  if (auto e = preferred(errs)) return map_exception(e, err, errlen);
  return kOk;
}

// Real BucketLayout::build + hash. Outputs: bucket_of[T], offset_of[T],
// ready_order[T], bucket_elems[<=T]; returns bucket count (or -code).
int ref_bucket_layout(const bo_spec_c* spec, const int* firsts, uint64_t bucket_bytes,
                      int* bucket_of, int64_t* offset_of, int* ready_order,
                      int64_t* bucket_elems, uint64_t* hash_out, char* err, int errlen) {
  try {
    refshim::ModelSpec ms = to_spec(spec);
    Model m;
    for (size_t t = 0; t < ms.names.size(); ++t) {
      m.index[ms.names[t]] = static_cast<int>(t);
      m.names.push_back(ms.names[t]);
      m.params.push_back(Tensor::zeros(ms.shapes[t]));
    }
    std::vector<int> f(firsts, firsts + spec->n_tensors);
    BucketLayout L = BucketLayout::build(m, f, bucket_bytes);
    for (int t = 0; t < spec->n_tensors; ++t) {
      bucket_of[t] = L.bucket_of[static_cast<size_t>(t)];
      offset_of[t] = static_cast<int64_t>(L.offset_of[static_cast<size_t>(t)]);
      ready_order[t] = L.ready_order[static_cast<size_t>(t)];
    }
    for (size_t b = 0; b < L.buckets.size(); ++b) {
      bucket_elems[b] = static_cast<int64_t>(L.buckets[b].elems);
    }
    if (hash_out) *hash_out = L.hash(m);
    return static_cast<int>(L.buckets.size());
  } catch (...) {
    return -map_exception(std::current_exception(), err, errlen);
  }
}

// CPU baseline: times the reference's own hot-path stages on a sample of the
// workload. Per rank (one thread, as the reference runs it):
//   K-1 accumulate passes          trainer.cpp:240-244 (fp32 tape gradients)
//   flatten into the fusion buckets trainer.cpp:186-203
//   ring_allreduce[_f16_wire] per bucket + x 1/world (real, InProcHub)
//                                  trainer.cpp:205-215, collective.hpp:53-99
//   unpack + the real lamb_step    trainer.cpp:356-366, lamb.cpp:23-84
// `groups` independent replicas (groups * world threads) run concurrently so
// that all host cores are used. seconds[s] is the wall time of timed step s
// between all-thread barriers; stage_seconds[4] sums rank 0 of group 0's
// accumulate / flatten / reduce / lamb time over the timed steps.
// shared_micros: the K fp32 micro-batch gradient sets are generated once and
// read by every rank thread (rank 0's values) instead of one copy per rank —
// the same bytes streamed per rank, K x 4 x P bytes less host memory per rank
// (the full BERT-large workload at world 8 would otherwise need ~110 GB).
int ref_stage_bench(int T, const int64_t* numels, const int* firsts, int world, int K,
                    uint64_t bucket_bytes, int f16, int groups, int warmup, int steps,
                    double* seconds, double* stage_seconds, char* err, int errlen,
                    int shared_micros) {
  try {
    if (world < 1 || K < 1 || groups < 1) throw InvalidConfig("bad bench config");
    const int nthreads = groups * world;
    auto make_micros = [&](int r) {
      std::vector<std::vector<Tensor>> micro(static_cast<size_t>(K));
      for (int t = 0; t < T; ++t) {
        for (int k = 0; k < K; ++k) {
          std::vector<float> g(static_cast<size_t>(numels[t]));
          const uint64_t base = bo_synth_base(1, static_cast<uint64_t>(r), 0, static_cast<uint64_t>(k));
          for (int64_t i = 0; i < numels[t]; ++i) {
            g[static_cast<size_t>(i)] = bo_synth_true_grad(base, static_cast<uint64_t>(i), 0, 1);
          }
          micro[static_cast<size_t>(k)].push_back(Tensor::from({numels[t]}, std::move(g)));
        }
      }
      return micro;
    };
    std::vector<std::vector<Tensor>> shared;
    if (shared_micros) shared = make_micros(0);
    std::vector<std::shared_ptr<InProcHub>> hubs;
    for (int g = 0; g < groups; ++g) hubs.push_back(std::make_shared<InProcHub>(world));
    std::barrier<> bar(nthreads);
    std::vector<std::exception_ptr> errs(static_cast<size_t>(nthreads));
    std::vector<std::thread> th;
    using clk = std::chrono::steady_clock;
    for (int id = 0; id < nthreads; ++id) {
      th.emplace_back([&, id] {
        const int grp = id / world, r = id % world;
        try {
          std::unique_ptr<InProcTransport> tr;
          WorkerGroup wg;
          wg.rank = r;
          wg.world = world;
          if (world > 1) {
            tr = std::make_unique<InProcTransport>(hubs[static_cast<size_t>(grp)], r);
            tr->set_watchdog(3600.0);
            wg.transport = tr.get();
          }
          Model m;
          for (int t = 0; t < T; ++t) {
            m.names.push_back("t" + std::to_string(t));
            m.params.push_back(Tensor::randn({numels[t]}, 1000 + static_cast<uint64_t>(t), 0.02f));
          }
          std::vector<std::vector<Tensor>> own;
          if (!shared_micros) own = make_micros(r);
          const std::vector<std::vector<Tensor>>& micro = shared_micros ? shared : own;
          std::vector<int> fs(firsts, firsts + T);
          const BucketLayout L = BucketLayout::build(m, fs, static_cast<size_t>(bucket_bytes));
          LambState st;
          LambConfig lc;
          std::vector<std::vector<float>> accum(static_cast<size_t>(T));
          std::vector<std::vector<float>> flat(L.buckets.size());
          const float inv = 1.0f / (static_cast<float>(K) * 1.0f);
          double acc_s = 0, flat_s = 0, red_s = 0, lamb_s = 0;
          for (int it = 0; it < warmup + steps; ++it) {
            bar.arrive_and_wait();
            const auto t0 = clk::now();
            for (int k = 0; k + 1 < K; ++k) {  // trainer.cpp:240-244
              for (int t = 0; t < T; ++t) {
                const Tensor& g = micro[static_cast<size_t>(k)][static_cast<size_t>(t)];
                std::vector<float>& a = accum[static_cast<size_t>(t)];
                if (a.empty()) a.assign(g.data.size(), 0.0f);
                for (size_t i = 0; i < g.data.size(); ++i) a[i] += g.data[i];
              }
            }
            const auto t1 = clk::now();
            for (size_t b = 0; b < L.buckets.size(); ++b) flat[b].assign(L.buckets[b].elems, 0.0f);
            for (int p : L.ready_order) {  // flatten_param, trainer.cpp:186-203
              const size_t sp = static_cast<size_t>(p);
              float* dst = flat[static_cast<size_t>(L.bucket_of[sp])].data() + L.offset_of[sp];
              const float* live = micro[static_cast<size_t>(K - 1)][sp].data.data();
              const float* summed = accum[sp].empty() ? nullptr : accum[sp].data();
              for (int64_t i = 0; i < numels[p]; ++i) {
                float v = live[i];
                if (summed) v += summed[i];
                dst[i] = v * inv;
              }
            }
            const auto t2 = clk::now();
            if (world > 1) {  // reduce_bucket, trainer.cpp:205-215
              for (size_t b = 0; b < flat.size(); ++b) {
                const uint32_t tag = static_cast<uint32_t>((it * flat.size() + b) & 0x7fffffffu);
                if (f16) ring_allreduce_f16_wire(wg, flat[b].data(), flat[b].size(), tag);
                else ring_allreduce<float>(wg, flat[b].data(), flat[b].size(), tag);
                const float invn = 1.0f / static_cast<float>(world);
                for (float& v : flat[b]) v *= invn;
              }
            }
            const auto t3 = clk::now();
            std::vector<Tensor> gvec(static_cast<size_t>(T));
            for (int t = 0; t < T; ++t) {  // unpack, trainer.cpp:356-365
              Tensor g = Tensor::zeros({numels[t]});
              const std::vector<float>& fb = flat[static_cast<size_t>(L.bucket_of[static_cast<size_t>(t)])];
              std::copy_n(fb.data() + L.offset_of[static_cast<size_t>(t)], numels[t], g.data.data());
              gvec[static_cast<size_t>(t)] = std::move(g);
            }
            lamb_step(m.params, gvec, st, lc);
            for (auto& a : accum) a.clear();
            const auto t4 = clk::now();
            bar.arrive_and_wait();
            const auto t5 = clk::now();
            if (it >= warmup) {
              if (id == 0) {
                seconds[it - warmup] = std::chrono::duration<double>(t5 - t0).count();
                acc_s += std::chrono::duration<double>(t1 - t0).count();
                flat_s += std::chrono::duration<double>(t2 - t1).count();
                red_s += std::chrono::duration<double>(t3 - t2).count();
                lamb_s += std::chrono::duration<double>(t4 - t3).count();
              }
            }
          }
          if (id == 0) {
            stage_seconds[0] = acc_s;
            stage_seconds[1] = flat_s;
            stage_seconds[2] = red_s;
            stage_seconds[3] = lamb_s;
          }
        } catch (...) {
          errs[static_cast<size_t>(id)] = std::current_exception();
          bar.arrive_and_drop();
        }
      });
    }
    for (auto& t : th) t.join();
    if (auto e = preferred(errs)) return map_exception(e, err, errlen);
    return kOk;
  } catch (...) {
    return map_exception(std::current_exception(), err, errlen);
  }
}

// Initial parameters exactly as the restated build_model draws them.
int ref_build_params(const bo_spec_c* spec, uint64_t seed, float* out) {
  Model m = refshim::build_model_from_spec(to_spec(spec), seed);
  size_t off = 0;
  for (const Tensor& t : m.params) {
    std::memcpy(out + off, t.data.data(), t.data.size() * 4);
    off += t.data.size();
  }
  return kOk;
}

// Full data-parallel run of the REAL DistributedTrainer::train_step with the
// builder-defined dynamic loss-scaler extension:
//   * micro k of rank r at step t gets fp16 gradients h = f32_to_f16(g * S_t)
//     from the synthetic spec (synth_grad.h), overridden by injections;
//   * the synthetic forward makes the trainer's live gradient exactly
//     widen(h) (the loss is multiplied by S_t through tape.scalar_mul);
//   * found_inf := train_step threw NonFiniteGradient (lamb.cpp:61-65: the
//     reduced gradient lamb_step consumes held a non-finite). The step is then
//     skipped: params / m / v / step are restored to their pre-step values;
//   * scaler: found_inf -> S = max(S*backoff, min), good = 0;
//     else good++, good == interval -> S = min(S*growth, max), good = 0.
//     With dynamic == 0 the scale never changes (skips still apply).
// inj is [n_inj][5] = (step, rank, micro, flat_index, f16 bits).
int ref_train(const bo_spec_c* spec, uint64_t init_seed, int world, int K,
              uint64_t bucket_bytes, int f16_exchange, int overlap, const float* lamb6,
              const bo_scaler_c* sc, uint64_t grad_seed, uint32_t spike_ppm, int spike_exp,
              const int64_t* inj, int n_inj, int steps, float* params_out, float* m_out,
              float* v_out, int64_t* lamb_step_out, float* scale_used, int* found_inf,
              float* final_scale, int* final_good, char* err, int errlen,
              double* step_seconds) {
  try {
    const refshim::ModelSpec ms = to_spec(spec);
    const int T = spec->n_tensors;
    std::vector<int> first_use(spec->first_use, spec->first_use + T);
    std::vector<int64_t> numel(static_cast<size_t>(T));
    std::vector<int64_t> flat_off(static_cast<size_t>(T));
    int64_t P = 0;
    for (int t = 0; t < T; ++t) {
      int64_t n = 1;
      for (int64_t e : ms.shapes[static_cast<size_t>(t)]) n *= e;
      numel[static_cast<size_t>(t)] = n;
      flat_off[static_cast<size_t>(t)] = P;
      P += n;
    }
    auto hub = world > 1 ? std::make_shared<InProcHub>(world) : nullptr;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(world));
    std::vector<uint64_t> hashes(static_cast<size_t>(world));
    std::vector<float> scales(static_cast<size_t>(world));
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r) {
      th.emplace_back([&, r] {
        try {
          std::unique_ptr<InProcTransport> tr;
          WorkerGroup g;
          g.rank = r;
          g.world = world;
          g.gpu = r;
          if (world > 1) {
            tr = std::make_unique<InProcTransport>(hub, r);
            tr->set_watchdog(600.0);
            g.transport = tr.get();
          }
          Model m = refshim::build_model_from_spec(ms, init_seed);
          TrainerConfig tc;
          tc.lamb = to_lamb(lamb6);
          tc.accumulation = K;
          tc.bucket_bytes = static_cast<size_t>(bucket_bytes);
          tc.overlap = overlap != 0;
          tc.f16_exchange = f16_exchange != 0;
          LambState saved;
          float S = sc->init_scale;
          int good = 0;
          std::vector<refshim::SynthMicro> micros(static_cast<size_t>(K));
          for (int step = 0; step < steps; ++step) {
            std::vector<Batch> batches(static_cast<size_t>(K));
            for (int k = 0; k < K; ++k) {
              refshim::SynthMicro& sm = micros[static_cast<size_t>(k)];
              sm.first_use_order = first_use;
              sm.G.assign(static_cast<size_t>(T), {});
              const uint64_t base = bo_synth_base(grad_seed, static_cast<uint64_t>(r),
                                                  static_cast<uint64_t>(step),
                                                  static_cast<uint64_t>(k));
              for (int t = 0; t < T; ++t) {
                std::vector<float>& G = sm.G[static_cast<size_t>(t)];
                G.resize(static_cast<size_t>(numel[static_cast<size_t>(t)]));
                for (int64_t i = 0; i < numel[static_cast<size_t>(t)]; ++i) {
                  const int64_t fi = flat_off[static_cast<size_t>(t)] + i;
                  const float gt = bo_synth_true_grad(base, static_cast<uint64_t>(fi),
                                                      spike_ppm, spike_exp);
                  uint16_t h = f32_to_f16(gt * S).bits;
                  for (int q = 0; q < n_inj; ++q) {
                    const int64_t* e = inj + 5 * q;
                    if (e[0] == step && e[1] == r && e[2] == k && e[3] == fi) {
                      h = static_cast<uint16_t>(e[4]);
                    }
                  }
                  G[static_cast<size_t>(i)] = f16_to_f32(Binary16{h}) / S;
                }
              }
              const int64_t handle = (static_cast<int64_t>(r) << 40) |
                                     (static_cast<int64_t>(step) << 8) | k;
              refshim::register_micro(handle, &sm);
              batches[static_cast<size_t>(k)].ids = {handle};
            }
            const std::vector<Tensor> saved_params = m.params;
            tc.loss_scale = S;
            if (r == 0) scale_used[step] = S;
            bool found = false;
            {
              DistributedTrainer trainer(g, m, tc);
              trainer.state() = saved;
              try {
                const auto ts0 = std::chrono::steady_clock::now();
                (void)trainer.train_step(batches);
                if (r == 0 && step_seconds) {
                  // rank 0's wall time of the real DistributedTrainer::train_step
                  // (synthetic forward/backward + accumulate, flatten, ring, lamb_step)
                  step_seconds[step] =
                      std::chrono::duration<double>(std::chrono::steady_clock::now() - ts0).count();
                }
                saved = trainer.state();
              } catch (const NonFiniteGradient&) {
                found = true;
                for (size_t p = 0; p < m.params.size(); ++p) {
                  m.params[p].data = saved_params[p].data;
                }
              }
            }
            for (int k = 0; k < K; ++k) {
              refshim::unregister_micro((static_cast<int64_t>(r) << 40) |
                                        (static_cast<int64_t>(step) << 8) | k);
            }
            if (r == 0) found_inf[step] = found ? 1 : 0;
            if (sc->dynamic) {
              if (found) {
                S = std::max(S * sc->backoff_factor, sc->min_scale);
                good = 0;
              } else if (++good == sc->growth_interval) {
                S = std::min(S * sc->growth_factor, sc->max_scale);
                good = 0;
              }
            }
          }
          hashes[static_cast<size_t>(r)] = model_param_hash(m);
          scales[static_cast<size_t>(r)] = S;
          if (r == 0) {
            size_t off = 0;
            for (size_t p = 0; p < m.params.size(); ++p) {
              const size_t n = m.params[p].data.size();
              std::memcpy(params_out + off, m.params[p].data.data(), n * 4);
              if (!saved.m.empty()) {
                std::memcpy(m_out + off, saved.m[p].data.data(), n * 4);
                std::memcpy(v_out + off, saved.v[p].data.data(), n * 4);
              } else {
                std::memset(m_out + off, 0, n * 4);
                std::memset(v_out + off, 0, n * 4);
              }
              off += n;
            }
            *lamb_step_out = saved.step;
            *final_scale = S;
            *final_good = good;
          }
        } catch (...) {
          errs[static_cast<size_t>(r)] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    if (auto e = preferred(errs)) return map_exception(e, err, errlen);
    for (int r = 1; r < world; ++r) {
      if (hashes[static_cast<size_t>(r)] != hashes[0] || scales[static_cast<size_t>(r)] != scales[0]) {
        throw Error("replica divergence across ranks");
      }
    }
    return kOk;
  } catch (...) {
    return map_exception(std::current_exception(), err, errlen);
  }
}

}  // extern "C"
