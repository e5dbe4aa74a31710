// TEST INFRASTRUCTURE — CPU restatement of the reference hot path, used ONLY
// as the checker by tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline leg. It is never linked into, imported by, or called from the
// product path (paper_2008_00177_b200/).
//
// Parity pinned: tests/test_oracle_*.py check every function here against the
// real reference compiled from /root/reference (oracle/_ref, when present) and
// against the golden fixtures tests/golden/*.npz generated from it
// (tests/golden/make_golden.py).
//
// Compile without -march/-mfma and with -ffp-contract=off: the reference build
// has no FMA (proj/CMakeLists.txt:13-14), so neither may its restatement.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

extern "C" {
#include "synth_grad.h"
}

namespace {

// ---------------------------------------------------------------- binary16
// Round-to-nearest-even narrowing (restates half.cpp:23-61). Written as a
// "round the magnitude on the binary16 grid" routine: pick the grid quantum for
// the target binade, split off the remainder, round half to even.
uint16_t f32_to_f16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const uint16_t sign = static_cast<uint16_t>((u >> 16) & 0x8000u);
  const uint32_t mag = u & 0x7FFFFFFFu;
  if (mag > 0x7F800000u) return sign | 0x7E00u;    // NaN -> quiet NaN, sign kept
  if (mag >= 0x477FF000u) return sign | 0x7C00u;   // >= 65520 (incl. inf) -> inf
  if (mag < 0x33000001u) return sign;              // <= 2^-25 -> zero (tie to even)
  const int exp32 = static_cast<int>(mag >> 23);   // biased binary32 exponent
  uint32_t sig = (mag & 0x7FFFFFu) | (exp32 ? 0x800000u : 0u);
  // Number of low significand bits below the binary16 quantum.
  int drop;
  uint32_t hbase;
  if (exp32 >= 113) {  // normal binary16 target (2^-14 and up)
    drop = 13;
    hbase = static_cast<uint32_t>(exp32 - 112) << 10;  // biased f16 exponent
    sig &= 0x7FFFFFu;                                  // implicit bit lives in hbase
  } else {             // subnormal target: quantum 2^-24
    drop = 126 - exp32;  // 14..25
    hbase = 0;
  }
  const uint32_t q = sig >> drop;
  const uint32_t rem = sig & ((1u << drop) - 1u);
  const uint32_t half = 1u << (drop - 1);
  uint32_t h = hbase + q;
  if (rem > half || (rem == half && (q & 1u))) h += 1;  // carry may bump exponent
  return static_cast<uint16_t>(sign | h);
}

// Exact widening (restates half.cpp:63-77).
float f16_to_f32(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu;
  const uint32_t m = h & 0x3FFu;
  uint32_t bits;
  if (e == 0) {
    float v = std::ldexp(static_cast<float>(m), -24);
    std::memcpy(&bits, &v, 4);
    bits |= sign;
  } else if (e == 31) {
    bits = sign | 0x7F800000u | (m << 13);
  } else {
    bits = sign | ((e + 112u) << 23) | (m << 13);
  }
  float out;
  std::memcpy(&out, &bits, 4);
  return out;
}

float f16_round(float x) { return f16_to_f32(f32_to_f16(x)); }

// --------------------------------------------------------------------- misc
uint64_t fnv1a(const void* data, size_t len, uint64_t h = 14695981039346656037ull) {
  const auto* p = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < len; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

size_t ceil_div(size_t n, size_t d) { return (n + d - 1) / d; }

// Host threads for or_train's elementwise loops (OR_THREADS, default all
// cores). Only loops whose iterations are independent are split; every
// reduction keeps the reference's sequential order, so the result is
// bit-identical to the single-threaded restatement for any thread count.
int n_threads() {
  if (const char* e = std::getenv("OR_THREADS")) return std::max(1, std::atoi(e));
  return std::max(1u, std::thread::hardware_concurrency());
}

// f(lo, hi) over [0, n) in contiguous slices, one per thread.
template <typename F>
void pfor(int64_t n, F&& f, int64_t grain = 1 << 16) {
  const int nt = static_cast<int>(std::min<int64_t>(n_threads(), std::max<int64_t>(1, n / grain)));
  if (nt <= 1) {
    if (n > 0) f(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (int i = 0; i < nt; ++i) {
    const int64_t lo = i * per, hi = std::min(n, lo + per);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : th) t.join();
}

// f(i) for i in [0, n), items handed out dynamically (uneven item costs).
template <typename F>
void pfor_items(int n, F&& f) {
  const int nt = std::min(n_threads(), n);
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> th;
  for (int k = 0; k < nt; ++k) {
    th.emplace_back([&] {
      for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) f(i);
    });
  }
  for (auto& t : th) t.join();
}

struct Lamb {
  float lr, beta1, beta2, eps, wd, clip;
};

Lamb lamb_from(const float* c) { return Lamb{c[0], c[1], c[2], c[3], c[4], c[5]}; }

// Returns 0, or 2 (NonFiniteGradient) with the reference's partial-update
// side effects (restates lamb.cpp:23-84 operation by operation).
int lamb_step(int T, const int64_t* numel, float* w, const float* g, float* m, float* v,
              int64_t* step, const Lamb& c) {
  *step += 1;  // lamb.cpp:40 — incremented before any tensor is checked
  const double t = static_cast<double>(*step);
  const double bc1 = 1.0 - std::pow(static_cast<double>(c.beta1), t);
  const double bc2 = 1.0 - std::pow(static_cast<double>(c.beta2), t);
  const float omb1 = 1.0f - c.beta1;
  const float omb2 = 1.0f - c.beta2;
  std::vector<float> u;
  size_t off = 0;
  for (int i = 0; i < T; ++i) {
    const size_t n = static_cast<size_t>(numel[i]);
    float* W = w + off;
    const float* G = g + off;
    float* M = m + off;
    float* V = v + off;
    u.resize(n);
    double wn = 0.0, un = 0.0;
    for (size_t j = 0; j < n; ++j) {
      const float gj = G[j];
      if (!std::isfinite(gj)) return 2;
      M[j] = c.beta1 * M[j] + omb1 * gj;
      V[j] = c.beta2 * V[j] + (omb2 * gj) * gj;
      const float mh = static_cast<float>(static_cast<double>(M[j]) / bc1);
      const float vh = static_cast<float>(static_cast<double>(V[j]) / bc2);
      u[j] = mh / (std::sqrt(vh) + c.eps) + c.wd * W[j];
      wn += static_cast<double>(W[j]) * static_cast<double>(W[j]);
      un += static_cast<double>(u[j]) * static_cast<double>(u[j]);
    }
    float r = 1.0f;
    if (wn > 0.0 && un > 0.0) {
      r = static_cast<float>(std::sqrt(wn) / std::sqrt(un));
      r = std::min(std::max(r, 0.0f), c.clip);
    }
    const float s = c.lr * r;
    for (size_t j = 0; j < n; ++j) W[j] = W[j] - s * u[j];
    off += n;
  }
  return 0;
}

// lamb_step for a gradient already known to be finite (or_train checks
// found_inf first, so the NonFiniteGradient partial update cannot occur), as
// three passes: the per-element moments and update u (independent elements,
// split across threads), the per-tensor fp64 norms summed sequentially in the
// reference's element order (tensors in parallel), and w -= (lr * r) * u.
// Every value is computed by the same expression as lamb_step, so the result
// is bit-identical to it.
void lamb_step_finite(int T, const int64_t* numel, float* w, const float* g, float* m, float* v,
                      int64_t* step, const Lamb& c, std::vector<float>& u) {
  *step += 1;  // lamb.cpp:40
  const double t = static_cast<double>(*step);
  const double bc1 = 1.0 - std::pow(static_cast<double>(c.beta1), t);
  const double bc2 = 1.0 - std::pow(static_cast<double>(c.beta2), t);
  const float omb1 = 1.0f - c.beta1;
  const float omb2 = 1.0f - c.beta2;
  std::vector<int64_t> off(static_cast<size_t>(T) + 1, 0);
  for (int i = 0; i < T; ++i) off[static_cast<size_t>(i) + 1] = off[static_cast<size_t>(i)] + numel[i];
  const int64_t P = off[static_cast<size_t>(T)];
  u.resize(static_cast<size_t>(P));
  pfor(P, [&](int64_t lo, int64_t hi) {
    for (int64_t j = lo; j < hi; ++j) {
      const float gj = g[j];
      m[j] = c.beta1 * m[j] + omb1 * gj;
      v[j] = c.beta2 * v[j] + (omb2 * gj) * gj;
      const float mh = static_cast<float>(static_cast<double>(m[j]) / bc1);
      const float vh = static_cast<float>(static_cast<double>(v[j]) / bc2);
      u[static_cast<size_t>(j)] = mh / (std::sqrt(vh) + c.eps) + c.wd * w[j];
    }
  });
  std::vector<float> s(static_cast<size_t>(T));
  pfor_items(T, [&](int i) {
    double wn = 0.0, un = 0.0;
    for (int64_t j = off[static_cast<size_t>(i)]; j < off[static_cast<size_t>(i) + 1]; ++j) {
      wn += static_cast<double>(w[j]) * static_cast<double>(w[j]);
      un += static_cast<double>(u[static_cast<size_t>(j)]) * static_cast<double>(u[static_cast<size_t>(j)]);
    }
    float r = 1.0f;
    if (wn > 0.0 && un > 0.0) {
      r = static_cast<float>(std::sqrt(wn) / std::sqrt(un));
      r = std::min(std::max(r, 0.0f), c.clip);
    }
    s[static_cast<size_t>(i)] = c.lr * r;
  });
  pfor(P, [&](int64_t lo, int64_t hi) {
    size_t i = static_cast<size_t>(std::upper_bound(off.begin(), off.end(), lo) - off.begin()) - 1;
    for (int64_t j = lo; j < hi; ++j) {
      while (j >= off[i + 1]) ++i;
      w[j] = w[j] - s[i] * u[static_cast<size_t>(j)];
    }
  });
}

// Emulated ring reduce-scatter + all-gather of one bucket over `world`
// ranks, all in this thread. xs[r] is rank r's length-n vector; on return
// every xs[r] holds the identical reduced result (collective.hpp:53-99 for
// fp32, collective.cpp:37-86 for the binary16 wire).
void ring_allreduce_emulated(std::vector<float*>& xs, size_t n, bool f16_wire) {
  const int N = static_cast<int>(xs.size());
  if (N == 1 || n == 0) return;
  const size_t c = ceil_div(n, static_cast<size_t>(N));
  std::vector<float> out(c * static_cast<size_t>(N), 0.0f);
  auto at = [&](int r, size_t idx) -> float { return idx < n ? xs[static_cast<size_t>(r)][idx] : 0.0f; };
  for (int k = 0; k < N; ++k) {     // chunk k is folded along ranks k, k+1, ..., k-1
    for (size_t i = 0; i < c; ++i) {
      const size_t idx = static_cast<size_t>(k) * c + i;
      float p = at(k, idx);
      for (int j = 1; j < N; ++j) {
        const float local = at((k + j) % N, idx);
        const float incoming = f16_wire ? f16_round(p) : p;  // hop narrows the partial
        p = incoming + local;
      }
      out[idx] = f16_wire ? f16_round(p) : p;  // owner re-round (collective.cpp:79-83)
    }
  }
  for (int r = 0; r < N; ++r) std::memcpy(xs[static_cast<size_t>(r)], out.data(), n * 4);
}

struct Layout {
  std::vector<int> bucket_of;
  std::vector<int64_t> offset_of;
  std::vector<int> ready;
  std::vector<std::vector<int>> buckets;
  std::vector<int64_t> elems;
};

// Greedy fusion-buffer layout in gradient-ready order (restates
// trainer.cpp:73-116): descending first-consumer id, ties by index; a bucket
// closes before it would exceed bucket_bytes; an oversized tensor goes alone.
Layout build_layout(int T, const int64_t* numel, const int* firsts, uint64_t bucket_bytes) {
  Layout L;
  L.ready.resize(static_cast<size_t>(T));
  std::iota(L.ready.begin(), L.ready.end(), 0);
  std::stable_sort(L.ready.begin(), L.ready.end(), [&](int a, int b) {
    return firsts[a] > firsts[b];  // stable sort keeps ascending index on ties
  });
  L.bucket_of.assign(static_cast<size_t>(T), -1);
  L.offset_of.assign(static_cast<size_t>(T), 0);
  uint64_t bytes = 0;
  for (int p : L.ready) {
    const uint64_t b = static_cast<uint64_t>(numel[p]) * 4u;
    if (L.buckets.empty() || (!L.buckets.back().empty() && bytes + b > bucket_bytes)) {
      L.buckets.emplace_back();
      L.elems.push_back(0);
      bytes = 0;
    }
    L.bucket_of[static_cast<size_t>(p)] = static_cast<int>(L.buckets.size()) - 1;
    L.offset_of[static_cast<size_t>(p)] = L.elems.back();
    L.buckets.back().push_back(p);
    L.elems.back() += numel[p];
    bytes += b;
  }
  return L;
}

}  // namespace

extern "C" {

struct or_scaler {
  float init_scale, growth_factor, backoff_factor, min_scale, max_scale;
  int growth_interval;
  int dynamic;
};

void or_f32_to_f16(const float* x, uint16_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = f32_to_f16(x[i]);
}

void or_f16_to_f32(const uint16_t* h, float* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = f16_to_f32(h[i]);
}

uint64_t or_fnv1a(const void* data, size_t len, uint64_t seed) { return fnv1a(data, len, seed); }

size_t or_ring_chunk_elems(size_t n, int world) { return ceil_div(n, static_cast<size_t>(world)); }

// Per-rank payload bytes of one ring all-reduce (collective.cpp:31-35).
uint64_t or_ring_allreduce_bytes(size_t n, int world, size_t e) {
  if (world <= 1 || n == 0) return 0;
  return 2ull * static_cast<uint64_t>(world - 1) * or_ring_chunk_elems(n, world) * e;
}

int or_bucket_layout(int T, const int64_t* numel, const int* firsts, uint64_t bucket_bytes,
                     int* bucket_of, int64_t* offset_of, int* ready_order, int64_t* bucket_elems) {
  if (bucket_bytes == 0) return -5;  // InvalidConfig
  Layout L = build_layout(T, numel, firsts, bucket_bytes);
  for (int t = 0; t < T; ++t) {
    bucket_of[t] = L.bucket_of[static_cast<size_t>(t)];
    offset_of[t] = L.offset_of[static_cast<size_t>(t)];
    ready_order[t] = L.ready[static_cast<size_t>(t)];
  }
  for (size_t b = 0; b < L.elems.size(); ++b) bucket_elems[b] = L.elems[b];
  return static_cast<int>(L.elems.size());
}

// BucketLayout::hash (trainer.cpp:118-134) over names + shapes.
uint64_t or_layout_hash(int T, const char* const* names, const int* ndims, const int64_t* dims,
                        const int* bucket_of, int n_buckets, const int* ready_order,
                        const int64_t* bucket_elems) {
  std::vector<size_t> dim_off(static_cast<size_t>(T) + 1, 0);
  for (int t = 0; t < T; ++t) dim_off[static_cast<size_t>(t) + 1] = dim_off[static_cast<size_t>(t)] + static_cast<size_t>(ndims[t]);
  uint64_t h = fnv1a("bucket-layout", 13);
  const uint64_t nb = static_cast<uint64_t>(n_buckets);
  h = fnv1a(&nb, 8, h);
  for (int b = 0; b < n_buckets; ++b) {
    for (int q = 0; q < T; ++q) {
      const int p = ready_order[q];
      if (bucket_of[p] != b) continue;
      h = fnv1a(names[p], std::strlen(names[p]), h);
      for (size_t d = dim_off[static_cast<size_t>(p)]; d < dim_off[static_cast<size_t>(p) + 1]; ++d) {
        const int64_t e = dims[d];
        h = fnv1a(&e, 8, h);
      }
    }
    const uint64_t el = static_cast<uint64_t>(bucket_elems[b]);
    h = fnv1a(&el, 8, h);
  }
  return h;
}

// fused_optimizer_step (graph.cpp:458-487) as run_fused_kernel executes it:
// apply_block (graph.cpp:296-347) rounds every attribute to float
// (`const float c = static_cast<float>(attr)`) and each of the 17 body
// instructions to fp32, in body order. In place on n elements of (w, g, m, v).
// Parity: graph.cpp needs Eigen (absent), so this restatement is pinned by the
// reference's own tests (test_graph.cpp:395-452, restated in
// tests/test_fused_optimizer.py), not by the compiled reference.
void or_fused_optimizer_step(int64_t n, float* w, const float* g, float* m, float* v, float lr,
                             float beta1, float beta2, float eps, float weight_decay, int step) {
  const double bc1 = 1.0 / (1.0 - std::pow(static_cast<double>(beta1), step));
  const double bc2 = 1.0 / (1.0 - std::pow(static_cast<double>(beta2), step));
  const float c_b1 = static_cast<float>(static_cast<double>(beta1));
  const float c_omb1 = static_cast<float>(1.0 - static_cast<double>(beta1));
  const float c_b2 = static_cast<float>(static_cast<double>(beta2));
  const float c_omb2 = static_cast<float>(1.0 - static_cast<double>(beta2));
  const float c_bc1 = static_cast<float>(bc1), c_bc2 = static_cast<float>(bc2);
  const float c_eps = static_cast<float>(static_cast<double>(eps));
  const float c_wd = static_cast<float>(static_cast<double>(weight_decay));
  const float c_nlr = static_cast<float>(-static_cast<double>(lr));
  for (int64_t i = 0; i < n; ++i) {
    const float r4 = c_b1 * m[i];           // kScalarMul m, beta1
    const float r5 = c_omb1 * g[i];         // kScalarMul g, 1 - beta1
    const float r6 = r4 + r5;               // m'
    const float r7 = g[i] * g[i];           // kMul g, g
    const float r8 = c_b2 * v[i];
    const float r9 = c_omb2 * r7;
    const float r10 = r8 + r9;              // v'
    const float r11 = c_bc1 * r6;
    const float r12 = c_bc2 * r10;
    const float r13 = std::sqrt(r12);
    const float r14 = r13 + c_eps;
    const float r15 = 1.0f / r14;
    const float r16 = r11 * r15;
    const float r17 = c_wd * w[i];
    const float r18 = r16 + r17;            // u
    const float r19 = c_nlr * r18;
    const float r20 = w[i] + r19;           // w'
    w[i] = r20;
    m[i] = r6;
    v[i] = r10;
  }
}

// quantize_inplace of a binary16 tensor: f16_round = widen(narrow(x)) RNE.
void or_f16_round(float* x, size_t n) {
  for (size_t i = 0; i < n; ++i) x[i] = f16_to_f32(f32_to_f16(x[i]));
}

int or_lamb_step(int T, const int64_t* numel, float* w, const float* g, float* m, float* v,
                 int64_t* step, const float* lamb6) {
  return lamb_step(T, numel, w, g, m, v, step, lamb_from(lamb6));
}

// data is [world][n]; kind 0 fp32 wire, 1 binary16 wire, 2 int64.
int or_ring_allreduce(int world, size_t n, void* data, int kind) {
  if (kind == 2) {
    auto* d = static_cast<int64_t*>(data);
    for (size_t i = 0; i < n; ++i) {
      int64_t s = 0;
      for (int r = 0; r < world; ++r) s += d[static_cast<size_t>(r) * n + i];
      for (int r = 0; r < world; ++r) d[static_cast<size_t>(r) * n + i] = s;
    }
    return 0;
  }
  std::vector<float*> xs;
  for (int r = 0; r < world; ++r) xs.push_back(static_cast<float*>(data) + static_cast<size_t>(r) * n);
  ring_allreduce_emulated(xs, n, kind == 1);
  return 0;
}

// Box-Muller initialisation (restates tensor.cpp:72-92 and the per-tensor
// seed draws of model.cpp:124-176). init: 0 randn(σ=0.02), 1 ones, 2 zeros.
void or_build_params(int T, const int64_t* numel, const int* init, uint64_t seed, float* out) {
  // the per-tensor seeds are drawn in tensor order first (model.cpp's
  // sequence), then the tensors are filled independently
  std::mt19937_64 seeds(seed);
  std::vector<uint64_t> tseed(static_cast<size_t>(T), 0);
  std::vector<size_t> toff(static_cast<size_t>(T), 0);
  size_t off = 0;
  for (int t = 0; t < T; ++t) {
    if (init[t] == 0) tseed[static_cast<size_t>(t)] = seeds();
    toff[static_cast<size_t>(t)] = off;
    off += static_cast<size_t>(numel[t]);
  }
  pfor_items(T, [&](int t) {
    const size_t n = static_cast<size_t>(numel[t]);
    float* o = out + toff[static_cast<size_t>(t)];
    if (init[t] == 0) {
      std::mt19937_64 rng(tseed[static_cast<size_t>(t)]);
      const double two_pi = 6.283185307179586476925286766559;
      size_t i = 0;
      while (i < n) {
        double u1;
        do { u1 = static_cast<double>(rng() >> 11) * 0x1.0p-53; } while (u1 <= 0.0);
        const double u2 = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        const double rad = std::sqrt(-2.0 * std::log(u1));
        o[i++] = static_cast<float>(rad * std::cos(two_pi * u2) * 0.02f);
        if (i < n) o[i++] = static_cast<float>(rad * std::sin(two_pi * u2) * 0.02f);
      }
    } else {
      const float fill = init[t] == 1 ? 1.0f : 0.0f;
      std::fill(o, o + n, fill);
    }
  });
}

// fp16 gradient bits of one (rank, step, micro), model-order flat layout.
void or_synth_grads(int64_t P, uint64_t seed, int rank, int step, int micro, float scale,
                    uint32_t spike_ppm, int spike_exp, uint16_t* out) {
  const uint64_t base = bo_synth_base(seed, static_cast<uint64_t>(rank),
                                      static_cast<uint64_t>(step), static_cast<uint64_t>(micro));
  pfor(P, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      out[i] = f32_to_f16(bo_synth_true_grad(base, static_cast<uint64_t>(i), spike_ppm, spike_exp) * scale);
    }
  });
}

// The whole gradient-to-update pipeline for `world` ranks, emulated in one
// thread. Restates DistributedTrainer::train_step (trainer.cpp:217-373):
//   acc   = ((0 + g0) + g1) + ... + g_{K-2}          (trainer.cpp:240-244)
//   x     = (g_{K-1} [+ acc]) * (1/(K*S))             (trainer.cpp:186-203)
//   bucket ring all-reduce, then * (1/world)          (trainer.cpp:205-215)
//   lamb_step on the reduced gradient                 (lamb.cpp:23-84)
// plus the dynamic loss-scaler extension (found_inf := the reduced gradient
// holds a non-finite -> skip the LAMB step entirely).
// grads_in: optional caller-supplied fp16 inputs [steps][world][K][P]; when
// null the synthetic spec is used (with injections inj[n_inj][5]).
int or_train(int T, const int64_t* numel, const int* firsts, const float* params_in, int world,
             int K, uint64_t bucket_bytes, int f16_wire, const float* lamb6, const or_scaler* sc,
             uint64_t grad_seed, uint32_t spike_ppm, int spike_exp, const int64_t* inj, int n_inj,
             const uint16_t* grads_in, int steps, float* params_out, float* m_out, float* v_out,
             int64_t* lamb_step_out, float* scale_used, int* found_inf, float* final_scale,
             int* final_good) {
  if (world < 1 || K < 1 || bucket_bytes == 0) return 5;
  int64_t P = 0;
  std::vector<int64_t> toff(static_cast<size_t>(T));
  for (int t = 0; t < T; ++t) { toff[static_cast<size_t>(t)] = P; P += numel[t]; }
  const Layout L = build_layout(T, numel, firsts, bucket_bytes);
  const Lamb lc = lamb_from(lamb6);
  std::vector<float> w(params_in, params_in + P), m(static_cast<size_t>(P), 0.0f), v(static_cast<size_t>(P), 0.0f);
  int64_t lstep = 0;
  float S = sc->init_scale;
  int good = 0;
  std::vector<std::vector<float>> x(static_cast<size_t>(world), std::vector<float>(static_cast<size_t>(P)));
  std::vector<float> acc(static_cast<size_t>(P));
  std::vector<uint16_t> h(static_cast<size_t>(P));
  std::vector<float> u;
  for (int step = 0; step < steps; ++step) {
    scale_used[step] = S;
    const float inv = 1.0f / (static_cast<float>(K) * S);
    for (int r = 0; r < world; ++r) {
      for (int k = 0; k < K; ++k) {
        if (grads_in) {
          const size_t base = ((static_cast<size_t>(step) * world + r) * K + k) * static_cast<size_t>(P);
          std::memcpy(h.data(), grads_in + base, static_cast<size_t>(P) * 2);
        } else {
          or_synth_grads(P, grad_seed, r, step, k, S, spike_ppm, spike_exp, h.data());
          for (int q = 0; q < n_inj; ++q) {
            const int64_t* e = inj + 5 * q;
            if (e[0] == step && e[1] == r && e[2] == k) h[static_cast<size_t>(e[3])] = static_cast<uint16_t>(e[4]);
          }
        }
        float* X = x[static_cast<size_t>(r)].data();
        pfor(P, [&](int64_t lo, int64_t hi) {
          for (int64_t i = lo; i < hi; ++i) {
            const float gi = f16_to_f32(h[static_cast<size_t>(i)]);
            if (k + 1 < K) {
              acc[static_cast<size_t>(i)] = (k == 0 ? 0.0f : acc[static_cast<size_t>(i)]) + gi;
            } else {
              const float val = K > 1 ? gi + acc[static_cast<size_t>(i)] : gi;
              X[i] = val * inv;
            }
          }
        });
      }
    }
    // Bucketed ring all-reduce: gather each bucket in layout order, reduce,
    // scatter back, scale by 1/world.
    if (world > 1) {
      const float invn = 1.0f / static_cast<float>(world);
      pfor_items(static_cast<int>(L.buckets.size()), [&](int bi) {  // buckets are disjoint
        const size_t b = static_cast<size_t>(bi);
        const size_t nb = static_cast<size_t>(L.elems[b]);
        std::vector<std::vector<float>> flat(static_cast<size_t>(world), std::vector<float>(nb));
        for (int r = 0; r < world; ++r) {
          size_t o = 0;
          for (int p : L.buckets[b]) {
            std::memcpy(flat[static_cast<size_t>(r)].data() + o, x[static_cast<size_t>(r)].data() + toff[static_cast<size_t>(p)],
                        static_cast<size_t>(numel[p]) * 4);
            o += static_cast<size_t>(numel[p]);
          }
        }
        std::vector<float*> ptrs;
        for (auto& f : flat) ptrs.push_back(f.data());
        ring_allreduce_emulated(ptrs, nb, f16_wire != 0);
        size_t o = 0;
        for (int p : L.buckets[b]) {
          float* dst = x[0].data() + toff[static_cast<size_t>(p)];
          for (int64_t i = 0; i < numel[p]; ++i) dst[i] = flat[0][o + static_cast<size_t>(i)] * invn;
          o += static_cast<size_t>(numel[p]);
        }
      });
    }
    const std::vector<float>& g = x[0];
    std::atomic<bool> any_bad{false};
    pfor(P, [&](int64_t lo, int64_t hi) {
      bool bad = false;
      for (int64_t i = lo; i < hi && !bad; ++i) bad = !std::isfinite(g[static_cast<size_t>(i)]);
      if (bad) any_bad = true;
    });
    const bool found = any_bad;
    if (!found) {
      lamb_step_finite(T, numel, w.data(), g.data(), m.data(), v.data(), &lstep, lc, u);
    }
    found_inf[step] = found ? 1 : 0;
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
  std::memcpy(params_out, w.data(), static_cast<size_t>(P) * 4);
  std::memcpy(m_out, m.data(), static_cast<size_t>(P) * 4);
  std::memcpy(v_out, v.data(), static_cast<size_t>(P) * 4);
  *lamb_step_out = lstep;
  *final_scale = S;
  *final_good = good;
  return 0;
}

}  // extern "C"
