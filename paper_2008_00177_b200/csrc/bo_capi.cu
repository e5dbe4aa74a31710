// C ABI of the pipeline context: creation, layout, communication, state, and
// the hot-path entry point bo_accumulate (see include/bertopt_b200.h).
#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bo_internal.hpp"

namespace bo {

namespace {
thread_local std::string g_last_error;
}

void fail(bo_status code, const std::string& msg) { throw Failure{code, msg}; }
void set_thread_error(const std::string& msg) { g_last_error = msg; }

void* dev_alloc(bo_ctx* c, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 256;
  BO_CUDA(cudaMalloc(&p, bytes));
  BO_CUDA(cudaMemsetAsync(p, 0, bytes, c->stream));
  c->allocations.push_back(p);
  c->device_bytes += bytes;
  return p;
}

template <typename T>
static T* upload(bo_ctx* c, const std::vector<T>& v) {
  T* d = static_cast<T*>(dev_alloc(c, v.size() * sizeof(T)));
  if (!v.empty()) {
    BO_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  }
  return d;
}

// Work tables: accumulate/finalize tiles over tensors, LAMB tiles over this
// rank's shard (split at tensor boundaries), ring tiles over the shard.
void upload_tables(bo_ctx* c) {
  const Layout& L = c->L;
  std::vector<TensorDev> td(static_cast<size_t>(L.T));
  std::vector<AccTile> acc_tiles;
  for (int t = 0; t < L.T; ++t) {
    td[static_cast<size_t>(t)] = TensorDev{L.acc_off[static_cast<size_t>(t)], L.flat_off[static_cast<size_t>(t)]};
    for (int64_t e = 0; e < L.numel[static_cast<size_t>(t)]; e += kTileElems) {
      const int64_t len = std::min<int64_t>(kTileElems, L.numel[static_cast<size_t>(t)] - e);
      acc_tiles.push_back(AccTile{t, static_cast<int32_t>(len), e});
    }
  }
  std::vector<LambTile> lamb_tiles;
  std::vector<int> tile_begin(static_cast<size_t>(L.T) + 1, 0);
  std::vector<std::vector<LambTile>> per_tensor(static_cast<size_t>(L.T));
  const int q = L.own;  // owned chunk
  for (int b = 0; b < L.B; ++b) {
    const int64_t cb = L.chunk[static_cast<size_t>(b)];
    const int64_t lo = q * cb;
    const int64_t hi = std::min<int64_t>((q + 1) * cb, L.elems[static_cast<size_t>(b)]);
    for (int p : L.buckets[static_cast<size_t>(b)]) {
      const int64_t t0 = L.offset_of[static_cast<size_t>(p)];
      const int64_t t1 = t0 + L.numel[static_cast<size_t>(p)];
      const int64_t a = std::max(lo, t0), z = std::min(hi, t1);
      for (int64_t e = a; e < z; e += kTileElems) {
        const int64_t len = std::min<int64_t>(kTileElems, z - e);
        per_tensor[static_cast<size_t>(p)].push_back(
            LambTile{L.shard_pos(b, p, e), L.flat_pos(b, p, e), static_cast<int32_t>(len), p});
      }
    }
  }
  // Tiles grouped per tensor so each tensor's partials are contiguous; within
  // a tensor, shard order.
  for (int t = 0; t < L.T; ++t) {
    tile_begin[static_cast<size_t>(t)] = static_cast<int>(lamb_tiles.size());
    for (const LambTile& lt : per_tensor[static_cast<size_t>(t)]) lamb_tiles.push_back(lt);
  }
  tile_begin[static_cast<size_t>(L.T)] = static_cast<int>(lamb_tiles.size());

  if (c->world == 1) {
    // Single-rank LAMB (bo_fused.cu): tiles of <= kTileElems elements of one
    // tensor, model order, in the aligned tensor layout; per-tensor tile
    // ranges for the fixed-order norm reduction.
    std::vector<FusedTile> ft;
    std::vector<int> ttiles(static_cast<size_t>(L.T) + 1);
    for (int t = 0; t < L.T; ++t) {
      const int64_t n = L.numel[static_cast<size_t>(t)];
      ttiles[static_cast<size_t>(t)] = static_cast<int>(ft.size());
      for (int64_t e = 0; e < n; e += kTileElems) {
        ft.push_back(FusedTile{L.acc_off[static_cast<size_t>(t)] + e, e,
                               static_cast<int32_t>(std::min<int64_t>(kTileElems, n - e)), t});
      }
    }
    ttiles[static_cast<size_t>(L.T)] = static_cast<int>(ft.size());
    c->d_fused_tiles = upload(c, ft);
    c->n_fused_tiles = static_cast<int>(ft.size());
    c->d_fused_tensor_tiles = upload(c, ttiles);
  }
  if (c->world > 1) {
    // Ring hops with the finalize fused in: for every chunk index q, the
    // valid (non-padding) elements of chunk q of every bucket, split at tensor
    // boundaries, in shard order.
    std::vector<HopXTile> hx;
    c->hopx_begin.assign(static_cast<size_t>(c->world) + 1, 0);
    c->hopx_bucket_begin.assign(static_cast<size_t>(c->world), std::vector<int>(static_cast<size_t>(L.B) + 1, 0));
    for (int qq = 0; qq < c->world; ++qq) {
      c->hopx_begin[static_cast<size_t>(qq)] = static_cast<int>(hx.size());
      for (int b = 0; b < L.B; ++b) {
        c->hopx_bucket_begin[static_cast<size_t>(qq)][static_cast<size_t>(b)] = static_cast<int>(hx.size());
        const int64_t cb = L.chunk[static_cast<size_t>(b)];
        const int64_t lo = qq * cb;
        const int64_t hi = std::min<int64_t>((qq + 1) * cb, L.elems[static_cast<size_t>(b)]);
        for (int p : L.buckets[static_cast<size_t>(b)]) {
          const int64_t t0 = L.offset_of[static_cast<size_t>(p)];
          const int64_t a = std::max(lo, t0), z = std::min(hi, t0 + L.numel[static_cast<size_t>(p)]);
          for (int64_t e = a; e < z; e += kTileElems) {
            hx.push_back(HopXTile{L.shoff[static_cast<size_t>(b)] + (e - lo), e - t0,
                                  static_cast<int32_t>(std::min<int64_t>(kTileElems, z - e)), p});
          }
        }
      }
      c->hopx_bucket_begin[static_cast<size_t>(qq)][static_cast<size_t>(L.B)] = static_cast<int>(hx.size());
    }
    c->hopx_begin[static_cast<size_t>(c->world)] = static_cast<int>(hx.size());
    c->d_hopx_tiles = upload(c, hx);

    // Communication groups for the overlapped sync micro: consecutive buckets
    // (layout order = gradient-ready order) merged up to >= BO_COMM_GROUP_ELEMS
    // elements (default 16 Mi = 64 MiB of fp32 gradient), so every group costs
    // N - 1 hop barriers; a pure function of the layout and the environment,
    // which must therefore match across ranks (it is part of the layout hash).
    int64_t group_elems = 16ll << 20;
    if (const char* e = std::getenv("BO_COMM_GROUP_ELEMS")) {
      group_elems = std::max<int64_t>(1, std::atoll(e));
    }
    c->comm_groups.clear();
    c->group_of_bucket.assign(static_cast<size_t>(L.B), 0);
    std::vector<AccTile> gacc;
    std::vector<int> first_acc_tile(static_cast<size_t>(L.T) + 1, 0);
    for (int t = 0, i = 0; t < L.T; ++t) {
      first_acc_tile[static_cast<size_t>(t)] = i;
      i += static_cast<int>((L.numel[static_cast<size_t>(t)] + kTileElems - 1) / kTileElems);
    }
    int b0 = 0;
    int64_t n = 0;
    for (int b = 0; b < L.B; ++b) {
      n += L.elems[static_cast<size_t>(b)];
      if (n >= group_elems || b == L.B - 1) {
        bo_ctx::CommGroup g{b0, b + 1, 0, static_cast<int>(gacc.size()), 0};
        for (int bb = b0; bb <= b; ++bb) {
          c->group_of_bucket[static_cast<size_t>(bb)] = static_cast<int>(c->comm_groups.size());
          for (int p : L.buckets[static_cast<size_t>(bb)]) {
            g.pending0 += 1;
            const int64_t nt = (L.numel[static_cast<size_t>(p)] + kTileElems - 1) / kTileElems;
            for (int64_t k = 0; k < nt; ++k) gacc.push_back(acc_tiles[static_cast<size_t>(first_acc_tile[static_cast<size_t>(p)] + k)]);
          }
        }
        g.acc1 = static_cast<int>(gacc.size());
        c->comm_groups.push_back(g);
        b0 = b + 1;
        n = 0;
      }
    }
    c->d_group_acc_tiles = upload(c, gacc);
  }
  c->d_tensors = upload(c, td);
  c->d_acc_tiles = upload(c, acc_tiles);
  c->n_acc_tiles = static_cast<int>(acc_tiles.size());
  c->d_lamb_tiles = upload(c, lamb_tiles);
  c->n_lamb_tiles = static_cast<int>(lamb_tiles.size());
  c->d_tensor_tile_begin = upload(c, tile_begin);
}

// Bias corrections bc_t = 1 - pow(double(beta), double(t)) evaluated on the
// host with the same libm the reference uses (lamb.cpp:158-161), with their
// reciprocals; the device indexes the table by its own step counter.
void grow_bc_table(bo_ctx* c, int64_t need) {
  if (need <= c->bc_cap) return;
  int64_t cap = std::max<int64_t>(4096, c->bc_cap * 2);
  while (cap < need) cap *= 2;
  std::vector<double> tab(static_cast<size_t>(cap) * 4);
  for (int64_t i = 0; i < cap; ++i) {
    const double t = static_cast<double>(i + 1);
    const double bc1 = 1.0 - std::pow(static_cast<double>(c->cfg.lamb.beta1), t);
    const double bc2 = 1.0 - std::pow(static_cast<double>(c->cfg.lamb.beta2), t);
    tab[static_cast<size_t>(4 * i)] = bc1;
    tab[static_cast<size_t>(4 * i + 1)] = bc2;
    tab[static_cast<size_t>(4 * i + 2)] = 1.0 / bc1;
    tab[static_cast<size_t>(4 * i + 3)] = 1.0 / bc2;
  }
  double* d = nullptr;
  BO_CUDA(cudaMalloc(&d, tab.size() * sizeof(double)));
  BO_CUDA(cudaMemcpyAsync(d, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  // The old table may still be read by queued kernels: keep it alive.
  if (c->bc_table) c->allocations.push_back(c->bc_table);
  BO_CUDA(cudaStreamSynchronize(c->stream));  // tab is pageable host memory
  c->bc_table = d;
  c->bc_cap = cap;
}

static cudaEvent_t take_event(bo_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  BO_CUDA(cudaEventCreate(&e));
  return e;
}

StageTimer::StageTimer(bo_ctx* ctx, int s) : StageTimer(ctx, s, ctx->stream) {}

StageTimer::StageTimer(bo_ctx* ctx, int s, cudaStream_t on) : c(ctx), stage(s), stream(on) {
  if (!c->profiling || !((c->profile_mask >> s) & 1)) return;
  b = take_event(c);
  BO_CUDA(cudaEventRecord(b, stream));
}

StageTimer::~StageTimer() {
  if (!c->profiling || !b) return;
  cudaEvent_t e = take_event(c);
  if (cudaEventRecord(e, stream) == cudaSuccess) c->marks.push_back({stage, b, e});
}

static void drain_marks(bo_ctx* c) {
  BO_CUDA(cudaStreamSynchronize(c->stream));
  if (c->comm_stream) BO_CUDA(cudaStreamSynchronize(c->comm_stream));
  for (const auto& mk : c->marks) {
    float ms = 0.0f;
    BO_CUDA(cudaEventElapsedTime(&ms, mk.a, mk.b));
    c->stage_ms[mk.stage] += ms;
    c->stage_count[mk.stage] += 1;
    c->event_pool.push_back(mk.a);
    c->event_pool.push_back(mk.b);
  }
  c->marks.clear();
}

static bool is_pow2(float s) {
  if (!(s > 0.0f) || !std::isfinite(s)) return false;
  int e = 0;
  return std::frexp(s, &e) == 0.5f;
}

static uint64_t fnv1a(const void* data, size_t len, uint64_t h) {
  const auto* p = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < len; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

// BucketLayout::hash (trainer.cpp:118-134) salted like ensure_layout
// (trainer.cpp:165-168). Without names, the tensor index stands in.
static uint64_t layout_hash(const Layout& L, const char* const* names, const int32_t* ndims,
                            const int64_t* dims, bool f16, int K) {
  std::vector<size_t> doff(static_cast<size_t>(L.T) + 1, 0);
  if (ndims) {
    for (int t = 0; t < L.T; ++t) doff[static_cast<size_t>(t) + 1] = doff[static_cast<size_t>(t)] + static_cast<size_t>(ndims[t]);
  }
  uint64_t h = fnv1a("bucket-layout", 13, 14695981039346656037ull);
  const uint64_t nb = static_cast<uint64_t>(L.B);
  h = fnv1a(&nb, 8, h);
  for (int b = 0; b < L.B; ++b) {
    for (int p : L.buckets[static_cast<size_t>(b)]) {
      if (names) {
        h = fnv1a(names[p], std::strlen(names[p]), h);
      } else {
        const int64_t id = p;
        h = fnv1a(&id, 8, h);
      }
      if (ndims && dims) {
        for (size_t d = doff[static_cast<size_t>(p)]; d < doff[static_cast<size_t>(p) + 1]; ++d) h = fnv1a(&dims[d], 8, h);
      } else {
        h = fnv1a(&L.numel[static_cast<size_t>(p)], 8, h);
      }
    }
    const uint64_t el = static_cast<uint64_t>(L.elems[static_cast<size_t>(b)]);
    h = fnv1a(&el, 8, h);
  }
  const bool f16b = f16;
  h = fnv1a(&f16b, sizeof(bool), h);
  const uint64_t salt = static_cast<uint64_t>(K);
  return fnv1a(&salt, 8, h);
}

static void validate(const bo_trainer_config& c) {
  if (c.accumulation < 1) fail(BO_ERR_INVALID_CONFIG, "accumulation must be >= 1");
  if (c.bucket_bytes == 0) fail(BO_ERR_INVALID_CONFIG, "bucket_bytes must be > 0");
  const bo_scaler_config& s = c.scaler;
  if (!is_pow2(s.init_scale)) fail(BO_ERR_INVALID_CONFIG, "loss scale must be a positive power of two");
  if (s.dynamic) {
    if (!is_pow2(s.min_scale) || !is_pow2(s.max_scale) || s.min_scale > s.max_scale ||
        !is_pow2(s.growth_factor) || !is_pow2(s.backoff_factor) || s.growth_interval < 1) {
      fail(BO_ERR_INVALID_CONFIG, "dynamic scaler needs power-of-two bounds/factors and interval >= 1");
    }
  }
  if (c.reduce_algo < 0 || c.reduce_algo > BO_REDUCE_NCCL) fail(BO_ERR_INVALID_CONFIG, "bad reduce_algo");
  if (c.reduce_algo == BO_REDUCE_NCCL && c.f16_exchange) {
    fail(BO_ERR_INVALID_CONFIG, "the binary16 wire needs the ring reduction (NCCL half sums differ)");
  }
}

struct StateHeader {
  char magic[4];
  uint32_t version;
  int32_t world, rank, own, T;
  int64_t P;
  uint64_t layout_hash;
  DevState st;
};

// Owned (shard) pieces: (shard index, model-order index, length).
template <typename F>
static void for_owned(const Layout& L, F&& f) {
  const int q = L.own;
  for (int b = 0; b < L.B; ++b) {
    const int64_t cb = L.chunk[static_cast<size_t>(b)];
    const int64_t lo = q * cb, hi = std::min<int64_t>((q + 1) * cb, L.elems[static_cast<size_t>(b)]);
    for (int p : L.buckets[static_cast<size_t>(b)]) {
      const int64_t t0 = L.offset_of[static_cast<size_t>(p)], t1 = t0 + L.numel[static_cast<size_t>(p)];
      const int64_t a = std::max(lo, t0), z = std::min(hi, t1);
      if (a < z) f(L.shard_pos(b, p, a), L.model_off[static_cast<size_t>(p)] + (a - t0), z - a);
    }
  }
}

}  // namespace bo

using namespace bo;

#define BO_GUARD_BEGIN try {
#define BO_GUARD_END                          \
  }                                           \
  catch (const Failure& f) {                  \
    set_thread_error(f.msg);                  \
    return f.code;                            \
  }                                           \
  catch (const std::exception& e) {           \
    set_thread_error(e.what());               \
    return BO_ERR_CUDA;                       \
  }                                           \
  return BO_OK;

extern "C" {

int32_t bo_abi_version(void) { return BO_ABI_VERSION; }

const char* bo_status_name(int32_t s) {
  switch (s) {
    case BO_OK: return "OK";
    case BO_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case BO_ERR_NON_FINITE_GRADIENT: return "NonFiniteGradient";
    case BO_ERR_OVERFLOW_DETECTED: return "OverflowDetected";
    case BO_ERR_LENGTH_MISMATCH: return "LengthMismatch";
    case BO_ERR_INVALID_CONFIG: return "InvalidConfig";
    case BO_ERR_BUCKET_LAYOUT_MISMATCH: return "BucketLayoutMismatch";
    case BO_ERR_PEER_DISCONNECTED: return "PeerDisconnected";
    case BO_ERR_WATCHDOG_TIMEOUT: return "WatchdogTimeout";
    case BO_ERR_PROTOCOL: return "ProtocolError";
    case BO_ERR_CUDA: return "CudaError";
    case BO_ERR_NCCL: return "NcclError";
    case BO_ERR_NO_DEVICE: return "NoDevice";
    default: return "Unknown";
  }
}

const char* bo_last_error(void) { return g_last_error.c_str(); }

void bo_default_config(bo_trainer_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->lamb = bo_lamb_config{1e-3f, 0.9f, 0.999f, 1e-6f, 0.01f, 10.0f};  // lamb.hpp:165-172
  cfg->accumulation = 1;
  cfg->bucket_bytes = 4ull << 20;  // trainer.hpp:78
  cfg->f16_exchange = 0;
  cfg->reduce_algo = BO_REDUCE_AUTO;
  cfg->scaler = bo_scaler_config{65536.0f, 2.0f, 0.5f, 1.0f, 16777216.0f, 2000, 1};
}

bo_status bo_bucket_layout(int32_t n_tensors, const int64_t* numels, const int32_t* firsts,
                           uint64_t bucket_bytes, const char* const* names, const int32_t* ndims,
                           const int64_t* dims, int32_t f16_exchange, int32_t accumulation,
                           int32_t* bucket_of, int64_t* offset_of, int32_t* ready_order,
                           int64_t* bucket_elems, int32_t* n_buckets, uint64_t* hash) {
  BO_GUARD_BEGIN
  if (!numels || !firsts) fail(BO_ERR_INVALID_CONFIG, "null argument");
  const Layout L = Layout::build(n_tensors, numels, firsts, bucket_bytes, 1, 0);
  for (int t = 0; t < L.T; ++t) {
    if (bucket_of) bucket_of[t] = L.bucket_of[static_cast<size_t>(t)];
    if (offset_of) offset_of[t] = L.offset_of[static_cast<size_t>(t)];
    if (ready_order) ready_order[t] = L.ready[static_cast<size_t>(t)];
  }
  if (bucket_elems) {
    for (int b = 0; b < L.B; ++b) bucket_elems[b] = L.elems[static_cast<size_t>(b)];
  }
  if (n_buckets) *n_buckets = L.B;
  if (hash) *hash = layout_hash(L, names, ndims, dims, f16_exchange != 0, accumulation);
  BO_GUARD_END
}

bo_status bo_shard_ranges(int32_t n_buckets, const int64_t* bucket_elems, int32_t world, int32_t rank,
                          int64_t* lo, int64_t* hi) {
  BO_GUARD_BEGIN
  if (world < 1 || rank < 0 || rank >= world) fail(BO_ERR_INVALID_CONFIG, "bad rank/world");
  for (int b = 0; b < n_buckets; ++b) {
    const int64_t c = (bucket_elems[b] + world - 1) / world;  // collective.cpp:50-52
    lo[b] = std::min<int64_t>(rank * c, bucket_elems[b]);
    hi[b] = std::min<int64_t>((rank + 1) * c, bucket_elems[b]);
  }
  BO_GUARD_END
}

bo_status bo_create(const bo_trainer_config* cfg, int32_t n_tensors, const int64_t* numels,
                    const int32_t* first_consumers, const char* const* names, const int32_t* ndims,
                    const int64_t* dims, int32_t device, int32_t rank, int32_t world, bo_ctx** out) {
  bo_ctx* c = nullptr;
  BO_GUARD_BEGIN
  *out = nullptr;
  if (!cfg || !numels || !first_consumers) fail(BO_ERR_INVALID_CONFIG, "null argument");
  validate(*cfg);
  if (n_tensors > kMaxTensors) fail(BO_ERR_INVALID_CONFIG, "more than 1024 tensors");
  if (world < 1 || world > 8) {
    fail(BO_ERR_INVALID_CONFIG, "world must be 1..8 (the GPUs of one NVSwitch node)");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    fail(BO_ERR_NO_DEVICE, "no CUDA device visible");
  }
  c = new bo_ctx();
  c->cfg = *cfg;
  c->device = device;
  c->rank = rank;
  c->world = world;
  if (const char* e = std::getenv("BO_UNFUSED")) c->force_unfused = std::strcmp(e, "0") != 0;
  if (const char* e = std::getenv("BO_RING_NCCL")) c->ring_via_nccl = std::strcmp(e, "0") != 0;
  if (const char* e = std::getenv("BO_FUSE_LAST")) c->fuse_last_hop = std::strcmp(e, "0") != 0;
  c->algo = cfg->reduce_algo == BO_REDUCE_AUTO ? (cfg->f16_exchange ? BO_REDUCE_RING : BO_REDUCE_NCCL)
                                               : cfg->reduce_algo;
  BO_CUDA(cudaSetDevice(device));
  BO_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  BO_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  c->L = Layout::build(n_tensors, numels, first_consumers, cfg->bucket_bytes, world, rank);
  c->L.hash = layout_hash(c->L, names, ndims, dims, cfg->f16_exchange != 0, cfg->accumulation);
  if (world > 1 && c->algo == BO_REDUCE_RING) c->L.own = (rank + 1) % world;
  const Layout& L = c->L;
  c->lamb = LambConsts{cfg->lamb.beta1, cfg->lamb.beta2, 1.0f - cfg->lamb.beta1, 1.0f - cfg->lamb.beta2,
                       cfg->lamb.eps, cfg->lamb.weight_decay, cfg->lamb.lr, cfg->lamb.trust_clip};
  c->scaler = ScalerConsts{cfg->scaler.growth_factor, cfg->scaler.backoff_factor, cfg->scaler.min_scale,
                           cfg->scaler.max_scale, cfg->scaler.growth_interval, cfg->scaler.dynamic};
  upload_tables(c);
  c->acc = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.acc_total) * 4));
  // the fusion buffer x and the fp32 reduced shard exist only where a kernel
  // materialises them: one rank's multi-kernel fallback and the NCCL wire (the
  // ring computes x inside its hops and LAMB reads the final wire buffer)
  if (world == 1 || c->algo == BO_REDUCE_NCCL) {
    c->x = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.flat_total) * 4));
    c->gshard = world == 1 ? c->x : static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
  }
  c->w = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.flat_total) * 4));
  c->m = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
  c->v = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
  // double-buffered moments: LAMB phase 1 writes the new m, v before the
  // step's overflow flag is final (DevState::parity picks the current set)
  c->m_alt = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
  c->v_alt = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
  c->sync_tab = new PtrTable{};
  c->delivered.assign(static_cast<size_t>(L.T), 0);
  if (world > 1) {
    BO_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    BO_CUDA(cudaEventCreateWithFlags(&c->comm_ready, cudaEventDisableTiming));
    BO_CUDA(cudaEventCreateWithFlags(&c->comm_done, cudaEventDisableTiming));
    c->wsh = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
    c->u = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
    c->d_barrier = static_cast<int*>(dev_alloc(c, 4));
  }
  if (world > 1 && c->algo == BO_REDUCE_RING) {
    const size_t e = cfg->f16_exchange ? 2 : 4;
    c->wire[0] = dev_alloc(c, static_cast<size_t>(L.shard_total) * e);
    c->wire[1] = dev_alloc(c, static_cast<size_t>(L.shard_total) * e);
  }
  c->tile_part = static_cast<double*>(
      dev_alloc(c, static_cast<size_t>(std::max({c->n_lamb_tiles, c->n_fused_tiles, 1})) * 16));
  if (world == 1) c->u = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.acc_total) * 4));
  c->rank_part = static_cast<double*>(dev_alloc(c, static_cast<size_t>(2 * L.T + 1) * 8));
  c->all_part = world == 1 ? c->rank_part
                           : static_cast<double*>(dev_alloc(c, static_cast<size_t>(world) * (2 * L.T + 1) * 8));
  c->trust = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.T) * 4));
  c->state = static_cast<DevState*>(dev_alloc(c, sizeof(DevState)));
  DevState st{};
  st.scale = cfg->scaler.init_scale;
  BO_CUDA(cudaMemcpyAsync(c->state, &st, sizeof(st), cudaMemcpyHostToDevice, c->stream));
  grow_bc_table(c, 16);
  BO_CUDA(cudaStreamSynchronize(c->stream));
  *out = c;
  c = nullptr;
  }
  catch (const Failure& f) {
    set_thread_error(f.msg);
    if (c) bo_destroy(c);
    return f.code;
  }
  return BO_OK;
}

void bo_destroy(bo_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (const auto& mk : c->marks) {
    cudaEventDestroy(mk.a);
    cudaEventDestroy(mk.b);
  }
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->comm_ready) cudaEventDestroy(c->comm_ready);
  if (c->comm_done) cudaEventDestroy(c->comm_done);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c->sync_tab;
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->comm) ncclCommDestroy(c->comm);
  for (void* p : c->allocations) cudaFree(p);
  if (c->bc_table) cudaFree(c->bc_table);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int32_t bo_layout_num_buckets(const bo_ctx* c) { return c ? c->L.B : 0; }

bo_status bo_layout_query(const bo_ctx* c, int32_t* bucket_of, int64_t* offset_of, int32_t* ready_order,
                          int64_t* bucket_elems) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  for (int t = 0; t < c->L.T; ++t) {
    if (bucket_of) bucket_of[t] = c->L.bucket_of[static_cast<size_t>(t)];
    if (offset_of) offset_of[t] = c->L.offset_of[static_cast<size_t>(t)];
    if (ready_order) ready_order[t] = c->L.ready[static_cast<size_t>(t)];
  }
  if (bucket_elems) {
    for (int b = 0; b < c->L.B; ++b) bucket_elems[b] = c->L.elems[static_cast<size_t>(b)];
  }
  BO_GUARD_END
}

uint64_t bo_layout_hash(const bo_ctx* c) { return c ? c->L.hash : 0; }
int64_t bo_shard_elems(const bo_ctx* c) {
  if (!c) return 0;
  int64_t s = 0;
  for (int b = 0; b < c->L.B; ++b) s += c->L.chunk[static_cast<size_t>(b)];
  return s;
}
uint64_t bo_device_bytes(const bo_ctx* c) { return c ? c->device_bytes : 0; }

bo_status bo_comm_unique_id(uint8_t* out128) {
  BO_GUARD_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  ncclUniqueId id;
  BO_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, 128);
  BO_GUARD_END
}

bo_status bo_comm_init(bo_ctx* c, const uint8_t* id128) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  if (c->world == 1) return BO_OK;
  BO_CUDA(cudaSetDevice(c->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  BO_NCCL(ncclCommInitRank(&c->comm, c->world, id, c->rank));
  // Layout agreement (trainer.cpp:169-183): all-gather the salted hash, and
  // a hash of the settings that shape the collective call sequence (reduce
  // algorithm, ring transport, communication groups of the overlapped sync
  // micro) so that ranks started with different BO_* environments fail here
  // instead of deadlocking later.
  uint64_t mine[2] = {c->L.hash, 1469598103934665603ull};
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) mine[1] = (mine[1] ^ ((v >> (8 * i)) & 0xFF)) * 1099511628211ull;
  };
  mix(static_cast<uint64_t>(c->algo));
  mix(c->ring_via_nccl ? 1 : 0);
  mix(c->comm_groups.size());
  for (const auto& g : c->comm_groups) mix(static_cast<uint64_t>(g.b1));
  uint64_t* d = static_cast<uint64_t*>(dev_alloc(c, static_cast<size_t>(2 * c->world + 2) * 8));
  BO_CUDA(cudaMemcpyAsync(d, mine, 16, cudaMemcpyHostToDevice, c->stream));
  BO_NCCL(ncclAllGather(d, d + 2, 2, ncclUint64, c->comm, c->stream));
  std::vector<uint64_t> all(static_cast<size_t>(2 * c->world));
  BO_CUDA(cudaMemcpyAsync(all.data(), d + 2, all.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  for (int r = 0; r < c->world; ++r) {
    if (all[static_cast<size_t>(2 * r)] != mine[0]) {
      fail(BO_ERR_BUCKET_LAYOUT_MISMATCH,
           "rank " + std::to_string(c->rank) + " bucket layout disagrees with peers");
    }
    if (all[static_cast<size_t>(2 * r + 1)] != mine[1]) {
      fail(BO_ERR_PROTOCOL, "rank " + std::to_string(c->rank) +
                                " collective settings (reduce algorithm, BO_RING_NCCL, "
                                "BO_COMM_GROUP_ELEMS) disagree with peers");
    }
  }
  // Map every rank's flat parameter replica into this process (CUDA IPC over
  // NVLink/NVSwitch): LAMB phase 2 stores each updated shard element straight
  // into all replicas, which replaces the parameter all-gather.
  // The ring's two staging buffers are mapped too: a hop reads the left
  // neighbour's previous output in place over NVLink.
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  const bool ring = c->algo == BO_REDUCE_RING;
  auto map_all = [&](void* mine_ptr, std::vector<void*>& out) {
    cudaIpcMemHandle_t mine;
    BO_CUDA(cudaIpcGetMemHandle(&mine, mine_ptr));
    uint8_t* dh = static_cast<uint8_t*>(dev_alloc(c, static_cast<size_t>(c->world + 1) * 64));
    BO_CUDA(cudaMemcpyAsync(dh, &mine, 64, cudaMemcpyHostToDevice, c->stream));
    BO_NCCL(ncclAllGather(dh, dh + 64, 64, ncclUint8, c->comm, c->stream));
    std::vector<cudaIpcMemHandle_t> handles(static_cast<size_t>(c->world));
    BO_CUDA(cudaMemcpyAsync(handles.data(), dh + 64, handles.size() * 64, cudaMemcpyDeviceToHost,
                            c->stream));
    BO_CUDA(cudaStreamSynchronize(c->stream));
    out.assign(static_cast<size_t>(c->world), nullptr);
    for (int j = 0; j < c->world; ++j) {
      if (j == c->rank) {
        out[static_cast<size_t>(j)] = mine_ptr;
        continue;
      }
      void* p = nullptr;
      BO_CUDA(cudaIpcOpenMemHandle(&p, handles[static_cast<size_t>(j)], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(p);
      out[static_cast<size_t>(j)] = p;
    }
  };
  std::vector<void*> pw;
  map_all(c->w, pw);
  std::vector<float*> peers(pw.size());
  for (size_t j = 0; j < pw.size(); ++j) peers[j] = static_cast<float*>(pw[j]);
  if (ring) {
    for (int k = 0; k < 2; ++k) {
      std::vector<void*> pk;
      map_all(c->wire[k], pk);
      for (int j = 0; j < c->world; ++j) c->peer_wire[k][j] = pk[static_cast<size_t>(j)];
    }
  }
  c->d_peer_w = static_cast<float**>(dev_alloc(c, peers.size() * sizeof(float*)));
  BO_CUDA(cudaMemcpyAsync(c->d_peer_w, peers.data(), peers.size() * sizeof(float*),
                          cudaMemcpyHostToDevice, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  BO_GUARD_END
}

bo_status bo_set_stream(bo_ctx* c, void* s) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  BO_CUDA(cudaStreamSynchronize(c->stream));
  if (c->own_stream) BO_CUDA(cudaStreamDestroy(c->stream));
  if (s) {
    c->stream = static_cast<cudaStream_t>(s);
    c->own_stream = false;
  } else {
    BO_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  BO_GUARD_END
}

void* bo_get_stream(const bo_ctx* c) { return c ? c->stream : nullptr; }

bo_status bo_synchronize(bo_ctx* c) {
  BO_GUARD_BEGIN
  BO_CUDA(cudaStreamSynchronize(c->stream));
  BO_GUARD_END
}

bo_status bo_wait(bo_ctx* c, int64_t timeout_ms) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  BO_CUDA(cudaSetDevice(c->device));
  const auto t0 = std::chrono::steady_clock::now();
  const cudaStream_t streams[2] = {c->stream, c->comm_stream};
  for (;;) {
    bool pending = false;
    for (cudaStream_t s : streams) {
      if (!s) continue;
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaErrorNotReady) {
        pending = true;
      } else if (e != cudaSuccess) {
        fail(BO_ERR_CUDA, std::string("bo_wait: ") + cudaGetErrorString(e));
      }
    }
    if (!pending) break;
    if (c->comm) {
      ncclResult_t async = ncclSuccess;
      BO_NCCL(ncclCommGetAsyncError(c->comm, &async));
      if (async != ncclSuccess) {
        fail(BO_ERR_PEER_DISCONNECTED, std::string("rank ") + std::to_string(c->rank) +
                                           ": communicator failed: " + ncclGetErrorString(async));
      }
    }
    const auto waited = std::chrono::duration_cast<std::chrono::milliseconds>(
        std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms >= 0 && waited >= timeout_ms) {
      fail(BO_ERR_WATCHDOG_TIMEOUT, "rank " + std::to_string(c->rank) + ": step still pending after " +
                                        std::to_string(waited) + " ms");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  BO_GUARD_END
}

bo_status bo_load_params(bo_ctx* c, const float* src, int32_t on_host) {
  BO_GUARD_BEGIN
  const Layout& L = c->L;
  const cudaMemcpyKind k = on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  for (int t = 0; t < L.T; ++t) {
    BO_CUDA(cudaMemcpyAsync(c->w + L.flat_off[static_cast<size_t>(t)], src + L.model_off[static_cast<size_t>(t)],
                            static_cast<size_t>(L.numel[static_cast<size_t>(t)]) * 4, k, c->stream));
  }
  gather_shard(c);  // world > 1: the fp32 master shard of the owned chunks
  BO_CUDA(cudaStreamSynchronize(c->stream));
  BO_GUARD_END
}

bo_status bo_read_params(bo_ctx* c, float* dst, int32_t on_host) {
  BO_GUARD_BEGIN
  const Layout& L = c->L;
  const cudaMemcpyKind k = on_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  for (int t = 0; t < L.T; ++t) {
    BO_CUDA(cudaMemcpyAsync(dst + L.model_off[static_cast<size_t>(t)], c->w + L.flat_off[static_cast<size_t>(t)],
                            static_cast<size_t>(L.numel[static_cast<size_t>(t)]) * 4, k, c->stream));
  }
  BO_CUDA(cudaStreamSynchronize(c->stream));
  BO_GUARD_END
}

bo_status bo_read_moments(bo_ctx* c, float* m, float* v, int32_t on_host) {
  BO_GUARD_BEGIN
  const Layout& L = c->L;
  const cudaMemcpyKind k = on_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  DevState st;
  BO_CUDA(cudaMemcpyAsync(&st, c->state, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  const float* mc = st.parity ? c->m_alt : c->m;
  const float* vc = st.parity ? c->v_alt : c->v;
  const int q = L.own;
  for (int b = 0; b < L.B; ++b) {
    const int64_t cb = L.chunk[static_cast<size_t>(b)];
    const int64_t lo = q * cb, hi = std::min<int64_t>((q + 1) * cb, L.elems[static_cast<size_t>(b)]);
    for (int p : L.buckets[static_cast<size_t>(b)]) {
      const int64_t t0 = L.offset_of[static_cast<size_t>(p)], t1 = t0 + L.numel[static_cast<size_t>(p)];
      const int64_t a = std::max(lo, t0), z = std::min(hi, t1);
      if (a >= z) continue;
      const int64_t s = L.shard_pos(b, p, a);
      const int64_t dsti = L.model_off[static_cast<size_t>(p)] + (a - t0);
      BO_CUDA(cudaMemcpyAsync(m + dsti, mc + s, static_cast<size_t>(z - a) * 4, k, c->stream));
      BO_CUDA(cudaMemcpyAsync(v + dsti, vc + s, static_cast<size_t>(z - a) * 4, k, c->stream));
    }
  }
  BO_CUDA(cudaStreamSynchronize(c->stream));
  BO_GUARD_END
}

bo_status bo_export_state(bo_ctx* c, void* blob, uint64_t* nbytes) {
  BO_GUARD_BEGIN
  if (!c || !nbytes) fail(BO_ERR_INVALID_CONFIG, "null argument");
  const uint64_t need = sizeof(StateHeader) + 3ull * static_cast<uint64_t>(c->L.P) * 4;
  if (!blob) {
    *nbytes = need;
    return BO_OK;
  }
  if (*nbytes < need) fail(BO_ERR_LENGTH_MISMATCH, "state blob too small");
  StateHeader h{};
  std::memcpy(h.magic, "BOST", 4);
  h.version = 1;
  h.world = c->world;
  h.rank = c->rank;
  h.own = c->L.own;
  h.T = c->L.T;
  h.P = c->L.P;
  h.layout_hash = c->L.hash;
  BO_CUDA(cudaMemcpyAsync(&h.st, c->state, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  auto* base = static_cast<uint8_t*>(blob);
  std::memcpy(base, &h, sizeof(h));
  float* w = reinterpret_cast<float*>(base + sizeof(h));
  float* m = w + c->L.P;
  float* v = m + c->L.P;
  std::memset(m, 0, static_cast<size_t>(c->L.P) * 8);
  bo_status s = bo_read_params(c, w, 1);
  if (s != BO_OK) return s;
  s = bo_read_moments(c, m, v, 1);
  if (s != BO_OK) return s;
  *nbytes = need;
  BO_GUARD_END
}

bo_status bo_import_state(bo_ctx* c, const void* blob, uint64_t nbytes) {
  BO_GUARD_BEGIN
  if (!c || !blob) fail(BO_ERR_INVALID_CONFIG, "null argument");
  StateHeader h;
  if (nbytes < sizeof(h)) fail(BO_ERR_LENGTH_MISMATCH, "state blob truncated");
  std::memcpy(&h, blob, sizeof(h));
  if (std::memcmp(h.magic, "BOST", 4) != 0 || h.version != 1) {
    fail(BO_ERR_INVALID_CONFIG, "not a bertopt_b200 state blob");
  }
  if (nbytes < sizeof(h) + 3ull * static_cast<uint64_t>(h.P) * 4) {
    fail(BO_ERR_LENGTH_MISMATCH, "state blob truncated");
  }
  if (h.world != c->world || h.rank != c->rank || h.own != c->L.own || h.T != c->L.T ||
      h.P != c->L.P || h.layout_hash != c->L.hash) {
    fail(BO_ERR_BUCKET_LAYOUT_MISMATCH, "state blob was written by a different layout or rank");
  }
  const auto* base = static_cast<const uint8_t*>(blob);
  const float* w = reinterpret_cast<const float*>(base + sizeof(h));
  const float* m = w + h.P;
  const float* v = m + h.P;
  bo_status s = bo_load_params(c, w, 1);
  if (s != BO_OK) return s;
  for_owned(c->L, [&](int64_t sp, int64_t mp, int64_t n) {
    BO_CUDA(cudaMemcpyAsync(c->m + sp, m + mp, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, c->stream));
    BO_CUDA(cudaMemcpyAsync(c->v + sp, v + mp, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, c->stream));
  });
  DevState st = h.st;
  st.parity = 0;  // moments were written into buffer set 0
  st.local_flag = 0;
  BO_CUDA(cudaMemcpyAsync(c->state, &st, sizeof(st), cudaMemcpyHostToDevice, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  grow_bc_table(c, st.lamb_step + 2);
  c->calls = std::max<int64_t>(c->calls, st.steps);
  c->next_micro = 0;
  BO_GUARD_END
}

bo_status bo_get_status(bo_ctx* c, bo_step_status* out) {
  BO_GUARD_BEGIN
  DevState st;
  BO_CUDA(cudaMemcpyAsync(&st, c->state, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  out->loss_scale = st.scale;
  out->good_steps = st.good;
  out->lamb_step = st.lamb_step;
  out->steps = st.steps;
  out->skipped_steps = st.skipped;
  out->found_inf = st.found_inf;
  out->reserved = 0;
  BO_GUARD_END
}

bo_status bo_param_ptr(bo_ctx* c, int32_t t, float** out) {
  BO_GUARD_BEGIN
  if (t < 0 || t >= c->L.T) fail(BO_ERR_SHAPE_MISMATCH, "tensor index out of range");
  *out = c->w + c->L.flat_off[static_cast<size_t>(t)];
  BO_GUARD_END
}

bo_status bo_profile_enable(bo_ctx* c, int32_t enable) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  c->profiling = enable != 0;
  // BO_PROFILE_STAGES: bit mask of the stages to bracket (default all); timing
  // one stage alone shows what the events between all stages cost
  c->profile_mask = ~0u;
  if (const char* e = std::getenv("BO_PROFILE_STAGES")) c->profile_mask = static_cast<unsigned>(std::strtoul(e, nullptr, 0));
  BO_GUARD_END
}

bo_status bo_profile_read(bo_ctx* c, double* stage_ms, int64_t* stage_count, int32_t reset) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  drain_marks(c);
  for (int s = 0; s < BO_NUM_STAGES; ++s) {
    if (stage_ms) stage_ms[s] = c->stage_ms[s];
    if (stage_count) stage_count[s] = c->stage_count[s];
    if (reset) {
      c->stage_ms[s] = 0.0;
      c->stage_count[s] = 0;
    }
  }
  BO_GUARD_END
}

int64_t bo_launch_count(const bo_ctx* c) { return c ? c->launches : 0; }

int32_t bo_path_flags(const bo_ctx* c) { return c ? c->path : 0; }

bo_status bo_accumulate(bo_ctx* c, int32_t micro, const uint16_t* const* grads) {
  BO_GUARD_BEGIN
  if (!c || !grads) fail(BO_ERR_INVALID_CONFIG, "null argument");
  const int K = c->cfg.accumulation;
  if (micro < 0 || micro >= K) fail(BO_ERR_INVALID_CONFIG, "micro index outside [0, K)");
  if (c->world > 1 && !c->comm) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init has not run");
  PtrTable tab;
  bool aligned = true;
  for (int t = 0; t < c->L.T; ++t) {
    tab.p[t] = grads[t];
    if (!grads[t]) fail(BO_ERR_SHAPE_MISMATCH, "null gradient for tensor " + std::to_string(t));
    aligned &= (reinterpret_cast<uintptr_t>(grads[t]) & 15u) == 0;
  }
  if (c->sync_open) fail(BO_ERR_PROTOCOL, "an overlapped sync micro (bo_sync_ready) is in progress");
  if (micro != c->next_micro) {
    fail(BO_ERR_PROTOCOL, "micro " + std::to_string(micro) + " out of order (expected " +
                              std::to_string(c->next_micro) + ")");
  }
  if (micro + 1 < K) {
    launch_accumulate(c, micro, tab, aligned);
    c->next_micro = micro + 1;
    return BO_OK;
  }
  c->next_micro = 0;
  grow_bc_table(c, c->calls + 2);
  c->path = 0;
  if (c->world == 1 && aligned && !c->force_unfused) {
    c->path = BO_PATH_ONE_RANK_FUSED;
    run_fused_single_rank(c, tab);
  } else {
    if (c->world == 1) c->path = BO_PATH_ONE_RANK_STAGED;
    // the ring fuses flatten_param into its hops; NCCL needs the fusion buffer
    if (c->world == 1 || c->algo == BO_REDUCE_NCCL) launch_finalize(c, tab);
    run_reduce(c, tab);
    run_lamb(c, tab);  // world > 1: includes the fused parameter all-gather (IPC push)
  }
  c->calls += 1;
  BO_GUARD_END
}

bo_status bo_train_step(bo_ctx* c, const uint16_t* const* grads) {
  BO_GUARD_BEGIN
  if (!c || !grads) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (c->world > 1 && !c->comm) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init has not run");
  if (c->sync_open) fail(BO_ERR_PROTOCOL, "an overlapped sync micro (bo_sync_ready) is in progress");
  if (c->next_micro != 0) fail(BO_ERR_PROTOCOL, "bo_train_step inside a step fed by bo_accumulate");
  const int K = c->cfg.accumulation, T = c->L.T;
  bool aligned = true;
  for (int i = 0; i < K * T; ++i) {
    if (!grads[i]) fail(BO_ERR_SHAPE_MISMATCH, "null gradient for micro " + std::to_string(i / T) +
                                                   ", tensor " + std::to_string(i % T));
    aligned &= (reinterpret_cast<uintptr_t>(grads[i]) & 15u) == 0;
  }
  // The resident-micro kernels read all K gradient sets in the sync pass
  // (no accumulator round trips): one rank's fused path and the ring. Other
  // configurations (NCCL wire, unaligned slots, K == 1, K > 8) take the
  // per-micro path; the results are identical either way.
  const bool resident = K > 1 && K <= kMaxResident && aligned &&
                        (c->world == 1 ? !c->force_unfused : c->algo == BO_REDUCE_RING);
  if (!resident) {
    for (int k = 0; k < K; ++k) {
      const bo_status st = bo_accumulate(c, k, grads + static_cast<size_t>(k) * T);
      if (st != BO_OK) return st;
    }
    return BO_OK;
  }
  if (c->micro_tab_cap < K * T) {
    c->d_micro_tab = static_cast<const uint16_t**>(dev_alloc(c, static_cast<size_t>(K) * T * sizeof(void*)));
    c->micro_tab_cap = K * T;
  }
  // pageable source: staged by the driver before the call returns; ordered
  // on the stream after the previous step's kernels that read the table
  BO_CUDA(cudaMemcpyAsync(c->d_micro_tab, grads, static_cast<size_t>(K) * T * sizeof(void*),
                          cudaMemcpyHostToDevice, c->stream));
  PtrTable tab;
  for (int t = 0; t < T; ++t) tab.p[t] = grads[static_cast<size_t>(K - 1) * T + t];  // the live micro
  grow_bc_table(c, c->calls + 2);
  c->ms = MicroSrc{c->d_micro_tab, K, T};
  c->path = BO_PATH_RESIDENT;
  try {
    if (c->world == 1) {
      c->path |= BO_PATH_ONE_RANK_FUSED;
      run_fused_single_rank(c, tab, c->ms);
    } else {
      run_reduce(c, tab);
      run_lamb(c, tab);
    }
  } catch (...) {
    c->ms = MicroSrc{nullptr, 0, 0};
    throw;
  }
  c->ms = MicroSrc{nullptr, 0, 0};
  c->calls += 1;
  BO_GUARD_END
}

bo_status bo_sync_ready(bo_ctx* c, int32_t n, const int32_t* tensors, const uint16_t* const* grads) {
  BO_GUARD_BEGIN
  if (!c || (n > 0 && (!tensors || !grads))) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (c->world > 1 && !c->comm) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init has not run");
  const Layout& L = c->L;
  if (!c->sync_open) {
    if (c->next_micro != c->cfg.accumulation - 1) {
      fail(BO_ERR_PROTOCOL, "bo_sync_ready before micros 0.." + std::to_string(c->cfg.accumulation - 2) +
                                " went through bo_accumulate");
    }
    c->sync_open = true;
    c->n_delivered = 0;
    c->next_group = 0;
    c->sync_aligned = true;
    std::fill(c->delivered.begin(), c->delivered.end(), 0);
    c->group_pending.clear();
    for (const auto& g : c->comm_groups) c->group_pending.push_back(g.pending0);
    c->path = BO_PATH_OVERLAP;
    c->ring_last_in = nullptr;
    c->ring_result = nullptr;
  }
  for (int i = 0; i < n; ++i) {
    const int t = tensors[i];
    if (t < 0 || t >= L.T) fail(BO_ERR_SHAPE_MISMATCH, "tensor index out of range");
    if (!grads[i]) fail(BO_ERR_SHAPE_MISMATCH, "null gradient for tensor " + std::to_string(t));
    if (c->delivered[static_cast<size_t>(t)]) {
      fail(BO_ERR_PROTOCOL, "tensor " + std::to_string(t) + " delivered twice in one sync micro");
    }
    c->delivered[static_cast<size_t>(t)] = 1;
    c->sync_tab->p[t] = grads[i];
    c->sync_aligned &= (reinterpret_cast<uintptr_t>(grads[i]) & 15u) == 0;
    c->n_delivered += 1;
    if (c->world > 1) {
      c->group_pending[static_cast<size_t>(c->group_of_bucket[static_cast<size_t>(L.bucket_of[static_cast<size_t>(t)])])] -= 1;
    }
  }
  // reduce every group whose tensors are all final, in layout order (the
  // reference's comm thread, trainer.cpp:301-327), on the communication
  // stream after the caller's work so far (the gradients' producer)
  if (c->world > 1) {
    const int G = static_cast<int>(c->comm_groups.size());
    if (c->next_group < G && c->group_pending[static_cast<size_t>(c->next_group)] == 0) {
      BO_CUDA(cudaEventRecord(c->comm_ready, c->stream));
      BO_CUDA(cudaStreamWaitEvent(c->comm_stream, c->comm_ready, 0));
    }
    while (c->next_group < G && c->group_pending[static_cast<size_t>(c->next_group)] == 0) {
      const auto& g = c->comm_groups[static_cast<size_t>(c->next_group)];
      run_reduce_group(c, *c->sync_tab, g.b0, g.b1, g.acc0, g.acc1, c->comm_stream);
      c->next_group += 1;
    }
  }
  if (c->n_delivered < L.T) return BO_OK;
  // every gradient delivered: the rest of the step on the caller's stream
  c->sync_open = false;
  c->next_micro = 0;
  grow_bc_table(c, c->calls + 2);
  if (c->world == 1) {
    if (c->sync_aligned && !c->force_unfused) {
      c->path |= BO_PATH_ONE_RANK_FUSED;
      run_fused_single_rank(c, *c->sync_tab);
    } else {
      c->path |= BO_PATH_ONE_RANK_STAGED;
      launch_finalize(c, *c->sync_tab);
      run_reduce(c, *c->sync_tab);
      run_lamb(c, *c->sync_tab);
    }
  } else {
    BO_CUDA(cudaEventRecord(c->comm_done, c->comm_stream));
    BO_CUDA(cudaStreamWaitEvent(c->stream, c->comm_done, 0));
    run_lamb(c, *c->sync_tab);
  }
  c->calls += 1;
  BO_GUARD_END
}

}  // extern "C"
