// C ABI of the pipeline context: creation, layout, communication, state,
// profiling (see include/bertopt_b200.h); the hot-path entry points are in
// bo_step.cu, the work tables in bo_tables.cu.
#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

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

static const char* const kStageNames[BO_NUM_STAGES] = {"accumulate", "finalize", "reduce", "lamb_norms",
                                                       "trust", "lamb_update", "allgather", "hop_kernels",
                                                       "reserved"};

StageTimer::StageTimer(bo_ctx* ctx, int s) : StageTimer(ctx, s, ctx->stream) {}

StageTimer::StageTimer(bo_ctx* ctx, int s, cudaStream_t on) : c(ctx), stage(s), stream(on) {
  if (c->tracing) nvtxRangePushA(kStageNames[s]);  // host-side issue range for a timeline profiler
  if (!c->profiling || !((c->profile_mask >> s) & 1)) return;
  b = take_event(c);
  BO_CUDA(cudaEventRecord(b, stream));
}

StageTimer::~StageTimer() {
  if (c->tracing) nvtxRangePop();
  if (!c->profiling || !b) return;
  cudaEvent_t e = take_event(c);
  if (cudaEventRecord(e, stream) == cudaSuccess) c->marks.push_back({stage, b, e});
}

void trace(bo_ctx* c, const char* event, uint64_t bytes, cudaStream_t s) {
  if (!c->tracing) return;
  cudaEvent_t e = take_event(c);
  BO_CUDA(cudaEventRecord(e, s));
  c->trace_marks.push_back(bo_ctx::TraceMark{event, bytes, e});
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

// One rank's communication record (bo_comm_export): the salted layout hash,
// a hash of the settings that shape the cross-rank call sequence, and CUDA IPC
// handles of the buffers peers access (parameter replica, ring staging,
// flag block, norm partials).
struct CommRecord {
  char magic[8];
  int32_t rank, world, ring, reserved;
  uint64_t layout_hash, settings;
  cudaIpcMemHandle_t w, wire0, wire1, ctrl, part;
};

static uint64_t settings_hash(const bo_ctx* c) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) h = (h ^ ((v >> (8 * i)) & 0xFF)) * 1099511628211ull;
  };
  mix(static_cast<uint64_t>(c->algo));
  mix(c->ring_via_nccl ? 1 : 0);
  mix(c->ring_push ? 1 : 0);
  mix(c->nb_barrier ? 1 : 0);
  mix(c->comm_groups.size());
  for (const auto& g : c->comm_groups) mix(static_cast<uint64_t>(g.b1));
  mix(static_cast<uint64_t>(c->n_push_groups));  // bo_params_wait slots
  mix(c->lamb_groups.size());  // grouped LAMB: one partials barrier per group
  for (const auto& g : c->lamb_groups) mix(static_cast<uint64_t>(g.t1));
  return h;
}

static CommRecord make_record(bo_ctx* c) {
  if (c->world == 1) fail(BO_ERR_INVALID_CONFIG, "world 1 has no peers");
  BO_CUDA(cudaSetDevice(c->device));
  CommRecord r{};
  std::memcpy(r.magic, "BOCOMM1", 8);
  r.rank = c->rank;
  r.world = c->world;
  r.ring = c->algo == BO_REDUCE_RING;
  r.layout_hash = c->L.hash;
  r.settings = settings_hash(c);
  BO_CUDA(cudaIpcGetMemHandle(&r.w, c->w));
  if (r.ring) {
    BO_CUDA(cudaIpcGetMemHandle(&r.wire0, c->wire[0]));
    BO_CUDA(cudaIpcGetMemHandle(&r.wire1, c->wire[1]));
  }
  BO_CUDA(cudaIpcGetMemHandle(&r.ctrl, c->ctrl));
  BO_CUDA(cudaIpcGetMemHandle(&r.part, c->all_part));
  return r;
}

// Layout agreement (trainer.cpp:169-183 — BucketLayoutMismatch), settings
// agreement (ProtocolError: ranks started with different BO_* environments
// would otherwise deadlock), then every peer buffer mapped into this process
// over NVLink/NVSwitch (CUDA IPC; ranks sharing one GPU map each other too).
static void import_records(bo_ctx* c, const CommRecord* all) {
  if (c->world == 1) return;
  if (c->peers_mapped) fail(BO_ERR_PROTOCOL, "peers are already mapped");
  BO_CUDA(cudaSetDevice(c->device));
  const uint64_t settings = settings_hash(c);
  for (int j = 0; j < c->world; ++j) {
    const CommRecord& r = all[j];
    if (std::memcmp(r.magic, "BOCOMM1", 8) != 0 || r.world != c->world || r.rank != j) {
      fail(BO_ERR_PROTOCOL, "communication record " + std::to_string(j) + " is not rank " +
                                std::to_string(j) + " of a world of " + std::to_string(c->world));
    }
    if (r.layout_hash != c->L.hash) {
      fail(BO_ERR_BUCKET_LAYOUT_MISMATCH,
           "rank " + std::to_string(c->rank) + " bucket layout disagrees with peers");
    }
    if (r.settings != settings) {
      fail(BO_ERR_PROTOCOL, "rank " + std::to_string(c->rank) +
                                " collective settings (reduce algorithm, BO_RING_NCCL, BO_RING_PUSH, "
                                "BO_RING_BARRIER, BO_COMM_GROUP_ELEMS) disagree with peers");
    }
  }
  const bool ring = c->algo == BO_REDUCE_RING;
  if (!c->comm && (c->algo == BO_REDUCE_NCCL || (ring && (c->ring_via_nccl || !c->nb_barrier)))) {
    fail(BO_ERR_INVALID_CONFIG, "this configuration (NCCL reduce-scatter, BO_RING_NCCL=1 or "
                                "BO_RING_BARRIER=nccl) needs bo_comm_init");
  }
  auto open = [&](int j, const cudaIpcMemHandle_t& h, void* mine_ptr) -> void* {
    if (j == c->rank) return mine_ptr;
    void* p = nullptr;
    BO_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    return p;
  };
  std::vector<float*> peers(static_cast<size_t>(c->world));
  c->peer_ctrl = PeerFlags{{}, c->world, c->rank};
  for (int j = 0; j < c->world; ++j) {
    peers[static_cast<size_t>(j)] = static_cast<float*>(open(j, all[j].w, c->w));
    if (ring) {
      c->peer_wire[0][j] = open(j, all[j].wire0, c->wire[0]);
      c->peer_wire[1][j] = open(j, all[j].wire1, c->wire[1]);
    }
    c->peer_ctrl.f[j] = static_cast<unsigned*>(open(j, all[j].ctrl, c->ctrl));
    c->peer_part[j] = static_cast<double*>(open(j, all[j].part, c->all_part));
  }
  if (ring && c->nb_barrier) {
    // neighbour slots for the barrier between ring hops
    const int left = (c->rank - 1 + c->world) % c->world, right = (c->rank + 1) % c->world;
    c->nb_flags = c->ctrl + kCtrlFromLeft;
    c->nb_left_from_right = c->peer_ctrl.f[left] + kCtrlFromRight;
    c->nb_right_from_left = c->peer_ctrl.f[right] + kCtrlFromLeft;
  }
  c->d_peer_w = static_cast<float**>(dev_alloc(c, peers.size() * sizeof(float*)));
  BO_CUDA(cudaMemcpyAsync(c->d_peer_w, peers.data(), peers.size() * sizeof(float*),
                          cudaMemcpyHostToDevice, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  c->peers_mapped = true;
}

}  // namespace bo

using namespace bo;

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
    case BO_ERR_IO_FAILURE: return "IoFailure";
    case BO_ERR_CUDA: return "CudaError";
    case BO_ERR_NCCL: return "NcclError";
    case BO_ERR_NO_DEVICE: return "NoDevice";
    default: return "Unknown";
  }
}

const char* bo_last_error(void) { return g_last_error.c_str(); }

void bo_default_config(bo_trainer_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->lamb = bo_lamb_config{1e-3f, 0.9f, 0.999f, 1e-6f, 0.01f, 10.0f};  // lamb.hpp:30-37
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
    const int64_t c = (bucket_elems[b] + world - 1) / world;  // collective.cpp:27-29
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
  if (const char* e = std::getenv("BO_RING_PUSH")) c->ring_push = std::strcmp(e, "0") != 0;
  if (const char* e = std::getenv("BO_RING_BARRIER")) c->nb_barrier = std::strcmp(e, "nccl") != 0;
  if (const char* e = std::getenv("BO_FUSE_LAST")) c->fuse_last_hop = std::strcmp(e, "0") != 0;
  // AUTO: the device ring for both wires — bit-exact (the reference fold) and,
  // for fp32, faster than ncclReduceScatter at every bucket size measured
  // (BERT-large, 4 GPUs: 3.60 vs 4.33 ms per step at 4 MiB; profiles/r02_sweep_n4.json)
  c->algo = cfg->reduce_algo == BO_REDUCE_AUTO ? BO_REDUCE_RING : cfg->reduce_algo;
  BO_CUDA(cudaSetDevice(device));
  BO_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  c->p1r_prefetch = 4 * c->num_sms / 3;
  if (const char* e = std::getenv("BO_P1R_PREFETCH")) c->p1r_prefetch = std::max(0, std::atoi(e));
  c->push_posted_ctas = 128;  // measured best at 4 GPUs (80-128 on a plateau; profiles/r02_notes.md)
  if (const char* e = std::getenv("BO_PUSH_POSTED_CTAS")) c->push_posted_ctas = std::max(0, std::atoi(e));
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
    if (c->lamb_groups.size() > 1) c->wsh_alt = static_cast<float*>(dev_alloc(c, static_cast<size_t>(L.shard_total) * 4));
    c->d_barrier = static_cast<int*>(dev_alloc(c, 4));
    c->ctrl = static_cast<unsigned*>(dev_alloc(c, kCtrlWords * sizeof(unsigned)));
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
                           : static_cast<double*>(dev_alloc(c, 2 * static_cast<size_t>(world) * (2 * L.T + 1) * 8));
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
  for (const auto& m : c->trace_marks) cudaEventDestroy(m.e);
  if (c->trace_base) cudaEventDestroy(c->trace_base);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->comm_ready) cudaEventDestroy(c->comm_ready);
  if (c->comm_done) cudaEventDestroy(c->comm_done);
  if (c->params_done) cudaEventDestroy(c->params_done);
  if (c->comm_stream && !c->shared_stream) cudaStreamDestroy(c->comm_stream);
  if (c->push_stream) {
    cudaStreamSynchronize(c->push_stream);
    cudaStreamDestroy(c->push_stream);
  }
  for (cudaEvent_t e : c->group_events) cudaEventDestroy(e);
  delete c->sync_tab;
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->comm) ncclCommDestroy(c->comm);
  for (void* p : c->allocations) cudaFree(p);
  if (c->op_ws) cudaFree(c->op_ws);
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

bo_status bo_comm_export(bo_ctx* c, void* rec, uint64_t* nbytes) {
  BO_GUARD_BEGIN
  if (!c || !nbytes) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (!rec) {
    *nbytes = sizeof(CommRecord);
    return BO_OK;
  }
  if (*nbytes < sizeof(CommRecord)) fail(BO_ERR_LENGTH_MISMATCH, "communication record buffer too small");
  const CommRecord r = make_record(c);
  std::memcpy(rec, &r, sizeof(r));
  *nbytes = sizeof(CommRecord);
  BO_GUARD_END
}

bo_status bo_comm_import(bo_ctx* c, const void* recs, uint64_t nbytes_each) {
  BO_GUARD_BEGIN
  if (!c || !recs) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (nbytes_each != sizeof(CommRecord)) fail(BO_ERR_LENGTH_MISMATCH, "communication record size");
  import_records(c, static_cast<const CommRecord*>(recs));
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
  // the same records bo_comm_export / bo_comm_import exchange through the
  // host, all-gathered over the new communicator
  const CommRecord mine = make_record(c);
  uint8_t* d = static_cast<uint8_t*>(dev_alloc(c, (static_cast<size_t>(c->world) + 1) * sizeof(CommRecord)));
  BO_CUDA(cudaMemcpyAsync(d, &mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
  BO_NCCL(ncclAllGather(d, d + sizeof(CommRecord), sizeof(CommRecord), ncclUint8, c->comm, c->stream));
  std::vector<CommRecord> all(static_cast<size_t>(c->world));
  BO_CUDA(cudaMemcpyAsync(all.data(), d + sizeof(CommRecord), all.size() * sizeof(CommRecord),
                          cudaMemcpyDeviceToHost, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  import_records(c, all.data());
  BO_GUARD_END
}

bo_status bo_world_init_local(bo_ctx* const* ctxs, int32_t n) {
  BO_GUARD_BEGIN
  if (!ctxs || n < 2) fail(BO_ERR_INVALID_CONFIG, "a local world needs >= 2 contexts");
  for (int i = 0; i < n; ++i) {
    bo_ctx* c = ctxs[i];
    if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
    if (c->world != n || c->rank != i) {
      fail(BO_ERR_PROTOCOL, "context " + std::to_string(i) + " is not rank " + std::to_string(i) +
                                " of a world of " + std::to_string(n));
    }
    if (c->peers_mapped) fail(BO_ERR_PROTOCOL, "peers are already mapped");
    if (c->device != ctxs[0]->device) fail(BO_ERR_INVALID_CONFIG, "a lockstep world shares one device");
    if (c->L.hash != ctxs[0]->L.hash) {
      fail(BO_ERR_BUCKET_LAYOUT_MISMATCH, "rank " + std::to_string(i) + " bucket layout disagrees with peers");
    }
    if (settings_hash(c) != settings_hash(ctxs[0])) {
      fail(BO_ERR_PROTOCOL, "rank " + std::to_string(i) + " collective settings disagree with peers");
    }
    const bool ring = c->algo == BO_REDUCE_RING;
    if (!ring || c->ring_via_nccl || !c->nb_barrier) {
      fail(BO_ERR_INVALID_CONFIG, "a lockstep world runs the ring reduction without NCCL");
    }
  }
  BO_CUDA(cudaSetDevice(ctxs[0]->device));
  auto shared = std::make_shared<SharedStream>();
  BO_CUDA(cudaStreamCreateWithFlags(&shared->s, cudaStreamNonBlocking));
  auto bar = std::make_shared<HostBarrier>();
  bar->n = n;
  for (int i = 0; i < n; ++i) {
    bo_ctx* c = ctxs[i];
    BO_CUDA(cudaStreamSynchronize(c->stream));
    if (c->own_stream) BO_CUDA(cudaStreamDestroy(c->stream));
    if (c->comm_stream) {
      BO_CUDA(cudaStreamSynchronize(c->comm_stream));
      BO_CUDA(cudaStreamDestroy(c->comm_stream));
    }
    c->stream = shared->s;
    c->comm_stream = shared->s;  // the overlapped sync micro's hops join the one stream too
    c->own_stream = false;
    c->shared_stream = shared;
    c->lockstep = bar;
    // peers are plain pointers in this process (no IPC)
    std::vector<float*> peers(static_cast<size_t>(n));
    c->peer_ctrl = PeerFlags{{}, n, i};
    for (int j = 0; j < n; ++j) {
      peers[static_cast<size_t>(j)] = ctxs[j]->w;
      c->peer_wire[0][j] = ctxs[j]->wire[0];
      c->peer_wire[1][j] = ctxs[j]->wire[1];
      c->peer_ctrl.f[j] = ctxs[j]->ctrl;
      c->peer_part[j] = ctxs[j]->all_part;
    }
    const int left = (i - 1 + n) % n, right = (i + 1) % n;
    c->nb_flags = c->ctrl + kCtrlFromLeft;  // (the rendezvous replaces the flag waits)
    c->nb_left_from_right = ctxs[left]->ctrl + kCtrlFromRight;
    c->nb_right_from_left = ctxs[right]->ctrl + kCtrlFromLeft;
    c->d_peer_w = static_cast<float**>(dev_alloc(c, peers.size() * sizeof(float*)));
    BO_CUDA(cudaMemcpyAsync(c->d_peer_w, peers.data(), peers.size() * sizeof(float*),
                            cudaMemcpyHostToDevice, c->stream));
    c->peers_mapped = true;
  }
  BO_CUDA(cudaStreamSynchronize(shared->s));
  BO_GUARD_END
}

bo_status bo_set_watchdog(bo_ctx* c, double seconds) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  if (!(seconds > 0.0) || seconds > 1e7) fail(BO_ERR_INVALID_CONFIG, "watchdog must be in (0, 1e7] seconds");
  c->watchdog_ns = static_cast<uint64_t>(seconds * 1e9);
  BO_GUARD_END
}

bo_status bo_set_stream(bo_ctx* c, void* s) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  if (c->lockstep) fail(BO_ERR_PROTOCOL, "the ranks of a lockstep world share one stream");
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
  if (c->peers_mapped) {
    // a cross-rank barrier gave up waiting: the step was abandoned (no
    // update, scaler untouched); reported once, then cleared
    int32_t timed_out = 0;
    BO_CUDA(cudaMemcpy(&timed_out, &c->state->peer_timeout, sizeof(timed_out), cudaMemcpyDeviceToHost));
    if (timed_out) {
      const int32_t zero = 0;
      BO_CUDA(cudaMemcpy(&c->state->peer_timeout, &zero, sizeof(zero), cudaMemcpyHostToDevice));
      fail(BO_ERR_PEER_DISCONNECTED, "rank " + std::to_string(c->rank) +
                                         ": a peer did not reach a step barrier within the watchdog");
    }
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
  st.peer_timeout = 0;  // a reported (or stale) barrier timeout is not state
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

bo_status bo_trace_enable(bo_ctx* c, int32_t enable) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  BO_CUDA(cudaStreamSynchronize(c->stream));
  for (const auto& m : c->trace_marks) c->event_pool.push_back(m.e);
  c->trace_marks.clear();
  c->tracing = enable != 0;
  if (c->tracing) {
    if (!c->trace_base) BO_CUDA(cudaEventCreate(&c->trace_base));
    BO_CUDA(cudaEventRecord(c->trace_base, c->stream));
  }
  BO_GUARD_END
}

bo_status bo_trace_write(bo_ctx* c, const char* path) {
  BO_GUARD_BEGIN
  if (!c || !path) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (!c->trace_base) fail(BO_ERR_PROTOCOL, "bo_trace_enable has not run");
  BO_CUDA(cudaDeviceSynchronize());
  struct Line {
    double ts;
    const char* ev;
    uint64_t bytes;
  };
  std::vector<Line> lines;
  for (const auto& m : c->trace_marks) {
    float ms = 0.0f;
    BO_CUDA(cudaEventElapsedTime(&ms, c->trace_base, m.e));
    lines.push_back(Line{ms * 1e-3, m.event, m.bytes});
  }
  std::stable_sort(lines.begin(), lines.end(), [](const Line& a, const Line& b) { return a.ts < b.ts; });
  FILE* f = std::fopen(path, "w");
  if (!f) fail(BO_ERR_IO_FAILURE, std::string("cannot open ") + path);
  bool ok = true;
  for (const Line& l : lines) {
    // the reference's line format (trainer.cpp:58-71)
    ok &= std::fprintf(f, "{\"ts\":%.9f,\"rank\":%d,\"event\":\"%s\",\"bytes\":%llu}\n", l.ts, c->rank,
                       l.ev, static_cast<unsigned long long>(l.bytes)) > 0;
  }
  ok &= std::fclose(f) == 0;
  if (!ok) fail(BO_ERR_IO_FAILURE, std::string("write failed for ") + path);
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

}  // extern "C"
