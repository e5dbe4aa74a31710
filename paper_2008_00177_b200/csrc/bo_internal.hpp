// Internal declarations of the B200 gradient-to-update pipeline.
#ifndef BO_INTERNAL_HPP_
#define BO_INTERNAL_HPP_

#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "bertopt_b200.h"

namespace bo {

constexpr int kMaxTensors = 1024;     // per-micro pointer table travels as a kernel parameter
constexpr int kTileElems = 4096;      // elements per CTA work tile
constexpr int kAlignElems = 64;       // 256-byte alignment of every buffer region
constexpr int kThreads = 256;
constexpr int kMaxResident = 8;       // micro-batches bo_train_step reads in one pass

// Thrown inside the library, turned into a bo_status at the C boundary.
struct Failure {
  bo_status code;
  std::string msg;
};

[[noreturn]] void fail(bo_status code, const std::string& msg);
void set_thread_error(const std::string& msg);

#define BO_CUDA(expr)                                                          \
  do {                                                                         \
    cudaError_t e_ = (expr);                                                   \
    if (e_ != cudaSuccess)                                                     \
      ::bo::fail(BO_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define BO_NCCL(expr)                                                          \
  do {                                                                         \
    ncclResult_t r_ = (expr);                                                  \
    if (r_ != ncclSuccess)                                                     \
      ::bo::fail(BO_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- layout
// Fusion-buffer layout (restates BucketLayout::build, trainer.cpp:73-116)
// plus the HBM placement of every device buffer:
//   flat  : bucket b at base[b], N*chunk[b] elements (reference zero padding,
//           collective.hpp:58-60); tensor p at base[bucket_of[p]] + offset_of[p]
//   shard : rank r owns chunk r of every bucket, concatenated at shoff[b]
//   acc   : per-tensor fp32 accumulators at acc_off[p] (model order)
struct Layout {
  int T = 0, B = 0, N = 1, rank = 0;
  // Chunk index this rank owns in every bucket: r for the NCCL reduce-scatter,
  // (r+1) % N for the reference ring, whose fold for chunk k ends on rank k-1
  // (collective.hpp:65-80); the parameter push places it, so no hand-off hop.
  int own = 0;
  std::vector<int64_t> numel;
  std::vector<int> bucket_of, ready;
  std::vector<int64_t> offset_of;
  std::vector<std::vector<int>> buckets;
  std::vector<int64_t> elems, chunk, base, shoff;
  std::vector<int64_t> flat_off, acc_off, model_off;
  int64_t flat_total = 0, shard_total = 0, acc_total = 0, P = 0;
  uint64_t hash = 0;

  static Layout build(int T, const int64_t* numel, const int32_t* firsts, uint64_t bucket_bytes,
                      int world, int rank);

  // Positions of bucket-local element a of tensor p (bucket b) in the flat
  // (parameter / fusion) buffer and in this rank's shard (m, v, reduced g).
  int64_t flat_pos(int b, int p, int64_t a) const {
    return N == 1 ? flat_off[static_cast<size_t>(p)] + (a - offset_of[static_cast<size_t>(p)])
                  : base[static_cast<size_t>(b)] + a;
  }
  int64_t shard_pos(int b, int p, int64_t a) const {
    return N == 1 ? flat_pos(b, p, a)
                  : shoff[static_cast<size_t>(b)] + (a - own * chunk[static_cast<size_t>(b)]);
  }
};

// Work tiles (device tables, built once per context).
struct AccTile {        // a slice of one tensor, model order
  int32_t t;
  int32_t len;
  int64_t e0;           // element offset inside the tensor
};
struct LambTile {       // a slice of one tensor inside this rank's shard
  int64_t s0;           // shard index of the first element
  int64_t w0;           // flat index of the first element
  int32_t len;
  int32_t t;
};
// Ring hop with the finalize fused in: a slice of one tensor inside chunk q of
// one bucket. x = (h + acc) * inv is computed on the fly from the caller's
// binary16 gradient and the accumulator instead of a materialised fusion
// buffer (each element of x is needed by exactly one hop).
struct HopXTile {
  int64_t s0;           // shard (wire staging) index of the first element
  int64_t e0;           // element offset inside tensor t
  int32_t len;
  int32_t t;
};

// Single-rank LAMB (bo_fused.cu): a slice of one tensor; every per-tensor
// array uses the aligned tensor layout, so one index a0 serves acc, w, m, v
// and the update scratch u; e0 indexes the caller's gradient tensor.
struct FusedTile {
  int64_t a0;
  int64_t e0;
  int32_t len;
  int32_t t;
};

// Per-tensor constants used by the accumulate / finalize kernels.
struct TensorDev {
  int64_t acc_off;
  int64_t flat_off;
};

// Device-resident optimizer / scaler state (one per rank, replicated values).
struct DevState {
  float scale;
  int32_t good;
  int64_t lamb_step;
  int64_t steps;
  int64_t skipped;
  int32_t found_inf;
  int32_t do_update;
  int32_t local_flag;   // set by LAMB phase 1 on this rank
  int32_t parity;       // which moment buffer set is current (one rank: double-buffered)
  int32_t peer_timeout; // a cross-rank flag barrier gave up waiting (peer gone or
                        // stalled past the watchdog): the step is abandoned
                        // without touching w/m/v or the scaler; bo_wait reports it
  uint32_t epoch;       // the step's barrier epoch (k_trust), for graph-launched publishers
  double bc1, bc2, ibc1, ibc2;   // bias corrections of the current LAMB step
};

struct LambConsts {
  float beta1, beta2, omb1, omb2, eps, wd, lr, clip;
};

struct ScalerConsts {
  float growth, backoff, min_scale, max_scale;
  int32_t interval, dynamic;
};

// Cross-rank flag block of every rank (one cudaMalloc, mapped into every peer
// with CUDA IPC). Slots are 32-bit epochs, written by the rank named in the
// slot with st.release.sys and read by the owner with ld.acquire.sys.
constexpr int kCtrlFromLeft = 0;     // ring-neighbour barrier: epoch of the left neighbour
constexpr int kCtrlFromRight = 1;    //                          epoch of the right neighbour
constexpr int kCtrlPartials = 16;    // [8] partials barrier: rank j's norm partials are in
constexpr int kCtrlStepEnd = 32;     // [8] end-of-step barrier: rank j's parameter push landed
constexpr int kCtrlReady = 64;       // [kMaxPushGroups][8] rank j's push of parameter group g landed
constexpr int kMaxPushGroups = 112;
constexpr int kCtrlWords = kCtrlReady + 8 * kMaxPushGroups;

// Per-step destinations of this rank's norm partials: slot `rank` of every
// rank's all_part (this step's parity half). N == 0: local rank_part only.
struct PartDst {
  double* p[8];
  int n;
};
// Every rank's flag block (device pointers valid in this process).
struct PeerFlags {
  unsigned* f[8];
  int n, rank;
};

struct PtrTable {
  const uint16_t* p[kMaxTensors];
};

// Lockstep world (bo_world_init_local): all ranks of a world live in one
// process and share ONE stream; every cross-rank wait of the step (ring hop
// barriers, the partials barrier, the end-of-step barrier) becomes a
// rendezvous of the ranks' host threads between kernel launches, so the
// stream holds every rank's phase-i kernels before any rank's phase-i+1
// kernel — the device never has a kernel waiting for another one. Used to
// run a world larger than the box (world 8 on one B200) bit for bit.
struct HostBarrier {
  std::mutex m;
  std::condition_variable cv;
  int n = 0, count = 0;
  uint64_t gen = 0;
  bool wait(uint64_t timeout_ns);
};
struct SharedStream {
  cudaStream_t s = nullptr;
  ~SharedStream();
};

// All K micro-batches of a step resident (bo_train_step): micro k's gradient
// of tensor t is hk[k * T + t] (a device array). K == 0: not in use.
struct MicroSrc {
  const uint16_t* const* hk;
  int K, T;
};

}  // namespace bo

struct bo_ctx {
  bo_trainer_config cfg{};
  int device = 0, rank = 0, world = 1, algo = BO_REDUCE_NCCL;
  int num_sms = 148;
  bo::Layout L;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;

  // device tables
  bo::TensorDev* d_tensors = nullptr;
  bo::AccTile* d_acc_tiles = nullptr;
  int n_acc_tiles = 0;
  bo::LambTile* d_lamb_tiles = nullptr;
  int n_lamb_tiles = 0;
  int* d_tensor_tile_begin = nullptr;   // [T+1] lamb-tile ranges per tensor
  bo::HopXTile* d_hopx_tiles = nullptr; // ring hops with fused finalize, grouped by chunk
  std::vector<int> hopx_begin;          // [N+1] tile range of chunk q
  std::vector<std::vector<int>> hopx_bucket_begin;  // [N][B+1] first tile of chunk q, bucket b

  // Overlapped sync micro (bo_sync_ready; trainer.cpp:247-348 with overlap):
  // buckets reduced in layout order, in communication groups of whole buckets
  // (deterministic, identical on every rank), on comm_stream as soon as every
  // tensor of the group has been delivered.
  struct CommGroup {
    int b0, b1;      // bucket range
    int pending0;    // tensors in the group
    int acc0, acc1;  // NCCL wire: range in d_group_acc_tiles (finalize of the group's tensors)
  };
  std::vector<CommGroup> comm_groups;
  std::vector<int> group_of_bucket;
  bo::AccTile* d_group_acc_tiles = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comm_ready = nullptr, comm_done = nullptr;
  bool sync_open = false;
  bo::PtrTable* sync_tab = nullptr;     // host copy of the delivered pointers
  std::vector<uint8_t> delivered;
  std::vector<int> group_pending;
  int n_delivered = 0, next_group = 0;
  bool sync_aligned = true;

  // single-rank fused LAMB (world == 1)
  bo::FusedTile* d_fused_tiles = nullptr;
  int n_fused_tiles = 0;
  int* d_fused_tensor_tiles = nullptr;  // [T+1] fused-tile ranges per tensor
  float* u = nullptr;                   // LAMB update scratch
  // k_lamb_p1r / k_lamb_p1: bulk L2 prefetch of the tile this many CTAs
  // ahead (BO_P1R_PREFETCH, 0 = off; default 4/3 x the SM count, measured
  // best: profiles/r02_notes.md)
  int p1r_prefetch = 0;
  // grouped LAMB: the parameter push as this many persistent CTAs with
  // posted stores (k_push_posted; BO_PUSH_POSTED_CTAS, default 128; 0 = one
  // CTA per tile with bulk copies)
  int push_posted_ctas = 0;
  bool force_unfused = false;           // BO_UNFUSED=1: unfused kernels (one rank: multi-kernel LAMB; ring: staged last hop)

  // device buffers
  float* acc = nullptr;
  float* x = nullptr;        // finalized local gradients, flat layout
  float* gshard = nullptr;   // reduced gradient shard (aliases x when world == 1)
  float* w = nullptr;        // full parameter replica, flat layout
  float* m = nullptr;
  float* v = nullptr;
  float* m_alt = nullptr;    // second moment buffer set (double-buffered moments)
  float* v_alt = nullptr;
  // world > 1: fp32 master copy of this rank's parameter shard (shard layout,
  // aligned with m, v, u) and every rank's flat replica mapped through CUDA IPC
  float* wsh = nullptr;
  float** d_peer_w = nullptr;          // [world] device pointers to each rank's w
  void* peer_wire[2][8] = {};          // every rank's ring staging buffers (IPC), host-side
  void* ring_result = nullptr;         // staging buffer holding the owned reduced chunk
  const void* ring_last_in = nullptr;  // last hop fused into LAMB phase 1: its input
  int fuse_last_hop = -1;
  int path = 0;                        // BO_PATH_* bits of the last sync micro
  bo::MicroSrc ms{nullptr, 0, 0};      // resident micros of the step in flight (bo_train_step)
  const uint16_t** d_micro_tab = nullptr;  // device [K][T] gradient pointer table
  int micro_tab_cap = 0;              // BO_FUSE_LAST=0/1 overrides the per-world default
  bool ring_via_nccl = false;          // BO_RING_NCCL=1: hops over ncclSend/ncclRecv
  bool ring_push = true;               // BO_RING_PUSH=0: hops pull the left neighbour's buffer
  bool fuse_push_default = true;       // push form: fuse the (local) last hop into phase 1 by default
  std::vector<void*> ipc_opened;       // peer mappings to close
  int* d_barrier = nullptr;            // 4-byte NCCL all-reduce barrier (BO_RING_BARRIER=nccl)
  // Cross-rank flags (kCtrl* slots): this rank's block and every rank's
  // block mapped here; the ring-neighbour barrier (bo_ring.cu k_ring_barrier)
  // uses the two neighbour slots, the partials and end-of-step barriers
  // (bo_pipeline.cu) the all-rank slots. No NCCL on the default step.
  unsigned* ctrl = nullptr;
  bo::PeerFlags peer_ctrl{};
  unsigned* nb_flags = nullptr;        // == ctrl when the neighbour barrier is in use
  unsigned* nb_left_from_right = nullptr;
  unsigned* nb_right_from_left = nullptr;
  uint64_t nb_epoch = 0;
  uint64_t bar_epoch = 0;              // all-rank barrier epochs (one per step)
  uint64_t watchdog_ns = 120000000000ull;  // RunConfig::watchdog_s = 120 (trainer.hpp:144)
  bool nb_barrier = true;              // BO_RING_BARRIER=nccl: 4-byte NCCL all-reduce instead
  bool peers_mapped = false;           // bo_comm_import / bo_comm_init / bo_world_init_local done
  std::shared_ptr<bo::HostBarrier> lockstep;      // bo_world_init_local
  std::shared_ptr<bo::SharedStream> shared_stream;
  // Parameter groups of the push (world > 1): consecutive tensors in model
  // (= forward first-use) order; the push tiles are the LAMB tiles plus one
  // empty tile for every group this rank owns no element of, so that every
  // group has a last CTA that publishes "group g of this step landed" into
  // every rank's kCtrlReady slots (bo_params_wait).
  bo::LambTile* d_push_tiles = nullptr;
  int n_push_tiles = 0;
  int n_push_groups = 0;
  std::vector<int> push_group_of_tensor;
  int* d_push_group_of_tensor = nullptr;
  int* d_push_group_tiles = nullptr;   // [G] tiles of group g on this rank
  unsigned* d_push_count = nullptr;    // [G] cumulative finished tiles
  cudaEvent_t params_done = nullptr;   // world 1: the step's update, for bo_params_wait
  unsigned long long* hash_acc = nullptr;  // bo_replica_hash accumulator
  void* op_ws = nullptr;               // bo_ring_allreduce_* workspace (grow-only)
  size_t op_ws_bytes = 0;
  // Grouped LAMB (BO_LAMB_GROUP_ELEMS, world > 1): consecutive tensors (model
  // order), the push of each group speculative on push_stream, the master
  // shard double-buffered (wsh / wsh_alt by DevState::parity)
  struct LambGroup {
    int t0, t1;        // tensors [t0, t1)
    int tile0, tile1;  // their LAMB tiles (contiguous: tiles are in model order)
  };
  std::vector<LambGroup> lamb_groups;
  float* wsh_alt = nullptr;
  cudaStream_t push_stream = nullptr;
  std::vector<cudaEvent_t> group_events;

  double* peer_part[8] = {};           // every rank's all_part (IPC)
  void* wire[3] = {nullptr, nullptr, nullptr};  // ring staging (shard-sized)
  double* tile_part = nullptr;    // [n_lamb_tiles][2]
  double* rank_part = nullptr;    // [2T+1]
  double* all_part = nullptr;     // world > 1: [2][world][2T+1] (step parity halves); 1: rank_part
  float* trust = nullptr;         // [T]
  bo::DevState* state = nullptr;
  double* bc_table = nullptr;     // [bc_cap][4] (bc1, bc2, 1/bc1, 1/bc2) for steps 1..cap
  int64_t bc_cap = 0;
  int64_t calls = 0;              // sync micros issued (upper bound of lamb_step)
  int next_micro = 0;             // the micro bo_accumulate expects next (0..K-1)
  uint64_t device_bytes = 0;

  bo::LambConsts lamb{};
  bo::ScalerConsts scaler{};
  std::vector<void*> allocations;
  // measurement
  bool profiling = false;
  unsigned profile_mask = ~0u;
  int64_t launches = 0;
  struct Mark { int stage; cudaEvent_t a, b; };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> event_pool;
  double stage_ms[BO_NUM_STAGES] = {};
  int64_t stage_count[BO_NUM_STAGES] = {};
  std::vector<bool> ptr_aligned_cache;
  // tracing (bo_trace_enable): the reference's EventLog schema, device-timed
  bool tracing = false;
  cudaEvent_t trace_base = nullptr;
  struct TraceMark {
    const char* event;
    uint64_t bytes;
    cudaEvent_t e;
  };
  std::vector<TraceMark> trace_marks;
};

// Every C entry point: library failures become a bo_status plus the thread's
// last-error message.
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

namespace bo {
void* dev_alloc(bo_ctx* c, size_t bytes);
void upload_tables(bo_ctx* c);
void grow_bc_table(bo_ctx* c, int64_t need);

// kernels / pipeline stages (bo_pipeline.cu)
void launch_accumulate(bo_ctx* c, int micro, const PtrTable& tab, bool vec_ok);
void launch_finalize(bo_ctx* c, const PtrTable& tab);
void launch_finalize_tiles(bo_ctx* c, const AccTile* tiles, int n, const PtrTable& tab,
                           cudaStream_t stream);
void check_launch(bo_ctx* c, const char* what);  // counts the launch, raises on a launch error
void run_reduce(bo_ctx* c, const PtrTable& tab);
// one communication group of buckets [b0, b1) on `stream` (overlap mode)
void run_reduce_group(bo_ctx* c, const PtrTable& tab, int b0, int b1, int acc0, int acc1,
                      cudaStream_t stream);
void run_lamb(bo_ctx* c, const PtrTable& tab);
void gather_shard(bo_ctx* c);
// tracing: a device timestamp (an event on `s`) named like the reference's
// EventLog events (trainer.hpp:30-35), no-op unless bo_trace_enable
void trace(bo_ctx* c, const char* event, uint64_t bytes, cudaStream_t s);
// lockstep world: rendezvous of the ranks' host threads (no-op otherwise)
void lockstep_sync(bo_ctx* c, const char* where);
// the caller's stream waits for tensor's parameter group of the last step
void params_wait(bo_ctx* c, int tensor, cudaStream_t stream);
// needs the NCCL communicator (bo_comm_init): fail otherwise
void need_nccl(bo_ctx* c, const char* what);
// bo_ring_allreduce_* over the mapped ring staging buffers (bo_ring.cu)
bool ring_op_available(const bo_ctx* c);
void ring_allreduce_op(bo_ctx* c, float* data, size_t n, bool f16);
void run_fused_single_rank(bo_ctx* c, const PtrTable& tab, MicroSrc ms = MicroSrc{nullptr, 0, 0});

// Stage bracket: records events when profiling is on.
struct StageTimer {
  bo_ctx* c;
  int stage;
  cudaEvent_t b = nullptr;
  cudaStream_t stream;
  StageTimer(bo_ctx* ctx, int s);
  StageTimer(bo_ctx* ctx, int s, cudaStream_t on);
  ~StageTimer();
};
}  // namespace bo

#endif  // BO_INTERNAL_HPP_
