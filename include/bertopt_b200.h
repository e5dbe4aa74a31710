/*
 * bertopt_b200 — C ABI of the B200-native gradient-to-update pipeline.
 *
 * Drop-in boundary for the reference's hot path. The
 * reference C++ operator API in proj/core stays unchanged; a maintainer binds
 * these entry points behind it. Plain pointers and sizes
 * only: no torch or CUDA types appear in the signatures (streams are void*).
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj/core):
 *   bo_create / bo_layout_*      BucketLayout::build + hash    trainer.cpp:73-134
 *                                TrainerConfig                 trainer.hpp:75-85
 *   bo_comm_*                    WorkerGroup + Transport       collective.hpp:30-40,
 *                                                              transport.hpp:38-53
 *   bo_accumulate (micro<K-1)    accum_[p][i] += g[i]          trainer.cpp:240-244
 *   bo_accumulate (micro=K-1)    flatten_param + reduce_bucket trainer.cpp:186-215
 *                                + unpack + lamb_step          trainer.cpp:356-366
 *                                (the sync micro of train_step trainer.cpp:217-373)
 *   bo_lamb_step                 lamb_step                     lamb.hpp:47-48, lamb.cpp:23-84
 *   bo_ring_allreduce_f32        ring_allreduce<float>         collective.hpp:104-107
 *   bo_ring_allreduce_f16_wire   ring_allreduce_f16_wire       collective.hpp:113-114
 *   bo_unscale_gradients         unscale_gradients             half.hpp:77, half.cpp:105-115
 *   bo_narrow_f16 / bo_widen_f16 narrow/widen_f16_block        graph.hpp:160-163
 *   bo_scale_loss                scale_loss                    half.hpp:73
 *
 * Error convention: every call returns a bo_status whose values map 1:1 onto
 * the bertopt::Error subclasses (errors.hpp:35-48), plus CUDA/NCCL failures.
 * The C++ adapter (include/bertopt_b200_adapter.hpp) re-throws them as the
 * typed reference exceptions. One deliberate difference on the pipeline path:
 * a non-finite reduced gradient is not an error there — it sets the step's
 * found_inf flag, the LAMB step is skipped on device (no host sync) and the
 * dynamic loss scaler backs off (the scaler extension).
 */
#ifndef BERTOPT_B200_H_
#define BERTOPT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BO_ABI_VERSION 1

typedef enum {
  BO_OK = 0,
  BO_ERR_SHAPE_MISMATCH = 1,         /* bertopt::ShapeMismatch */
  BO_ERR_NON_FINITE_GRADIENT = 2,    /* bertopt::NonFiniteGradient */
  BO_ERR_OVERFLOW_DETECTED = 3,      /* bertopt::OverflowDetected */
  BO_ERR_LENGTH_MISMATCH = 4,        /* bertopt::LengthMismatch */
  BO_ERR_INVALID_CONFIG = 5,         /* bertopt::InvalidConfig */
  BO_ERR_BUCKET_LAYOUT_MISMATCH = 6, /* bertopt::BucketLayoutMismatch */
  BO_ERR_PEER_DISCONNECTED = 7,      /* bertopt::PeerDisconnected */
  BO_ERR_WATCHDOG_TIMEOUT = 8,       /* bertopt::WatchdogTimeout */
  BO_ERR_PROTOCOL = 9,               /* bertopt::ProtocolError */
  BO_ERR_IO_FAILURE = 10,            /* bertopt::IoFailure */
  BO_ERR_CUDA = 20,
  BO_ERR_NCCL = 21,
  BO_ERR_NO_DEVICE = 22
} bo_status;

/* bertopt::LambConfig (lamb.hpp:30-37); defaults via bo_default_config. */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay, trust_clip;
} bo_lamb_config;

/* Dynamic loss scaler (builder-defined extension; the reference scaler is
 * static, half.hpp:52-70). Scales stay powers of two. dynamic = 0 keeps
 * init_scale for the whole run (the reference behaviour). */
typedef struct {
  float init_scale, growth_factor, backoff_factor, min_scale, max_scale;
  int32_t growth_interval;
  int32_t dynamic;
} bo_scaler_config;

typedef enum {
  BO_REDUCE_AUTO = 0,  /* RING (measured faster than NCCL for the fp32 wire too) */
  BO_REDUCE_RING = 1,  /* reference ring order, bit-exact (fp32 or f16 wire) */
  BO_REDUCE_NCCL = 2   /* ncclReduceScatter (fp32 wire only; reassociated sum) */
} bo_reduce_algo;

/* bertopt::TrainerConfig (trainer.hpp:75-85) restricted to the hot path. */
typedef struct {
  bo_lamb_config lamb;
  int32_t accumulation;   /* K micro-batches per optimizer step */
  uint64_t bucket_bytes;  /* fusion-buffer threshold (4 MiB default) */
  int32_t f16_exchange;   /* binary16 wire for the gradient reduction */
  int32_t reduce_algo;    /* bo_reduce_algo */
  bo_scaler_config scaler;
} bo_trainer_config;

/* Device-resident step status (read back by bo_get_status; host sync). */
typedef struct {
  float loss_scale;       /* scale the NEXT step will use */
  int32_t good_steps;     /* consecutive finite steps since last change */
  int64_t lamb_step;      /* LambState::step (lamb.hpp:39-43) */
  int64_t steps;          /* optimizer steps attempted (incl. skipped) */
  int64_t skipped_steps;  /* steps skipped on overflow */
  int32_t found_inf;      /* last step's global overflow flag */
  int32_t reserved;
} bo_step_status;

typedef struct bo_ctx bo_ctx;

int32_t bo_abi_version(void);
const char* bo_status_name(int32_t status);
/* Last error message of the calling thread (any entry point). */
const char* bo_last_error(void);
void bo_default_config(bo_trainer_config* cfg);

/* ---- layout (host only, no device needed) -------------------------------- */
/* BucketLayout::build (trainer.cpp:73-116): fills bucket_of[T], offset_of[T],
 * ready_order[T], bucket_elems[T] (first *n_buckets entries valid) and the
 * salted layout hash (names/ndims/dims optional, as in bo_create). */
bo_status bo_bucket_layout(int32_t n_tensors, const int64_t* numels, const int32_t* first_consumers,
                           uint64_t bucket_bytes, const char* const* names, const int32_t* ndims,
                           const int64_t* dims, int32_t f16_exchange, int32_t accumulation,
                           int32_t* bucket_of, int64_t* offset_of, int32_t* ready_order,
                           int64_t* bucket_elems, int32_t* n_buckets, uint64_t* hash);
/* Elements rank `rank` of `world` owns: for every bucket b the range
 * [lo[b], hi[b]) of bucket-local element indices (chunk `rank` of the ring's
 * ceil(n_b/world) chunking, clipped to n_b). */
bo_status bo_shard_ranges(int32_t n_buckets, const int64_t* bucket_elems, int32_t world,
                          int32_t rank, int64_t* lo, int64_t* hi);

/* ---- context / layout -------------------------------------------------- */
/* One context per rank (one process or thread per GPU). numels and
 * first_consumers are in model parameter order; first_consumers[p] is the op
 * id of p's first consumer in the forward (gradients become final in
 * descending order, trainer.cpp:85-90). names/ndims/dims are optional (may be
 * NULL) and only feed the layout hash. */
bo_status bo_create(const bo_trainer_config* cfg, int32_t n_tensors, const int64_t* numels,
                    const int32_t* first_consumers, const char* const* names,
                    const int32_t* ndims, const int64_t* dims, int32_t device, int32_t rank,
                    int32_t world, bo_ctx** out);
void bo_destroy(bo_ctx* ctx);

int32_t bo_layout_num_buckets(const bo_ctx* ctx);
/* BucketLayout fields: bucket_of[T], offset_of[T], ready_order[T], bucket_elems[B]. */
bo_status bo_layout_query(const bo_ctx* ctx, int32_t* bucket_of, int64_t* offset_of,
                          int32_t* ready_order, int64_t* bucket_elems);
/* BucketLayout::hash salted with f16_exchange and K (trainer.cpp:161-168). */
uint64_t bo_layout_hash(const bo_ctx* ctx);
/* Elements of this rank's shard (sum of ceil(n_b / world) over buckets). */
int64_t bo_shard_elems(const bo_ctx* ctx);
/* Device bytes held by the context. */
uint64_t bo_device_bytes(const bo_ctx* ctx);

/* ---- communication (world > 1) ----------------------------------------- */
/* 128-byte NCCL unique id; rank 0 creates it, the host harness broadcasts it. */
bo_status bo_comm_unique_id(uint8_t* out128);
/* Collective over all ranks: NCCL communicator + layout-hash agreement
 * (BO_ERR_BUCKET_LAYOUT_MISMATCH on disagreement, trainer.cpp:169-183) + the
 * peer mappings of bo_comm_import. Needed for the NCCL reduce-scatter, the
 * ncclSend/Recv ring (BO_RING_NCCL=1), the NCCL hop barrier
 * (BO_RING_BARRIER=nccl) and the bo_ring_allreduce_* operators of a context
 * without mapped ring buffers. */
bo_status bo_comm_init(bo_ctx* ctx, const uint8_t* id128);
/* NCCL-free initialisation of the default (binary16 / fp32 ring) step, which
 * runs without any collective library: every rank exports a fixed-size
 * record (layout hash, settings hash, CUDA IPC handles of its parameter
 * replica, ring staging buffers, flag block and norm partials), the host
 * harness all-gathers the records in rank order over any channel (the
 * reference's WorkerGroup transport, torch.distributed, MPI, a file), and
 * every rank imports all of them. bo_comm_export(ctx, NULL, &n) returns the
 * record size. Import fails with BO_ERR_BUCKET_LAYOUT_MISMATCH / BO_ERR_PROTOCOL
 * when ranks disagree (trainer.cpp:169-183). Several ranks may share one GPU. */
bo_status bo_comm_export(bo_ctx* ctx, void* record, uint64_t* nbytes);
bo_status bo_comm_import(bo_ctx* ctx, const void* records, uint64_t nbytes_each);
/* A whole world in THIS process (the reference's run_data_parallel: one host
 * thread per rank, trainer.cpp:397-470), all contexts on one device: peers
 * are mapped directly, all contexts share one stream, and every cross-rank
 * wait of the step becomes a rendezvous of the ranks' host threads between
 * kernel launches (lockstep) — no kernel ever waits for another. Each rank's
 * thread then calls the step entry points as usual, concurrently. Runs a
 * world larger than the machine (world 8 on one B200) with the same kernels
 * and bit-identical results; ring reduction only (no NCCL). */
bo_status bo_world_init_local(bo_ctx* const* ctxs, int32_t n);
/* Bound of every cross-rank wait inside a step (RunConfig::watchdog_s,
 * trainer.hpp:144; default 120 s). A peer that misses it abandons the step on
 * this rank (no update, loss scaler untouched) and the next bo_wait returns
 * BO_ERR_PEER_DISCONNECTED. */
bo_status bo_set_watchdog(bo_ctx* ctx, double seconds);

/* ---- streams ----------------------------------------------------------- */
/* Stream contract: every hot-path call is asynchronous on the context stream
 * and reads the caller's gradient buffers there; the library does not
 * synchronise with any other stream. The caller must produce the gradients on
 * the context stream (bo_set_stream to the producer's stream — the simplest),
 * or order the context stream after the producer (an event), and keep the
 * buffers alive and unmodified until the step's work has run (bo_synchronize,
 * bo_wait, or an event recorded on the context stream). */
/* Run all work of ctx on the caller's cudaStream_t (NULL: ctx's own stream). */
bo_status bo_set_stream(bo_ctx* ctx, void* cuda_stream);
void* bo_get_stream(const bo_ctx* ctx);
bo_status bo_synchronize(bo_ctx* ctx);
/* Watchdog wait (the reference's transport watchdog, transport.cpp:113-132 /
 * 336-383): block until the context's queued work has completed, at most
 * timeout_ms milliseconds (< 0: no limit). BO_ERR_PEER_DISCONNECTED when the
 * communicator reports a remote failure (ncclCommGetAsyncError) or a ring
 * neighbour never reached a hop barrier (its step was then skipped),
 * BO_ERR_WATCHDOG_TIMEOUT when the work is still pending at the deadline (a
 * stalled or dead peer keeps a collective from completing). Nothing is
 * cancelled: the caller decides whether to keep waiting or to tear the rank
 * down (the reference's run_data_parallel then reports the root cause,
 * trainer.cpp:473-487). */
bo_status bo_wait(bo_ctx* ctx, int64_t timeout_ms);

/* ---- state ------------------------------------------------------------- */
/* Parameters in model order, flat (all tensors concatenated). */
bo_status bo_load_params(bo_ctx* ctx, const float* src, int32_t src_on_host);
bo_status bo_read_params(bo_ctx* ctx, float* dst, int32_t dst_on_host);
/* LAMB moments of the elements this rank owns, scattered into model-order
 * flat arrays (elements owned by other ranks are left untouched). */
bo_status bo_read_moments(bo_ctx* ctx, float* m, float* v, int32_t dst_on_host);
/* Replica hash, the device counterpart of the reference's per-step replica
 * divergence check (DistributedTrainer::param_hash, trainer.cpp:136-142,
 * 375-377, checked across ranks at trainer.cpp:442-453): sum mod 2^64 of
 * mix64(mix64(t << 40 | i) ^ bits(param[t][i])) over this rank's parameter
 * replica (splitmix64 finaliser), one pass over the replica on the device,
 * after the context stream's work so far; synchronous. Equal on every rank
 * whose replica is bit-identical. (The reference's own FNV-1a value is
 * sequential by construction: the C++ adapter's GradPipeline::param_hash()
 * computes it from a host copy.) */
bo_status bo_replica_hash(bo_ctx* ctx, uint64_t* out);
bo_status bo_get_status(bo_ctx* ctx, bo_step_status* out);
/* Checkpoint / resume of the device state (the reference
 * BCKP checkpoint, model.cpp:360-425, keeps only parameters). The blob holds
 * the parameter replica and the moments of the elements this rank owns (both
 * in model order), the LAMB step and the loss-scaler state; every rank of a
 * world exports / imports its own blob. bo_export_state(ctx, NULL, &n) returns
 * the size. Import requires the same tensors, world and ownership. Syncs. */
bo_status bo_export_state(bo_ctx* ctx, void* blob, uint64_t* nbytes);
bo_status bo_import_state(bo_ctx* ctx, const void* blob, uint64_t nbytes);
/* Per-tensor device pointer into the full-replica parameter buffer. */
bo_status bo_param_ptr(bo_ctx* ctx, int32_t tensor, float** out);

/* ---- hot path ------------------------------------------------------------ */
/* Feed micro-batch `micro` (0..K-1) of the current optimizer step. grads[p]
 * is a device pointer to tensor p's binary16 gradient (loss-scaled by the
 * current scale). Micros 0..K-2 accumulate in fp32. micro == K-1 is the sync
 * micro: finalize (accumulate + unscale + overflow check + pack into the
 * fusion buffer) -> reduce-scatter -> sharded LAMB (per-tensor norms, trust
 * ratio; skipped on overflow) -> loss-scaler update -> all-gather of the
 * updated parameters. Asynchronous on the context stream. */
bo_status bo_accumulate(bo_ctx* ctx, int32_t micro, const uint16_t* const* grads);
/* One whole optimizer step, DistributedTrainer::train_step(micros)
 * (trainer.cpp:217-373): grads[k * n_tensors + p] is micro k's binary16
 * gradient of tensor p, for k = 0..K-1, all resident in HBM until the step's
 * work has run on the context stream. With every micro at hand the sync pass
 * reads the K gradient sets directly — summed in the reference's order,
 * ((0 + g0) + g1) + ... + g_{K-2}, then + g_{K-1} — instead of materialising
 * an fp32 accumulator (24 B/param of accumulator traffic saved at K = 4).
 * Bit-identical to K bo_accumulate calls. */
bo_status bo_train_step(bo_ctx* ctx, const uint16_t* const* grads);
/* The sync micro with bucket-level overlap (TrainerConfig::overlap,
 * trainer.cpp:247-348; readiness = Tape::backward's progress hook,
 * tensor.hpp:94-106): deliver the sync micro's gradients as they become final,
 * n tensors per call (tensor indices + device pointers, any chunking, each
 * tensor once). Buckets are reduced in layout order, in communication groups
 * of whole buckets, on an internal stream as soon as every tensor of the group
 * has been delivered — overlapping the caller's remaining backward work on the
 * context stream. The call that delivers the last tensor runs the rest of the
 * step. Results are bit-identical to bo_accumulate(ctx, K-1, grads). Micros
 * 0..K-2 still go through bo_accumulate. */
bo_status bo_sync_ready(bo_ctx* ctx, int32_t n, const int32_t* tensors, const uint16_t* const* grads);

/* The next step's forward overlapping this step's parameter all-gather:
 * enqueue on `stream` (a cudaStream_t, typically the forward's) a wait until
 * the parameters of `tensor`'s parameter group, as updated by the most
 * recently enqueued step, are in this rank's replica (bo_param_ptr) — every
 * rank pushes its updated shard into every replica group by group, in model
 * (= forward first-use) order, and publishes each group as it lands. Kernels
 * enqueued on `stream` afterwards read the new values; the rest of the push
 * continues on the context stream. The parameters read must not be those of
 * a later step still in flight. World 1: the stream waits for the whole
 * step. With the grouped LAMB (the default at world >= 4, where the push
 * overlaps the next tensor group's phase 1 inside the step instead) the
 * groups are published together at the end of the step. Bounded by the
 * watchdog (bo_set_watchdog). */
bo_status bo_params_wait(bo_ctx* ctx, int32_t tensor, void* stream);
/* Parameter group of a tensor (world 1: 0; -1 for a bad index). */
int32_t bo_param_group(const bo_ctx* ctx, int32_t tensor);

/* ---- measurement ---------------------------------------------------------- */
/* Stage timing with CUDA events recorded on the context stream around every
 * stage of bo_accumulate (off by default). Stages: */
#define BO_STAGE_ACCUMULATE 0   /* micros 0..K-2 */
#define BO_STAGE_FINALIZE 1     /* unscale + pack into the fusion buffer (NCCL wire) */
#define BO_STAGE_REDUCE 2       /* reduce-scatter (ring hops with fused finalize, or NCCL) */
#define BO_STAGE_LAMB_NORMS 3   /* LAMB phase 1: moments, update, norm partials */
#define BO_STAGE_TRUST 4        /* norm reduction, partials all-gather, trust/scaler */
#define BO_STAGE_LAMB_UPDATE 5  /* LAMB phase 2 (world > 1: + parameter push to all replicas) */
#define BO_STAGE_ALLGATHER 6    /* world > 1: replica-completion barrier */
#define BO_STAGE_FLAG 7         /* ring hop kernels alone (nested inside REDUCE) */
#define BO_STAGE_LAMB_FUSED 8   /* reserved */
#define BO_NUM_STAGES 9
bo_status bo_profile_enable(bo_ctx* ctx, int32_t enable);
/* Total milliseconds and event count per stage since the last reset; syncs. */
bo_status bo_profile_read(bo_ctx* ctx, double* stage_ms, int64_t* stage_count, int32_t reset);
/* Kernels this library has launched on ctx (NCCL kernels not included). */
int64_t bo_launch_count(const bo_ctx* ctx);
/* Which implementation the last sync micro ran (bit set; 0 before the first). */
#define BO_PATH_ONE_RANK_FUSED 1     /* one rank: k_lamb_p1 / k_lamb_trust / k_lamb_p2 */
#define BO_PATH_ONE_RANK_STAGED 2    /* one rank: finalize + multi-kernel LAMB */
#define BO_PATH_RING_P2P 4           /* ring hops reading the left neighbour over CUDA IPC */
#define BO_PATH_RING_SENDRECV 8      /* ring hops over ncclSend/ncclRecv */
#define BO_PATH_LAST_HOP_FUSED 16    /* the ring's last hop ran inside LAMB phase 1 */
#define BO_PATH_NCCL_RS 32           /* ncclReduceScatter of the fusion buffer */
#define BO_PATH_OVERLAP 64           /* sync micro delivered through bo_sync_ready */
#define BO_PATH_RESIDENT 128         /* bo_train_step: the K micros read in the sync pass */
#define BO_PATH_RING_PUSH 256        /* ring hops push their output into the right neighbour's buffer over NVLink */
#define BO_PATH_LAMB_GROUPED 512     /* LAMB in tensor groups, the push of group g overlapping phase 1 of g+1 */
int32_t bo_path_flags(const bo_ctx* ctx);

/* Event timeline in the reference's EventLog schema (trainer.cpp:43-71,
 * events trainer.hpp:30-35): one JSON line per event,
 *   {"ts":<seconds since bo_trace_enable>,"rank":<r>,"event":"<name>","bytes":<n>}
 * with device timestamps (CUDA events on the stream that carries the work):
 * micro_ready (a micro-batch's gradients entered the step; bytes: binary16
 * gradient bytes), bucket_ready (bo_sync_ready: a communication group's
 * gradients are final), comm_start / comm_end (the reduce-scatter, or one
 * group of it; bytes: what this rank sends over NVLink), lamb_start,
 * step_end. NVTX ranges name the stages for a timeline profiler while
 * tracing is on. bo_trace_write syncs and writes the lines, oldest first
 * (BO_ERR_IO_FAILURE if the file cannot be written). */
bo_status bo_trace_enable(bo_ctx* ctx, int32_t enable);
bo_status bo_trace_write(bo_ctx* ctx, const char* path);

/* ---- operator-level drop-ins -------------------------------------------- */
/* lamb_step (lamb.cpp:23-84) over device tensors; exact reference numerics
 * and error behaviour (step incremented first; on a non-finite gradient the
 * tensors before it are updated and BO_ERR_NON_FINITE_GRADIENT returned). */
bo_status bo_lamb_step(int32_t n_tensors, const int64_t* numels, float* const* params,
                       const float* const* grads, float* const* m, float* const* v,
                       int64_t* step, const bo_lamb_config* cfg, void* stream);
/* In-place elementwise sum over all ranks of ctx's world, reference fold
 * order (chunk k folded over ranks k, k+1, ..., k-1; binary16 wire rounding
 * per hop and the owner re-round for the f16 variant), identical bits on
 * every rank. data is a device pointer; every rank calls with the same n.
 * Runs over the context's own NVLink ring staging buffers (push form, a
 * neighbour barrier per hop, chunks larger than the buffers in slices) once
 * the peers are mapped (bo_comm_import / bo_comm_init / bo_world_init_local
 * with the ring reduce algorithm), else over ncclSend/ncclRecv (bo_comm_init).
 * Returns with the data reduced (the context stream is synchronised);
 * BO_ERR_PROTOCOL while a bo_sync_ready micro is open. */
bo_status bo_ring_allreduce_f32(bo_ctx* ctx, float* data, size_t n);
bo_status bo_ring_allreduce_f16_wire(bo_ctx* ctx, float* data, size_t n);
/* unscale_gradients: BO_ERR_OVERFLOW_DETECTED (and no change) if any entry is
 * non-finite, else divide by scale when enabled. BO_ERR_INVALID_CONFIG when
 * scale is not a positive power of two. Device pointer; synchronizes. */
bo_status bo_unscale_gradients(float* grads, size_t n, float scale, int32_t enabled,
                               void* stream);
bo_status bo_narrow_f16(const float* src, uint16_t* dst, size_t n, void* stream);
bo_status bo_widen_f16(const uint16_t* src, float* dst, size_t n, void* stream);
/* SURVEY §8(f) rank 4, the paper's fused elementwise optimizer: the
 * Adam-form FusedKernel fused_optimizer_step(lr, beta1, beta2, eps,
 * weight_decay, step) (graph.cpp:458-487) as run_fused_kernel executes it on
 * (w, g, m, v) -> (w', m', v') in fp32 (apply_block, graph.cpp:296-347: every
 * attribute a double rounded to float, one rounding per instruction), applied
 * in place over n_tensors device tensors. */
bo_status bo_fused_optimizer_step(int32_t n_tensors, const int64_t* numels, float* const* params,
                                  const float* const* grads, float* const* m, float* const* v,
                                  float lr, float beta1, float beta2, float eps,
                                  float weight_decay, int32_t step, void* stream);
/* The AMP cast (Tape::cast to f16, ops.cpp:655-668 -> quantize_inplace):
 * x = binary16_RNE(x) in place (f16_round, half.cpp:79). */
bo_status bo_f16_round(float* x, size_t n, void* stream);
float bo_scale_loss(float loss, float scale, int32_t enabled);

/* ---- device memory for hosts without the CUDA toolkit (cgo / JNI / C++) -- */
bo_status bo_malloc(void** ptr, size_t bytes, int32_t device);
bo_status bo_free(void* ptr);
/* kind: 0 host->device, 1 device->host, 2 device->device; synchronous. */
bo_status bo_memcpy(void* dst, const void* src, size_t bytes, int32_t kind);

/* ---- synthetic workload (bench / test harness utility) ------------------- */
/* fp16 gradient bits of the synthetic spec
 * for elements [flat_begin, flat_begin + n) of model-order flat index space,
 * written to dst (device). */
bo_status bo_synth_grads(uint16_t* dst, int64_t flat_begin, int64_t n, uint64_t seed,
                         int32_t rank, int32_t step, int32_t micro, float scale,
                         uint32_t spike_ppm, int32_t spike_exp, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BERTOPT_B200_H_ */
