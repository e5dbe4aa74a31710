// The reference ring's reduce-scatter on the device (collective.hpp:53-99,
// binary16 wire collective.cpp:37-86), flatten_param fused into every hop:
//   k_hopx       one hop over the chunk of every bucket this rank adds at hop s
//   run_reduce   hop 0 (pack) + N-1 hops reading the left neighbour's staging
//                buffer over NVLink (CUDA IPC), or grouped ncclSend/ncclRecv,
//                or ncclReduceScatter for the NCCL wire
// Bit-level contract as in bo_pipeline.cu (--fmad=false, explicit _rn).
#include <cuda_fp16.h>

#include <algorithm>

#include "bo_device.cuh"
#include "bo_internal.hpp"

namespace bo {
namespace {

// --------------------------------------------------------------- ring hops
// Ring hop with flatten_param fused in (trainer.cpp:186-203 + collective.hpp:65-80
// / collective.cpp:47-62): x = (h + acc) * inv for the elements of chunk q,
// out = wire(x) (combine == 0, the first send) or wire(from_wire(in) + x).
// KR > 0 (bo_train_step): x from the KR resident micros instead of h + acc.
template <typename W, int KR>
__global__ void __launch_bounds__(kThreads) k_hopx(const HopXTile* __restrict__ tiles,
                                                   const TensorDev* __restrict__ td,
                                                   const __grid_constant__ PtrTable tab, MicroSrc ms,
                                                   const float* __restrict__ acc,
                                                   const DevState* __restrict__ st, int K,
                                                   const W* __restrict__ in, W* __restrict__ out,
                                                   int combine) {
  const HopXTile tile = tiles[blockIdx.x];
  const float inv = __fdiv_rn(1.0f, __fmul_rn(static_cast<float>(K), st->scale));
  const uint16_t* __restrict__ h = tab.p[tile.t] + tile.e0;
  const float* __restrict__ a = acc + td[tile.t].acc_off + tile.e0;
  constexpr bool resident = KR > 0;
  __shared__ const uint16_t* mp[KR > 0 ? KR : 1];  // the tile's KR micro pointers
  if constexpr (resident) {
    if (static_cast<int>(threadIdx.x) < KR) mp[threadIdx.x] = ms.hk[threadIdx.x * ms.T + tile.t] + tile.e0;
    __syncthreads();
  }
  // (h + acc) * inv, or the resident micros' sum * inv, for element e / e..e+3
  auto x1 = [&](int e) {
    if constexpr (resident) return __fmul_rn(micro_sum1(mp, KR, e), inv);
    const float g = widen(__ldcs(h + e));
    return __fmul_rn(K > 1 ? __fadd_rn(g, __ldcs(a + e)) : g, inv);
  };
  auto x4 = [&](int e, float (&x)[4]) {
    if constexpr (resident) {
      micro_sum4_k<KR>(mp, e, x);
    } else {
      const uint2 hv = __ldcs(reinterpret_cast<const uint2*>(h + e));
      x[0] = widen(static_cast<uint16_t>(hv.x & 0xFFFFu));
      x[1] = widen(static_cast<uint16_t>(hv.x >> 16));
      x[2] = widen(static_cast<uint16_t>(hv.y & 0xFFFFu));
      x[3] = widen(static_cast<uint16_t>(hv.y >> 16));
      if (K > 1) {
        const float4 a4 = __ldcs(reinterpret_cast<const float4*>(a + e));
        x[0] = __fadd_rn(x[0], a4.x);
        x[1] = __fadd_rn(x[1], a4.y);
        x[2] = __fadd_rn(x[2], a4.z);
        x[3] = __fadd_rn(x[3], a4.w);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = __fmul_rn(x[i], inv);
  };
  // Vector path when the tensor side (h, acc) and the shard side (in, out)
  // share their 4-element alignment (the common case: BERT tensor sizes and
  // chunk lengths are multiples of 4): scalar head to the boundary, float4 /
  // 4 x binary16 body, scalar tail. Caller slots are 16-byte aligned (all K
  // of them in resident mode, checked by bo_train_step).
  if (((tile.e0 - tile.s0) & 3) == 0 && (resident || (reinterpret_cast<uintptr_t>(tab.p[tile.t]) & 15) == 0)) {
    const int head = min(static_cast<int>((4 - (tile.s0 & 3)) & 3), tile.len);
    const int nv = (tile.len - head) >> 2;
    auto one = [&](int e) {
      float p = x1(e);
      if (combine) p = __fadd_rn(from_wire(in[tile.s0 + e]), p);
      out[tile.s0 + e] = to_wire<W>(p);
    };
    if (threadIdx.x < head) one(threadIdx.x);
    const int tail0 = head + 4 * nv;
    if (threadIdx.x >= 32 && static_cast<int>(threadIdx.x) - 32 < tile.len - tail0) {
      one(tail0 + static_cast<int>(threadIdx.x) - 32);
    }
#pragma unroll 4
    for (int q = threadIdx.x; q < nv; q += kThreads) {
      const int e = head + 4 * q;
      float iv[4] = {0.f, 0.f, 0.f, 0.f};
      if (combine) {
        if constexpr (sizeof(W) == 2) {
          const uint2 w2 = __ldcs(reinterpret_cast<const uint2*>(in + tile.s0 + e));
          iv[0] = widen(static_cast<uint16_t>(w2.x & 0xFFFFu));
          iv[1] = widen(static_cast<uint16_t>(w2.x >> 16));
          iv[2] = widen(static_cast<uint16_t>(w2.y & 0xFFFFu));
          iv[3] = widen(static_cast<uint16_t>(w2.y >> 16));
        } else {
          const float4 w4 = __ldcs(reinterpret_cast<const float4*>(in + tile.s0 + e));
          iv[0] = w4.x; iv[1] = w4.y; iv[2] = w4.z; iv[3] = w4.w;
        }
      }
      float xv[4];
      x4(e, xv);
      W o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float p = xv[i];
        if (combine) p = __fadd_rn(iv[i], p);
        o[i] = to_wire<W>(p);
      }
      if constexpr (sizeof(W) == 2) {
        uint2 w2;
        w2.x = static_cast<uint32_t>(o[0]) | (static_cast<uint32_t>(o[1]) << 16);
        w2.y = static_cast<uint32_t>(o[2]) | (static_cast<uint32_t>(o[3]) << 16);
        *reinterpret_cast<uint2*>(out + tile.s0 + e) = w2;
      } else {
        *reinterpret_cast<float4*>(out + tile.s0 + e) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    return;
  }
  constexpr int kPer = kTileElems / kThreads;
  float xv[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * kThreads;
    xv[j] = e < tile.len ? x1(e) : 0.0f;
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * kThreads;
    if (e < tile.len) {
      float p = xv[j];
      if (combine) p = __fadd_rn(from_wire(__ldcs(in + tile.s0 + e)), p);
      out[tile.s0 + e] = to_wire<W>(p);
    }
  }
}

// Neighbour barrier between ring hops: this rank's previous hop kernel has
// completed (stream order), so its stores — including the NVLink pushes — are
// performed; publish that to both ring neighbours (a flag in each of their
// memories) and wait until both have published the same epoch. A hop only
// exchanges data with its neighbours (reads what the left pushed, pushes into
// the right's buffer after the right read it), so this replaces a global
// barrier. The wait is bounded by the watchdog (RunConfig::watchdog_s,
// trainer.hpp:144; bo_set_watchdog): a neighbour that never arrives sets
// peer_timeout — the step is then abandoned without an update and without
// touching the loss scaler (k_trust), and bo_wait reports PeerDisconnected.
__global__ void k_ring_barrier(unsigned* left_from_right, unsigned* right_from_left, const unsigned* mine,
                               unsigned epoch, DevState* st, uint64_t timeout_ns) {
  if (st->peer_timeout) return;  // an earlier barrier of this step gave up
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(left_from_right), "r"(epoch) : "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(right_from_left), "r"(epoch) : "memory");
  const uint64_t t0 = global_ns();
  for (int i = 0; i < 2; ++i) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + i) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (global_ns() - t0 > timeout_ns) {
        st->peer_timeout = 1;
        return;
      }
      __nanosleep(64);
    }
  }
}

}  // namespace

// Barrier before a ring hop: the neighbour flags when mapped, else a 4-byte
// NCCL all-reduce.
static void hop_barrier(bo_ctx* c, cudaStream_t st) {
  if (c->lockstep) {
    lockstep_sync(c, "ring hop");
    return;
  }
  if (c->nb_flags) {
    c->nb_epoch += 1;
    k_ring_barrier<<<1, 1, 0, st>>>(c->nb_left_from_right, c->nb_right_from_left, c->nb_flags,
                                    static_cast<unsigned>(c->nb_epoch), c->state, c->watchdog_ns);
    check_launch(c, "k_ring_barrier");
  } else {
    need_nccl(c, "BO_RING_BARRIER=nccl");
    BO_NCCL(ncclAllReduce(c->d_barrier, c->d_barrier, 1, ncclInt32, ncclSum, c->comm, st));
  }
}

// The reference ring's reduce-scatter phase (collective.hpp:65-80, binary16
// wire collective.cpp:47-62) over buckets [b0, b1), with flatten_param fused
// into every hop: the local addend x of chunk q is computed from the sync
// micro's binary16 input and the accumulator as the hop needs it.
template <typename W>
static void ring_reduce_scatter(bo_ctx* c, const PtrTable& tab, ncclDataType_t dt, int b0, int b1,
                                cudaStream_t st) {
  const int N = c->world, r = c->rank;
  const int right = (r + 1) % N, left = (r - 1 + N) % N;
  const Layout& L = c->L;
  const int64_t sh0 = L.shoff[static_cast<size_t>(b0)];
  const int64_t sh1 = b1 < L.B ? L.shoff[static_cast<size_t>(b1)] : L.shard_total;
  W* a = static_cast<W*>(c->wire[0]);
  W* b = static_cast<W*>(c->wire[1]);
  const int K = c->cfg.accumulation;
  auto hop = [&](int q, const W* in, W* out, int combine) {
    const std::vector<int>& qb = c->hopx_bucket_begin[static_cast<size_t>(q)];
    const int t0 = qb[static_cast<size_t>(b0)], t1 = qb[static_cast<size_t>(b1)];
    if (t1 > t0) {
      StageTimer timer(c, BO_STAGE_FLAG, st);
      auto go = [&](auto kern) {
        kern<<<t1 - t0, kThreads, 0, st>>>(c->d_hopx_tiles + t0, c->d_tensors, tab, c->ms, c->acc, c->state, K,
                                           in, out, combine);
      };
      switch (c->ms.K) {
        case 0: go(k_hopx<W, 0>); break;
        case 2: go(k_hopx<W, 2>); break;
        case 3: go(k_hopx<W, 3>); break;
        case 4: go(k_hopx<W, 4>); break;
        case 5: go(k_hopx<W, 5>); break;
        case 6: go(k_hopx<W, 6>); break;
        case 7: go(k_hopx<W, 7>); break;
        case 8: go(k_hopx<W, 8>); break;
        default: fail(BO_ERR_INVALID_CONFIG, "resident micro count outside 2..8");
      }
      check_launch(c, "k_hopx");
    }
  };
  // The last hop completes the owned chunk. It can run inside LAMB phase 1
  // (k_p1w<W, true, true>), which then reads the left neighbour's partial
  // directly: one staged write + read of the chunk less, but the NVLink
  // latency is exposed inside an HBM-bound kernel. Measured on BERT-large
  // (profiles/r01_notes.md): a net win at world 2 (1.10 vs 1.18 ms), a loss
  // at world 4 (0.67 vs 0.62 ms), so the default fuses only at world 2 —
  // and never in the overlapped sync micro, where a staged last hop runs
  // under the caller's backward instead of inside the exposed LAMB.
  // That is the pull form (BO_RING_PUSH=0), where it also never fuses with
  // resident micros (staged measured 2.93 vs 3.13 ms per step at world 2).
  // The push form (default) fuses at every world size, resident micros
  // included (world 2: 2.50 vs 2.65 ms, world 4: 2.84 vs 2.89 ms).
  const bool p2p = c->peer_wire[0][left] && !c->ring_via_nccl;
  const bool push = p2p && c->ring_push;
  // Push form: the last hop's input is local (what the left neighbour
  // pushed), so fusing it into phase 1 costs no NVLink latency there; it is
  // fused with the per-micro accumulator or K = 2 / 4 resident micros.
  const bool fuse_ok = push ? (c->ms.K == 0 || c->ms.K == 2 || c->ms.K == 4) : c->ms.K == 0;
  const bool fuse_default = push ? c->fuse_push_default : N == 2;
  const bool fuse_last = !c->force_unfused && fuse_ok &&
                         (c->fuse_last_hop >= 0 ? c->fuse_last_hop != 0 : (fuse_default && !c->sync_open));
  c->path |= p2p ? BO_PATH_RING_P2P : BO_PATH_RING_SENDRECV;
  if (push) {
    // Push form: every hop writes its output straight into the RIGHT
    // neighbour's staging buffer over NVLink and reads its input locally
    // (what the left neighbour pushed). With every rank sending and
    // receiving at once, NVLink stores sustain ~700 GB/s per direction where
    // remote reads (the pull form below) stall at ~540 GB/s. The barrier
    // before each hop orders the pushes into a buffer before its reader and
    // its reader before the next push into it; the last hop completes this
    // rank's owned chunk locally.
    // Hop 0 writes into the right neighbour's staging buffer 0 without a
    // barrier of its own. Write-after-read safety against that neighbour's
    // previous step (whose fused last hop, or unfused hop N-1, read that
    // buffer in place) comes from the previous step's partials barrier in
    // k_trust: this rank only gets here after every rank has published its
    // partials, i.e. after every rank's phase 1 — the last reader — finished
    // (tests/test_ring_protocol.py checks two consecutive steps). In the
    // overlapped sync micro the hops run on comm_stream after an event on
    // the context stream, which carries that same k_trust.
    hop(r, nullptr, static_cast<W*>(c->peer_wire[0][right]), 0);
    c->path |= BO_PATH_RING_PUSH;
    for (int s = 0; s < N - 1; ++s) {
      hop_barrier(c, st);
      const W* in = static_cast<const W*>(c->wire[s % 2]);
      if (s == N - 2 && fuse_last) {
        c->ring_last_in = in;  // the last hop runs inside LAMB phase 1, reading locally
        c->path |= BO_PATH_LAST_HOP_FUSED;
        return;
      }
      W* out = s == N - 2 ? static_cast<W*>(c->wire[(s + 1) % 2]) : static_cast<W*>(c->peer_wire[(s + 1) % 2][right]);
      hop((r - s - 1 + 2 * N) % N, in, out, 1);  // chunk added at hop s (collective.hpp:70-71)
    }
    c->ring_result = c->wire[(N - 1) % 2];
    return;
  }
  hop(r, nullptr, a, 0);  // hop 0 payload: this rank's own chunk r (collective.cpp:52)
  if (p2p) {
    // Peer-to-peer hops: hop s reads the left neighbour's hop s-1 output in
    // place over NVLink (CUDA IPC mapping) and writes the other local buffer.
    // A 4-byte all-reduce before each hop is the barrier that orders a
    // buffer's writer before its reader and its reader before its next writer
    // (buckets of different groups occupy disjoint positions).
    for (int s = 0; s < N - 1; ++s) {
      hop_barrier(c, st);
      const W* in = static_cast<const W*>(c->peer_wire[s % 2][left]);
      if (s == N - 2 && fuse_last) {
        c->ring_last_in = in;  // the last hop runs inside LAMB phase 1
        c->path |= BO_PATH_LAST_HOP_FUSED;
        return;
      }
      W* out = static_cast<W*>(c->wire[(s + 1) % 2]);
      hop((r - s - 1 + 2 * N) % N, in, out, 1);  // chunk added at hop s (collective.hpp:70-71)
    }
    c->ring_result = c->wire[(N - 1) % 2];
  } else {
    need_nccl(c, "ring hops over ncclSend/ncclRecv (BO_RING_NCCL=1)");
    for (int s = 0; s < N - 1; ++s) {
      BO_NCCL(ncclGroupStart());
      BO_NCCL(ncclSend(a + sh0, static_cast<size_t>(sh1 - sh0), dt, right, c->comm, st));
      BO_NCCL(ncclRecv(b + sh0, static_cast<size_t>(sh1 - sh0), dt, left, c->comm, st));
      BO_NCCL(ncclGroupEnd());
      if (s == N - 2 && fuse_last) {
        c->ring_last_in = b;
        c->path |= BO_PATH_LAST_HOP_FUSED;
        return;
      }
      hop((r - s - 1 + 2 * N) % N, b, a, 1);  // chunk received at hop s (collective.hpp:70-71)
    }
    c->ring_result = a;
  }
  // Unfused: after N-1 hops the result buffer holds the finished chunk
  // (r+1) % N, already wire-rounded (the owner re-round of
  // collective.cpp:79-83): the chunk this rank owns (Layout::own). LAMB
  // reads it in place.
}

static void nccl_reduce_scatter(bo_ctx* c, int b0, int b1, cudaStream_t st) {
  need_nccl(c, "the NCCL reduce-scatter (BO_REDUCE_NCCL)");
  c->path |= BO_PATH_NCCL_RS;
  BO_NCCL(ncclGroupStart());
  for (int b = b0; b < b1; ++b) {
    if (c->L.chunk[static_cast<size_t>(b)] == 0) continue;  // a bucket of empty tensors
    BO_NCCL(ncclReduceScatter(c->x + c->L.base[static_cast<size_t>(b)], c->gshard + c->L.shoff[static_cast<size_t>(b)],
                              static_cast<size_t>(c->L.chunk[static_cast<size_t>(b)]), ncclFloat, ncclSum,
                              c->comm, st));
  }
  BO_NCCL(ncclGroupEnd());
}

// NVLink bytes this rank sends for buckets [b0, b1): (N-1) hops of one chunk each
static uint64_t comm_bytes(const bo_ctx* c, int b0, int b1) {
  const size_t e = c->algo == BO_REDUCE_RING && c->cfg.f16_exchange ? 2 : 4;
  uint64_t n = 0;
  for (int b = b0; b < b1; ++b) n += static_cast<uint64_t>(c->L.chunk[static_cast<size_t>(b)]);
  return n * static_cast<uint64_t>(c->world - 1) * e;
}

void run_reduce(bo_ctx* c, const PtrTable& tab) {
  if (c->world == 1) return;
  StageTimer timer(c, BO_STAGE_REDUCE);
  const uint64_t bytes = comm_bytes(c, 0, c->L.B);
  trace(c, "comm_start", bytes, c->stream);
  struct End {
    bo_ctx* c;
    uint64_t bytes;
    ~End() {
      try {
        trace(c, "comm_end", bytes, c->stream);
      } catch (...) {  // a failing event record must not escape a destructor
      }
    }
  } end{c, bytes};
  c->ring_last_in = nullptr;
  c->ring_result = nullptr;
  if (c->algo == BO_REDUCE_NCCL) {
    nccl_reduce_scatter(c, 0, c->L.B, c->stream);
  } else if (c->cfg.f16_exchange) {
    ring_reduce_scatter<uint16_t>(c, tab, ncclFloat16, 0, c->L.B, c->stream);
  } else {
    ring_reduce_scatter<float>(c, tab, ncclFloat32, 0, c->L.B, c->stream);
  }
}

void run_reduce_group(bo_ctx* c, const PtrTable& tab, int b0, int b1, int acc0, int acc1,
                      cudaStream_t stream) {
  StageTimer timer(c, BO_STAGE_REDUCE, stream);
  const uint64_t bytes = comm_bytes(c, b0, b1);
  trace(c, "comm_start", bytes, stream);
  struct End {
    bo_ctx* c;
    uint64_t bytes;
    cudaStream_t s;
    ~End() {
      try {
        trace(c, "comm_end", bytes, s);
      } catch (...) {
      }
    }
  } end{c, bytes, stream};
  if (c->algo == BO_REDUCE_NCCL) {
    launch_finalize_tiles(c, c->d_group_acc_tiles + acc0, acc1 - acc0, tab, stream);
    nccl_reduce_scatter(c, b0, b1, stream);
  } else if (c->cfg.f16_exchange) {
    ring_reduce_scatter<uint16_t>(c, tab, ncclFloat16, b0, b1, stream);
  } else {
    ring_reduce_scatter<float>(c, tab, ncclFloat32, b0, b1, stream);
  }
}

// ------------------------------------------------- operator drop-ins
// ring_allreduce<float> / ring_allreduce_f16_wire (collective.hpp:53-99,
// collective.cpp:37-86) on caller device data, over the context's mapped ring
// staging buffers (CUDA IPC / NVLink) in push form: every hop writes its
// output straight into the right neighbour's staging buffer and a neighbour
// barrier orders it before the reader. Chunk k = ceil(n/N) elements, zero
// padded (collective.hpp:44-60), folded over ranks k, k+1, ..., k-1 with the
// wire rounding per hop; the owner's chunk is re-rounded (collective.cpp:79-83)
// and the all-gather forwards the owner's wire bits, so every rank ends with
// the same bits. Chunks larger than the staging buffers run in slices of the
// chunk (the fold order per element is unchanged).
namespace {
template <typename W>
__global__ void k_op_rs(const float* __restrict__ data, int64_t n, int64_t base, int64_t len,
                        const W* __restrict__ in, W* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = base + e;
    const float x = i < n ? data[i] : 0.0f;  // zero padding past n
    out[e] = to_wire<W>(in ? __fadd_rn(from_wire(in[e]), x) : x);
  }
}
// The owner: the chunk's last addition, its wire rounding (the owner
// re-round), and the first all-gather push.
template <typename W>
__global__ void k_op_own(float* __restrict__ data, int64_t n, int64_t base, int64_t len,
                         const W* __restrict__ in, W* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = base + e;
    const W w = to_wire<W>(__fadd_rn(from_wire(in[e]), i < n ? data[i] : 0.0f));
    out[e] = w;
    if (i < n) data[i] = from_wire(w);
  }
}
// All-gather: store the chunk received from the left and forward its bits
// (out == nullptr: the last hop, store only).
template <typename W>
__global__ void k_op_fwd(float* __restrict__ data, int64_t n, int64_t base, int64_t len,
                         const W* __restrict__ in, W* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const W w = in[e];
    if (out) out[e] = w;
    if (base + e < n) data[base + e] = from_wire(w);
  }
}
int op_grid(int64_t len) {
  return static_cast<int>(std::min<int64_t>(std::max<int64_t>((len + kThreads - 1) / kThreads, 1), 148 * 8));
}
}  // namespace

bool ring_op_available(const bo_ctx* c) {
  return c->world > 1 && c->peers_mapped && c->wire[0] && c->peer_wire[0][(c->rank + 1) % c->world] &&
         !c->ring_via_nccl;
}

template <typename W>
static void ring_allreduce_op_t(bo_ctx* c, float* data, size_t n) {
  const int N = c->world, r = c->rank, right = (r + 1) % N;
  if (c->sync_open) fail(BO_ERR_PROTOCOL, "bo_ring_allreduce_* while a sync micro (bo_sync_ready) is open");
  cudaStream_t st = c->stream;
  const int64_t ch = static_cast<int64_t>((n + static_cast<size_t>(N) - 1) / static_cast<size_t>(N));
  const size_t wire_bytes = static_cast<size_t>(c->L.shard_total) * (c->cfg.f16_exchange ? 2 : 4);
  const int64_t cap = static_cast<int64_t>(wire_bytes / sizeof(W));
  if (cap <= 0) fail(BO_ERR_INVALID_CONFIG, "ring staging buffers are empty");
  W* mine[2] = {static_cast<W*>(c->wire[0]), static_cast<W*>(c->wire[1])};
  W* theirs[2] = {static_cast<W*>(c->peer_wire[0][right]), static_cast<W*>(c->peer_wire[1][right])};
  auto chunk = [&](int k) { return static_cast<int64_t>(((k % N) + N) % N) * ch; };
  for (int64_t o = 0; o < ch; o += cap) {
    const int64_t len = std::min(cap, ch - o);
    const int g = op_grid(len);
    // every neighbour is done with its staging buffers (previous slice,
    // operator call or step) before this rank pushes into them
    hop_barrier(c, st);
    int h = 0;  // hop counter: hop h pushes into the right's staging[h % 2]
    for (int s = 0; s < N - 1; ++s, ++h) {  // reduce-scatter (collective.hpp:65-80)
      if (s > 0) hop_barrier(c, st);
      k_op_rs<W><<<g, kThreads, 0, st>>>(data, static_cast<int64_t>(n), chunk(r - s) + o, len,
                                         s == 0 ? nullptr : mine[(h - 1) % 2], theirs[h % 2]);
      check_launch(c, "k_op_rs");
    }
    hop_barrier(c, st);
    k_op_own<W><<<g, kThreads, 0, st>>>(data, static_cast<int64_t>(n), chunk(r + 1) + o, len,
                                        mine[(h - 1) % 2], theirs[h % 2]);
    check_launch(c, "k_op_own");
    ++h;
    for (int t = 1; t < N; ++t, ++h) {  // all-gather (collective.hpp:83-96)
      hop_barrier(c, st);
      k_op_fwd<W><<<g, kThreads, 0, st>>>(data, static_cast<int64_t>(n), chunk(r - t + 1) + o, len,
                                          mine[(h - 1) % 2], t < N - 1 ? theirs[h % 2] : nullptr);
      check_launch(c, "k_op_fwd");
    }
  }
  // the neighbours' last reads are done before anything else pushes here
  hop_barrier(c, st);
}

void ring_allreduce_op(bo_ctx* c, float* data, size_t n, bool f16) {
  if (f16) {
    ring_allreduce_op_t<uint16_t>(c, data, n);
  } else {
    ring_allreduce_op_t<float>(c, data, n);
  }
}

}  // namespace bo
