// B200 gradient-to-update pipeline: accumulate / finalize kernels and the
// sharded (world > 1) LAMB with the fused parameter all-gather.
//
// Stage map onto the reference (proj/core/src, read-only):
//   k_accumulate     accum_[p][i] += g[i]                trainer.cpp:240-244
//   k_finalize       flatten_param: (live + accum) * inv trainer.cpp:186-203
//   (ring hops: bo_ring.cu; one rank's fused LAMB: bo_fused.cu)
//   k_p1w            lamb_step moments, u + fp64 norm partials on the shard
//                                                        lamb.cpp:59-73
//   k_norm_reduce / k_trust  trust ratio (lamb.cpp:75-79), found_inf and
//                    the loss scaler
//   k_shard_p2_push  w -= (lr * r) * u (lamb.cpp:80-81) + the push into
//                    every replica (the all-gather)
//   k_lamb_norms / k_lamb_update  one rank with unaligned inputs
//
// Bit-level contract: every float operation uses an
// explicit round-to-nearest intrinsic and the file is compiled with
// --fmad=false, so nothing contracts into an FMA the reference does not have.
#include <cuda_fp16.h>

#include <chrono>

#include "bo_device.cuh"
#include "bo_internal.hpp"

namespace bo {
namespace {

// ------------------------------------------------------------ accumulate
// acc = (micro == 0 ? 0 + g : acc + g) over one tensor slice; 16-byte loads of
// 8 binary16 values, 2 x 16-byte fp32 accesses (trainer.cpp:240-244: the
// accumulator starts at 0.0f, so -0 becomes +0 exactly as in the reference).
template <bool kVec>
__global__ void __launch_bounds__(kThreads) k_accumulate(const AccTile* __restrict__ tiles,
                                                         const TensorDev* __restrict__ td,
                                                         const __grid_constant__ PtrTable tab,
                                                         float* __restrict__ acc, int first,
                                                         DevState* __restrict__ st, int reverse) {
  // reverse: the last micro before the sync micro walks the tiles backwards,
  // so the accumulator lines still in L2 when it ends are the ones the sync
  // micro's first CTAs read (and then drop from L2, see k_lamb_p1)
  const AccTile tile = tiles[reverse ? gridDim.x - 1 - blockIdx.x : blockIdx.x];
  const uint16_t* __restrict__ src = tab.p[tile.t] + tile.e0;
  float* __restrict__ dst = acc + td[tile.t].acc_off + tile.e0;
  const int len = tile.len;
  int done = 0;
  bool bad = false;
  if (kVec) {
    const int nvec = len >> 3;
#pragma unroll 2
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      const uint4 hv = __ldcs(reinterpret_cast<const uint4*>(src) + i);
      float4* d4 = reinterpret_cast<float4*>(dst) + 2 * i;
      float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
      if (!first) {
        a0 = d4[0];
        a1 = d4[1];
      }
      bad |= pair_nonfinite(hv.x) | pair_nonfinite(hv.y) | pair_nonfinite(hv.z) |
             pair_nonfinite(hv.w);
      const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
      float g[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        g[2 * j] = widen(static_cast<uint16_t>(hw[j] & 0xFFFFu));
        g[2 * j + 1] = widen(static_cast<uint16_t>(hw[j] >> 16));
      }
      a0.x = __fadd_rn(a0.x, g[0]); a0.y = __fadd_rn(a0.y, g[1]);
      a0.z = __fadd_rn(a0.z, g[2]); a0.w = __fadd_rn(a0.w, g[3]);
      a1.x = __fadd_rn(a1.x, g[4]); a1.y = __fadd_rn(a1.y, g[5]);
      a1.z = __fadd_rn(a1.z, g[6]); a1.w = __fadd_rn(a1.w, g[7]);
      d4[0] = a0;
      d4[1] = a1;
    }
    done = nvec << 3;
  }
  for (int i = done + threadIdx.x; i < len; i += kThreads) {
    const float a = first ? 0.0f : dst[i];
    const float g = widen(src[i]);
    bad |= !finite(g);
    dst[i] = __fadd_rn(a, g);
  }
  raise_flag(bad, st);
}

// -------------------------------------------------------------- finalize
// The sync micro's flatten_param (trainer.cpp:186-203): v = live (+ summed),
// dst = v * inv with inv = 1/(K*S) in float, S the current (device) scale.
// Writes the fusion-buffer position of every element (the packer).
// KR > 0 (bo_train_step): v = the KR resident micros' sum in the reference's
// order (live + ((0 + g0) + ... + g_{K-2})), no accumulator.
template <int KR>
__global__ void __launch_bounds__(kThreads) k_finalize(const AccTile* __restrict__ tiles,
                                                       const TensorDev* __restrict__ td,
                                                       const __grid_constant__ PtrTable tab, MicroSrc ms,
                                                       const float* __restrict__ acc,
                                                       float* __restrict__ x,
                                                       const DevState* __restrict__ st, int K) {
  const AccTile tile = tiles[blockIdx.x];
  const float inv = __fdiv_rn(1.0f, __fmul_rn(static_cast<float>(K), st->scale));
  const uint16_t* __restrict__ src = tab.p[tile.t] + tile.e0;
  const float* __restrict__ a = acc + td[tile.t].acc_off + tile.e0;
  float* __restrict__ dst = x + td[tile.t].flat_off + tile.e0;
  if constexpr (KR > 0) {
    __shared__ const uint16_t* mp[KR];
    if (static_cast<int>(threadIdx.x) < KR) mp[threadIdx.x] = ms.hk[threadIdx.x * ms.T + tile.t] + tile.e0;
    __syncthreads();
    if ((td[tile.t].flat_off & 3) == 0) {  // resident slots are 16-byte aligned (bo_train_step)
      const int nv = tile.len >> 2;
#pragma unroll 2
      for (int q = threadIdx.x; q < nv; q += kThreads) {
        float g[4];
        micro_sum4_k<KR>(mp, 4 * q, g);
        reinterpret_cast<float4*>(dst)[q] = make_float4(__fmul_rn(g[0], inv), __fmul_rn(g[1], inv),
                                                        __fmul_rn(g[2], inv), __fmul_rn(g[3], inv));
      }
      for (int e = 4 * nv + threadIdx.x; e < tile.len; e += kThreads) dst[e] = __fmul_rn(micro_sum1(mp, KR, e), inv);
    } else {
      for (int e = threadIdx.x; e < tile.len; e += kThreads) dst[e] = __fmul_rn(micro_sum1(mp, KR, e), inv);
    }
    return;
  }
  if (((td[tile.t].flat_off & 3) | (reinterpret_cast<uintptr_t>(tab.p[tile.t]) & 15)) == 0) {
    // the tensor's fusion-buffer offset is 16-byte aligned: float4 path
    const int nv = tile.len >> 2;
#pragma unroll 4
    for (int q = threadIdx.x; q < nv; q += kThreads) {
      const uint2 hv = __ldcs(reinterpret_cast<const uint2*>(src) + q);
      float g[4] = {widen(static_cast<uint16_t>(hv.x & 0xFFFFu)), widen(static_cast<uint16_t>(hv.x >> 16)),
                    widen(static_cast<uint16_t>(hv.y & 0xFFFFu)), widen(static_cast<uint16_t>(hv.y >> 16))};
      if (K > 1) {
        const float4 a4 = __ldcs(reinterpret_cast<const float4*>(a) + q);
        g[0] = __fadd_rn(g[0], a4.x);
        g[1] = __fadd_rn(g[1], a4.y);
        g[2] = __fadd_rn(g[2], a4.z);
        g[3] = __fadd_rn(g[3], a4.w);
      }
      reinterpret_cast<float4*>(dst)[q] = make_float4(__fmul_rn(g[0], inv), __fmul_rn(g[1], inv),
                                                      __fmul_rn(g[2], inv), __fmul_rn(g[3], inv));
    }
    for (int e = 4 * nv + threadIdx.x; e < tile.len; e += kThreads) {
      const float g = widen(src[e]);
      dst[e] = __fmul_rn(K > 1 ? __fadd_rn(g, a[e]) : g, inv);
    }
    return;
  }
  constexpr int kPer = kTileElems / kThreads;
  float gv[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * kThreads;
    gv[j] = 0.0f;
    if (e < tile.len) {
      const float g = widen(__ldcs(src + e));
      gv[j] = K > 1 ? __fadd_rn(g, __ldcs(a + e)) : g;
    }
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * kThreads;
    if (e < tile.len) dst[e] = __fmul_rn(gv[j], inv);
  }
}

// ------------------------------------------------------------------- LAMB
// Phase 1: per-tile fp64 partials of ||w||^2 and ||u||^2 and the non-finite
// flag of the reduced gradient (lamb.cpp:59-73; the flag is the
// NonFiniteGradient condition, lamb.cpp:61-65). Nothing is written to w/m/v.
template <typename G>
__global__ void __launch_bounds__(kThreads) k_lamb_norms(const LambTile* __restrict__ tiles,
                                                         const G* __restrict__ g,
                                                         const float* __restrict__ w,
                                                         const float* m0, const float* v0,
                                                         const float* m1, const float* v1,
                                                         DevState* __restrict__ st, LambConsts c,
                                                         const double* __restrict__ bc_table,
                                                         float invn, int scale_g,
                                                         double* __restrict__ tile_part) {
  const LambTile tile = tiles[blockIdx.x];
  const float* __restrict__ m = st->parity ? m1 : m0;  // current moment buffers
  const float* __restrict__ v = st->parity ? v1 : v0;
  __shared__ double bc[4];
  __shared__ double red[2][kThreads / 32];
  __shared__ int bad_any;
  if (threadIdx.x < 4) bc[threadIdx.x] = bc_table[4 * st->lamb_step + threadIdx.x];
  if (threadIdx.x == 0) bad_any = 0;
  __syncthreads();
  constexpr int kPer = kTileElems / kThreads;
  double wn = 0.0, un = 0.0;
  bool bad = false;
#pragma unroll 4
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * kThreads;
    if (e < tile.len) {
      float gi = from_wire(__ldcs(g + tile.s0 + e));
      if (scale_g) gi = __fmul_rn(gi, invn);
      const float wi = w[tile.w0 + e];
      bad |= !finite(gi);
      const Moments o = lamb_elem(gi, wi, __ldcs(m + tile.s0 + e), __ldcs(v + tile.s0 + e), c, bc);
      wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wi), static_cast<double>(wi)));
      un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u), static_cast<double>(o.u)));
    }
  }
  wn = warp_sum(wn);
  un = warp_sum(un);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = wn;
    red[1][wid] = un;
  }
  if (bad) bad_any = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      a += red[0][i];
      b += red[1][i];
    }
    tile_part[2 * blockIdx.x] = a;
    tile_part[2 * blockIdx.x + 1] = b;
    if (bad_any) atomicOr(&st->local_flag, 1);
  }
}

// Per-tensor sums of the tile partials in a fixed order (deterministic), plus
// this rank's flag, into rank_part[2T+1] — or, world > 1, straight into this
// rank's slot of every rank's all_part over NVLink (CUDA IPC): the partials
// all-gather without a collective; k_trust's barrier then orders these
// stores before every reader.
__global__ void __launch_bounds__(kThreads) k_norm_reduce(const int* __restrict__ tile_begin,
                                                          const double* __restrict__ tile_part,
                                                          const DevState* __restrict__ st, int T,
                                                          double* __restrict__ rank_part,
                                                          const PartDst dst, int t_first = 0) {
  const int t = t_first + static_cast<int>(blockIdx.x);  // grouped LAMB: tensors [t_first, ...)
  const int b0 = tile_begin[t], b1 = tile_begin[t + 1];
  double a = 0.0, b = 0.0;
  for (int i = b0 + threadIdx.x; i < b1; i += kThreads) {
    a += tile_part[2 * i];
    b += tile_part[2 * i + 1];
  }
  __shared__ double red[2][kThreads];
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x < (dst.n > 0 ? dst.n : 1)) {
    double* out = dst.n > 0 ? dst.p[threadIdx.x] : rank_part;
    out[2 * t] = red[0][0];
    out[2 * t + 1] = red[1][0];
    if (blockIdx.x == 0) out[2 * T] = st->local_flag ? 1.0 : 0.0;  // (cumulative over groups)
  }
}

// One thread: publish `epoch` into slot `rank` of every rank's flag block
// (after the stores of this stream's previous kernels, which have completed)
// and wait until every rank has published it into this rank's block. Bounded
// by the watchdog: a rank that never arrives sets peer_timeout and the step is
// abandoned (no update, scaler untouched); bo_wait reports PeerDisconnected.
// Returns false on timeout (or when an earlier barrier of the step timed out).
__device__ bool all_rank_barrier(const PeerFlags& pf, int slot0, unsigned epoch, DevState* st,
                                 uint64_t timeout_ns) {
  if (st->peer_timeout) return false;
  __threadfence_system();
  for (int j = 0; j < pf.n; ++j) {
    unsigned* f = pf.f[j] + slot0 + pf.rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
  const unsigned* mine = pf.f[pf.rank] + slot0;
  const uint64_t t0 = global_ns();
  for (int j = 0; j < pf.n; ++j) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + j) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (global_ns() - t0 > timeout_ns) {
        st->peer_timeout = 1;
        return false;
      }
      __nanosleep(32);
    }
  }
  return true;
}

// End-of-step barrier: every rank's parameter push into every replica has
// landed (each rank publishes after its k_shard_p2_push completed).
__global__ void k_step_end_barrier(PeerFlags pf, unsigned epoch, DevState* st, uint64_t timeout_ns) {
  all_rank_barrier(pf, kCtrlStepEnd, epoch, st, timeout_ns);
}

// Global decision: found_inf = any rank flagged; trust ratios from the
// rank-ordered sums (identical on every rank); LAMB step counter; dynamic
// loss-scaler state machine.
// world > 1: first the partials barrier (every rank's k_norm_reduce stored
// its partials into this rank's all_part), then the sums.
// Grouped LAMB (group_mode, tensors [t0, t1)): the barrier and that group's
// trust ratios only, computed whatever the flags (the push of the group is
// speculative); the step's decision and state update is k_step_final's.
__global__ void __launch_bounds__(1024) k_trust(const double* __restrict__ all_part, int N, int T,
                                                DevState* __restrict__ st, LambConsts c,
                                                ScalerConsts sc, float* __restrict__ trust,
                                                int flip_parity, PeerFlags pf, unsigned epoch,
                                                uint64_t timeout_ns, int group_mode = 0, int t0 = 0,
                                                int t1 = 0) {
  __shared__ int found, abandoned;
  if (group_mode) {
    if (threadIdx.x == 0) abandoned = pf.n > 0 && !all_rank_barrier(pf, kCtrlPartials, epoch, st, timeout_ns);
    __syncthreads();
    if (abandoned) return;
    for (int t = t0 + static_cast<int>(threadIdx.x); t < t1; t += blockDim.x) {
      double W = 0.0, U = 0.0;
      for (int r = 0; r < N; ++r) {
        W = __dadd_rn(W, __ldcv(all_part + static_cast<size_t>(r) * (2 * T + 1) + 2 * t));
        U = __dadd_rn(U, __ldcv(all_part + static_cast<size_t>(r) * (2 * T + 1) + 2 * t + 1));
      }
      float r = 1.0f;
      if (W > 0.0 && U > 0.0) {
        r = __double2float_rn(__ddiv_rn(__dsqrt_rn(W), __dsqrt_rn(U)));
        r = fminf(fmaxf(r, 0.0f), c.clip);
      }
      trust[t] = r;
    }
    return;
  }
  if (threadIdx.x == 0) {
    st->epoch = epoch;
    abandoned = pf.n > 0 && !all_rank_barrier(pf, kCtrlPartials, epoch, st, timeout_ns);
    int f = 0;
    for (int r = 0; r < N; ++r) f |= __ldcv(all_part + static_cast<size_t>(r) * (2 * T + 1) + 2 * T) != 0.0;
    found = f;
  }
  __syncthreads();
  if (abandoned) {
    // a peer never arrived: no update, step counters and scaler untouched
    if (threadIdx.x == 0) {
      st->do_update = 0;
      st->local_flag = 0;
    }
    return;
  }
  if (!found) {
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      double W = 0.0, U = 0.0;
      for (int r = 0; r < N; ++r) {
        W = __dadd_rn(W, __ldcv(all_part + static_cast<size_t>(r) * (2 * T + 1) + 2 * t));
        U = __dadd_rn(U, __ldcv(all_part + static_cast<size_t>(r) * (2 * T + 1) + 2 * t + 1));
      }
      float r = 1.0f;
      if (W > 0.0 && U > 0.0) {
        r = __double2float_rn(__ddiv_rn(__dsqrt_rn(W), __dsqrt_rn(U)));
        r = fminf(fmaxf(r, 0.0f), c.clip);
      }
      trust[t] = r;
    }
  }
  if (threadIdx.x == 0) {
    st->found_inf = found;
    st->do_update = !found;
    st->steps += 1;
    st->local_flag = 0;
    if (found) {
      st->skipped += 1;
    } else {
      st->lamb_step += 1;
      if (flip_parity) st->parity ^= 1;  // double-buffered moments written by phase 1
    }
    if (sc.dynamic) {
      if (found) {
        st->scale = fmaxf(__fmul_rn(st->scale, sc.backoff), sc.min_scale);
        st->good = 0;
      } else if (++st->good == sc.interval) {
        st->scale = fminf(__fmul_rn(st->scale, sc.growth), sc.max_scale);
        st->good = 0;
      }
    }
  }
}

// Phase 2: recompute the element (bit-identical to phase 1) and apply
// w -= (lr * r) * u, storing w, m, v (lamb.cpp:80-81). Skipped steps exit.
template <typename G>
__global__ void __launch_bounds__(kThreads) k_lamb_update(const LambTile* __restrict__ tiles,
                                                          const G* __restrict__ g,
                                                          float* __restrict__ w,
                                                          float* m0, float* v0, float* m1,
                                                          float* v1,
                                                          const DevState* __restrict__ st,
                                                          LambConsts c,
                                                          const double* __restrict__ bc_table,
                                                          float invn, int scale_g,
                                                          const float* __restrict__ trust) {
  if (!st->do_update) return;
  const LambTile tile = tiles[blockIdx.x];
  float* __restrict__ m = st->parity ? m1 : m0;  // current moment buffers (updated in place)
  float* __restrict__ v = st->parity ? v1 : v0;
  __shared__ double bc[4];
  if (threadIdx.x < 4) bc[threadIdx.x] = bc_table[4 * (st->lamb_step - 1) + threadIdx.x];
  __syncthreads();
  const float step_scale = __fmul_rn(c.lr, trust[tile.t]);
  constexpr int kPer = kTileElems / kThreads;
#pragma unroll 4
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * kThreads;
    if (e < tile.len) {
      float gi = from_wire(__ldcs(g + tile.s0 + e));
      if (scale_g) gi = __fmul_rn(gi, invn);
      const float wi = w[tile.w0 + e];
      const Moments o = lamb_elem(gi, wi, m[tile.s0 + e], v[tile.s0 + e], c, bc);
      w[tile.w0 + e] = __fsub_rn(wi, __fmul_rn(step_scale, o.u));
      m[tile.s0 + e] = o.m;
      v[tile.s0 + e] = o.v;
    }
  }
}

// ------------------------------------------------ sharded LAMB (world > 1)
// All of g (the reduced shard, wire type G), wsh, m, v and u share the shard
// layout, so a tile is split into a scalar head up to the next 16-byte
// boundary, an aligned float4 body and a scalar tail.
struct Split {
  int head, nv, tail;
};
__device__ __forceinline__ Split split_tile(int64_t s0, int len) {
  const int head = min(static_cast<int>((4 - (s0 & 3)) & 3), len);
  return Split{head, (len - head) >> 2, (len - head) & 3};
}
// ------------------------------------------------ phase 1 (world > 1)
// Phase 1 on this rank's shard: the reduced gradient g (trainer.cpp:212
// scaling), the NonFiniteGradient flag (lamb.cpp:61-65), m', v' into the other
// moment buffer set (double-buffered: found_inf is global, known only after
// every rank's phase 1), the update u, and per-tile fp64 partials of
// ||w||^2 and ||u||^2 (lamb.cpp:59-73).
struct P1Args {
  const TensorDev* td;
  const float* acc;
  int K;
  float invn;
  const float* wsh;
  float *m0, *v0, *m1, *v1, *u;
  const float* wsh_alt;  // grouped LAMB: the master shard is double-buffered (parity)
  DevState* st;
  LambConsts c;
  const double* bc_table;
  double* tile_part;
  MicroSrc ms;  // KR > 0: the resident micros (bo_train_step)
};

// Phase 1 with one WARP per tile (<= 4096 elements, up to 128 per lane): the
// tile's setup, its norm reduction (one warp_sum, no block barrier) and the
// flag are amortised over 16x more elements per thread than with a CTA per
// tile, which at 8 elements per thread spent about a quarter of its
// instructions on them (profiles/r01_notes.md).
//   kIn && kX : the fused last ring hop, g = wire(in + x) / N
//   kIn       : the staged ring / NCCL shard, g = in / N
//   kX        : one rank, g = x
// with x = (h + acc) * inv from the sync micro's binary16 gradient and the
// accumulator (flatten_param, trainer.cpp:186-203).
constexpr int kWarpTileCTA = 256;
// KR > 0 (with kX): x from the KR resident micros in the reference's order
// instead of h + acc.
template <typename W, bool kIn, bool kX, int U = 2, int kMinBlocks = 4, int KR = 0, bool kDbl = false>
__global__ void __launch_bounds__(kWarpTileCTA, kMinBlocks) k_p1w(const LambTile* __restrict__ tiles,
                                                          int n_tiles,
                                                          const __grid_constant__ PtrTable tab,
                                                          const W* __restrict__ in, P1Args A) {
  static_assert(kIn || kX, "a gradient source");
  const int wt = static_cast<int>((blockIdx.x * kWarpTileCTA + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (wt >= n_tiles) return;
  DevState* __restrict__ st = A.st;
  // one rank: an earlier micro overflowed, the step is skipped
  if constexpr (!kIn) {
    if (st->local_flag) return;
  }
  const LambTile t = tiles[wt];
  const int par = st->parity;
  const float* __restrict__ m = par ? A.m1 : A.m0;
  const float* __restrict__ v = par ? A.v1 : A.v0;
  float* __restrict__ mn = par ? A.m0 : A.m1;
  float* __restrict__ vn = par ? A.v0 : A.v1;
  // kDbl (grouped LAMB): the master shard is double-buffered by parity
  // (an arithmetic select: a branchy one made ptxas spill 64 more bytes)
  const float* __restrict__ wsh =
      (kDbl ? reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(A.wsh) +
                                             (reinterpret_cast<uintptr_t>(A.wsh_alt) -
                                              reinterpret_cast<uintptr_t>(A.wsh)) * static_cast<uintptr_t>(par != 0))
           : A.wsh) + t.s0;
  float* __restrict__ u = A.u + t.s0;
  m += t.s0;
  v += t.s0;
  mn += t.s0;
  vn += t.s0;
  const W* __restrict__ gin = kIn ? in + t.s0 : nullptr;
  const double* bcp = A.bc_table + 4 * st->lamb_step;
  const double ibc1 = bcp[2], ibc2 = bcp[3];
  const int K = A.K;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const uint16_t* __restrict__ h = nullptr;
  const float* __restrict__ a = nullptr;
  float inv = 0.0f;
  bool vec = true;
  const uint16_t* hk[KR > 0 ? KR : 1];
  if constexpr (kX) {
    const TensorDev d = A.td[t.t];
    const int64_t e0t = t.w0 - d.flat_off;  // element offset of the tile inside its tensor
    h = tab.p[t.t] + e0t;
    a = A.acc + d.acc_off + e0t;
    inv = __fdiv_rn(1.0f, __fmul_rn(static_cast<float>(K), st->scale));
    vec = ((e0t - t.s0) & 3) == 0 && (reinterpret_cast<uintptr_t>(tab.p[t.t]) & 7) == 0;
    if constexpr (KR > 0) {
#pragma unroll
      for (int k = 0; k < KR; ++k) hk[k] = A.ms.hk[k * A.ms.T + t.t] + e0t;
      vec = ((e0t - t.s0) & 3) == 0;  // resident slots are 16-byte aligned (bo_train_step)
    }
  }
  // xs: the flattened gradient before the unscale (h + acc)
  auto grad = [&](float win, float xs) {
    if constexpr (kX) {
      const float x = __fmul_rn(xs, inv);
      if constexpr (kIn) {
        return __fmul_rn(from_wire(to_wire<W>(__fadd_rn(win, x))), A.invn);
      } else {
        return x;
      }
    } else {
      return __fmul_rn(win, A.invn);
    }
  };
  double wn = 0.0, un = 0.0;
  bool bad = false;
  auto scalar = [&](int e) {
    float xs = 0.0f, win = 0.0f;
    if constexpr (kX && KR > 0) {
      xs = micro_sum1(hk, KR, e);
    } else if constexpr (kX) {
      xs = widen(h[e]);
      if (K > 1) xs = __fadd_rn(xs, a[e]);
    }
    if constexpr (kIn) win = from_wire(gin[e]);
    const float gi = grad(win, xs);
    bad |= !finite(gi);
    const float wi = wsh[e];
    const Moments o = lamb_elem(gi, wi, m[e], v[e], A.c, bcp);
    mn[e] = o.m;
    vn[e] = o.v;
    u[e] = o.u;
    wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wi), static_cast<double>(wi)));
    un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u), static_cast<double>(o.u)));
  };
  if (!vec) {
    for (int e = lane; e < t.len; e += 32) scalar(e);
  } else {
    const Split sp = split_tile(t.s0, t.len);
    if (lane < sp.head) scalar(lane);
    if (lane >= 8 && lane - 8 < sp.tail) scalar(sp.head + 4 * sp.nv + lane - 8);
    for (int q0 = 0; q0 < sp.nv; q0 += 32 * U) {
      float iv[U][4], av[U][4];
      uint2 hv[U];
      uint2 hr[U][KR > 0 ? KR : 1];
      float4 wv[U], mv[U], vv[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int q = q0 + lane + 32 * j;
        if (q < sp.nv) {
          const int e = sp.head + 4 * q;
          if constexpr (kIn) {
            if constexpr (sizeof(W) == 2) {
              widen4(__ldcs(reinterpret_cast<const uint2*>(gin + e)), iv[j]);
            } else {
              const float4 x = __ldcs(reinterpret_cast<const float4*>(gin + e));
              iv[j][0] = x.x; iv[j][1] = x.y; iv[j][2] = x.z; iv[j][3] = x.w;
            }
          }
          if constexpr (kX && KR > 0) {
#pragma unroll
            for (int k = 0; k < KR; ++k) hr[j][k] = ld2u(hk[k] + e, pf);
          } else if constexpr (kX) {
            hv[j] = ld2u(h + e, pf);
            if (K > 1) {
              const float4 a4 = ld4(a + e, pf);
              av[j][0] = a4.x; av[j][1] = a4.y; av[j][2] = a4.z; av[j][3] = a4.w;
            }
          }
          wv[j] = ld4(wsh + e, pl);
          mv[j] = ld4(m + e, pf);
          vv[j] = ld4(v + e, pf);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int q = q0 + lane + 32 * j;
        if (q < sp.nv) {
          const int e = sp.head + 4 * q;
          const float wa[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
          const float ma[4] = {mv[j].x, mv[j].y, mv[j].z, mv[j].w};
          const float va[4] = {vv[j].x, vv[j].y, vv[j].z, vv[j].w};
          float ga[4];
          float xr[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          if constexpr (kX && KR > 0) {
            // live + (((0 + g0) + g1) + ... + g_{K-2}) (trainer.cpp:240-244, 196-201)
            float acc4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int k = 0; k + 1 < KR; ++k) {
              float f[4];
              widen4(hr[j][k], f);
#pragma unroll
              for (int i = 0; i < 4; ++i) acc4[i] = __fadd_rn(acc4[i], f[i]);
            }
            widen4(hr[j][KR - 1], xr);
#pragma unroll
            for (int i = 0; i < 4; ++i) xr[i] = __fadd_rn(xr[i], acc4[i]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float xs = 0.0f, win = 0.0f;
            if constexpr (kX && KR > 0) {
              xs = xr[i];
            } else if constexpr (kX) {
              const uint32_t hw = i < 2 ? hv[j].x : hv[j].y;
              xs = widen(static_cast<uint16_t>(hw >> (16 * (i & 1))));
              if (K > 1) xs = __fadd_rn(xs, av[j][i]);
            }
            if constexpr (kIn) win = iv[j][i];
            ga[i] = grad(win, xs);
            bad |= !finite(ga[i]);
          }
          const Lamb4 o = lamb_elem4(ga, wa, ma, va, A.c, bcp, ibc1, ibc2);
          st4(mn + e, make_float4(o.m[0], o.m[1], o.m[2], o.m[3]), pf);
          st4(vn + e, make_float4(o.v[0], o.v[1], o.v[2], o.v[3]), pf);
          st4(u + e, make_float4(o.u[0], o.u[1], o.u[2], o.u[3]), pl);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wa[i]), static_cast<double>(wa[i])));
            un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u[i]), static_cast<double>(o.u[i])));
          }
        }
      }
    }
  }
  wn = warp_sum(wn);
  un = warp_sum(un);
  if (lane == 0) {
    A.tile_part[2 * wt] = wn;
    A.tile_part[2 * wt + 1] = un;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&st->local_flag, 1);
}

// Phase 2 fused with the parameter all-gather: w -= (lr * r) * u on the
// master shard (lamb.cpp:80-81), and the new value written into every
// rank's flat parameter replica over NVLink (CUDA IPC mappings) at the
// element's fusion-buffer position. The replica writes are bulk asynchronous
// copies (cp.async.bulk, the TMA engine) from a shared-memory copy of the
// tile, staged at its 16-byte phase in the flat replica: one bulk copy per
// destination moves the aligned middle of the tile and the SMs only issue the
// <= 3 + 3 edge elements. The arithmetic reads the shard with 16-byte loads.
// Skipped steps exit.
__device__ __forceinline__ void bulk_s2g(float* gdst, const float* ssrc, uint32_t bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
// Parameter groups (bo_params_wait): the tiles run in model order, grouped by
// parameter group; the last CTA of group g to finish publishes "group g of
// step `epoch` landed in every replica" into slot `rank` of every rank's
// kCtrlReady[g] flags — after its own bulk copies completed and with a
// system-scope fence behind every CTA's stores of the group.
struct PushGroups {
  const int* group_of_tensor;
  const int* group_tiles;
  unsigned* count;
  PeerFlags pf;
  unsigned epoch;
};

// Thread 0, once every store of a finished tile has completed (bulk copies
// waited for, the CTA's edge stores ordered by a barrier): count the tile;
// the group's last tile publishes the group into every rank's flags.
__device__ __forceinline__ void push_tile_done(const PushGroups& G, int tensor) {
  __threadfence_system();
  const int g = G.group_of_tensor[tensor];
  const unsigned done = atomicAdd(G.count + g, 1u) + 1u;
  if (done % static_cast<unsigned>(G.group_tiles[g]) == 0u) {
    __threadfence_system();
    for (int j = 0; j < G.pf.n; ++j) {
      unsigned* f = G.pf.f[j] + kCtrlReady + 8 * g + G.pf.rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(G.epoch) : "memory");
    }
  }
}

// One CTA per tile (model order, so parameter groups complete front to back):
// the hardware keeps ~8 CTAs — 8 tiles' bulk copies — in flight per SM and
// launches the next CTA the moment one retires. Measured faster than every
// persistent form tried (two or four shared-memory tile buffers, TMA-fed
// input ring, 24-1184 CTAs: 20 % to 10x slower; profiles/r02_notes.md).
// Grouped LAMB (wsh_alt != null): speculative — runs before the step's
// decision, reads the current master shard (parity) and writes the other one
// (k_step_final flips, k_rollback undoes the replicas on a skipped step).
__global__ void __launch_bounds__(kThreads) k_shard_p2_push(const LambTile* __restrict__ tiles,
                                                            int n_tiles, float* wsh_main,
                                                            const float* __restrict__ u,
                                                            const DevState* __restrict__ st,
                                                            LambConsts c,
                                                            const float* __restrict__ trust,
                                                            float* const* __restrict__ peer_w,
                                                            int N, const PushGroups G,
                                                            float* wsh_alt = nullptr) {
  __shared__ __align__(128) float buf[kTileElems + 4];
  __shared__ float* dst[8];
  if (threadIdx.x < N) dst[threadIdx.x] = peer_w[threadIdx.x];
  const bool speculative = wsh_alt != nullptr;
  const bool update = speculative || st->do_update != 0;
  const int par = speculative ? st->parity : 0;
  const float* __restrict__ wsrc = par ? wsh_alt : wsh_main;
  float* __restrict__ wdst = speculative ? (par ? wsh_main : wsh_alt) : wsh_main;
  const int i = blockIdx.x;
  const LambTile t = tiles[i];
  __syncthreads();
  int64_t a0 = 0, a1 = 0;
  if (update && t.len > 0) {
    const float step_scale = __fmul_rn(c.lr, trust[t.t]);
    const int off = static_cast<int>(t.w0 & 3);  // buf[off + e] <-> flat element w0 + e
    const Split sp = split_tile(t.s0, t.len);
    auto one = [&](int e) {
      const int64_t s = t.s0 + e;
      const float nw = __fsub_rn(wsrc[s], __fmul_rn(step_scale, u[s]));
      wdst[s] = nw;
      buf[off + e] = nw;
    };
    if (static_cast<int>(threadIdx.x) < sp.head) one(threadIdx.x);
    if (threadIdx.x >= 32 && static_cast<int>(threadIdx.x) - 32 < sp.tail) {
      one(sp.head + 4 * sp.nv + static_cast<int>(threadIdx.x) - 32);
    }
    for (int q = threadIdx.x; q < sp.nv; q += kThreads) {
      const int e = sp.head + 4 * q;
      const int64_t s = t.s0 + e;
      const float4 w4 = *reinterpret_cast<const float4*>(wsrc + s);
      const float4 u4 = __ldcs(reinterpret_cast<const float4*>(u + s));
      const float4 n4 = make_float4(__fsub_rn(w4.x, __fmul_rn(step_scale, u4.x)),
                                    __fsub_rn(w4.y, __fmul_rn(step_scale, u4.y)),
                                    __fsub_rn(w4.z, __fmul_rn(step_scale, u4.z)),
                                    __fsub_rn(w4.w, __fmul_rn(step_scale, u4.w)));
      *reinterpret_cast<float4*>(wdst + s) = n4;
      buf[off + e] = n4.x;
      buf[off + e + 1] = n4.y;
      buf[off + e + 2] = n4.z;
      buf[off + e + 3] = n4.w;
    }
    // make the generic-proxy shared-memory writes visible to the bulk copies
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // flat elements [w0, w0 + len): aligned middle [a0, a1) by bulk copy
    a0 = (t.w0 + 3) & ~static_cast<int64_t>(3);
    a1 = (t.w0 + t.len) & ~static_cast<int64_t>(3);
    if (a1 > a0 && threadIdx.x == 0) {
      // destinations in a per-tile rotated order, so the CTAs of all ranks
      // spread their pushes over every peer's NVLink ingress at any moment
      for (int k = 0; k < N; ++k) {
        const int j = (i + k) % N;
        bulk_s2g(dst[j] + a0, buf + off + (a0 - t.w0), static_cast<uint32_t>(a1 - a0) * 4u);
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    // edges (and tiles shorter than one aligned 16-byte group)
    const int nhead = static_cast<int>(a1 > a0 ? a0 - t.w0 : t.len);
    const int ntail = static_cast<int>(a1 > a0 ? t.w0 + t.len - a1 : 0);
    if (static_cast<int>(threadIdx.x) < nhead * N) {
      const int e = threadIdx.x % nhead, j = threadIdx.x / nhead;
      dst[j][t.w0 + e] = buf[off + e];
    } else if (static_cast<int>(threadIdx.x) >= 128 && static_cast<int>(threadIdx.x) - 128 < ntail * N) {
      const int k = static_cast<int>(threadIdx.x) - 128;
      const int e = static_cast<int>(a1 - t.w0) + k % ntail, j = k / ntail;
      dst[j][t.w0 + e] = buf[off + e];
    }
  }
  // the shared-memory tile must outlive the copies (wait for their writes,
  // not only their smem reads, so the group count below covers them)
  __syncthreads();  // the edge stores
  if (threadIdx.x == 0) {
    if (a1 > a0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    push_tile_done(G, t.t);
  }
}

// bo_params_wait: one thread on the caller's stream waits until every rank
// published parameter group g of step `epoch` (bounded by the watchdog).
__global__ void k_params_wait(const unsigned* __restrict__ slots, int N, unsigned epoch,
                              DevState* st, uint64_t timeout_ns) {
  const uint64_t t0 = global_ns();
  for (int j = 0; j < N; ++j) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(slots + j) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (global_ns() - t0 > timeout_ns) {
        st->peer_timeout = 1;
        return;
      }
      __nanosleep(64);
    }
  }
}

// Owned chunk positions of the flat replica -> the master shard (load time).
// Grouped LAMB, after every group's speculative push: the step's decision
// from the last group's exchange (each rank's cumulative flag), then the same
// state transitions as k_trust — the parity flip now also makes the pushed
// master shard current.
__global__ void k_step_final(const double* __restrict__ all_part, int N, int T, DevState* st,
                             ScalerConsts sc, unsigned epoch) {
  st->epoch = epoch;
  if (st->peer_timeout) {  // abandoned: no update, counters and scaler untouched
    st->do_update = 0;
    st->local_flag = 0;
    return;
  }
  int found = 0;
  for (int r = 0; r < N; ++r) found |= __ldcv(all_part + static_cast<size_t>(r) * (2 * T + 1) + 2 * T) != 0.0;
  st->found_inf = found;
  st->do_update = !found;
  st->steps += 1;
  st->local_flag = 0;
  if (found) {
    st->skipped += 1;
  } else {
    st->lamb_step += 1;
    st->parity ^= 1;  // moments written by phase 1, master shard written by the push
  }
  if (sc.dynamic) {
    if (found) {
      st->scale = fmaxf(__fmul_rn(st->scale, sc.backoff), sc.min_scale);
      st->good = 0;
    } else if (++st->good == sc.interval) {
      st->scale = fminf(__fmul_rn(st->scale, sc.growth), sc.max_scale);
      st->good = 0;
    }
  }
}

// The parameter push as persistent CTAs with posted stores (grouped LAMB,
// BO_PUSH_POSTED_CTAS, default 128): each thread takes one float4 of a tile
// (grid-stride over the tiles, two in flight) and stores the new value into
// the master shard and — plain 16-byte stores, no completion wait — into
// every rank's replica (rotated per tile). Posted stores let even 24-64 CTAs
// of 1024 threads drive ~650-700 GB/s of NVLink while phase 1 of the next
// group streams HBM on the other SMs (tools/nvl_partition.cu,
// profiles/r02_notes.md); the one-CTA-per-tile bulk-copy push, which waits
// for its copies, needs every SM. Same arithmetic and destinations as
// k_shard_p2_push; tiles whose shard and replica 16-byte phases differ go
// scalar. Kernel completion performs the posted stores before the stream's
// next work (the end-of-step barrier, k_rollback).
constexpr int kPostThreads = 1024;
static_assert(kPostThreads * 4 == kTileElems, "one float4 per thread per tile");
__global__ void __launch_bounds__(kPostThreads, 1) k_push_posted(const LambTile* __restrict__ tiles,
                                                                 int n_tiles, float* wsh_main,
                                                                 const float* __restrict__ u,
                                                                 const DevState* __restrict__ st,
                                                                 LambConsts c,
                                                                 const float* __restrict__ trust,
                                                                 float* const* __restrict__ peer_w, int N,
                                                                 float* wsh_alt) {
  __shared__ float* dst[8];
  if (static_cast<int>(threadIdx.x) < N) dst[threadIdx.x] = peer_w[threadIdx.x];
  const bool speculative = wsh_alt != nullptr;
  const bool update = speculative || st->do_update != 0;
  const int par = speculative ? st->parity : 0;
  const float* __restrict__ wsrc = par ? wsh_alt : wsh_main;
  float* __restrict__ wdst = speculative ? (par ? wsh_main : wsh_alt) : wsh_main;
  __syncthreads();
  if (!update) return;
  // two tiles per iteration (i and i + G), all their loads issued first
  const int G = static_cast<int>(gridDim.x);
  for (int i0 = static_cast<int>(blockIdx.x); i0 < n_tiles; i0 += 2 * G) {
    float4 w4[2], u4[2];
    bool body[2] = {false, false};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = i0 + k * G;
      if (i >= n_tiles) continue;
      const LambTile t = tiles[i];
      if (((t.s0 - t.w0) & 3) != 0) continue;
      const Split sp = split_tile(t.s0, t.len);
      body[k] = static_cast<int>(threadIdx.x) < sp.nv;
      if (body[k]) {
        const int64_t s = t.s0 + sp.head + 4 * static_cast<int64_t>(threadIdx.x);
        w4[k] = *reinterpret_cast<const float4*>(wsrc + s);
        u4[k] = __ldcs(reinterpret_cast<const float4*>(u + s));
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = i0 + k * G;
      if (i >= n_tiles) continue;
      const LambTile t = tiles[i];
      const float sc = __fmul_rn(c.lr, trust[t.t]);
      auto one = [&](int e) {
        const int64_t s = t.s0 + e;
        const float nw = __fsub_rn(wsrc[s], __fmul_rn(sc, u[s]));
        wdst[s] = nw;
        for (int q = 0; q < N; ++q) dst[(i + q) % N][t.w0 + e] = nw;
      };
      if (((t.s0 - t.w0) & 3) != 0) {  // shard and replica 16-byte phases differ
        for (int e = threadIdx.x; e < t.len; e += kPostThreads) one(e);
        continue;
      }
      const Split sp = split_tile(t.s0, t.len);
      if (body[k]) {
        const int e = sp.head + 4 * static_cast<int>(threadIdx.x);
        const float4 n4 = make_float4(__fsub_rn(w4[k].x, __fmul_rn(sc, u4[k].x)),
                                      __fsub_rn(w4[k].y, __fmul_rn(sc, u4[k].y)),
                                      __fsub_rn(w4[k].z, __fmul_rn(sc, u4[k].z)),
                                      __fsub_rn(w4[k].w, __fmul_rn(sc, u4[k].w)));
        *reinterpret_cast<float4*>(wdst + t.s0 + e) = n4;
        for (int q = 0; q < N; ++q) __stcs(reinterpret_cast<float4*>(dst[(i + q) % N] + t.w0 + e), n4);
      }
      if (static_cast<int>(threadIdx.x) < sp.head) one(threadIdx.x);
      if (threadIdx.x >= 32 && static_cast<int>(threadIdx.x) - 32 < sp.tail) {
        one(sp.head + 4 * sp.nv + static_cast<int>(threadIdx.x) - 32);
      }
    }
  }
}


// A skipped (or abandoned) grouped step: the speculative pushes are undone by
// pushing the unchanged current master shard into every replica again. Exits
// at once on a normal step.
__global__ void __launch_bounds__(kThreads) k_rollback(const LambTile* __restrict__ tiles, int n_tiles,
                                                       const float* __restrict__ wsh0,
                                                       const float* __restrict__ wsh1,
                                                       float* const* __restrict__ peer_w, int N,
                                                       const DevState* __restrict__ st) {
  if (st->do_update) return;
  const float* __restrict__ wsh = st->parity ? wsh1 : wsh0;
  for (int i = blockIdx.x; i < n_tiles; i += gridDim.x) {
    const LambTile t = tiles[i];
    for (int e = threadIdx.x; e < t.len; e += blockDim.x) {
      const float v = wsh[t.s0 + e];
      for (int j = 0; j < N; ++j) peer_w[j][t.w0 + e] = v;
    }
  }
}

// Grouped LAMB: every parameter group is published once the step's decision
// (and any rollback) is final — the pushes themselves are speculative.
__global__ void k_publish_all(PeerFlags pf, int n_groups, unsigned epoch) {
  __threadfence_system();
  for (int g = threadIdx.x; g < n_groups; g += blockDim.x) {
    for (int j = 0; j < pf.n; ++j) {
      unsigned* f = pf.f[j] + kCtrlReady + 8 * g + pf.rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
    }
  }
}

__global__ void k_gather_shard(const LambTile* __restrict__ tiles, const float* __restrict__ w,
                               float* __restrict__ wsh, float* __restrict__ wsh_alt) {
  const LambTile t = tiles[blockIdx.x];
  for (int e = threadIdx.x; e < t.len; e += blockDim.x) {
    const float v = w[t.w0 + e];
    wsh[t.s0 + e] = v;
    if (wsh_alt) wsh_alt[t.s0 + e] = v;
  }
}

}  // namespace

void check_launch(bo_ctx* c, const char* what) {
  c->launches += 1;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(BO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}


void launch_accumulate(bo_ctx* c, int micro, const PtrTable& tab, bool vec_ok) {
  StageTimer timer(c, BO_STAGE_ACCUMULATE);
  const int reverse = micro == c->cfg.accumulation - 2;
  if (vec_ok) {
    k_accumulate<true><<<c->n_acc_tiles, kThreads, 0, c->stream>>>(c->d_acc_tiles, c->d_tensors,
                                                                    tab, c->acc, micro == 0, c->state,
                                                                    reverse);
  } else {
    k_accumulate<false><<<c->n_acc_tiles, kThreads, 0, c->stream>>>(c->d_acc_tiles, c->d_tensors,
                                                                     tab, c->acc, micro == 0, c->state,
                                                                     reverse);
  }
  check_launch(c, "k_accumulate");
}

void launch_finalize_tiles(bo_ctx* c, const AccTile* tiles, int n, const PtrTable& tab,
                           cudaStream_t stream) {
  if (n == 0) return;
  StageTimer timer(c, BO_STAGE_FINALIZE, stream);
  auto go = [&](auto kern) {
    kern<<<n, kThreads, 0, stream>>>(tiles, c->d_tensors, tab, c->ms, c->acc, c->x, c->state, c->cfg.accumulation);
  };
  switch (c->ms.K) {
    case 0: go(k_finalize<0>); break;
    case 2: go(k_finalize<2>); break;
    case 3: go(k_finalize<3>); break;
    case 4: go(k_finalize<4>); break;
    case 5: go(k_finalize<5>); break;
    case 6: go(k_finalize<6>); break;
    case 7: go(k_finalize<7>); break;
    case 8: go(k_finalize<8>); break;
    default: fail(BO_ERR_INVALID_CONFIG, "resident micro count outside 2..8");
  }
  check_launch(c, "k_finalize");
}

void launch_finalize(bo_ctx* c, const PtrTable& tab) {
  launch_finalize_tiles(c, c->d_acc_tiles, c->n_acc_tiles, tab, c->stream);
}

// One rank's multi-kernel fallback (inputs not 16-byte aligned): recompute
// LAMB in phase 2, moments updated in place.
template <typename G>
static void lamb_shard(bo_ctx* c, const G* g) {
  const int T = c->L.T;
  const float invn = 1.0f / static_cast<float>(c->world);  // trainer.cpp:212
  const int scale_g = c->world > 1;
  {
  StageTimer timer(c, BO_STAGE_LAMB_NORMS);
  k_lamb_norms<G><<<c->n_lamb_tiles, kThreads, 0, c->stream>>>(c->d_lamb_tiles, g, c->w, c->m, c->v,
                                                                c->m_alt, c->v_alt,
                                                                c->state, c->lamb, c->bc_table, invn,
                                                                scale_g, c->tile_part);
  check_launch(c, "k_lamb_norms");
  }
  {
  StageTimer timer(c, BO_STAGE_TRUST);
  k_norm_reduce<<<T, kThreads, 0, c->stream>>>(c->d_tensor_tile_begin, c->tile_part, c->state, T,
                                                c->rank_part, PartDst{{}, 0});
  check_launch(c, "k_norm_reduce");
  k_trust<<<1, 1024, 0, c->stream>>>(c->all_part, c->world, T, c->state, c->lamb, c->scaler,
                                     c->trust, 0, PeerFlags{{}, 0, 0}, 0u, 0ull);
  check_launch(c, "k_trust");
  }
  StageTimer timer(c, BO_STAGE_LAMB_UPDATE);
  k_lamb_update<G><<<c->n_lamb_tiles, kThreads, 0, c->stream>>>(c->d_lamb_tiles, g, c->w, c->m, c->v,
                                                                 c->m_alt, c->v_alt,
                                                                 c->state, c->lamb, c->bc_table, invn,
                                                                 scale_g, c->trust);
  check_launch(c, "k_lamb_update");
}

// world > 1: phase 1 on the shard -> per-tensor partials -> all-gather of
// the partials and flags (2T+1 doubles per rank, summed in rank order so all
// ranks agree) -> trust ratios, found_inf, scaler -> phase 2 pushing the new
// parameters into every rank's replica -> barrier.
template <typename W, bool kHop, bool kDbl>
static void launch_p1w(bo_ctx* c, const PtrTable& tab, const W* in, const P1Args& A, int tile0, int n) {
  if (n <= 0) return;
  P1Args a = A;
  a.tile_part = A.tile_part + 2 * static_cast<size_t>(tile0);  // partials at global tile indices
  const LambTile* tiles = c->d_lamb_tiles + tile0;
  const int grid = (n * 32 + kWarpTileCTA - 1) / kWarpTileCTA;
  auto go = [&](auto kern) { kern<<<grid, kWarpTileCTA, 0, c->stream>>>(tiles, n, tab, in, a); };
  if constexpr (!kHop) {
    go(k_p1w<W, true, false, 1, 4, 0, kDbl>);
  } else if (c->ms.K == 0) {
    go(k_p1w<W, true, true, 1, 4, 0, kDbl>);
  } else if (c->ms.K == 2) {
    go(k_p1w<W, true, true, 1, 4, 2, kDbl>);
  } else if (c->ms.K == 4) {
    go(k_p1w<W, true, true, 1, 4, 4, kDbl>);
  } else {
    fail(BO_ERR_INVALID_CONFIG, "fused last hop with resident micros: K must be 2 or 4");
  }
  check_launch(c, "k_p1w");
}

// Grouped LAMB (BO_LAMB_GROUP_ELEMS): the shard's LAMB in groups of
// consecutive tensors (model order), each group's parameter push speculative
// and on its own stream, so the push of group g (NVLink) overlaps phase 1 of
// group g + 1 (HBM):
//   compute stream: p1w(g) -> norm partials(g) -> k_trust(g) [all-rank barrier,
//                   trust ratios of g] -> event(g)            for g = 0..G-1
//   push stream:    wait event(g) -> push(g) (reads the current master shard,
//                   writes the other one + every replica)      for g = 0..G-1
//   then:           k_step_final (found_inf from every rank's cumulative flag,
//                   counters, scaler, parity flip), k_rollback (a skipped step
//                   re-pushes the unchanged master shard), publish, barrier.
// Same arithmetic per element as the serial path; only the order of the
// independent tensor groups changes.
template <typename W, bool kHop>
static void lamb_grouped(bo_ctx* c, const PtrTable& tab, const W* in) {
  c->path |= BO_PATH_LAMB_GROUPED;
  const int T = c->L.T;
  const float invn = 1.0f / static_cast<float>(c->world);  // trainer.cpp:212
  const P1Args A{c->d_tensors, c->acc, c->cfg.accumulation, invn, c->wsh, c->m, c->v,
                 c->m_alt, c->v_alt, c->u, c->wsh_alt, c->state, c->lamb, c->bc_table, c->tile_part, c->ms};
  const size_t slot = static_cast<size_t>(2 * T + 1);
  const int G = static_cast<int>(c->lamb_groups.size());
  cudaStream_t ps = c->lockstep ? c->stream : c->push_stream;
  if (!c->lockstep && !c->push_stream) {
    BO_CUDA(cudaStreamCreateWithPriority(&c->push_stream, cudaStreamNonBlocking, -1));
    ps = c->push_stream;
    c->group_events.assign(static_cast<size_t>(G) + 1, nullptr);
    for (auto& e : c->group_events) BO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  PushGroups none{c->d_push_group_of_tensor, c->d_push_group_tiles, c->d_push_count, PeerFlags{{}, 0, c->rank}, 0u};
  unsigned epoch = 0;
  size_t half = 0;
  {
  StageTimer timer(c, BO_STAGE_LAMB_NORMS);
  auto p1 = [&](int g) {
    const bo_ctx::LambGroup& lg = c->lamb_groups[static_cast<size_t>(g)];
    launch_p1w<W, kHop, true>(c, tab, in, A, lg.tile0, lg.tile1 - lg.tile0);
  };
  auto norms = [&](int g) {
    const bo_ctx::LambGroup& lg = c->lamb_groups[static_cast<size_t>(g)];
    c->bar_epoch += 1;
    epoch = static_cast<unsigned>(c->bar_epoch);
    half = (c->bar_epoch & 1) * static_cast<size_t>(c->world) * slot;
    PartDst dst{{}, c->world};
    for (int j = 0; j < c->world; ++j) dst.p[j] = c->peer_part[j] + half + static_cast<size_t>(c->rank) * slot;
    if (lg.t1 > lg.t0) {
      k_norm_reduce<<<lg.t1 - lg.t0, kThreads, 0, c->stream>>>(c->d_tensor_tile_begin, c->tile_part, c->state, T,
                                                               c->rank_part, dst, lg.t0);
      check_launch(c, "k_norm_reduce");
    }
  };
  auto trust_push = [&](int g) {
    const bo_ctx::LambGroup& lg = c->lamb_groups[static_cast<size_t>(g)];
    PeerFlags pf = c->peer_ctrl;
    if (c->lockstep) {
      lockstep_sync(c, "partials");
      pf.n = 0;
    }
    k_trust<<<1, 1024, 0, c->stream>>>(c->all_part + half, c->world, T, c->state, c->lamb, c->scaler,
                                       c->trust, 0, pf, epoch, c->watchdog_ns, 1, lg.t0, lg.t1);
    check_launch(c, "k_trust");
    if (!c->lockstep) {
      BO_CUDA(cudaEventRecord(c->group_events[static_cast<size_t>(g)], c->stream));
      BO_CUDA(cudaStreamWaitEvent(ps, c->group_events[static_cast<size_t>(g)], 0));
    }
    if (lg.tile1 > lg.tile0 && c->push_posted_ctas > 0) {
      k_push_posted<<<std::min(c->push_posted_ctas, lg.tile1 - lg.tile0), kPostThreads, 0, ps>>>(
          c->d_lamb_tiles + lg.tile0, lg.tile1 - lg.tile0, c->wsh, c->u, c->state, c->lamb, c->trust,
          c->d_peer_w, c->world, c->wsh_alt);
      check_launch(c, "k_push_posted");
    } else if (lg.tile1 > lg.tile0) {
      k_shard_p2_push<<<lg.tile1 - lg.tile0, kThreads, 0, ps>>>(
          c->d_lamb_tiles + lg.tile0, lg.tile1 - lg.tile0, c->wsh, c->u, c->state, c->lamb, c->trust,
          c->d_peer_w, c->world, none, c->wsh_alt);
      check_launch(c, "k_shard_p2_push");
    }
  };
  // compute stream: p1(g) norms(g) trust(g) [event -> push(g) on ps] p1(g+1)
  // ... (issuing p1(g+1) ahead of trust(g) was measured slower: the push of
  // g, the bottleneck, then starts a phase 1 later; profiles/r02_notes.md)
  for (int g = 0; g < G; ++g) {
    p1(g);
    norms(g);
    trust_push(g);
  }
  if (!c->lockstep) {
    BO_CUDA(cudaEventRecord(c->group_events[static_cast<size_t>(G)], ps));
    BO_CUDA(cudaStreamWaitEvent(c->stream, c->group_events[static_cast<size_t>(G)], 0));
  }
  }
  StageTimer timer(c, BO_STAGE_ALLGATHER);
  k_step_final<<<1, 1, 0, c->stream>>>(c->all_part + half, c->world, T, c->state, c->scaler, epoch);
  check_launch(c, "k_step_final");
  if (c->n_lamb_tiles > 0) {
    k_rollback<<<std::min(c->n_lamb_tiles, 2 * c->num_sms), kThreads, 0, c->stream>>>(
        c->d_lamb_tiles, c->n_lamb_tiles, c->wsh, c->wsh_alt, c->d_peer_w, c->world, c->state);
    check_launch(c, "k_rollback");
  }
  k_publish_all<<<1, 128, 0, c->stream>>>(c->peer_ctrl, c->n_push_groups, epoch);
  check_launch(c, "k_publish_all");
  if (c->lockstep) {
    lockstep_sync(c, "end of step");
    return;
  }
  k_step_end_barrier<<<1, 1, 0, c->stream>>>(c->peer_ctrl, epoch, c->state, c->watchdog_ns);
  check_launch(c, "k_step_end_barrier");
}

template <typename W, bool kHop>
static void lamb_sharded(bo_ctx* c, const PtrTable& tab, const W* in) {
  if (c->lamb_groups.size() > 1) {
    lamb_grouped<W, kHop>(c, tab, in);
    return;
  }
  const int T = c->L.T;
  const float invn = 1.0f / static_cast<float>(c->world);  // trainer.cpp:212
  {
  StageTimer timer(c, BO_STAGE_LAMB_NORMS);
  const P1Args A{c->d_tensors, c->acc, c->cfg.accumulation, invn, c->wsh, c->m, c->v,
                 c->m_alt, c->v_alt, c->u, nullptr, c->state, c->lamb, c->bc_table, c->tile_part, c->ms};
  const int grid = (c->n_lamb_tiles * 32 + kWarpTileCTA - 1) / kWarpTileCTA;
  auto go = [&](auto kern) {
    kern<<<grid, kWarpTileCTA, 0, c->stream>>>(c->d_lamb_tiles, c->n_lamb_tiles, tab, in, A);
  };
  if (c->n_lamb_tiles > 0) {  // a rank of a tiny model can own no element
    if constexpr (!kHop) {
      go(k_p1w<W, true, false, 1, 4>);
    } else if (c->ms.K == 0) {
      go(k_p1w<W, true, true, 1, 4>);
    } else if (c->ms.K == 2) {  // the last ring hop fused in, x from the resident micros
      go(k_p1w<W, true, true, 1, 4, 2>);
    } else if (c->ms.K == 4) {
      go(k_p1w<W, true, true, 1, 4, 4>);
    } else {
      fail(BO_ERR_INVALID_CONFIG, "fused last hop with resident micros: K must be 2 or 4");
    }
  }
  check_launch(c, "k_p1w");
  }
  // The partials all-gather without a collective: k_norm_reduce stores this
  // rank's 2T+1 partials into its slot of every rank's all_part (this step's
  // parity half, so a fast rank's next step cannot overwrite a slow rank's
  // current read), k_trust's all-rank flag barrier orders them before the sums.
  c->bar_epoch += 1;
  const unsigned epoch = static_cast<unsigned>(c->bar_epoch);
  const size_t slot = static_cast<size_t>(2 * T + 1);
  const size_t half = (c->bar_epoch & 1) * static_cast<size_t>(c->world) * slot;
  {
  StageTimer timer(c, BO_STAGE_TRUST);
  PartDst dst{{}, c->world};
  for (int j = 0; j < c->world; ++j) dst.p[j] = c->peer_part[j] + half + static_cast<size_t>(c->rank) * slot;
  k_norm_reduce<<<T, kThreads, 0, c->stream>>>(c->d_tensor_tile_begin, c->tile_part, c->state, T,
                                                c->rank_part, dst);
  check_launch(c, "k_norm_reduce");
  PeerFlags pf = c->peer_ctrl;
  if (c->lockstep) {  // every rank's k_norm_reduce is on the shared stream before any k_trust
    lockstep_sync(c, "partials");
    pf.n = 0;
  }
  k_trust<<<1, 1024, 0, c->stream>>>(c->all_part + half, c->world, T, c->state, c->lamb, c->scaler,
                                     c->trust, 1, pf, epoch, c->watchdog_ns);
  check_launch(c, "k_trust");
  }
  {
  StageTimer timer(c, BO_STAGE_LAMB_UPDATE);
  const PushGroups G{c->d_push_group_of_tensor, c->d_push_group_tiles, c->d_push_count, c->peer_ctrl, epoch};
  k_shard_p2_push<<<c->n_push_tiles, kThreads, 0, c->stream>>>(c->d_push_tiles, c->n_push_tiles, c->wsh, c->u,
                                                                c->state, c->lamb, c->trust, c->d_peer_w,
                                                                c->world, G);
  check_launch(c, "k_shard_p2_push");
  }
  // every rank's pushes into every replica have landed once all ranks are
  // past their phase 2 (kernel completion flushes the NVLink stores): an
  // all-rank flag barrier, no collective
  StageTimer timer(c, BO_STAGE_ALLGATHER);
  if (c->lockstep) {
    lockstep_sync(c, "end of step");
    return;
  }
  k_step_end_barrier<<<1, 1, 0, c->stream>>>(c->peer_ctrl, epoch, c->state, c->watchdog_ns);
  check_launch(c, "k_step_end_barrier");
}

void run_lamb(bo_ctx* c, const PtrTable& tab) {
  trace(c, "lamb_start", 0, c->stream);
  if (c->world == 1) {
    lamb_shard<float>(c, c->gshard);
  } else if (c->algo == BO_REDUCE_RING) {
    // the owned chunk: the left neighbour's last partial (last hop fused into
    // phase 1) or the ring's final wire buffer (wire-exact values)
    if (c->cfg.f16_exchange) {
      if (c->ring_last_in) {
        lamb_sharded<uint16_t, true>(c, tab, static_cast<const uint16_t*>(c->ring_last_in));
      } else {
        lamb_sharded<uint16_t, false>(c, tab, static_cast<const uint16_t*>(c->ring_result));
      }
    } else {
      if (c->ring_last_in) {
        lamb_sharded<float, true>(c, tab, static_cast<const float*>(c->ring_last_in));
      } else {
        lamb_sharded<float, false>(c, tab, static_cast<const float*>(c->ring_result));
      }
    }
  } else {
    lamb_sharded<float, false>(c, tab, c->gshard);
  }
}

bool HostBarrier::wait(uint64_t timeout_ns) {
  std::unique_lock<std::mutex> lk(m);
  const uint64_t g = gen;
  if (++count == n) {
    count = 0;
    ++gen;
    cv.notify_all();
    return true;
  }
  return cv.wait_for(lk, std::chrono::nanoseconds(timeout_ns), [&] { return gen != g; });
}

SharedStream::~SharedStream() {
  if (s) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
}

void lockstep_sync(bo_ctx* c, const char* where) {
  if (!c->lockstep) return;
  if (!c->lockstep->wait(c->watchdog_ns)) {
    fail(BO_ERR_PEER_DISCONNECTED, "rank " + std::to_string(c->rank) + ": a rank thread of the lockstep "
                                       "world did not reach the " + where + " rendezvous within the watchdog");
  }
}

void params_wait(bo_ctx* c, int tensor, cudaStream_t stream) {
  if (c->world == 1 || c->lockstep) {
    // one rank (or a lockstep world on one stream): the update runs on the
    // context stream; order the caller's stream after the most recent step
    if (!c->params_done) BO_CUDA(cudaEventCreateWithFlags(&c->params_done, cudaEventDisableTiming));
    BO_CUDA(cudaEventRecord(c->params_done, c->stream));
    BO_CUDA(cudaStreamWaitEvent(stream, c->params_done, 0));
    return;
  }
  if (c->bar_epoch == 0) return;  // no step enqueued yet
  const int g = c->push_group_of_tensor[static_cast<size_t>(tensor)];
  k_params_wait<<<1, 1, 0, stream>>>(c->ctrl + kCtrlReady + 8 * g, c->world,
                                     static_cast<unsigned>(c->bar_epoch), c->state, c->watchdog_ns);
  check_launch(c, "k_params_wait");
}

void need_nccl(bo_ctx* c, const char* what) {
  if (!c->comm) {
    fail(BO_ERR_INVALID_CONFIG, std::string(what) +
                                    " needs the NCCL communicator: initialise with bo_comm_init "
                                    "(bo_comm_export / bo_comm_import map peers without NCCL)");
  }
}

void gather_shard(bo_ctx* c) {
  if (c->world == 1) return;
  if (c->n_lamb_tiles == 0) return;
  k_gather_shard<<<c->n_lamb_tiles, kThreads, 0, c->stream>>>(c->d_lamb_tiles, c->w, c->wsh, c->wsh_alt);
  check_launch(c, "k_gather_shard");
}

}  // namespace bo
