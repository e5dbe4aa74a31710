// Single-rank sync micro: the whole LAMB step (lamb.cpp:23-84) with the
// flatten_param unscale (trainer.cpp:186-203) fused in.
//
//   k_lamb_p1     g = (h + acc) * inv; m', v', u (one pass, vectorised);
//                 stores m', v' into the OTHER moment buffer set (double
//                 buffering: the step's overflow flag — micros 0..K-2 from
//                 k_accumulate, micro K-1 checked here — is only final at the
//                 end of this pass) and the update u; per-tile fp64 partials
//                 of ||w||^2 and ||u||^2                                   30 B/elem
//   k_lamb_trust  per-tensor fixed-order sums of the tile partials ->
//                 trust ratios (lamb.cpp:75-79)
//   k_lamb_p2     w -= (lr * r) * u, tiles in reverse order so the update
//                 and weights phase 1 wrote last are still in L2; the dead
//                 u lines are then dropped from L2 (discard.global.L2)      12 B/elem
//   k_lamb_p1r    the same with the K micro-batches resident (bo_train_step):
//                 g = micro sum * inv, no accumulator               2K + 24 B/elem
//   k_fused_epilogue  step counters, the moment-buffer flip and the
//                 loss-scaler state machine
//
// Every per-tensor array (acc, w, m, v, u) uses the aligned tensor layout, so
// a tile index a0 serves all of them and every access is a 16-byte vector.
// Measured alternatives (profiles/r01_notes.md): one persistent kernel that
// re-read w and u from L2 per group (TMA-fed or not) made every group a
// grid-wide rendezvous and streamed at 2.2-3.3 TB/s; two plain passes with no
// inter-CTA waiting stream faster.
#include <cuda_fp16.h>

#include "bo_device.cuh"
#include "bo_internal.hpp"

namespace bo {
namespace {

constexpr int kP1Threads = 512;               // 8 elements (2 float4) per thread per tile
constexpr int kP2Threads = 256;               // 16 elements (4 float4) per thread per tile
static_assert(kTileElems == 2 * 4 * kP1Threads, "tile = 2 float4 per P1 thread");
static_assert(kTileElems == 4 * 4 * kP2Threads, "tile = 4 float4 per P2 thread");

__device__ __forceinline__ float at(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ void put(float4& v, int i, float x) {
  if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
}

// Phase 1, one tile per CTA (the fused tiles are 16-byte aligned slices of one
// tensor). Elements past len inside the last float4 keep their old m/v bits.
__global__ void __launch_bounds__(kP1Threads, 2) k_lamb_p1(
    const FusedTile* __restrict__ tiles, const __grid_constant__ PtrTable tab,
    const float* __restrict__ acc, const float* __restrict__ w, float* m0, float* v0, float* m1,
    float* v1, float* __restrict__ u, DevState* __restrict__ st, LambConsts c,
    const double* __restrict__ bc_table, int K, double* __restrict__ tile_part, int pref) {
  if (st->local_flag) return;  // an earlier micro overflowed: the step is skipped
  // double-buffered moments: read the current set, write the other one; the
  // epilogue makes it current only if the step's overflow flag stays clear
  const int par = st->parity;
  const float* __restrict__ m = par ? m1 : m0;
  const float* __restrict__ v = par ? v1 : v0;
  float* __restrict__ mn = par ? m0 : m1;
  float* __restrict__ vn = par ? v0 : v1;
  __shared__ double red[2][kP1Threads / 32];
  const double* bcp = bc_table + 4 * st->lamb_step;
  const double bc1 = bcp[0], bc2 = bcp[1], ibc1 = bcp[2], ibc2 = bcp[3];
  const FusedTile t = tiles[blockIdx.x];
  const float inv = __fdiv_rn(1.0f, __fmul_rn(static_cast<float>(K), st->scale));
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const uint16_t* __restrict__ hsrc = tab.p[t.t] + t.e0;
  float4 wv[2], mv[2], vv[2], av[2];
  uint2 hv[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e0 = 4 * (threadIdx.x + j * kP1Threads);
    if (e0 < t.len) {
      const int64_t a = t.a0 + e0;
      hv[j] = ld_h4(hsrc + e0, t.len - e0, pf);  // no load past the tensor's end
      av[j] = K > 1 ? ld4(acc + a, pf) : make_float4(0.f, 0.f, 0.f, 0.f);
      wv[j] = ld4(w + a, pl);
      mv[j] = ld4(m + a, pf);
      vv[j] = ld4(v + a, pf);
    }
  }
  // bulk L2 prefetch of the tile `pref` CTAs ahead (as k_lamb_p1r)
  if (pref > 0 && threadIdx.x < 5 && blockIdx.x + pref < gridDim.x) {
    const FusedTile nt = tiles[blockIdx.x + pref];
    if (threadIdx.x == 0) {
      prefetch_l2(tab.p[nt.t] + nt.e0, 2ull * nt.len);
    } else if (threadIdx.x == 1) {
      if (K > 1) prefetch_l2(acc + nt.a0, 4ull * nt.len);
    } else {
      const int which = threadIdx.x - 2;
      prefetch_l2((which == 0 ? w : which == 1 ? m : v) + nt.a0, 4ull * nt.len);
    }
  }
  double wn = 0.0, un = 0.0;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e0 = 4 * (threadIdx.x + j * kP1Threads);
    if (e0 >= t.len) continue;
    const int n = min(4, t.len - e0);  // < 4 only in a tensor's last float4
    // the sync micro's overflow check (micros 0..K-2: k_accumulate)
    if (n == 4) {
      bad |= pair_nonfinite(hv[j].x) | pair_nonfinite(hv[j].y);
    } else {
      const uint32_t hw[2] = {hv[j].x, hv[j].y};
      for (int i = 0; i < n; ++i) bad |= ((hw[i >> 1] >> (16 * (i & 1))) & 0x7C00u) == 0x7C00u;
    }
    const float hg[4] = {widen(static_cast<uint16_t>(hv[j].x & 0xFFFFu)),
                         widen(static_cast<uint16_t>(hv[j].x >> 16)),
                         widen(static_cast<uint16_t>(hv[j].y & 0xFFFFu)),
                         widen(static_cast<uint16_t>(hv[j].y >> 16))};
    const float wa[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
    const float ma[4] = {mv[j].x, mv[j].y, mv[j].z, mv[j].w};
    const float va[4] = {vv[j].x, vv[j].y, vv[j].z, vv[j].w};
    const float aa[4] = {av[j].x, av[j].y, av[j].z, av[j].w};
    float ga[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) ga[i] = __fmul_rn(K > 1 ? __fadd_rn(hg[i], aa[i]) : hg[i], inv);
    const Lamb4 o = lamb_elem4(ga, wa, ma, va, c, bc1, bc2, ibc1, ibc2);
    float4 mo = make_float4(o.m[0], o.m[1], o.m[2], o.m[3]);
    float4 vo = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
    float4 uo = make_float4(o.u[0], o.u[1], o.u[2], o.u[3]);
    if (n == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wa[i]), static_cast<double>(wa[i])));
        un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u[i]), static_cast<double>(o.u[i])));
      }
    } else {
      // padding lanes past len keep their old m/v bits and contribute nothing
      for (int i = n; i < 4; ++i) {
        put(mo, i, ma[i]);
        put(vo, i, va[i]);
        put(uo, i, 0.0f);
      }
      for (int i = 0; i < n; ++i) {
        wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wa[i]), static_cast<double>(wa[i])));
        un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u[i]), static_cast<double>(o.u[i])));
      }
    }
    const int64_t a = t.a0 + e0;
    st4(mn + a, mo, pf);
    st4(vn + a, vo, pf);
    st4(u + a, uo, pl);
  }
  raise_flag(bad, st);
  wn = warp_sum(wn);
  un = warp_sum(un);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = wn;
    red[1][wid] = un;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int i = 0; i < kP1Threads / 32; ++i) {
      A += red[0][i];
      B += red[1][i];
    }
    tile_part[2 * blockIdx.x] = A;
    tile_part[2 * blockIdx.x + 1] = B;
  }
}

// Phase 1 with the K micro-batches resident (bo_train_step): g = the micro
// sum * inv straight from the K binary16 gradients, no accumulator. K is a
// template parameter so the K loads of both float4 groups of a thread are
// issued up front like k_lamb_p1's; the tile's K gradient pointers sit in
// shared memory. 2K + 24 B/elem.
template <int K>
__global__ void __launch_bounds__(kP1Threads, 2) k_lamb_p1r(
    const FusedTile* __restrict__ tiles, MicroSrc ms, const float* __restrict__ w, float* m0,
    float* v0, float* m1, float* v1, float* __restrict__ u, DevState* __restrict__ st, LambConsts c,
    const double* __restrict__ bc_table, double* __restrict__ tile_part, int pref) {
  const FusedTile t = tiles[blockIdx.x];
  __shared__ const uint16_t* sp[K];
  __shared__ double red[2][kP1Threads / 32];
  if (threadIdx.x < K) sp[threadIdx.x] = ms.hk[threadIdx.x * ms.T + t.t] + t.e0;
  const int par = st->parity;
  const float* __restrict__ m = par ? m1 : m0;
  const float* __restrict__ v = par ? v1 : v0;
  float* __restrict__ mn = par ? m0 : m1;
  float* __restrict__ vn = par ? v0 : v1;
  const double* bcp = bc_table + 4 * st->lamb_step;
  const double ibc1 = bcp[2], ibc2 = bcp[3];
  const float inv = __fdiv_rn(1.0f, __fmul_rn(static_cast<float>(K), st->scale));
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  __syncthreads();
  float4 wv[2], mv[2], vv[2];
  uint2 hv[2][K];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e0 = 4 * (threadIdx.x + j * kP1Threads);
    if (e0 < t.len) {
      const int64_t a = t.a0 + e0;
#pragma unroll
      for (int k = 0; k < K; ++k) hv[j][k] = ld_h4(sp[k] + e0, t.len - e0, pf);
      wv[j] = ld4(w + a, pl);
      mv[j] = ld4(m + a, pf);
      vv[j] = ld4(v + a, pf);
    }
  }
  // Bulk L2 prefetch of the inputs of the tile `pref` CTAs ahead (one bulk
  // request per array, issued by K + 3 threads): with two 512-thread CTAs
  // per SM holding their loads in registers, the DRAM otherwise idles while
  // both compute; the prefetched tile's loads then hit L2. BERT-large K = 4:
  // 1.79 -> 1.65 ms at a distance of 4/3 x the SM count (profiles/r02_notes.md).
  if (pref > 0 && threadIdx.x < K + 3 && blockIdx.x + pref < gridDim.x) {
    const FusedTile nt = tiles[blockIdx.x + pref];
    if (static_cast<int>(threadIdx.x) < K) {
      prefetch_l2(ms.hk[threadIdx.x * ms.T + nt.t] + nt.e0, 2ull * nt.len);
    } else {
      const int which = threadIdx.x - K;
      prefetch_l2((which == 0 ? w : which == 1 ? m : v) + nt.a0, 4ull * nt.len);
    }
  }
  double wn = 0.0, un = 0.0;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e0 = 4 * (threadIdx.x + j * kP1Threads);
    if (e0 >= t.len) continue;
    const int n = min(4, t.len - e0);  // < 4 only in a tensor's last float4
    // live + (((0 + g0) + g1) + ... + g_{K-2}) (trainer.cpp:240-244, 196-201)
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f}, xs[4];
#pragma unroll
    for (int k = 0; k + 1 < K; ++k) {
      float f[4];
      widen4(hv[j][k], f);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], f[i]);
    }
    widen4(hv[j][K - 1], xs);
    float ga[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      xs[i] = __fadd_rn(xs[i], acc[i]);
      ga[i] = __fmul_rn(xs[i], inv);
      // a non-finite input makes the fp32 sum non-finite (K finite binary16
      // values cannot overflow fp32): the step's overflow check
      if (i < n) bad |= !finite(xs[i]);
    }
    const float wa[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
    const float ma[4] = {mv[j].x, mv[j].y, mv[j].z, mv[j].w};
    const float va[4] = {vv[j].x, vv[j].y, vv[j].z, vv[j].w};
    const Lamb4 o = lamb_elem4(ga, wa, ma, va, c, bcp, ibc1, ibc2);
    float4 mo = make_float4(o.m[0], o.m[1], o.m[2], o.m[3]);
    float4 vo = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
    float4 uo = make_float4(o.u[0], o.u[1], o.u[2], o.u[3]);
    if (n == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wa[i]), static_cast<double>(wa[i])));
        un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u[i]), static_cast<double>(o.u[i])));
      }
    } else {
      for (int i = n; i < 4; ++i) {  // padding lanes keep their old m/v bits
        put(mo, i, ma[i]);
        put(vo, i, va[i]);
        put(uo, i, 0.0f);
      }
      for (int i = 0; i < n; ++i) {
        wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wa[i]), static_cast<double>(wa[i])));
        un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u[i]), static_cast<double>(o.u[i])));
      }
    }
    const int64_t a = t.a0 + e0;
    st4(mn + a, mo, pf);
    st4(vn + a, vo, pf);
    st4(u + a, uo, pl);
  }
  raise_flag(bad, st);
  wn = warp_sum(wn);
  un = warp_sum(un);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = wn;
    red[1][wid] = un;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int i = 0; i < kP1Threads / 32; ++i) {
      A += red[0][i];
      B += red[1][i];
    }
    tile_part[2 * blockIdx.x] = A;
    tile_part[2 * blockIdx.x + 1] = B;
  }
}

// Trust ratio of tensor t from its tiles' partials (lamb.cpp:75-79) in a
// fixed order: threads 0..kThreads-1 stride over the tiles, warp sums, then
// thread 0 adds the warps in order. Every thread of the CTA must call it;
// the result is valid in thread 0. red: [2][>= kThreads / 32] shared doubles.
__device__ __forceinline__ float trust_ratio(const int* __restrict__ tensor_tiles,
                                             const double* __restrict__ tile_part, int t, float clip,
                                             double* red0, double* red1) {
  if (threadIdx.x < kThreads) {
    double A = 0.0, B = 0.0;
    for (int i = tensor_tiles[t] + threadIdx.x; i < tensor_tiles[t + 1]; i += kThreads) {
      A += __ldcg(tile_part + 2 * i);
      B += __ldcg(tile_part + 2 * i + 1);
    }
    A = warp_sum(A);
    B = warp_sum(B);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
      red0[wid] = A;
      red1[wid] = B;
    }
  }
  __syncthreads();
  float r = 1.0f;
  if (threadIdx.x == 0) {
    double W = 0.0, U = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      W += red0[i];
      U += red1[i];
    }
    if (W > 0.0 && U > 0.0) {
      r = __double2float_rn(__ddiv_rn(__dsqrt_rn(W), __dsqrt_rn(U)));
      r = fminf(fmaxf(r, 0.0f), clip);
    }
  }
  return r;
}

// Trust ratio of tensor blockIdx.x (two-pass form).
__global__ void __launch_bounds__(kThreads) k_lamb_trust(const int* __restrict__ tensor_tiles,
                                                         const double* __restrict__ tile_part,
                                                         const DevState* __restrict__ st,
                                                         LambConsts c, float* __restrict__ trust) {
  if (st->local_flag) return;
  __shared__ double red[2][kThreads / 32];
  const float r = trust_ratio(tensor_tiles, tile_part, blockIdx.x, c.clip, red[0], red[1]);
  if (threadIdx.x == 0) trust[blockIdx.x] = r;
}

// Phase 2 (lamb.cpp:80-81): tiles in reverse order (block b takes tile
// n-1-b) so the most recently written w and u are L2 hits.
__global__ void __launch_bounds__(kP2Threads) k_lamb_p2(const FusedTile* __restrict__ tiles,
                                                        int n_tiles, float* __restrict__ w,
                                                        float* __restrict__ u,
                                                        const DevState* __restrict__ st,
                                                        LambConsts c,
                                                        const float* __restrict__ trust) {
  if (st->local_flag) return;
  const FusedTile t = tiles[n_tiles - 1 - blockIdx.x];
  const float step_scale = __fmul_rn(c.lr, trust[t.t]);
  const uint64_t pf = policy_evict_first();
  float4 wv[4], uv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e0 = 4 * (threadIdx.x + j * kP2Threads);
    if (e0 < t.len) {
      wv[j] = ld4(w + t.a0 + e0, pf);
      uv[j] = ld4(u + t.a0 + e0, pf);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e0 = 4 * (threadIdx.x + j * kP2Threads);
    if (e0 >= t.len) continue;
    const int n = min(4, t.len - e0);
    float4 o = wv[j];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < n) put(o, i, __fsub_rn(at(wv[j], i), __fmul_rn(step_scale, at(uv[j], i))));
    }
    st4(w + t.a0 + e0, o, pf);
  }
  // the u scratch of this tile is dead: drop its L2 lines without write-back
  __syncthreads();
  const int nlines = (t.len * 4 + 127) / 128;
  if (threadIdx.x < nlines) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(u + t.a0 + 32 * threadIdx.x) : "memory");
  }
}

// Step bookkeeping: counters and the loss-scaler state machine (the same
// transitions as k_trust).
__device__ __forceinline__ void step_epilogue(DevState* st, const ScalerConsts& sc) {
  const int found = st->local_flag != 0;
  st->found_inf = found;
  st->do_update = !found;
  st->steps += 1;
  st->local_flag = 0;
  if (found) {
    st->skipped += 1;
  } else {
    st->lamb_step += 1;
    st->parity ^= 1;  // the moments phase 1 wrote become current
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

__global__ void k_fused_epilogue(DevState* st, ScalerConsts sc) { step_epilogue(st, sc); }

void check(bo_ctx* c, const char* what) {
  c->launches += 1;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(BO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void run_fused_single_rank(bo_ctx* c, const PtrTable& tab, MicroSrc ms) {
  trace(c, "lamb_start", 0, c->stream);
  {
    StageTimer timer(c, BO_STAGE_LAMB_NORMS);
    if (ms.K > 0) {
      auto launch = [&](auto kern) {
        kern<<<c->n_fused_tiles, kP1Threads, 0, c->stream>>>(c->d_fused_tiles, ms, c->w, c->m, c->v, c->m_alt,
                                                             c->v_alt, c->u, c->state, c->lamb, c->bc_table,
                                                             c->tile_part, c->p1r_prefetch);
      };
      switch (ms.K) {
        case 2: launch(k_lamb_p1r<2>); break;
        case 3: launch(k_lamb_p1r<3>); break;
        case 4: launch(k_lamb_p1r<4>); break;
        case 5: launch(k_lamb_p1r<5>); break;
        case 6: launch(k_lamb_p1r<6>); break;
        case 7: launch(k_lamb_p1r<7>); break;
        default: launch(k_lamb_p1r<8>); break;
      }
      check(c, "k_lamb_p1r");
    } else {
      k_lamb_p1<<<c->n_fused_tiles, kP1Threads, 0, c->stream>>>(
          c->d_fused_tiles, tab, c->acc, c->w, c->m, c->v, c->m_alt, c->v_alt, c->u, c->state, c->lamb,
          c->bc_table, c->cfg.accumulation, c->tile_part, c->p1r_prefetch);
      check(c, "k_lamb_p1");
    }
  }
  {
    StageTimer timer(c, BO_STAGE_TRUST);
    k_lamb_trust<<<c->L.T, kThreads, 0, c->stream>>>(c->d_fused_tensor_tiles, c->tile_part, c->state,
                                                     c->lamb, c->trust);
    check(c, "k_lamb_trust");
  }
  {
    StageTimer timer(c, BO_STAGE_LAMB_UPDATE);
    k_lamb_p2<<<c->n_fused_tiles, kP2Threads, 0, c->stream>>>(c->d_fused_tiles, c->n_fused_tiles,
                                                              c->w, c->u, c->state, c->lamb, c->trust);
    check(c, "k_lamb_p2");
  }
  StageTimer timer(c, BO_STAGE_TRUST);
  k_fused_epilogue<<<1, 1, 0, c->stream>>>(c->state, c->scaler);
  check(c, "k_fused_epilogue");
}

}  // namespace bo
