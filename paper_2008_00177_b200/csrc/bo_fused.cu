// Single-rank sync micro: the whole LAMB step (lamb.cpp:140-201) with the
// flatten_param unscale (trainer.cpp:186-203) fused in, as one persistent
// TMA-fed kernel.
//
//   k_flag        overflow pre-check of the sync micro's binary16 inputs
//                 (found_inf must be known before the moments are written)
//   k_lamb_fused  one CTA per SM: a producer warp claims work tiles in order
//                 and streams them into a 3-stage shared-memory ring with
//                 cp.async.bulk (TMA bulk copies, mbarrier completion); 16
//                 consumer warps compute from shared memory.
//                   phase 1 of a tile: g = (h + acc) * inv; m', v', u; store
//                     m', v' and u; fp64 partials of ||w||^2, ||u||^2
//                   the CTA completing a group's phase 1 reduces the partials
//                     (fixed order) into that group's trust ratios
//                   phase 2 of a tile: w -= (lr * r) * u, once published
//                 Tiles are claimed P1(g0) P1(g1) P2(g0) P1(g2) P2(g1) ..., so
//                 a phase-2 tile's w and u are still in L2; u lines are then
//                 discarded from L2 so the scratch never reaches DRAM.
//   k_fused_epilogue  step counters and the loss-scaler state machine
#include <cuda_fp16.h>

#include "bo_device.cuh"
#include "bo_internal.hpp"

namespace bo {
namespace {

constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kFusedThreads = kConsumers + 32;  // + one producer warp
constexpr int kStages = 3;
// stage layout (bytes): h[4096] u16 | acc | w | m | v  (fp32 [4096] each)
constexpr int kOffH = 0;
constexpr int kOffAcc = kTileElems * 2;
constexpr int kOffW = kOffAcc + kTileElems * 4;
constexpr int kOffM = kOffW + kTileElems * 4;
constexpr int kOffV = kOffM + kTileElems * 4;
constexpr int kStageBytes = kOffV + kTileElems * 4;                 // 73728
constexpr int kSmemBytes = kStages * kStageBytes + 2048;            // + barriers / headers / partials
constexpr int kPerThread = kTileElems / kConsumers;                 // 8 elements
static_assert(kPerThread == 8, "two float4 per consumer thread");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// TMA bulk copy global -> shared, completion counted on mbarrier b.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b,
                                          uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st4(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float at(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ void put(float4& v, int i, float x) {
  if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
}
__device__ __forceinline__ uint32_t round16(uint32_t b) { return (b + 15u) & ~15u; }

__global__ void __launch_bounds__(kThreads) k_flag(const AccTile* __restrict__ tiles,
                                                   const __grid_constant__ PtrTable tab,
                                                   DevState* __restrict__ st) {
  const AccTile tile = tiles[blockIdx.x];
  const uint16_t* __restrict__ src = tab.p[tile.t] + tile.e0;
  bool bad = false;
  const int nvec = tile.len >> 3;
#pragma unroll 2
  for (int i = threadIdx.x; i < nvec; i += kThreads) {
    const uint4 hv = __ldcs(reinterpret_cast<const uint4*>(src) + i);
    bad |= pair_nonfinite(hv.x) | pair_nonfinite(hv.y) | pair_nonfinite(hv.z) | pair_nonfinite(hv.w);
  }
  for (int i = (nvec << 3) + threadIdx.x; i < tile.len; i += kThreads) bad |= !finite(widen(src[i]));
  raise_flag(bad, st);
}

// Per-stage header the producer fills before it arms the stage's barrier.
struct StageHdr {
  int item;
  uint32_t wk;
  float trust;  // phase 2: the tile's trust ratio
  int pad;
  FusedTile t;
};

__global__ void __launch_bounds__(kFusedThreads, 1) k_lamb_fused(
    const FusedTile* __restrict__ tiles, const FusedGroup* __restrict__ groups,
    const int* __restrict__ tensor_tiles, const int* __restrict__ tensor_ids,
    const uint32_t* __restrict__ work, int n_work, const __grid_constant__ PtrTable tab,
    const float* __restrict__ acc, float* __restrict__ w, float* __restrict__ m,
    float* __restrict__ v, float* __restrict__ u, const DevState* __restrict__ st, LambConsts c,
    const double* __restrict__ bc_table, int K, double* __restrict__ tile_part,
    float* __restrict__ trust, unsigned long long* __restrict__ sync, int n_groups,
    const int* __restrict__ sb_tiles, const int* __restrict__ tensor_sbs,
    double* __restrict__ sb_part, int n_sb) {
  if (st->local_flag) return;  // overflow: the step is skipped (epilogue backs off)
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* tail = smem + kStages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty = full + kStages;
  StageHdr* hdr = reinterpret_cast<StageHdr*>(tail + 64);                  // [kStages]
  double* part = reinterpret_cast<double*>(tail + 256);                      // [kStages][16][2]
  int* cnt = reinterpret_cast<int*>(tail + 256 + kStages * kConsumerWarps * 16);  // [kStages]
  // sync = [group done | work counter | superblock done] (reset per launch) [ready epochs]
  unsigned long long* done = sync;
  unsigned long long* counter = sync + n_groups;
  unsigned long long* sb_done = sync + n_groups + 1;
  unsigned long long* ready = sync + n_groups + 1 + n_sb;
  const unsigned long long epoch = static_cast<unsigned long long>(st->steps) + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
      cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      // Static interleaved schedule: CTA b takes items b, b+G, b+2G, ... of the
      // ordered work list (so every CTA walks the P1/P2 order in step), with
      // the next item's descriptor fetched while the current stage drains.
      const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
      int item = blockIdx.x;
      uint32_t wk_next = item < n_work ? work[item] : 0u;
      FusedTile t_next = item < n_work ? tiles[wk_next >> 1] : FusedTile{};
      (void)counter;
      for (int it = 0;; ++it, item += gridDim.x) {
        const int s = it % kStages;
        const uint32_t wk = wk_next;
        const FusedTile t = t_next;
        if (item + static_cast<int>(gridDim.x) < n_work) {
          wk_next = __ldg(work + item + gridDim.x);
          t_next = tiles[wk_next >> 1];
        }
        mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        StageHdr& h = hdr[s];
        h.item = item;
        if (item >= n_work) {
          mbar_arrive(&full[s]);  // sentinel: consumers stop
          break;
        }
        h.wk = wk;
        h.t = t;
        unsigned char* base = smem + s * kStageBytes;
        const uint32_t nb4 = round16(static_cast<uint32_t>(t.len) * 4u);
        if ((wk & 1u) == 0) {
          const uint32_t nb2 = round16(static_cast<uint32_t>(t.len) * 2u);
          mbar_arrive_tx(&full[s], nb2 + (K > 1 ? nb4 : 0u) + 3u * nb4);
          bulk_load(base + kOffH, tab.p[t.t] + t.e0, nb2, &full[s], pf);
          if (K > 1) bulk_load(base + kOffAcc, acc + t.a0, nb4, &full[s], pf);
          bulk_load(base + kOffW, w + t.a0, nb4, &full[s], pl);
          bulk_load(base + kOffM, m + t.a0, nb4, &full[s], pf);
          bulk_load(base + kOffV, v + t.a0, nb4, &full[s], pf);
        } else {
          while (ld_acquire(&ready[t.g]) < epoch) __nanosleep(64);
          asm volatile("fence.proxy.async.global;" ::: "memory");
          h.trust = __ldcg(trust + t.t);
          mbar_arrive_tx(&full[s], 2u * nb4);
          bulk_load(base + kOffW, w + t.a0, nb4, &full[s], pf);
          bulk_load(base + kOffM, u + t.a0, nb4, &full[s], pf);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  // Warps run independently: no CTA-wide barrier in the loop. The last warp to
  // finish a phase-1 tile (a shared-memory counter per stage) sums the warps'
  // partials, publishes the tile and, if it completes the group, computes the
  // group's trust ratios.
  double bc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) bc[i] = bc_table[4 * st->lamb_step + i];
  const float inv = __fdiv_rn(1.0f, __fmul_rn(static_cast<float>(K), st->scale));
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (int it = 0;; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (it / kStages) & 1);
    const StageHdr& h = hdr[s];
    if (h.item >= n_work) break;
    const uint32_t wk = h.wk;
    const FusedTile t = h.t;
    const unsigned char* base = smem + s * kStageBytes;
    const float4* sw = reinterpret_cast<const float4*>(base + kOffW);
    const int q0 = threadIdx.x;  // float4 index; second one at q0 + kConsumers
    if ((wk & 1u) == 0) {
      // ---------------- phase 1
      const uint2* sh = reinterpret_cast<const uint2*>(base + kOffH);
      const float4* sa = reinterpret_cast<const float4*>(base + kOffAcc);
      const float4* sm = reinterpret_cast<const float4*>(base + kOffM);
      const float4* sv = reinterpret_cast<const float4*>(base + kOffV);
      float4 wv[2], mv[2], vv[2], av[2];
      uint2 hv[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = q0 + j * kConsumers;
        hv[j] = sh[q];
        av[j] = K > 1 ? sa[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        wv[j] = sw[q];
        mv[j] = sm[q];
        vv[j] = sv[q];
      }
      double wn = 0.0, un = 0.0;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e0 = 4 * (q0 + j * kConsumers);
        if (e0 >= t.len) continue;
        const float hg[4] = {widen(static_cast<uint16_t>(hv[j].x & 0xFFFFu)),
                             widen(static_cast<uint16_t>(hv[j].x >> 16)),
                             widen(static_cast<uint16_t>(hv[j].y & 0xFFFFu)),
                             widen(static_cast<uint16_t>(hv[j].y >> 16))};
        float4 mo = mv[j], vo = vv[j], uo = make_float4(0.f, 0.f, 0.f, 0.f);
        const int n = min(4, t.len - e0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < n) {
            const float g = __fmul_rn(K > 1 ? __fadd_rn(hg[i], at(av[j], i)) : hg[i], inv);
            const float wi = at(wv[j], i);
            const Moments o = lamb_elem(g, wi, at(mv[j], i), at(vv[j], i), c, bc);
            put(mo, i, o.m);
            put(vo, i, o.v);
            put(uo, i, o.u);
            wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wi), static_cast<double>(wi)));
            un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u), static_cast<double>(o.u)));
          }
        }
        const int64_t a = t.a0 + e0;  // padding lanes past len keep old m/v bits
        st4(m + a, mo, pf);
        st4(v + a, vo, pf);
        st4(u + a, uo, pl);
      }
      wn = warp_sum(wn);
      un = warp_sum(un);
      int last = 0;
      if (lane == 0) {
        part[(s * kConsumerWarps + warp) * 2] = wn;
        part[(s * kConsumerWarps + warp) * 2 + 1] = un;
        __threadfence_block();
        last = atomicAdd(&cnt[s], 1) == kConsumerWarps - 1;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        int group_last = 0;
        if (lane == 0) {
          __threadfence_block();
          double A = 0.0, B = 0.0;
          for (int i = 0; i < kConsumerWarps; ++i) {
            A += reinterpret_cast<volatile double*>(part)[(s * kConsumerWarps + i) * 2];
            B += reinterpret_cast<volatile double*>(part)[(s * kConsumerWarps + i) * 2 + 1];
          }
          cnt[s] = 0;
          tile_part[2 * (wk >> 1)] = A;
          tile_part[2 * (wk >> 1) + 1] = B;
          // every warp's u of this tile (ordered by the block-scope counter) and
          // the partials become visible GPU-wide, to generic and async proxies
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          group_last = atomicAdd(&sb_done[t.sb], 1ull) + 1 ==
                       static_cast<unsigned long long>(sb_tiles[t.sb + 1] - sb_tiles[t.sb]);
        }
        // superblock complete: its <= 32 tile partials, one per lane
        if (__shfl_sync(0xffffffffu, group_last, 0)) {
          __threadfence();
          const int i = sb_tiles[t.sb] + lane;
          double A = 0.0, B = 0.0;
          if (i < sb_tiles[t.sb + 1]) {
            A = __ldcg(tile_part + 2 * i);
            B = __ldcg(tile_part + 2 * i + 1);
          }
          A = warp_sum(A);
          B = warp_sum(B);
          group_last = 0;
          if (lane == 0) {
            sb_part[2 * t.sb] = A;
            sb_part[2 * t.sb + 1] = B;
            __threadfence();
            const FusedGroup gr = groups[t.g];
            group_last = atomicAdd(&done[t.g], 1ull) + 1 ==
                         static_cast<unsigned long long>(gr.sb_end - gr.sb_begin);
          }
        } else {
          group_last = 0;
        }
        group_last = __shfl_sync(0xffffffffu, group_last, 0);
        if (group_last) {
          // this warp completed the group: trust ratios (lamb.cpp:192-196)
          __threadfence();
          const FusedGroup gr = groups[t.g];
          for (int f = gr.t_begin; f < gr.t_end; ++f) {
            double W = 0.0, U = 0.0;
            for (int i = tensor_sbs[f] + lane; i < tensor_sbs[f + 1]; i += 32) {
              W += __ldcg(sb_part + 2 * i);
              U += __ldcg(sb_part + 2 * i + 1);
            }
            W = warp_sum(W);
            U = warp_sum(U);
            if (lane == 0) {
              float r = 1.0f;
              if (W > 0.0 && U > 0.0) {
                r = __double2float_rn(__ddiv_rn(__dsqrt_rn(W), __dsqrt_rn(U)));
                r = fminf(fmaxf(r, 0.0f), c.clip);
              }
              trust[tensor_ids[f]] = r;
            }
          }
          if (lane == 0) {
            __threadfence();
            atomicExch(&ready[t.g], epoch);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    } else {
      // ---------------- phase 2
      const float4* su = reinterpret_cast<const float4*>(base + kOffM);
      float4 wv[2], uv[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        wv[j] = sw[q0 + j * kConsumers];
        uv[j] = su[q0 + j * kConsumers];
      }
      const float step_scale = __fmul_rn(c.lr, h.trust);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // stage data now in registers
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e0 = 4 * (q0 + j * kConsumers);
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
      const int nlines = (t.len * 4 + 127) / 128;
      if (threadIdx.x < nlines) {
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(u + t.a0 + 32 * threadIdx.x) : "memory");
      }
    }
  }
}

// Step bookkeeping after the fused kernel: counters and the loss-scaler state
// machine (the same transitions as k_trust).
__global__ void k_fused_epilogue(DevState* st, ScalerConsts sc) {
  const int found = st->local_flag != 0;
  st->found_inf = found;
  st->do_update = !found;
  st->steps += 1;
  st->local_flag = 0;
  if (found) {
    st->skipped += 1;
  } else {
    st->lamb_step += 1;
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

void check(bo_ctx* c, const char* what) {
  c->launches += 1;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(BO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

int fused_occupancy(int) {
  BO_CUDA(cudaFuncSetAttribute(k_lamb_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  int nb = 0;
  BO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_lamb_fused, kFusedThreads, kSmemBytes));
  return nb;
}

void run_fused_single_rank(bo_ctx* c, const PtrTable& tab) {
  {
    StageTimer timer(c, BO_STAGE_FLAG);
    k_flag<<<c->n_acc_tiles, kThreads, 0, c->stream>>>(c->d_acc_tiles, tab, c->state);
    check(c, "k_flag");
  }
  StageTimer timer(c, BO_STAGE_LAMB_FUSED);
  BO_CUDA(cudaMemsetAsync(c->d_fused_sync, 0,
                          static_cast<size_t>(c->n_fused_groups + 1 + c->n_fused_sb) * 8, c->stream));
  const int K = c->cfg.accumulation;
  const float* acc = c->acc;
  int n_work = c->n_fused_work, n_groups = c->n_fused_groups, n_sb = c->n_fused_sb;
  void* args[] = {&c->d_fused_tiles, &c->d_fused_groups, &c->d_fused_tensor_tiles,
                  &c->d_fused_tensor_ids, &c->d_fused_work, &n_work, const_cast<PtrTable*>(&tab),
                  &acc, &c->w, &c->m, &c->v, &c->u, &c->state, &c->lamb, &c->bc_table,
                  const_cast<int*>(&K), &c->tile_part, &c->trust, &c->d_fused_sync, &n_groups,
                  &c->d_fused_sb_tiles, &c->d_fused_tensor_sbs, &c->sb_part, &n_sb};
  BO_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_lamb_fused), c->fused_blocks,
                                      kFusedThreads, args, kSmemBytes, c->stream));
  check(c, "k_lamb_fused");
  k_fused_epilogue<<<1, 1, 0, c->stream>>>(c->state, c->scaler);
  check(c, "k_fused_epilogue");
}

}  // namespace bo
