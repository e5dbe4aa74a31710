// Operator-level drop-ins for the reference's hot-path functions, each with
// the reference's argument meaning and error behaviour, plus the synthetic
// gradient generator used by the bench and the tests.
//
//   bo_lamb_step               lamb_step              lamb.cpp:23-84
//   bo_ring_allreduce_f32      ring_allreduce<float>  collective.hpp:53-99
//   bo_ring_allreduce_f16_wire ring_allreduce_f16_wire collective.cpp:37-86
//   bo_unscale_gradients       unscale_gradients      half.cpp:105-115
//   bo_narrow_f16/bo_widen_f16 narrow/widen_f16_block graph.cpp:176-199
//   bo_fused_optimizer_step    fused_optimizer_step   graph.cpp:458-487 run by
//                              run_fused_kernel (apply_block, graph.cpp:296-347)
//   bo_f16_round               quantize_inplace of a binary16 tensor (Tape::cast,
//                              ops.cpp:655-668; f16_round, half.cpp:79)
#include <cmath>
#include <cstring>
#include <memory>

#include "bo_device.cuh"
#include "bo_internal.hpp"

namespace bo {
namespace {

struct OpTensor {
  float* w;
  const float* g;
  float* m;
  float* v;
  int64_t n;
};

struct OpTile {
  int32_t t;
  int32_t len;
  int64_t e0;
};

// Smallest (tensor, element) key holding a non-finite gradient.
__global__ void k_first_nonfinite(const OpTile* tiles, const OpTensor* ts,
                                  unsigned long long* key) {
  const OpTile tile = tiles[blockIdx.x];
  const float* g = ts[tile.t].g + tile.e0;
  for (int e = threadIdx.x; e < tile.len; e += blockDim.x) {
    if (!finite(g[e])) {
      const unsigned long long k = (static_cast<unsigned long long>(tile.t) << 40) |
                                   static_cast<unsigned long long>(tile.e0 + e);
      atomicMin(key, k);
    }
  }
}

__global__ void k_op_norms(const OpTile* tiles, const OpTensor* ts, int limit_t, LambConsts c,
                           const double* bc, double* part) {
  const OpTile tile = tiles[blockIdx.x];
  double wn = 0.0, un = 0.0;
  if (tile.t < limit_t) {
    const OpTensor T = ts[tile.t];
    for (int e = threadIdx.x; e < tile.len; e += blockDim.x) {
      const int64_t i = tile.e0 + e;
      const float wi = T.w[i];
      const Moments o = lamb_elem(T.g[i], wi, T.m[i], T.v[i], c, bc);
      wn = __dadd_rn(wn, __dmul_rn(static_cast<double>(wi), static_cast<double>(wi)));
      un = __dadd_rn(un, __dmul_rn(static_cast<double>(o.u), static_cast<double>(o.u)));
    }
  }
  __shared__ double red[2][kThreads];
  red[0][threadIdx.x] = wn;
  red[1][threadIdx.x] = un;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = red[0][0];
    part[2 * blockIdx.x + 1] = red[1][0];
  }
}

__global__ void k_op_trust(const int* tile_begin, const double* part, int T, float clip,
                           float* trust) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    double W = 0.0, U = 0.0;
    for (int i = tile_begin[t]; i < tile_begin[t + 1]; ++i) {
      W = __dadd_rn(W, part[2 * i]);
      U = __dadd_rn(U, part[2 * i + 1]);
    }
    float r = 1.0f;
    if (W > 0.0 && U > 0.0) {
      r = __double2float_rn(__ddiv_rn(__dsqrt_rn(W), __dsqrt_rn(U)));
      r = fminf(fmaxf(r, 0.0f), clip);
    }
    trust[t] = r;
  }
}

// Full update for tensors < limit_t; for tensor limit_t, only the moments of
// the elements before the offending one (the reference's partial loop).
__global__ void k_op_update(const OpTile* tiles, const OpTensor* ts, int limit_t, int64_t limit_e,
                            LambConsts c, const double* bc, const float* trust) {
  const OpTile tile = tiles[blockIdx.x];
  if (tile.t > limit_t) return;
  const OpTensor T = ts[tile.t];
  const float step_scale = __fmul_rn(c.lr, tile.t < limit_t ? trust[tile.t] : 0.0f);
  for (int e = threadIdx.x; e < tile.len; e += blockDim.x) {
    const int64_t i = tile.e0 + e;
    if (tile.t == limit_t && i >= limit_e) continue;
    const float wi = T.w[i];
    const Moments o = lamb_elem(T.g[i], wi, T.m[i], T.v[i], c, bc);
    T.m[i] = o.m;
    T.v[i] = o.v;
    if (tile.t < limit_t) T.w[i] = __fsub_rn(wi, __fmul_rn(step_scale, o.u));
  }
}

__global__ void k_any_nonfinite(const float* g, size_t n, int* flag) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (!finite(g[i])) *flag = 1;
  }
}

__global__ void k_scale(float* g, size_t n, float inv) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    g[i] = __fmul_rn(g[i], inv);
  }
}

__global__ void k_narrow(const float* s, uint16_t* d, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    d[i] = narrow(s[i]);
  }
}

__global__ void k_widen(const uint16_t* s, float* d, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    d[i] = widen(s[i]);
  }
}

// mine = widen(in) + mine (f16) or in + mine (fp32): collective.cpp:58-61
template <typename W>
__global__ void k_ring_add(const W* in, float* mine, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float w;
    if constexpr (sizeof(W) == 2) w = widen(in[i]); else w = in[i];
    mine[i] = __fadd_rn(w, mine[i]);
  }
}

// fused_optimizer_step's constants exactly as apply_block sees them: every
// attribute is a double cast to float at use (graph.cpp:297).
struct AdamConsts {
  float b1, omb1, b2, omb2, bc1, bc2, eps, wd, nlr;
};

struct AdamTensor {
  float* w;
  const float* g;
  float* m;
  float* v;
  int64_t n;
  int32_t vec;  // all four arrays 16-byte aligned
};

// The 17 instructions of the fused kernel body in order, each rounded to
// fp32 (no contraction): m' = b1 m + (1-b1) g; v' = b2 v + (1-b2) g g;
// u = (bc1 m') * (1 / (sqrt(bc2 v') + eps)) + wd w; w' = w + (-lr) u.
__device__ __forceinline__ void adam_elem(const AdamConsts& k, float w, float g, float m, float v,
                                          float& wo, float& mo, float& vo) {
  mo = __fadd_rn(__fmul_rn(k.b1, m), __fmul_rn(k.omb1, g));
  vo = __fadd_rn(__fmul_rn(k.b2, v), __fmul_rn(k.omb2, __fmul_rn(g, g)));
  const float re = __fdiv_rn(1.0f, __fadd_rn(__fsqrt_rn(__fmul_rn(k.bc2, vo)), k.eps));
  const float u = __fadd_rn(__fmul_rn(__fmul_rn(k.bc1, mo), re), __fmul_rn(k.wd, w));
  wo = __fadd_rn(w, __fmul_rn(k.nlr, u));
}

// The tensor table travels as a kernel parameter (CUDA 12.1+: up to 32 KB),
// so calls need no device scratch and no synchronisation; larger lists are
// processed in batches of kAdamBatch tensors.
constexpr int kAdamBatch = 512;
struct AdamTable {
  AdamTensor t[kAdamBatch];
  int64_t cstart[kAdamBatch + 1];  // first chunk of each tensor; cstart[T] = total
  int T;
};
static_assert(sizeof(AdamTable) + sizeof(AdamConsts) < 32000, "kernel parameter limit");

// One CTA per 4096-element chunk of one tensor, grid-stride over the chunks
// of all tensors; chunk c belongs to the tensor t with cstart[t] <= c <
// cstart[t + 1] (binary search).
__global__ void __launch_bounds__(kThreads) k_fused_adam(const __grid_constant__ AdamTable tab,
                                                         AdamConsts k) {
  const int T = tab.T;
  const int64_t total = tab.cstart[T];
  for (int64_t c = blockIdx.x; c < total; c += gridDim.x) {
    int lo = 0, hi = T - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tab.cstart[mid] <= c) lo = mid; else hi = mid - 1;
    }
    const AdamTensor Tn = tab.t[lo];
    const int64_t e0 = (c - tab.cstart[lo]) * kTileElems;
    const int64_t rem = Tn.n - e0;
    const int len = static_cast<int>(rem < kTileElems ? rem : kTileElems);
    float* __restrict__ w = Tn.w + e0;
    const float* __restrict__ g = Tn.g + e0;
    float* __restrict__ m = Tn.m + e0;
    float* __restrict__ v = Tn.v + e0;
    int done = 0;
    if (Tn.vec) {  // e0 is a multiple of 4096: 16-byte aligned like the tensor
      const int nv = len >> 2;
#pragma unroll 2
      for (int q = threadIdx.x; q < nv; q += kThreads) {
        const float4 w4 = __ldcs(reinterpret_cast<const float4*>(w) + q);
        const float4 g4 = __ldcs(reinterpret_cast<const float4*>(g) + q);
        const float4 m4 = __ldcs(reinterpret_cast<const float4*>(m) + q);
        const float4 v4 = __ldcs(reinterpret_cast<const float4*>(v) + q);
        float4 wo, mo, vo;
        adam_elem(k, w4.x, g4.x, m4.x, v4.x, wo.x, mo.x, vo.x);
        adam_elem(k, w4.y, g4.y, m4.y, v4.y, wo.y, mo.y, vo.y);
        adam_elem(k, w4.z, g4.z, m4.z, v4.z, wo.z, mo.z, vo.z);
        adam_elem(k, w4.w, g4.w, m4.w, v4.w, wo.w, mo.w, vo.w);
        __stcs(reinterpret_cast<float4*>(w) + q, wo);
        __stcs(reinterpret_cast<float4*>(m) + q, mo);
        __stcs(reinterpret_cast<float4*>(v) + q, vo);
      }
      done = nv << 2;
    }
    for (int e = done + threadIdx.x; e < len; e += kThreads) {
      float wo, mo, vo;
      adam_elem(k, w[e], g[e], m[e], v[e], wo, mo, vo);
      w[e] = wo;
      m[e] = mo;
      v[e] = vo;
    }
  }
}

__global__ void k_round_f16(float* d, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    d[i] = widen(narrow(d[i]));
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Synthetic spec: g = ±(1 + mant/1024) 2^E, E in [-24, -15] (or the
// spike exponent), h = binary16_RNE(g * S). Independent of oracle/synth_grad.h;
// tests check the two agree bit for bit.
__global__ void k_synth(uint16_t* dst, int64_t begin, int64_t n, uint64_t base, float scale,
                        uint32_t spike_ppm, int spike_exp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t z = mix64(base + static_cast<uint64_t>(begin + i));
    const uint32_t sign = static_cast<uint32_t>(z & 1u);
    int e = -24 + static_cast<int>((z >> 1) % 10u);
    const uint32_t mant = static_cast<uint32_t>((z >> 8) & 0x3FFu);
    if (spike_ppm && ((z >> 32) % 1000000u) < spike_ppm) e = spike_exp;
    const uint32_t bits = (sign << 31) | (static_cast<uint32_t>(e + 127) << 23) | (mant << 13);
    dst[i] = narrow(__fmul_rn(__uint_as_float(bits), scale));
  }
}

// Replica hash (the device counterpart of the reference's per-step
// param_hash divergence check, trainer.cpp:136-142, 442-453): the sum mod 2^64
// of mix64(mix64(t << 40 | i) ^ bits(w[t][i])) over every element i of every
// tensor t of this rank's parameter replica. Integer addition is order-free,
// so the value is deterministic and identical on ranks with identical
// replicas, whatever the layout; one differing bit changes it.
__global__ void __launch_bounds__(kThreads) k_replica_hash(const AccTile* __restrict__ tiles,
                                                           const TensorDev* __restrict__ td,
                                                           const float* __restrict__ w,
                                                           unsigned long long* __restrict__ out) {
  const AccTile tile = tiles[blockIdx.x];
  const float* src = w + td[tile.t].flat_off + tile.e0;
  unsigned long long h = 0;
  for (int e = threadIdx.x; e < tile.len; e += kThreads) {
    const uint64_t key = (static_cast<uint64_t>(tile.t) << 40) | static_cast<uint64_t>(tile.e0 + e);
    h += mix64(mix64(key) ^ static_cast<uint64_t>(__float_as_uint(src[e])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

int grid_for(size_t n) {
  const size_t b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(std::min<size_t>(std::max<size_t>(b, 1), 148 * 16));
}

void check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(BO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// A view of part of a workspace.
struct View {
  void* p;
  template <typename T> T* as() { return static_cast<T*>(p); }
};

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { BO_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
  ~DevBuf() { if (p) cudaFree(p); }
  template <typename T> T* as() { return static_cast<T*>(p); }
};

bool is_pow2(float s) {
  if (!(s > 0.0f) || !std::isfinite(s)) return false;
  int e = 0;
  return std::frexp(s, &e) == 0.5f;
}

template <typename W>
void ring_allreduce_impl(bo_ctx* c, float* data, size_t n, bool f16) {
  const int N = c->world, r = c->rank;
  if (N == 1 || n == 0) return;
  if (ring_op_available(c)) {
    // the library's own ring over NVLink (push form, neighbour barriers)
    ring_allreduce_op(c, data, n, f16);
    BO_CUDA(cudaStreamSynchronize(c->stream));  // returns with the data reduced, as the reference
    return;
  }
  need_nccl(c, "bo_ring_allreduce_* without mapped ring buffers");
  cudaStream_t s = c->stream;
  const size_t ch = (n + static_cast<size_t>(N) - 1) / static_cast<size_t>(N);  // collective.cpp:27-29
  // one grow-only workspace per context (the padded buffer, the outgoing
  // and the incoming wire chunk) instead of three allocations per call
  const size_t need = ch * static_cast<size_t>(N) * 4 + 2 * align_up(static_cast<int64_t>(ch * sizeof(W)), 256);
  if (c->op_ws_bytes < need) {
    if (c->op_ws) BO_CUDA(cudaFree(c->op_ws));
    c->op_ws = nullptr;
    BO_CUDA(cudaMalloc(&c->op_ws, need));
    c->op_ws_bytes = need;
  }
  uint8_t* ws = static_cast<uint8_t*>(c->op_ws);
  View buf{ws};
  View wire{ws + ch * static_cast<size_t>(N) * 4};
  View in{ws + ch * static_cast<size_t>(N) * 4 + align_up(static_cast<int64_t>(ch * sizeof(W)), 256)};
  float* B = buf.as<float>();
  BO_CUDA(cudaMemsetAsync(B, 0, ch * static_cast<size_t>(N) * 4, s));
  BO_CUDA(cudaMemcpyAsync(B, data, n * 4, cudaMemcpyDeviceToDevice, s));
  const ncclDataType_t dt = f16 ? ncclFloat16 : ncclFloat32;
  const int right = (r + 1) % N, left = (r - 1 + N) % N;
  auto send_recv = [&](const float* chunk) {
    const void* out = chunk;
    if (f16) {
      k_narrow<<<grid_for(ch), kThreads, 0, s>>>(chunk, wire.as<uint16_t>(), ch);
      check("k_narrow");
      out = wire.p;
    }
    BO_NCCL(ncclGroupStart());
    BO_NCCL(ncclSend(out, ch, dt, right, c->comm, s));
    BO_NCCL(ncclRecv(in.p, ch, dt, left, c->comm, s));
    BO_NCCL(ncclGroupEnd());
  };
  for (int st = 0; st < N - 1; ++st) {  // reduce-scatter (collective.hpp:65-80)
    const size_t send_idx = static_cast<size_t>((r - st + 2 * N) % N);
    const size_t recv_idx = static_cast<size_t>((r - st - 1 + 2 * N) % N);
    send_recv(B + send_idx * ch);
    k_ring_add<W><<<grid_for(ch), kThreads, 0, s>>>(in.as<W>(), B + recv_idx * ch, ch);
    check("k_ring_add");
  }
  for (int st = 0; st < N - 1; ++st) {  // all-gather (collective.hpp:83-96)
    const size_t send_idx = static_cast<size_t>((r + 1 - st + 2 * N) % N);
    const size_t recv_idx = static_cast<size_t>((r - st + 2 * N) % N);
    send_recv(B + send_idx * ch);
    if (f16) {
      k_widen<<<grid_for(ch), kThreads, 0, s>>>(in.as<uint16_t>(), B + recv_idx * ch, ch);
      check("k_widen");
    } else {
      BO_CUDA(cudaMemcpyAsync(B + recv_idx * ch, in.p, ch * 4, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (f16) {  // owner re-round (collective.cpp:79-83)
    k_round_f16<<<grid_for(ch), kThreads, 0, s>>>(B + static_cast<size_t>((r + 1) % N) * ch, ch);
    check("k_round_f16");
  }
  BO_CUDA(cudaMemcpyAsync(data, B, n * 4, cudaMemcpyDeviceToDevice, s));
  BO_CUDA(cudaStreamSynchronize(s));
}

}  // namespace
}  // namespace bo

using namespace bo;

#define BO_OP_BEGIN try {
#define BO_OP_END                \
  }                              \
  catch (const Failure& f) {     \
    set_thread_error(f.msg);     \
    return f.code;               \
  }                              \
  return BO_OK;

extern "C" {

bo_status bo_lamb_step(int32_t T, const int64_t* numels, float* const* params,
                       const float* const* grads, float* const* m, float* const* v, int64_t* step,
                       const bo_lamb_config* cfg, void* stream) {
  BO_OP_BEGIN
  if (T < 0 || !numels || !params || !grads || !m || !v || !step || !cfg) {
    fail(BO_ERR_SHAPE_MISMATCH, "lamb_step: null argument");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  *step += 1;  // lamb.cpp:40, before any check
  const double t = static_cast<double>(*step);
  double bc[4];
  bc[0] = 1.0 - std::pow(static_cast<double>(cfg->beta1), t);
  bc[1] = 1.0 - std::pow(static_cast<double>(cfg->beta2), t);
  bc[2] = 1.0 / bc[0];
  bc[3] = 1.0 / bc[1];
  if (T == 0) return BO_OK;
  std::vector<OpTensor> ts(static_cast<size_t>(T));
  std::vector<OpTile> tiles;
  std::vector<int> tile_begin(static_cast<size_t>(T) + 1);
  for (int i = 0; i < T; ++i) {
    ts[static_cast<size_t>(i)] = OpTensor{params[i], grads[i], m[i], v[i], numels[i]};
    tile_begin[static_cast<size_t>(i)] = static_cast<int>(tiles.size());
    for (int64_t e = 0; e < numels[i]; e += kTileElems) {
      tiles.push_back(OpTile{i, static_cast<int32_t>(std::min<int64_t>(kTileElems, numels[i] - e)), e});
    }
  }
  tile_begin[static_cast<size_t>(T)] = static_cast<int>(tiles.size());
  const size_t nt = tiles.size();
  DevBuf d_ts(ts.size() * sizeof(OpTensor)), d_tiles(nt * sizeof(OpTile)), d_tb(tile_begin.size() * 4),
      d_bc(32), d_key(8), d_part(std::max<size_t>(nt, 1) * 16), d_trust(static_cast<size_t>(T) * 4);
  BO_CUDA(cudaMemcpyAsync(d_ts.p, ts.data(), ts.size() * sizeof(OpTensor), cudaMemcpyHostToDevice, s));
  if (nt) BO_CUDA(cudaMemcpyAsync(d_tiles.p, tiles.data(), nt * sizeof(OpTile), cudaMemcpyHostToDevice, s));
  BO_CUDA(cudaMemcpyAsync(d_tb.p, tile_begin.data(), tile_begin.size() * 4, cudaMemcpyHostToDevice, s));
  BO_CUDA(cudaMemcpyAsync(d_bc.p, bc, 32, cudaMemcpyHostToDevice, s));
  BO_CUDA(cudaMemsetAsync(d_key.p, 0xFF, 8, s));
  unsigned long long key = ~0ull;
  if (nt) {
    k_first_nonfinite<<<static_cast<int>(nt), kThreads, 0, s>>>(d_tiles.as<OpTile>(), d_ts.as<OpTensor>(),
                                                               d_key.as<unsigned long long>());
    check("k_first_nonfinite");
    BO_CUDA(cudaMemcpyAsync(&key, d_key.p, 8, cudaMemcpyDeviceToHost, s));
    BO_CUDA(cudaStreamSynchronize(s));
  }
  int limit_t = T;
  int64_t limit_e = 0;
  if (key != ~0ull) {
    limit_t = static_cast<int>(key >> 40);
    limit_e = static_cast<int64_t>(key & ((1ull << 40) - 1));
  }
  const LambConsts lc{cfg->beta1, cfg->beta2, 1.0f - cfg->beta1, 1.0f - cfg->beta2, cfg->eps,
                      cfg->weight_decay, cfg->lr, cfg->trust_clip};
  if (nt) {
    k_op_norms<<<static_cast<int>(nt), kThreads, 0, s>>>(d_tiles.as<OpTile>(), d_ts.as<OpTensor>(), limit_t, lc,
                                                        d_bc.as<double>(), d_part.as<double>());
    check("k_op_norms");
    k_op_trust<<<(T + 255) / 256, 256, 0, s>>>(d_tb.as<int>(), d_part.as<double>(), T, cfg->trust_clip,
                                              d_trust.as<float>());
    check("k_op_trust");
    k_op_update<<<static_cast<int>(nt), kThreads, 0, s>>>(d_tiles.as<OpTile>(), d_ts.as<OpTensor>(), limit_t,
                                                         limit_e, lc, d_bc.as<double>(), d_trust.as<float>());
    check("k_op_update");
  }
  BO_CUDA(cudaStreamSynchronize(s));
  if (limit_t < T) {
    fail(BO_ERR_NON_FINITE_GRADIENT, "non-finite gradient in tensor " + std::to_string(limit_t));
  }
  BO_OP_END
}

bo_status bo_fused_optimizer_step(int32_t T, const int64_t* numels, float* const* params,
                                  const float* const* grads, float* const* m, float* const* v,
                                  float lr, float beta1, float beta2, float eps,
                                  float weight_decay, int32_t step, void* stream) {
  BO_OP_BEGIN
  if (T < 0 || (T > 0 && (!numels || !params || !grads || !m || !v))) {
    fail(BO_ERR_SHAPE_MISMATCH, "fused_optimizer_step: null argument");
  }
  if (T == 0) return BO_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // graph.cpp:460-462 and the attributes of the body (graph.cpp:468-483)
  const double bc1 = 1.0 / (1.0 - std::pow(static_cast<double>(beta1), step));
  const double bc2 = 1.0 / (1.0 - std::pow(static_cast<double>(beta2), step));
  const AdamConsts k{static_cast<float>(static_cast<double>(beta1)),
                     static_cast<float>(1.0 - static_cast<double>(beta1)),
                     static_cast<float>(static_cast<double>(beta2)),
                     static_cast<float>(1.0 - static_cast<double>(beta2)),
                     static_cast<float>(bc1), static_cast<float>(bc2),
                     static_cast<float>(static_cast<double>(eps)),
                     static_cast<float>(static_cast<double>(weight_decay)),
                     static_cast<float>(-static_cast<double>(lr))};
  int device = 0;
  BO_CUDA(cudaGetDevice(&device));
  int sms = 148;
  BO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  auto tab = std::make_unique<AdamTable>();
  for (int base = 0; base < T; base += kAdamBatch) {
    const int nb = std::min(kAdamBatch, T - base);
    tab->T = nb;
    tab->cstart[0] = 0;
    for (int j = 0; j < nb; ++j) {
      const int i = base + j;
      if (numels[i] < 0) fail(BO_ERR_SHAPE_MISMATCH, "fused_optimizer_step: negative size");
      const bool vec = ((reinterpret_cast<uintptr_t>(params[i]) | reinterpret_cast<uintptr_t>(grads[i]) |
                         reinterpret_cast<uintptr_t>(m[i]) | reinterpret_cast<uintptr_t>(v[i])) & 15u) == 0;
      tab->t[j] = AdamTensor{params[i], grads[i], m[i], v[i], numels[i], vec ? 1 : 0};
      tab->cstart[j + 1] = tab->cstart[j] + (numels[i] + kTileElems - 1) / kTileElems;
    }
    if (tab->cstart[nb] == 0) continue;
    const int grid = static_cast<int>(std::min<int64_t>(tab->cstart[nb], static_cast<int64_t>(sms) * 8));
    k_fused_adam<<<grid, kThreads, 0, s>>>(*tab, k);
    check("k_fused_adam");
  }
  BO_OP_END
}

bo_status bo_f16_round(float* x, size_t n, void* stream) {
  BO_OP_BEGIN
  if (!x && n) fail(BO_ERR_SHAPE_MISMATCH, "f16_round: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n) {
    k_round_f16<<<grid_for(n), kThreads, 0, s>>>(x, n);
    check("k_round_f16");
  }
  BO_OP_END
}

bo_status bo_replica_hash(bo_ctx* c, uint64_t* out) {
  BO_OP_BEGIN
  if (!c || !out) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (c->sync_open) fail(BO_ERR_PROTOCOL, "bo_replica_hash while a sync micro (bo_sync_ready) is open");
  if (!c->hash_acc) c->hash_acc = static_cast<unsigned long long*>(dev_alloc(c, sizeof(unsigned long long)));
  BO_CUDA(cudaMemsetAsync(c->hash_acc, 0, sizeof(unsigned long long), c->stream));
  if (c->n_acc_tiles > 0) {
    k_replica_hash<<<c->n_acc_tiles, kThreads, 0, c->stream>>>(c->d_acc_tiles, c->d_tensors, c->w, c->hash_acc);
    check_launch(c, "k_replica_hash");
  }
  unsigned long long h = 0;
  BO_CUDA(cudaMemcpyAsync(&h, c->hash_acc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  BO_CUDA(cudaStreamSynchronize(c->stream));
  *out = static_cast<uint64_t>(h);
  BO_OP_END
}

bo_status bo_ring_allreduce_f32(bo_ctx* c, float* data, size_t n) {
  BO_OP_BEGIN
  ring_allreduce_impl<float>(c, data, n, false);
  BO_OP_END
}

bo_status bo_ring_allreduce_f16_wire(bo_ctx* c, float* data, size_t n) {
  BO_OP_BEGIN
  ring_allreduce_impl<uint16_t>(c, data, n, true);
  BO_OP_END
}

bo_status bo_unscale_gradients(float* g, size_t n, float scale, int32_t enabled, void* stream) {
  BO_OP_BEGIN
  if (!is_pow2(scale)) {
    fail(BO_ERR_INVALID_CONFIG, "loss scale must be a positive power of two");  // half.cpp:94-99
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return BO_OK;
  DevBuf flag(4);
  BO_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
  k_any_nonfinite<<<grid_for(n), kThreads, 0, s>>>(g, n, flag.as<int>());
  check("k_any_nonfinite");
  int h = 0;
  BO_CUDA(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, s));
  BO_CUDA(cudaStreamSynchronize(s));
  if (h) fail(BO_ERR_OVERFLOW_DETECTED, "non-finite gradient before unscale");
  if (!enabled) return BO_OK;
  k_scale<<<grid_for(n), kThreads, 0, s>>>(g, n, 1.0f / scale);
  check("k_scale");
  BO_CUDA(cudaStreamSynchronize(s));
  BO_OP_END
}

bo_status bo_narrow_f16(const float* src, uint16_t* dst, size_t n, void* stream) {
  BO_OP_BEGIN
  if (n) {
    k_narrow<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
    check("k_narrow");
  }
  BO_OP_END
}

bo_status bo_widen_f16(const uint16_t* src, float* dst, size_t n, void* stream) {
  BO_OP_BEGIN
  if (n) {
    k_widen<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
    check("k_widen");
  }
  BO_OP_END
}

float bo_scale_loss(float loss, float scale, int32_t enabled) { return enabled ? loss * scale : loss; }

bo_status bo_malloc(void** ptr, size_t bytes, int32_t device) {
  BO_OP_BEGIN
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) fail(BO_ERR_NO_DEVICE, "no CUDA device visible");
  BO_CUDA(cudaSetDevice(device));
  BO_CUDA(cudaMalloc(ptr, std::max<size_t>(bytes, 1)));
  BO_OP_END
}

bo_status bo_free(void* ptr) {
  BO_OP_BEGIN
  if (ptr) BO_CUDA(cudaFree(ptr));
  BO_OP_END
}

bo_status bo_memcpy(void* dst, const void* src, size_t bytes, int32_t kind) {
  BO_OP_BEGIN
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                           : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (bytes) BO_CUDA(cudaMemcpy(dst, src, bytes, k));
  BO_OP_END
}

bo_status bo_synth_grads(uint16_t* dst, int64_t begin, int64_t n, uint64_t seed, int32_t rank,
                         int32_t step, int32_t micro, float scale, uint32_t spike_ppm,
                         int32_t spike_exp, void* stream) {
  BO_OP_BEGIN
  auto mix = [](uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  uint64_t h = mix(seed);
  h = mix(h ^ static_cast<uint64_t>(rank));
  h = mix(h ^ static_cast<uint64_t>(step));
  h = mix(h ^ static_cast<uint64_t>(micro));
  if (n > 0) {
    k_synth<<<grid_for(static_cast<size_t>(n)), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        dst, begin, n, h, scale, spike_ppm, spike_exp);
    check("k_synth");
  }
  BO_OP_END
}

}  // extern "C"
