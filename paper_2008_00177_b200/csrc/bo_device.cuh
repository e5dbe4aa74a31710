// Device helpers shared by the pipeline and the operator-level kernels.
// All float arithmetic is explicitly round-to-nearest (no FMA contraction):
// the reference is compiled without FMA (proj/CMakeLists.txt:13-14).
#ifndef BO_DEVICE_CUH_
#define BO_DEVICE_CUH_

#include <cuda_fp16.h>

#include "bo_internal.hpp"

namespace bo {

__device__ __forceinline__ float widen(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ uint16_t narrow(float x) { return __half_as_ushort(__float2half_rn(x)); }

__device__ __forceinline__ bool finite(float x) { return fabsf(x) <= 3.402823466e38f; }

// Wall-clock nanoseconds (the watchdog bound of the cross-rank barriers).
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// float(double(x) / d) with the reference's double rounding (lamb.cpp:68-69),
// computed as a multiply by the host-rounded reciprocal. The product is within
// ~3 double ulps of RN_d(x/d); only when it lies that close to a binary32
// rounding midpoint (or in the binary32 subnormal range) can the two round to
// different floats, and then the exact IEEE division is used instead.
__device__ __forceinline__ float div_to_float(float x, double d, double inv_d) {
  double q = __dmul_rn(static_cast<double>(x), inv_d);
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(q));
  const int low = static_cast<int>(b & 0x1FFFFFFFull) - 0x10000000;
  const unsigned e = static_cast<unsigned>((b >> 52) & 0x7FF);
  if (e < 898u || (low >= -16 && low <= 16)) q = __ddiv_rn(static_cast<double>(x), d);
  return __double2float_rn(q);
}

// Fast path of div_to_float: the product and whether the exact division is
// needed (result within 16 double-ulps of a binary32 midpoint, or binary32
// subnormal range).
__device__ __forceinline__ float div_to_float_fast(float x, double inv_d, bool& need_exact) {
  const double q = __dmul_rn(static_cast<double>(x), inv_d);
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(q));
  const unsigned low = static_cast<unsigned>(b & 0x1FFFFFFFull) - 0x0FFFFFF0u;  // in [0, 32] near a midpoint
  const unsigned e = static_cast<unsigned>((b >> 52) & 0x7FF);
  need_exact |= (e < 898u) | (low <= 32u);
  return __double2float_rn(q);
}

// Four LAMB elements (lamb.cpp:66-70, operation order kept) with one rarely
// taken branch for the exact double divisions instead of one per value.
struct Lamb4 {
  float m[4], v[4], u[4];
};

template <typename C>
__device__ __forceinline__ Lamb4 lamb_elem4(const float (&g)[4], const float (&w)[4],
                                            const float (&m)[4], const float (&v)[4], const C& c,
                                            double bc1, double bc2, double ibc1, double ibc2) {
  Lamb4 o;
  float mh[4], vh[4];
  bool need = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o.m[i] = __fadd_rn(__fmul_rn(c.beta1, m[i]), __fmul_rn(c.omb1, g[i]));
    o.v[i] = __fadd_rn(__fmul_rn(c.beta2, v[i]), __fmul_rn(__fmul_rn(c.omb2, g[i]), g[i]));
    mh[i] = div_to_float_fast(o.m[i], ibc1, need);
    vh[i] = div_to_float_fast(o.v[i], ibc2, need);
  }
  if (__builtin_expect(need, 0)) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mh[i] = __double2float_rn(__ddiv_rn(static_cast<double>(o.m[i]), bc1));
      vh[i] = __double2float_rn(__ddiv_rn(static_cast<double>(o.v[i]), bc2));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float den = __fadd_rn(__fsqrt_rn(vh[i]), c.eps);
    o.u[i] = __fadd_rn(__fdiv_rn(mh[i], den), __fmul_rn(c.wd, w[i]));
  }
  return o;
}

// The same with the exact-division operands read from memory only on the rare
// path (bcp -> {bc1, bc2}), which keeps two doubles out of the register file.
template <typename C>
__device__ __forceinline__ Lamb4 lamb_elem4(const float (&g)[4], const float (&w)[4],
                                            const float (&m)[4], const float (&v)[4], const C& c,
                                            const double* bcp, double ibc1, double ibc2) {
  Lamb4 o;
  float mh[4], vh[4];
  bool need = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o.m[i] = __fadd_rn(__fmul_rn(c.beta1, m[i]), __fmul_rn(c.omb1, g[i]));
    o.v[i] = __fadd_rn(__fmul_rn(c.beta2, v[i]), __fmul_rn(__fmul_rn(c.omb2, g[i]), g[i]));
    mh[i] = div_to_float_fast(o.m[i], ibc1, need);
    vh[i] = div_to_float_fast(o.v[i], ibc2, need);
  }
  if (__builtin_expect(need, 0)) {
    const double bc1 = bcp[0], bc2 = bcp[1];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mh[i] = __double2float_rn(__ddiv_rn(static_cast<double>(o.m[i]), bc1));
      vh[i] = __double2float_rn(__ddiv_rn(static_cast<double>(o.v[i]), bc2));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float den = __fadd_rn(__fsqrt_rn(vh[i]), c.eps);
    o.u[i] = __fadd_rn(__fdiv_rn(mh[i], den), __fmul_rn(c.wd, w[i]));
  }
  return o;
}

struct Moments {
  float m, v, u;
};

// One element of lamb_step's fused loop (lamb.cpp:66-70), operation order kept.
__device__ __forceinline__ Moments lamb_elem(float g, float w, float m, float v, const LambConsts& c,
                                             const double* bc) {
  Moments o;
  o.m = __fadd_rn(__fmul_rn(c.beta1, m), __fmul_rn(c.omb1, g));
  o.v = __fadd_rn(__fmul_rn(c.beta2, v), __fmul_rn(__fmul_rn(c.omb2, g), g));
  const float mh = div_to_float(o.m, bc[0], bc[2]);
  const float vh = div_to_float(o.v, bc[1], bc[3]);
  const float den = __fadd_rn(__fsqrt_rn(vh), c.eps);
  o.u = __fadd_rn(__fdiv_rn(mh, den), __fmul_rn(c.wd, w));
  return o;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Any binary16 in the packed pair x has an all-ones exponent (inf or NaN).
__device__ __forceinline__ bool pair_nonfinite(uint32_t x) {
  const uint32_t e = x & 0x7C007C00u;
  return (e & 0xFFFFu) == 0x7C00u || (e >> 16) == 0x7C00u;
}

// The step's overflow flag accumulates across micro-batches: a non-finite
// binary16 input makes the accumulated gradient non-finite (an fp32 sum of at
// most K values <= 65504 cannot overflow on its own), so OR-ing the inputs'
// flags equals checking the finalized gradient lamb_step would see
// (lamb.cpp:61-65) on a single rank.
__device__ __forceinline__ void raise_flag(bool bad, DevState* st) {
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->local_flag, 1);
}

// All K micro-batches of one step resident (bo_train_step). p[k] points at
// micro k's gradient of the current tile (a per-CTA/per-warp table in shared
// memory); the flattened sync gradient before the unscale is the reference's
// live + summed, summed = ((0 + g0) + g1) + ... + g_{K-2} (trainer.cpp:240-244,
// 196-201): the same additions in the same order as the accumulator path.
__device__ __forceinline__ void widen4(uint2 x, float (&o)[4]) {
  o[0] = widen(static_cast<uint16_t>(x.x & 0xFFFFu));
  o[1] = widen(static_cast<uint16_t>(x.x >> 16));
  o[2] = widen(static_cast<uint16_t>(x.y & 0xFFFFu));
  o[3] = widen(static_cast<uint16_t>(x.y >> 16));
}

__device__ __forceinline__ float micro_sum1(const uint16_t* const* p, int K, int e) {
  float acc = 0.0f;
  for (int k = 0; k + 1 < K; ++k) acc = __fadd_rn(acc, widen(p[k][e]));
  const float live = widen(p[K - 1][e]);
  return K > 1 ? __fadd_rn(live, acc) : live;
}

// Elements e..e+3 with K known at compile time (all K loads first).
template <int K>
__device__ __forceinline__ void micro_sum4_k(const uint16_t* const* p, int e, float (&o)[4]) {
  uint2 x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = __ldcs(reinterpret_cast<const uint2*>(p[k] + e));
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k + 1 < K; ++k) {
    float f[4];
    widen4(x[k], f);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], f[i]);
  }
  widen4(x[K - 1], o);
  if (K > 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = __fadd_rn(o[i], acc[i]);
  }
}

// Ring wire element type W (float or binary16 bits).
template <typename W>
__device__ __forceinline__ W to_wire(float p);
template <>
__device__ __forceinline__ float to_wire<float>(float p) { return p; }
template <>
__device__ __forceinline__ uint16_t to_wire<uint16_t>(float p) { return narrow(p); }
__device__ __forceinline__ float from_wire(float w) { return w; }
__device__ __forceinline__ float from_wire(uint16_t w) { return widen(w); }

// Streaming accesses with explicit L2 eviction priority (no L1 allocation):
// evict_first for data read once, evict_last for what the next pass re-reads.
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
__device__ __forceinline__ float4 ld4(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ld2u(const uint16_t* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
// Four binary16 values starting at p when n >= 4 valid elements remain, else
// only the n < 4 valid ones (the rest zero): a caller's gradient tensor may
// end right at its allocation, so the last group of a tensor never loads past
// it.
__device__ __forceinline__ uint2 ld_h4(const uint16_t* p, int n, uint64_t pol) {
  if (n >= 4) return ld2u(p, pol);
  uint32_t h[4] = {0u, 0u, 0u, 0u};
  for (int i = 0; i < n; ++i) h[i] = p[i];
  return make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
}
// Bulk L2 prefetch of the 16-byte aligned part of [p, p + bytes) (a hint:
// no data moves into the SM; never touches memory outside the range).
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t bytes) {
  const uintptr_t lo = (reinterpret_cast<uintptr_t>(p) + 15) & ~static_cast<uintptr_t>(15);
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes) & ~static_cast<uintptr_t>(15);
  if (hi > lo) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(static_cast<uint32_t>(hi - lo))
                 : "memory");
  }
}
__device__ __forceinline__ void st4(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol));
}

}  // namespace bo

#endif  // BO_DEVICE_CUH_
