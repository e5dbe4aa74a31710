/*
 * TEST INFRASTRUCTURE — synthetic-gradient specification shared by the two
 * CPU oracles (oracle/bo_oracle.cpp and the compiled reference harness in
 * oracle/ref/). The GPU product carries its own, independent implementation
 * of the same spec (paper_2008_00177_b200/csrc/synth.cu); tests check the two
 * agree bit for bit.
 *
 * Spec ("Synthetic gradients"): a counter-based generator so
 * CPU and GPU produce identical fp16 gradient bits without shipping data.
 *   base  = mix(mix(mix(mix(seed) ^ rank) ^ step) ^ micro)
 *   z     = mix(base + flat_index)          flat_index: model-order element id
 *   sign  = z & 1
 *   E     = -24 + ((z >> 1) % 10)           true |g| in [2^-24, 2^-14)
 *   mant  = (z >> 8) & 0x3FF
 *   spike : if spike_ppm && ((z >> 32) % 1000000) < spike_ppm, E = spike_exp
 *   g     = (-1)^sign * (1 + mant/1024) * 2^E       (exact binary32)
 *   h     = f32_to_f16(g * S)                RNE; S = current loss scale
 * The log-uniform magnitudes follow proj/tests/test_half.cpp:143-153.
 */
#ifndef BO_ORACLE_SYNTH_GRAD_H_
#define BO_ORACLE_SYNTH_GRAD_H_

#include <stdint.h>
#include <string.h>

static inline uint64_t bo_mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t bo_synth_base(uint64_t seed, uint64_t rank,
                                     uint64_t step, uint64_t micro) {
  uint64_t h = bo_mix64(seed);
  h = bo_mix64(h ^ rank);
  h = bo_mix64(h ^ step);
  return bo_mix64(h ^ micro);
}

/* True (unscaled) gradient value for one element. */
static inline float bo_synth_true_grad(uint64_t base, uint64_t flat_index,
                                       uint32_t spike_ppm, int spike_exp) {
  const uint64_t z = bo_mix64(base + flat_index);
  const uint32_t sign = (uint32_t)(z & 1u);
  int e = -24 + (int)((z >> 1) % 10u);
  const uint32_t mant = (uint32_t)((z >> 8) & 0x3FFu);
  if (spike_ppm && ((z >> 32) % 1000000u) < spike_ppm) e = spike_exp;
  const uint32_t bits = (sign << 31) | ((uint32_t)(e + 127) << 23) | (mant << 13);
  float g;
  memcpy(&g, &bits, 4);
  return g;
}

#endif /* BO_ORACLE_SYNTH_GRAD_H_ */
