// Fusion-buffer layout and HBM placement (host side, built once per context).
//
// The bucket assignment restates BucketLayout::build (reference
// proj/core/src/trainer.cpp:73-116): parameters sorted by descending
// first-consumer id (ties by index), packed greedily; a bucket closes before
// it would exceed bucket_bytes and an oversized parameter sits alone. The
// per-bucket chunking is the ring's c_b = ceil(n_b / world) with zero padding
// to world * c_b (collective.hpp:44-60), so chunk boundaries — and therefore
// the reference's per-element fold order — are preserved exactly.
#include <algorithm>
#include <numeric>

#include "bo_internal.hpp"

namespace bo {

Layout Layout::build(int T, const int64_t* numel, const int32_t* firsts, uint64_t bucket_bytes,
                     int world, int rank) {
  if (T <= 0) fail(BO_ERR_INVALID_CONFIG, "n_tensors must be > 0");
  if (bucket_bytes == 0) fail(BO_ERR_INVALID_CONFIG, "bucket_bytes must be > 0");
  if (world < 1 || rank < 0 || rank >= world) fail(BO_ERR_INVALID_CONFIG, "bad rank/world");
  Layout L;
  L.T = T;
  L.N = world;
  L.rank = rank;
  L.own = rank;
  L.numel.assign(numel, numel + T);
  // Zero-element tensors are legal (the reference's Tensor allows them:
  // they join a bucket with 0 bytes, own no tiles and get trust ratio 1); a
  // model without any element is not.
  int64_t total = 0;
  for (int t = 0; t < T; ++t) {
    if (numel[t] < 0) fail(BO_ERR_SHAPE_MISMATCH, "tensor " + std::to_string(t) + " has a negative size");
    total += numel[t];
  }
  if (total == 0) fail(BO_ERR_SHAPE_MISMATCH, "the model has no parameter elements");
  L.ready.resize(static_cast<size_t>(T));
  std::iota(L.ready.begin(), L.ready.end(), 0);
  std::stable_sort(L.ready.begin(), L.ready.end(),
                   [&](int a, int b) { return firsts[a] > firsts[b]; });
  L.bucket_of.assign(static_cast<size_t>(T), -1);
  L.offset_of.assign(static_cast<size_t>(T), 0);
  uint64_t cur_bytes = 0;
  for (int p : L.ready) {
    const uint64_t bytes = static_cast<uint64_t>(numel[p]) * sizeof(float);
    if (L.buckets.empty() || cur_bytes + bytes > bucket_bytes) {  // close before exceeding
      L.buckets.emplace_back();
      L.elems.push_back(0);
      cur_bytes = 0;
    }
    L.bucket_of[static_cast<size_t>(p)] = static_cast<int>(L.buckets.size()) - 1;
    L.offset_of[static_cast<size_t>(p)] = L.elems.back();
    L.buckets.back().push_back(p);
    L.elems.back() += numel[p];
    cur_bytes += bytes;
  }
  L.B = static_cast<int>(L.buckets.size());

  L.chunk.resize(static_cast<size_t>(L.B));
  L.base.resize(static_cast<size_t>(L.B));
  L.shoff.resize(static_cast<size_t>(L.B));
  int64_t flat = 0, shard = 0;
  for (int b = 0; b < L.B; ++b) {
    const int64_t c = (L.elems[static_cast<size_t>(b)] + world - 1) / world;
    L.chunk[static_cast<size_t>(b)] = c;
    L.base[static_cast<size_t>(b)] = flat;
    L.shoff[static_cast<size_t>(b)] = shard;
    flat += align_up(c * world, kAlignElems);
    shard += align_up(c, kAlignElems);
  }
  L.flat_total = flat;
  L.shard_total = shard;

  L.flat_off.resize(static_cast<size_t>(T));
  L.acc_off.resize(static_cast<size_t>(T));
  L.model_off.resize(static_cast<size_t>(T));
  int64_t acc = 0, model = 0;
  for (int t = 0; t < T; ++t) {
    L.flat_off[static_cast<size_t>(t)] =
        L.base[static_cast<size_t>(L.bucket_of[static_cast<size_t>(t)])] + L.offset_of[static_cast<size_t>(t)];
    L.acc_off[static_cast<size_t>(t)] = acc;
    L.model_off[static_cast<size_t>(t)] = model;
    acc += align_up(numel[t], kAlignElems);
    model += numel[t];
  }
  L.acc_total = acc;
  L.P = model;
  if (world == 1) {
    // One rank: no collective touches the fusion buffer, so every per-tensor
    // array (params, moments, gradients) uses the 256-byte aligned tensor
    // layout and the LAMB kernels run fully vectorised. The bucket layout
    // itself (bucket_of / offset_of / hash) is unchanged.
    L.flat_off = L.acc_off;
    L.flat_total = L.acc_total;
    L.shard_total = L.acc_total;
  }
  return L;
}

}  // namespace bo
