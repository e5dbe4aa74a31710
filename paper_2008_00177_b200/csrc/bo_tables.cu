// Work tables of a context: accumulate / LAMB / ring-hop tiles, communication
// groups of the overlapped sync micro, and the bias-correction table.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "bo_internal.hpp"

namespace bo {

template <typename T>
static T* upload(bo_ctx* c, const std::vector<T>& v) {
  T* d = static_cast<T*>(dev_alloc(c, v.size() * sizeof(T)));
  if (!v.empty()) {
    BO_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  }
  return d;
}

// Work tables: accumulate/finalize tiles over tensors, LAMB tiles over this
// rank's shard (split at tensor boundaries), ring tiles over the shard.
void upload_tables(bo_ctx* c) {
  const Layout& L = c->L;
  std::vector<TensorDev> td(static_cast<size_t>(L.T));
  std::vector<AccTile> acc_tiles;
  for (int t = 0; t < L.T; ++t) {
    td[static_cast<size_t>(t)] = TensorDev{L.acc_off[static_cast<size_t>(t)], L.flat_off[static_cast<size_t>(t)]};
    for (int64_t e = 0; e < L.numel[static_cast<size_t>(t)]; e += kTileElems) {
      const int64_t len = std::min<int64_t>(kTileElems, L.numel[static_cast<size_t>(t)] - e);
      acc_tiles.push_back(AccTile{t, static_cast<int32_t>(len), e});
    }
  }
  std::vector<LambTile> lamb_tiles;
  std::vector<int> tile_begin(static_cast<size_t>(L.T) + 1, 0);
  std::vector<std::vector<LambTile>> per_tensor(static_cast<size_t>(L.T));
  const int q = L.own;  // owned chunk
  for (int b = 0; b < L.B; ++b) {
    const int64_t cb = L.chunk[static_cast<size_t>(b)];
    const int64_t lo = q * cb;
    const int64_t hi = std::min<int64_t>((q + 1) * cb, L.elems[static_cast<size_t>(b)]);
    for (int p : L.buckets[static_cast<size_t>(b)]) {
      const int64_t t0 = L.offset_of[static_cast<size_t>(p)];
      const int64_t t1 = t0 + L.numel[static_cast<size_t>(p)];
      const int64_t a = std::max(lo, t0), z = std::min(hi, t1);
      for (int64_t e = a; e < z; e += kTileElems) {
        const int64_t len = std::min<int64_t>(kTileElems, z - e);
        per_tensor[static_cast<size_t>(p)].push_back(
            LambTile{L.shard_pos(b, p, e), L.flat_pos(b, p, e), static_cast<int32_t>(len), p});
      }
    }
  }
  // Tiles grouped per tensor so each tensor's partials are contiguous; within
  // a tensor, shard order.
  for (int t = 0; t < L.T; ++t) {
    tile_begin[static_cast<size_t>(t)] = static_cast<int>(lamb_tiles.size());
    for (const LambTile& lt : per_tensor[static_cast<size_t>(t)]) lamb_tiles.push_back(lt);
  }
  tile_begin[static_cast<size_t>(L.T)] = static_cast<int>(lamb_tiles.size());

  if (c->world == 1) {
    // Single-rank LAMB (bo_fused.cu): tiles of <= kTileElems elements of one
    // tensor, model order, in the aligned tensor layout; per-tensor tile
    // ranges for the fixed-order norm reduction.
    std::vector<FusedTile> ft;
    std::vector<int> ttiles(static_cast<size_t>(L.T) + 1);
    for (int t = 0; t < L.T; ++t) {
      const int64_t n = L.numel[static_cast<size_t>(t)];
      ttiles[static_cast<size_t>(t)] = static_cast<int>(ft.size());
      for (int64_t e = 0; e < n; e += kTileElems) {
        ft.push_back(FusedTile{L.acc_off[static_cast<size_t>(t)] + e, e,
                               static_cast<int32_t>(std::min<int64_t>(kTileElems, n - e)), t});
      }
    }
    ttiles[static_cast<size_t>(L.T)] = static_cast<int>(ft.size());
    c->d_fused_tiles = upload(c, ft);
    c->n_fused_tiles = static_cast<int>(ft.size());
    c->d_fused_tensor_tiles = upload(c, ttiles);
  }
  if (c->world > 1) {
    // Ring hops with the finalize fused in: for every chunk index q, the
    // valid (non-padding) elements of chunk q of every bucket, split at tensor
    // boundaries, in shard order.
    std::vector<HopXTile> hx;
    c->hopx_begin.assign(static_cast<size_t>(c->world) + 1, 0);
    c->hopx_bucket_begin.assign(static_cast<size_t>(c->world), std::vector<int>(static_cast<size_t>(L.B) + 1, 0));
    for (int qq = 0; qq < c->world; ++qq) {
      c->hopx_begin[static_cast<size_t>(qq)] = static_cast<int>(hx.size());
      for (int b = 0; b < L.B; ++b) {
        c->hopx_bucket_begin[static_cast<size_t>(qq)][static_cast<size_t>(b)] = static_cast<int>(hx.size());
        const int64_t cb = L.chunk[static_cast<size_t>(b)];
        const int64_t lo = qq * cb;
        const int64_t hi = std::min<int64_t>((qq + 1) * cb, L.elems[static_cast<size_t>(b)]);
        for (int p : L.buckets[static_cast<size_t>(b)]) {
          const int64_t t0 = L.offset_of[static_cast<size_t>(p)];
          const int64_t a = std::max(lo, t0), z = std::min(hi, t0 + L.numel[static_cast<size_t>(p)]);
          for (int64_t e = a; e < z; e += kTileElems) {
            hx.push_back(HopXTile{L.shoff[static_cast<size_t>(b)] + (e - lo), e - t0,
                                  static_cast<int32_t>(std::min<int64_t>(kTileElems, z - e)), p});
          }
        }
      }
      c->hopx_bucket_begin[static_cast<size_t>(qq)][static_cast<size_t>(L.B)] = static_cast<int>(hx.size());
    }
    c->hopx_begin[static_cast<size_t>(c->world)] = static_cast<int>(hx.size());
    c->d_hopx_tiles = upload(c, hx);

    // Communication groups for the overlapped sync micro: consecutive buckets
    // (layout order = gradient-ready order) merged up to >= BO_COMM_GROUP_ELEMS
    // elements (default 16 Mi = 64 MiB of fp32 gradient), so every group costs
    // N - 1 hop barriers; a pure function of the layout and the environment,
    // which must therefore match across ranks (it is part of the layout hash).
    int64_t group_elems = 16ll << 20;
    if (const char* e = std::getenv("BO_COMM_GROUP_ELEMS")) {
      group_elems = std::max<int64_t>(1, std::atoll(e));
    }
    c->comm_groups.clear();
    c->group_of_bucket.assign(static_cast<size_t>(L.B), 0);
    std::vector<AccTile> gacc;
    std::vector<int> first_acc_tile(static_cast<size_t>(L.T) + 1, 0);
    for (int t = 0, i = 0; t < L.T; ++t) {
      first_acc_tile[static_cast<size_t>(t)] = i;
      i += static_cast<int>((L.numel[static_cast<size_t>(t)] + kTileElems - 1) / kTileElems);
    }
    int b0 = 0;
    int64_t n = 0;
    for (int b = 0; b < L.B; ++b) {
      n += L.elems[static_cast<size_t>(b)];
      if (n >= group_elems || b == L.B - 1) {
        bo_ctx::CommGroup g{b0, b + 1, 0, static_cast<int>(gacc.size()), 0};
        for (int bb = b0; bb <= b; ++bb) {
          c->group_of_bucket[static_cast<size_t>(bb)] = static_cast<int>(c->comm_groups.size());
          for (int p : L.buckets[static_cast<size_t>(bb)]) {
            g.pending0 += 1;
            const int64_t nt = (L.numel[static_cast<size_t>(p)] + kTileElems - 1) / kTileElems;
            for (int64_t k = 0; k < nt; ++k) gacc.push_back(acc_tiles[static_cast<size_t>(first_acc_tile[static_cast<size_t>(p)] + k)]);
          }
        }
        g.acc1 = static_cast<int>(gacc.size());
        c->comm_groups.push_back(g);
        b0 = b + 1;
        n = 0;
      }
    }
    c->d_group_acc_tiles = upload(c, gacc);

    // Parameter groups of the push, in model order (the forward's first-use
    // order: embeddings, layer 0, ..., heads), >= BO_PUSH_GROUP_ELEMS elements
    // each (default 8 Mi), at most kMaxPushGroups. Every rank derives the same
    // groups from the layout.
    int64_t push_elems = 8ll << 20;
    if (const char* e = std::getenv("BO_PUSH_GROUP_ELEMS")) push_elems = std::max<int64_t>(1, std::atoll(e));
    push_elems = std::max<int64_t>(push_elems, (L.P + kMaxPushGroups - 1) / kMaxPushGroups);
    c->push_group_of_tensor.assign(static_cast<size_t>(L.T), 0);
    int G = 0;
    int64_t acc_n = 0;
    for (int t = 0; t < L.T; ++t) {
      c->push_group_of_tensor[static_cast<size_t>(t)] = G;
      acc_n += L.numel[static_cast<size_t>(t)];
      if (acc_n >= push_elems && t + 1 < L.T) {
        G += 1;
        acc_n = 0;
      }
    }
    c->n_push_groups = G + 1;
    std::vector<LambTile> push;
    std::vector<int> gtiles(static_cast<size_t>(c->n_push_groups), 0);
    int gcur = 0, first_t = 0;
    auto close_group = [&](int g, int t_first) {
      if (gtiles[static_cast<size_t>(g)] == 0) {  // nothing owned here: one empty tile publishes
        push.push_back(LambTile{0, 0, 0, t_first});
        gtiles[static_cast<size_t>(g)] = 1;
      }
    };
    for (int t = 0; t < L.T; ++t) {
      const int g = c->push_group_of_tensor[static_cast<size_t>(t)];
      if (g != gcur) {
        close_group(gcur, first_t);
        gcur = g;
        first_t = t;
      }
      for (int i = tile_begin[static_cast<size_t>(t)]; i < tile_begin[static_cast<size_t>(t) + 1]; ++i) {
        push.push_back(lamb_tiles[static_cast<size_t>(i)]);
        gtiles[static_cast<size_t>(g)] += 1;
      }
    }
    close_group(gcur, first_t);
    c->d_push_tiles = upload(c, push);
    c->n_push_tiles = static_cast<int>(push.size());
    c->d_push_group_of_tensor = upload(c, c->push_group_of_tensor);
    c->d_push_group_tiles = upload(c, gtiles);
    c->d_push_count = static_cast<unsigned*>(dev_alloc(c, static_cast<size_t>(c->n_push_groups) * sizeof(unsigned)));

    // Grouped LAMB: consecutive tensors in model order, >= BO_LAMB_GROUP_ELEMS
    // elements each (0: one group, the serial path). Default: eight groups at
    // world >= 4, where the parameter push (NVLink) is the largest stage and
    // the posted push of group g hides phase 1 of group g + 1 (BERT-large,
    // 4 B200s: 2.60 vs 2.85 ms per step); serial below (2 B200s: within
    // box-to-box variance, profiles/r02_notes.md).
    int64_t lg_elems = L.N >= 4 ? (L.P + 7) / 8 : 0;
    if (lg_elems > 0) {
      // The posted push stores 16-byte vectors only where a rank's shard and
      // the replica share their 16-byte phase, i.e. where owner * c_b is a
      // multiple of 4; other chunks go element by element, which made the
      // step 1.8x slower with 1 GiB buckets (two buckets, odd chunk sizes;
      // profiles/r02_notes.md). Those layouts keep the serial path (its
      // bulk-copy push stages every tile at the replica's phase). Decided
      // from the layout alone, so every rank agrees.
      int64_t odd = 0;
      for (int b = 0; b < L.B; ++b) {
        if (L.chunk[static_cast<size_t>(b)] % 4 != 0) odd += L.elems[static_cast<size_t>(b)];
      }
      if (odd * 10 > L.P) lg_elems = 0;  // > 10 % of the elements (64 MiB at 4 GPUs: 4 %, grouped still faster)
    }
    if (const char* e = std::getenv("BO_LAMB_GROUP_ELEMS")) lg_elems = std::max<int64_t>(0, std::atoll(e));
    c->lamb_groups.clear();
    if (lg_elems > 0) {
      int t0 = 0;
      int64_t n = 0;
      for (int t = 0; t < L.T; ++t) {
        n += L.numel[static_cast<size_t>(t)];
        if (n >= lg_elems || t == L.T - 1) {
          c->lamb_groups.push_back(bo_ctx::LambGroup{t0, t + 1, tile_begin[static_cast<size_t>(t0)],
                                                     tile_begin[static_cast<size_t>(t) + 1]});
          t0 = t + 1;
          n = 0;
        }
      }
      if (c->lamb_groups.size() <= 1) c->lamb_groups.clear();
    }
  }
  c->d_tensors = upload(c, td);
  c->d_acc_tiles = upload(c, acc_tiles);
  c->n_acc_tiles = static_cast<int>(acc_tiles.size());
  c->d_lamb_tiles = upload(c, lamb_tiles);
  c->n_lamb_tiles = static_cast<int>(lamb_tiles.size());
  c->d_tensor_tile_begin = upload(c, tile_begin);
}

// Bias corrections bc_t = 1 - pow(double(beta), double(t)) evaluated on the
// host with the same libm the reference uses (lamb.cpp:41-44), with their
// reciprocals; the device indexes the table by its own step counter.
void grow_bc_table(bo_ctx* c, int64_t need) {
  if (need <= c->bc_cap) return;
  int64_t cap = std::max<int64_t>(4096, c->bc_cap * 2);
  while (cap < need) cap *= 2;
  std::vector<double> tab(static_cast<size_t>(cap) * 4);
  for (int64_t i = 0; i < cap; ++i) {
    const double t = static_cast<double>(i + 1);
    const double bc1 = 1.0 - std::pow(static_cast<double>(c->cfg.lamb.beta1), t);
    const double bc2 = 1.0 - std::pow(static_cast<double>(c->cfg.lamb.beta2), t);
    tab[static_cast<size_t>(4 * i)] = bc1;
    tab[static_cast<size_t>(4 * i + 1)] = bc2;
    tab[static_cast<size_t>(4 * i + 2)] = 1.0 / bc1;
    tab[static_cast<size_t>(4 * i + 3)] = 1.0 / bc2;
  }
  double* d = nullptr;
  BO_CUDA(cudaMalloc(&d, tab.size() * sizeof(double)));
  BO_CUDA(cudaMemcpyAsync(d, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  // The old table may still be read by queued kernels: keep it alive.
  if (c->bc_table) c->allocations.push_back(c->bc_table);
  BO_CUDA(cudaStreamSynchronize(c->stream));  // tab is pageable host memory
  c->bc_table = d;
  c->bc_cap = cap;
}

}  // namespace bo
