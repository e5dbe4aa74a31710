// Single-process probe of the world > 1 LAMB kernels on real BERT layouts:
// times k_lamb_p1 / k_p1w variants / k_hopx / k_shard_p2_push of rank `rank` of a
// `world`-rank layout, with the ring input either local or on a peer GPU
// (cudaDeviceEnablePeerAccess, no NCCL), so ncu can profile them in
// isolation. Values are synthetic (timing only, not a parity check).
//   make -C tools p1_probe && tools/p1_probe tools/bert_large.txt 2 0
#include "../paper_2008_00177_b200/csrc/bo_pipeline.cu"
#include "../paper_2008_00177_b200/csrc/bo_fused.cu"
#include "../paper_2008_00177_b200/csrc/bo_ring.cu"

#include <cstdio>
#include <fstream>
#include <vector>

using namespace bo;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

// Deterministic pseudo-random fill (splitmix64 of the index): realistic
// magnitudes so the LAMB arithmetic takes its common paths.
__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float rnd(uint64_t i, uint64_t salt) {  // uniform in (-1, 1)
  return static_cast<float>(static_cast<int64_t>(mix(i * 7 + salt)) >> 11) * 0x1.0p-52f;
}
__global__ void fill_f32(float* p, int64_t n, float scale, int positive, uint64_t salt) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
    const float r = rnd(i, salt);
    p[i] = scale * (positive ? fabsf(r) + 0.01f : r);
  }
}
__global__ void fill_f16(uint16_t* p, int64_t n, float scale, uint64_t salt) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) p[i] = narrow(scale * rnd(i, salt));
}

int main(int argc, char** argv) {
  if (argc < 4) { printf("usage: p1_probe spec.txt world rank [reps]\n"); return 2; }
  std::ifstream f(argv[1]);
  int T;
  f >> T;
  std::vector<int64_t> numel(T);
  std::vector<int32_t> first(T);
  for (int i = 0; i < T; ++i) f >> numel[i] >> first[i];
  const int world = atoi(argv[2]), rank = atoi(argv[3]);
  const int reps = argc > 4 ? atoi(argv[4]) : 10;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const bool peer = ndev > 1;
  bo_trainer_config cfg;
  bo_default_config(&cfg);
  cfg.accumulation = 4;
  cfg.f16_exchange = 1;
  cfg.reduce_algo = BO_REDUCE_RING;
  bo_ctx* c = nullptr;
  if (bo_create(&cfg, T, numel.data(), first.data(), nullptr, nullptr, nullptr, 0, rank, world, &c) != BO_OK) {
    printf("bo_create: %s\n", bo_last_error());
    return 1;
  }
  CK(cudaSetDevice(0));
  const Layout& L = c->L;
  if (world == 1) {  // one rank: the weights are the aligned flat replica, no staging
    c->wsh = c->w;
    c->wire[0] = c->x;
    c->wire[1] = c->x;
  }
  // caller gradients (binary16, one aligned slot per tensor)
  PtrTable tab{};
  int64_t tot = 0;
  for (int t = 0; t < T; ++t) tot += align_up(numel[t], 64);
  uint16_t* g16;
  CK(cudaMalloc(&g16, tot * 2));
  fill_f16<<<1024, 256>>>(g16, tot, 4096.0f * 0.01f, 1);
  int64_t o2 = 0;
  for (int t = 0; t < T; ++t) { tab.p[t] = g16 + o2; o2 += align_up(numel[t], 64); }
  fill_f32<<<1024, 256>>>(c->acc, L.acc_total, 4096.0f * 0.03f, 0, 2);
  if (world > 1) {
    fill_f16<<<1024, 256>>>(static_cast<uint16_t*>(c->wire[0]), L.shard_total, 0.01f, 3);
    fill_f16<<<1024, 256>>>(static_cast<uint16_t*>(c->wire[1]), L.shard_total, 0.01f, 4);
  }
  fill_f32<<<1024, 256>>>(c->wsh, L.shard_total, 0.05f, 0, 5);
  for (float* p : {c->m, c->m_alt}) fill_f32<<<1024, 256>>>(p, L.shard_total, 1e-3f, 0, 6);
  for (float* p : {c->v, c->v_alt}) fill_f32<<<1024, 256>>>(p, L.shard_total, 1e-6f, 1, 7);
  CK(cudaDeviceSynchronize());
  // a peer-resident copy of the staging buffer and of the flat replica
  void* pwire = c->wire[1];
  float* pw = nullptr;
  if (peer) {
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaMalloc(&pwire, L.shard_total * 2));
    fill_f16<<<1024, 256>>>(static_cast<uint16_t*>(pwire), L.shard_total, 0.01f, 8);
    CK(cudaDeviceSynchronize());
    CK(cudaMalloc(&pw, L.flat_total * 4));
    CK(cudaSetDevice(0));
  }
  float** d_peer_w;
  CK(cudaMalloc(&d_peer_w, 8 * sizeof(float*)));
  std::vector<float*> pws(8, c->w);
  // replicas of the other ranks on distinct GPUs where the box has them
  for (int r = 0, j = 0; r < world; ++r) {
    if (r == rank || !peer) continue;
    const int dev = 1 + (j++ % (ndev - 1));
    if (dev == 1) {
      pws[r] = pw;
    } else {
      CK(cudaDeviceEnablePeerAccess(dev, 0));
      CK(cudaSetDevice(dev));
      CK(cudaDeviceEnablePeerAccess(0, 0));
      CK(cudaMalloc(&pws[r], L.flat_total * 4));
      CK(cudaSetDevice(0));
    }
  }
  CK(cudaMemcpy(d_peer_w, pws.data(), 8 * sizeof(float*), cudaMemcpyHostToDevice));
  DevState st{};
  CK(cudaMemcpy(&st, c->state, sizeof(st), cudaMemcpyDeviceToHost));
  st.do_update = 1;
  st.lamb_step = 1000;  // a typical bias-correction regime
  grow_bc_table(c, 2048);
  CK(cudaMemcpy(c->state, &st, sizeof(st), cudaMemcpyHostToDevice));
  const float invn = 1.0f / world;
  const P1Args A{c->d_tensors, c->acc, c->cfg.accumulation, invn, c->wsh, c->m, c->v,
                 c->m_alt, c->v_alt, c->u, c->state, c->lamb, c->bc_table, c->tile_part};
  const uint16_t* lin = static_cast<const uint16_t*>(c->wire[1]);
  const uint16_t* pin = static_cast<const uint16_t*>(pwire);
  const int q = L.own;
  const double S = static_cast<double>(L.shard_total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, double hbm_b, double nvl_b, auto&& launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const cudaError_t e = cudaGetLastError();
    printf("%-34s %8.3f ms  HBM %6.0f GB/s  NVL %5.0f GB/s  %s\n", name, ms, hbm_b / ms / 1e6,
           nvl_b / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  printf("world %d rank %d: %d tensors, shard %lld elems, %d lamb tiles, peer %d\n", world, rank, T,
         (long long)L.shard_total, c->n_lamb_tiles, (int)peer);
  const int wgrid = (c->n_lamb_tiles * 32 + kWarpTileCTA - 1) / kWarpTileCTA;
  if (world == 1) {
    time("k_lamb_p1 (one rank)", 30 * S, 0, [&] {
      k_lamb_p1<<<c->n_fused_tiles, kP1Threads>>>(c->d_fused_tiles, tab, c->acc, c->w, c->m, c->v, c->m_alt,
                                                   c->v_alt, c->u, c->state, c->lamb, c->bc_table, 4,
                                                   c->tile_part);
    });
    time("k_p1w<x> U1 B4 (one rank)", 30 * S, 0, [&] {
      k_p1w<float, false, true, 1, 4><<<wgrid, kWarpTileCTA>>>(c->d_lamb_tiles, c->n_lamb_tiles, tab, nullptr, A);
    });
    {  // p1 right after the last accumulate micro (the pipeline's order)
      cudaEvent_t x0, x1, y0;
      cudaEventCreate(&x0); cudaEventCreate(&x1); cudaEventCreate(&y0);
      float tot = 0.0f, tacc = 0.0f;
      for (int i = 0; i < reps; ++i) {
        cudaEventRecord(y0);
        k_accumulate<true><<<c->n_acc_tiles, kThreads>>>(c->d_acc_tiles, c->d_tensors, tab, c->acc, 0, c->state, 1);
        cudaEventRecord(x0);
        k_lamb_p1<<<c->n_fused_tiles, kP1Threads>>>(c->d_fused_tiles, tab, c->acc, c->w, c->m, c->v, c->m_alt,
                                                     c->v_alt, c->u, c->state, c->lamb, c->bc_table, 4,
                                                     c->tile_part);
        cudaEventRecord(x1);
        cudaEventSynchronize(x1);
        float a, b;
        cudaEventElapsedTime(&a, y0, x0);
        cudaEventElapsedTime(&b, x0, x1);
        tacc += a;
        tot += b;
      }
      printf("%-34s %8.3f ms  (accumulate before it %.3f ms)\n", "k_lamb_p1 after k_accumulate", tot / reps,
             tacc / reps);
    }
    time("k_lamb_p2 (one rank)", 12 * S, 0, [&] {
      k_lamb_p2<<<c->n_fused_tiles, kP2Threads>>>(c->d_fused_tiles, c->n_fused_tiles, c->w, c->u, c->state,
                                                  c->lamb, c->trust);
    });
    bo_destroy(c);
    return 0;
  }
  const int t0 = c->hopx_begin[q], t1 = c->hopx_begin[q + 1];
  time("k_p1w<f16,in,x> U1 B4 local", 30 * S + 2 * S, 0, [&] {
    k_p1w<uint16_t, true, true, 1, 4><<<wgrid, kWarpTileCTA>>>(c->d_lamb_tiles, c->n_lamb_tiles, tab, lin, A);
  });
  time("k_p1w<f16,in,x> U1 B4 peer", 30 * S, 2 * S, [&] {
    k_p1w<uint16_t, true, true, 1, 4><<<wgrid, kWarpTileCTA>>>(c->d_lamb_tiles, c->n_lamb_tiles, tab, pin, A);
  });
  time("k_p1w<f16,in> U1 B4 staged local", 26 * S, 0, [&] {
    k_p1w<uint16_t, true, false, 1, 4><<<wgrid, kWarpTileCTA>>>(c->d_lamb_tiles, c->n_lamb_tiles, tab, lin, A);
  });
  time("k_hopx<f16> (own chunk) local", 10 * S, 0, [&] {
    k_hopx<uint16_t, 0><<<t1 - t0, kThreads>>>(c->d_hopx_tiles + t0, c->d_tensors, tab, MicroSrc{nullptr, 0, 0}, c->acc, c->state,
                                            4, lin, static_cast<uint16_t*>(c->wire[0]), 1);
  });
  time("k_hopx<f16> (own chunk) peer", 8 * S, 2 * S, [&] {
    k_hopx<uint16_t, 0><<<t1 - t0, kThreads>>>(c->d_hopx_tiles + t0, c->d_tensors, tab, MicroSrc{nullptr, 0, 0}, c->acc, c->state,
                                            4, pin, static_cast<uint16_t*>(c->wire[0]), 1);
  });
  // resident micros (bo_train_step): K = 4 binary16 gradient sets
  std::vector<const uint16_t*> mt(4 * static_cast<size_t>(T));
  for (int k = 0; k < 4; ++k) {
    uint16_t* gk;
    CK(cudaMalloc(&gk, tot * 2));
    fill_f16<<<1024, 256>>>(gk, tot, 4096.0f * 0.01f, 10 + k);
    int64_t o = 0;
    for (int t = 0; t < T; ++t) { mt[static_cast<size_t>(k) * T + t] = gk + o; o += align_up(numel[t], 64); }
  }
  const uint16_t** dmt;
  CK(cudaMalloc(&dmt, mt.size() * sizeof(void*)));
  CK(cudaMemcpy(dmt, mt.data(), mt.size() * sizeof(void*), cudaMemcpyHostToDevice));
  const MicroSrc ms4{dmt, 4, T};
  time("k_hopx<f16, K=4> pack (own chunk)", 10 * S, 0, [&] {
    k_hopx<uint16_t, 4><<<t1 - t0, kThreads>>>(c->d_hopx_tiles + t0, c->d_tensors, tab, ms4, c->acc, c->state,
                                              4, nullptr, static_cast<uint16_t*>(c->wire[0]), 0);
  });
  time("k_hopx<f16, K=4> (own chunk) peer", 10 * S, 2 * S, [&] {
    k_hopx<uint16_t, 4><<<t1 - t0, kThreads>>>(c->d_hopx_tiles + t0, c->d_tensors, tab, ms4, c->acc, c->state,
                                              4, pin, static_cast<uint16_t*>(c->wire[0]), 1);
  });
  time("k_hopx<f16> pack (own chunk)", 8 * S, 0, [&] {
    k_hopx<uint16_t, 0><<<t1 - t0, kThreads>>>(c->d_hopx_tiles + t0, c->d_tensors, tab, MicroSrc{nullptr, 0, 0}, c->acc, c->state,
                                            4, nullptr, static_cast<uint16_t*>(c->wire[0]), 0);
  });
  time("k_shard_p2_push (peer replicas)", 16 * S, 4.0 * (world - 1) * S, [&] {
    k_shard_p2_push<<<c->n_lamb_tiles, kThreads>>>(c->d_lamb_tiles, c->wsh, c->u, c->state, c->lamb,
                                                   c->trust, d_peer_w, world);
  });
  bo_destroy(c);
  return 0;
}
