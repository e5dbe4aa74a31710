// SM-partition probe: can a FEW SMs drive the NVLink parameter push (posted
// 16-byte stores to the peers) while the other SMs stream HBM (LAMB phase 1's
// byte mix)? GPU 0 writes a 336 MB / (N-1)-peer shard from HBM into every
// peer with a persistent grid of G CTAs, alone and concurrently with an
// HBM-streaming kernel on a second stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_partition tools/nvl_partition.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                                 \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

struct Dsts {
  float4* p[8];
  int n;
};

// persistent push: every thread keeps U independent 16-byte loads in flight
// and posts their stores to every peer (no completion wait)
template <int U>
__global__ void __launch_bounds__(1024) k_push(const float4* __restrict__ src, Dsts d, int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nv; i0 += U * stride) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < nv) x[u] = __ldcs(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < nv)
        for (int j = 0; j < d.n; ++j) __stcs(d.p[j] + i, x[u]);
    }
  }
}

// LAMB phase 1's mix: 5 arrays read, 3 written (32 B per element-equivalent)
__global__ void k_stream(const float4* a, const float4* b, const float4* c, float4* d, float4* e, float4* f,
                         int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = __ldcs(a + i), y = __ldcs(b + i), z = __ldcs(c + i);
    __stcs(d + i, make_float4(x.x + y.x * z.x, x.y + y.y * z.y, x.z + y.z * z.z, x.w + y.w * z.w));
    __stcs(e + i, x);
    __stcs(f + i, y);
  }
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const int N = ndev;
  const int64_t P = 336226108;
  const int64_t shard_bytes = P / N * 4;  // this rank's master shard
  const int64_t nv = shard_bytes / 16;
  std::vector<float4*> rep(N);
  for (int dv = 0; dv < N; ++dv) {
    CK(cudaSetDevice(dv));
    for (int pe = 0; pe < N; ++pe)
      if (pe != dv) CK(cudaDeviceEnablePeerAccess(pe, 0));
    CK(cudaMalloc(&rep[dv], shard_bytes));
    CK(cudaMemset(rep[dv], 0, shard_bytes));
  }
  CK(cudaSetDevice(0));
  float4* src;
  CK(cudaMalloc(&src, shard_bytes));
  CK(cudaMemset(src, 0, shard_bytes));
  const int64_t nv2 = P / N / 4 * 6 / 6;  // phase-1-sized stream: P/N elements ~ 32 B each
  float4* s[6];
  for (auto& x : s) CK(cudaMalloc(&x, nv2 * 16));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t sa, sb;
  CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  cudaEvent_t a0, a1, b0, b1;
  for (cudaEvent_t* ev : {&a0, &a1, &b0, &b1}) CK(cudaEventCreate(ev));
  Dsts d{};
  d.n = N - 1;
  for (int j = 1; j < N; ++j) d.p[j - 1] = rep[j];
  const double push_bytes = (double)shard_bytes * (N - 1);
  const double stream_bytes = (double)nv2 * 16 * 6;
  auto push = [&](int G, int T, cudaStream_t st) { k_push<4><<<G, T, 0, st>>>(src, d, nv); };
  auto strm = [&](int G, cudaStream_t st) { k_stream<<<G, 512, 0, st>>>(s[0], s[1], s[2], s[3], s[4], s[5], nv2); };
  // alone
  float ms;
  for (int w = 0; w < 3; ++w) strm(4 * sms, sb);
  CK(cudaEventRecord(b0, sb));
  for (int it = 0; it < 10; ++it) strm(4 * sms, sb);
  CK(cudaEventRecord(b1, sb));
  CK(cudaEventSynchronize(b1));
  CK(cudaEventElapsedTime(&ms, b0, b1));
  const float stream_alone = ms / 10;
  printf("world %d: push %.1f MB to %d peer(s); stream kernel alone %.3f ms (%.0f GB/s)\n", N, shard_bytes / 1e6, N - 1,
         stream_alone, stream_bytes / (stream_alone * 1e-3) / 1e9);
  for (int T : {512, 1024}) {
    for (int G : {8, 16, 24, 32, 48, 64, 96, 148, 296}) {
      if (T == 1024 && G > 148) continue;
      push(G, T, sa);
      CK(cudaStreamSynchronize(sa));
      CK(cudaEventRecord(a0, sa));
      for (int it = 0; it < 5; ++it) push(G, T, sa);
      CK(cudaEventRecord(a1, sa));
      CK(cudaEventSynchronize(a1));
      CK(cudaEventElapsedTime(&ms, a0, a1));
      const float pa = ms / 5;
      // concurrent: the push (G CTAs) and the stream kernel (all SMs) on two streams
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a0, sa));
      CK(cudaEventRecord(b0, sb));
      for (int it = 0; it < 5; ++it) push(G, T, sa);
      CK(cudaEventRecord(a1, sa));
      int kit = 0;
      while (cudaEventQuery(a1) == cudaErrorNotReady && kit < 400) {
        strm(4 * sms, sb);
        ++kit;
        CK(cudaStreamSynchronize(sb));
      }
      CK(cudaEventRecord(b1, sb));
      CK(cudaDeviceSynchronize());
      float pms, kms;
      CK(cudaEventElapsedTime(&pms, a0, a1));
      CK(cudaEventElapsedTime(&kms, b0, b1));
      printf("push G=%3d x %4d: alone %.3f ms (%.0f GB/s out) | with stream: push %.3f ms (%.0f GB/s), stream %.3f ms/launch (%.2fx alone)\n",
             G, T, pa, push_bytes / (pa * 1e-3) / 1e9, pms / 5, push_bytes / (pms / 5 * 1e-3) / 1e9, kit ? kms / kit : 0.f,
             kit ? kms / kit / stream_alone : 0.f);
    }
  }
  return 0;
}
