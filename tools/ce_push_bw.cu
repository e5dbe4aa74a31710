// Copy-engine push probe: can the parameter all-gather run on the copy
// engines at NVLink speed, leaving the SMs to LAMB phase 1? GPU 0 pushes the
// owned chunk of every bucket (nb chunks of `chunk` bytes, stride = N chunks,
// the fusion-buffer layout of a world of N) into GPU 1..N-1, as
//   (a) one contiguous copy per peer (the bound),
//   (b) one cudaMemcpyAsync per chunk per peer (round 2's CE graph form),
//   (c) one cudaMemcpyAsync per chunk per peer, one stream per peer,
// each alone and (d) while an HBM-streaming kernel runs on all SMs of GPU 0
// (the overlap the push would buy: the kernel's slowdown is the cost).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ce_push_bw tools/ce_push_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                       \
      return 1;                                                            \
    }                                                                      \
  } while (0)

// 32 B/elem streaming kernel (reads 5 arrays, writes 3: LAMB phase 1's mix)
__global__ void k_stream(const float4* a, const float4* b, const float4* c2, float4* d, float4* e, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = __ldcs(a + i), y = __ldcs(b + i), z = __ldcs(c2 + i);
    float4 o = make_float4(x.x + y.x * z.x, x.y + y.y * z.y, x.z + y.z * z.z, x.w + y.w * z.w);
    __stcs(d + i, o);
    __stcs(e + i, x);
  }
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const int N = ndev;                     // world
  const int nb = argc > 1 ? atoi(argv[1]) : 294;   // buckets
  const int64_t P = 336226108;            // BERT-large parameters
  const int64_t shard = P / N * 4;        // bytes this rank pushes to each peer
  const int64_t chunk = (shard / nb + 255) / 256 * 256;
  const int64_t flat = chunk * N * nb;
  std::vector<char*> rep(N);
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < N; ++p)
      if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&rep[d], flat));
    CK(cudaMemset(rep[d], 1, flat));
  }
  CK(cudaSetDevice(0));
  // stream kernel: the bytes of LAMB phase 1 on a shard (P/N x 32 B over 5 arrays)
  const int64_t nv2 = (int64_t)(P / N) * 2 / 5;
  float4 *a, *b, *c2, *d, *e;
  for (float4** x : {&a, &b, &c2, &d, &e}) CK(cudaMalloc(x, nv2 * 16));
  cudaStream_t sk, sc[8];
  CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
  for (int i = 0; i < 8; ++i) CK(cudaStreamCreateWithFlags(&sc[i], cudaStreamNonBlocking));
  cudaEvent_t e0, e1, k0, k1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&k0));
  CK(cudaEventCreate(&k1));
  const int own = 0;
  auto run = [&](int mode, cudaStream_t s) -> int {
    for (int p = 1; p < N; ++p) {
      cudaStream_t st = mode == 3 ? sc[(p - 1) % 8] : s;
      if (mode == 0) {
        CK(cudaMemcpyAsync(rep[p] + own * chunk * nb, rep[0] + own * chunk * nb, shard, cudaMemcpyDeviceToDevice, st));
      } else {
        for (int bk = 0; bk < nb; ++bk) {
          const int64_t off = (int64_t)bk * N * chunk + own * chunk;
          CK(cudaMemcpyAsync(rep[p] + off, rep[0] + off, chunk, cudaMemcpyDeviceToDevice, st));
        }
      }
    }
    if (mode == 3) {
      for (int i = 0; i < 8 && i < N - 1; ++i) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, sc[i]));
        CK(cudaStreamWaitEvent(s, ev, 0));
        CK(cudaEventDestroy(ev));
      }
    }
    return 0;
  };
  const char* names[] = {"one copy per peer", "cudaMemcpyAsync per chunk", "", "per chunk, one stream per peer"};
  printf("world %d, %d buckets, chunk %.2f MB, %.1f MB per peer\n", N, nb, chunk / 1e6, shard / 1e6);
  float kalone = 0.f;
  {
    for (int w = 0; w < 3; ++w) k_stream<<<148 * 4, 512, 0, sk>>>(a, b, c2, d, e, nv2);
    CK(cudaEventRecord(k0, sk));
    for (int it = 0; it < 10; ++it) k_stream<<<148 * 4, 512, 0, sk>>>(a, b, c2, d, e, nv2);
    CK(cudaEventRecord(k1, sk));
    CK(cudaEventSynchronize(k1));
    CK(cudaEventElapsedTime(&kalone, k0, k1));
    kalone /= 10;
    printf("stream kernel alone: %.3f ms (%.0f GB/s)\n", kalone, nv2 * 16.0 * 5 / (kalone * 1e-3) / 1e9);
  }
  for (int mode = 0; mode < 4; ++mode) {
    if (mode == 2) continue;
    cudaStream_t s = sc[7];
    for (int w = 0; w < 2; ++w)
      if (run(mode, s)) return 1;
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int it = 0; it < 5; ++it)
      if (run(mode, s)) return 1;
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    printf("%-34s alone: %.3f ms, %.0f GB/s out\n", names[mode], ms, shard * (N - 1) / (ms * 1e-3) / 1e9);
    // under the streaming kernel
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(k0, sk));
    CK(cudaEventRecord(e0, s));
    for (int it = 0; it < 5; ++it)
      if (run(mode, s)) return 1;
    CK(cudaEventRecord(e1, s));
    int kit = 0;
    while (cudaEventQuery(e1) == cudaErrorNotReady && kit < 200) {
      k_stream<<<148 * 4, 512, 0, sk>>>(a, b, c2, d, e, nv2);
      ++kit;
      CK(cudaStreamSynchronize(sk));
    }
    CK(cudaEventRecord(k1, sk));
    CK(cudaDeviceSynchronize());
    float ms2 = 0.f, kms = 0.f;
    CK(cudaEventElapsedTime(&ms2, e0, e1));
    CK(cudaEventElapsedTime(&kms, k0, k1));
    printf("%-34s under the kernel: %.3f ms per push (%.0f GB/s), kernel %.3f ms per launch (%d launches, alone %.3f)\n",
           names[mode], ms2 / 5, shard * (N - 1) / (ms2 / 5 * 1e-3) / 1e9, kit ? kms / kit : 0.f, kit, kalone);
  }
  return 0;
}
