// Raw NVLink bandwidth on this box: GPU 0 writes (SM stores, float4) or reads
// 1 GiB to/from 1..ngpu-1 peers at once, and the copy-engine equivalent.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_bw tools/nvl_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Dsts { float4* p[8]; int n; };

// element i goes to every destination (the all-gather push pattern)
__global__ void k_write_all(const float4* __restrict__ src, Dsts d, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = __ldcs(src + i);
    for (int j = 0; j < d.n; ++j) __stcs(d.p[j] + i, x);
  }
}
// scalar 4-byte stores of the same pattern
__global__ void k_write_all_scalar(const float* __restrict__ src, Dsts d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = __ldcs(src + i);
    for (int j = 0; j < d.n; ++j) __stcs(reinterpret_cast<float*>(d.p[j]) + i, x);
  }
}
__global__ void k_read(const float4* __restrict__ src, float4* __restrict__ dst, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x)
    __stcs(dst + i, __ldcs(src + i));
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("needs 2 GPUs\n"); return 0; }
  const int64_t bytes = 1ll << 30, nv = bytes / 16;
  std::vector<float4*> buf(ndev);
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    for (int pe = 0; pe < ndev; ++pe) if (pe != d) CK(cudaDeviceEnablePeerAccess(pe, 0));
    CK(cudaMalloc(&buf[d], bytes));
    CK(cudaMemset(buf[d], 0, bytes));
  }
  CK(cudaSetDevice(0));
  float4* src;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 0, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto&& f) {
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
  };
  for (int np = 1; np < ndev; ++np) {
    Dsts d{};
    d.n = np;
    for (int j = 0; j < np; ++j) d.p[j] = buf[j + 1];
    for (int grid : {sms, 2 * sms, 4 * sms, 8 * sms}) {
      float ms = timeit([&] { k_write_all<<<grid, 512>>>(src, d, nv); });
      printf("SM float4 stores to %d peer(s), grid %4d: %.3f ms  %.0f GB/s out\n", np, grid, ms, np * bytes / ms / 1e6);
    }
    float ms = timeit([&] { k_write_all_scalar<<<4 * sms, 512>>>(reinterpret_cast<float*>(src), d, bytes / 4); });
    printf("SM scalar stores to %d peer(s):        %.3f ms  %.0f GB/s out\n", np, ms, np * bytes / ms / 1e6);
    ms = timeit([&] { for (int j = 0; j < np; ++j) cudaMemcpyPeerAsync(buf[j + 1], j + 1, src, 0, bytes); });
    printf("copy engine to %d peer(s):             %.3f ms  %.0f GB/s out\n", np, ms, np * bytes / ms / 1e6);
  }
  for (int grid : {2 * sms, 8 * sms}) {
    float ms = timeit([&] { k_read<<<grid, 512>>>(buf[1], src, nv); });
    printf("SM float4 reads from 1 peer, grid %4d:  %.3f ms  %.0f GB/s in\n", grid, ms, bytes / ms / 1e6);
  }
  return 0;
}
