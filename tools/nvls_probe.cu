// NVSwitch multicast (NVLS) probe for the parameter all-gather: every GPU of
// the box writes its 1/N shard of a P-element fp32 replica into EVERY GPU's
// replica at once, (a) as unicast SM stores to each peer (the library's push
// pattern), (b) as one multimem.st per element to a multicast object bound to
// every GPU's replica (the switch replicates). Single process, one host
// thread per GPU. Prints support, the time of each form and a check.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                               \
    }                                                                         \
  } while (0)
#define CU(x)                                                                 \
  do {                                                                        \
    CUresult r_ = (x);                                                        \
    if (r_ != CUDA_SUCCESS) {                                                 \
      const char* s_ = nullptr;                                               \
      cuGetErrorString(r_, &s_);                                              \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?");       \
      return 1;                                                               \
    }                                                                         \
  } while (0)

struct Dsts {
  float4* p[8];
  int n;
};

__global__ void k_unicast(const float4* __restrict__ src, Dsts d, int64_t nv, int rot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = __ldcs(src + i);
    for (int k = 0; k < d.n; ++k) __stcs(d.p[(k + rot) % d.n] + i, x);
  }
}

__global__ void k_multicast(const float4* __restrict__ src, float4* mc, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = __ldcs(src + i);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(x.x), "f"(x.y),
                 "f"(x.z), "f"(x.w)
                 : "memory");
  }
}

__global__ void k_fill(float4* p, int64_t nv, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_float4(v, v + 1, v + 2, v + 3);
}

int main() {
  CU(cuInit(0));
  int N = 0;
  CK(cudaGetDeviceCount(&N));
  if (N < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  for (int d = 0; d < N; ++d) {
    int mcs = 0;
    CU(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
    printf("device %d multicast supported: %d\n", d, mcs);
    if (!mcs) return 0;
  }
  const int64_t P = 336226108;
  const int64_t shard_nv = (P / N + 3) / 4;  // float4 per shard
  // multicast object over N devices
  CUmulticastObjectProp mp{};
  mp.numDevices = N;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = 2ull << 20;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t bytes = ((size_t)shard_nv * N * 16 + gran - 1) / gran * gran;
  mp.size = bytes;
  printf("world %d, replica %.1f MB, multicast granularity %zu\n", N, bytes / 1e6, gran);
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < N; ++d) CU(cuMulticastAddDevice(mc, d));
  std::vector<CUmemGenericAllocationHandle> phys(N);
  std::vector<CUdeviceptr> uva(N), mva(N);
  std::vector<float4*> src(N);
  std::vector<cudaStream_t> st(N);
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < N; ++p)
      if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CU(cuMemCreate(&phys[d], bytes, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, phys[d], 0, bytes, 0));
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    // unicast view of this device's replica
    CU(cuMemAddressReserve(&uva[d], bytes, gran, 0, 0));
    CU(cuMemMap(uva[d], bytes, 0, phys[d], 0));
    CU(cuMemSetAccess(uva[d], bytes, &acc, 1));
    // multicast view (stores reach every device's replica)
    CU(cuMemAddressReserve(&mva[d], bytes, gran, 0, 0));
    CU(cuMemMap(mva[d], bytes, 0, mc, 0));
    CU(cuMemSetAccess(mva[d], bytes, &acc, 1));
    CK(cudaMalloc(&src[d], shard_nv * 16));
    k_fill<<<1184, 512>>>(src[d], shard_nv, 100.f * d);
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  // unicast views of every replica must be accessible from every device
  for (int d = 0; d < N; ++d) {
    CUmemAccessDesc acc[8]{};
    for (int p = 0; p < N; ++p) {
      acc[p].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc[p].location.id = p;
      acc[p].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CU(cuMemSetAccess(uva[d], bytes, acc, N));
  }
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  auto run = [&](int mode, int iters) -> double {
    std::vector<cudaEvent_t> e0(N), e1(N);
    std::vector<std::thread> th;
    std::vector<float> ms(N, 0.f);
    for (int d = 0; d < N; ++d) {
      th.emplace_back([&, d] {
        cudaSetDevice(d);
        cudaEventCreate(&e0[d]);
        cudaEventCreate(&e1[d]);
        Dsts ds{};
        ds.n = N;
        for (int p = 0; p < N; ++p) ds.p[p] = reinterpret_cast<float4*>(uva[p]) + d * shard_nv;
        cudaEventRecord(e0[d], st[d]);
        for (int it = 0; it < iters; ++it) {
          if (mode == 0)
            k_unicast<<<148 * 8, 256, 0, st[d]>>>(src[d], ds, shard_nv, d);
          else
            k_multicast<<<148 * 8, 256, 0, st[d]>>>(src[d], reinterpret_cast<float4*>(mva[d]) + d * shard_nv, shard_nv);
        }
        cudaEventRecord(e1[d], st[d]);
        cudaEventSynchronize(e1[d]);
        cudaEventElapsedTime(&ms[d], e0[d], e1[d]);
      });
    }
    for (auto& t : th) t.join();
    double mx = 0;
    for (int d = 0; d < N; ++d) mx = ms[d] > mx ? ms[d] : mx;
    return mx / iters;
  };
  for (int mode = 0; mode < 2; ++mode) {
    run(mode, 2);
    const double ms = run(mode, 10);
    const double in_bytes = (double)shard_nv * 16 * (N - 1);  // each GPU receives N-1 shards
    printf("%-10s all %d GPUs at once: %.3f ms per all-gather, %.0f GB/s in per GPU\n",
           mode ? "multicast" : "unicast", N, ms, in_bytes / (ms * 1e-3) / 1e9);
  }
  // check: every replica holds every shard
  int bad = 0;
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < N; ++q) {
      float4 v;
      CK(cudaMemcpy(&v, reinterpret_cast<float4*>(uva[d]) + q * shard_nv + 12345, 16, cudaMemcpyDeviceToHost));
      if (v.x != 100.f * q || v.w != 100.f * q + 3) ++bad;
    }
  }
  printf("replica check: %s\n", bad ? "MISMATCH" : "ok");
  return 0;
}
