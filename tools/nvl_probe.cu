// NVLink-read vs HBM-stream interference probe (2 GPUs, one process, no NCCL).
// Each GPU streams a phase-1-like pattern over n elements (reads h:2 B,
// acc/w/m/v: 16 B, writes m/v/u: 12 B) and optionally reads a binary16 array
// of n elements from the peer GPU at the same index. Both GPUs run at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvl_probe tools/nvl_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Bufs { const uint2* h; const float4 *acc, *w, *m, *v; float4 *mo, *vo, *uo; const uint2* peer; };

template <int kMode>  // 0 local only, 1 local + peer, 2 peer only (+h), 3 local + peer via smem prefetch-free ld.cg
__global__ void __launch_bounds__(512, 2) k_probe(Bufs b, int64_t nv) {
  for (int64_t q = blockIdx.x * 512 + threadIdx.x; q < nv; q += (int64_t)gridDim.x * 512) {
    uint2 hv = b.h[q];
    uint2 pv = make_uint2(0, 0);
    if (kMode >= 1) pv = __ldcs(b.peer + q);
    if (kMode == 2) { b.uo[q] = make_float4(__uint_as_float(hv.x ^ pv.x), __uint_as_float(hv.y ^ pv.y), 0.f, 0.f); continue; }
    float4 a = __ldcs(b.acc + q), w = __ldcs(b.w + q), m = __ldcs(b.m + q), v = __ldcs(b.v + q);
    float s = __uint_as_float(hv.x ^ pv.x) + __uint_as_float(hv.y ^ pv.y);
    __stcs(b.mo + q, make_float4(m.x + s, m.y, m.z, m.w + a.x));
    __stcs(b.vo + q, make_float4(v.x + s, v.y, v.z, v.w + a.y));
    __stcs(b.uo + q, make_float4(w.x + s, w.y, w.z, w.w + a.z));
  }
}

int main(int argc, char** argv) {
  const int64_t n = 96ll << 20;  // elements per GPU
  const int64_t nv = n / 4;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("needs 2 GPUs\n"); return 0; }
  Bufs B[2];
  cudaStream_t s[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    void* p;
    CK(cudaMalloc(&p, n * 2)); B[d].h = (const uint2*)p; cudaMemset(p, 0, n * 2);
    float4* f[7];
    for (int i = 0; i < 7; ++i) { CK(cudaMalloc(&p, n * 4)); cudaMemset(p, 0, n * 4); f[i] = (float4*)p; }
    B[d].acc = f[0]; B[d].w = f[1]; B[d].m = f[2]; B[d].v = f[3]; B[d].mo = f[4]; B[d].vo = f[5]; B[d].uo = f[6];
    CK(cudaStreamCreate(&s[d]));
    cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]);
  }
  B[0].peer = B[1].h; B[1].peer = B[0].h;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](int mode, int grid, const char* name, double bytes_local, double bytes_peer) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
      for (int d = 0; d < 2; ++d) {
        cudaSetDevice(d);
        cudaEventRecord(e0[d], s[d]);
        if (mode == 0) k_probe<0><<<grid, 512, 0, s[d]>>>(B[d], nv);
        if (mode == 1) k_probe<1><<<grid, 512, 0, s[d]>>>(B[d], nv);
        if (mode == 2) k_probe<2><<<grid, 512, 0, s[d]>>>(B[d], nv);
        cudaEventRecord(e1[d], s[d]);
      }
      float mx = 0;
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaEventSynchronize(e1[d]); float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); mx = ms > mx ? ms : mx; }
      best = mx < best ? mx : best;
    }
    printf("%-28s grid %6d  %.3f ms  local %.0f GB/s  peer %.0f GB/s\n", name, grid, best,
           bytes_local / best / 1e6, bytes_peer / best / 1e6);
  };
  for (int g : {2 * sms, 4 * sms, 16 * sms}) {
    run(0, g, "local p1-like", n * 30.0, 0);
    run(1, g, "local p1-like + peer read", n * 30.0, n * 2.0);
    run(2, g, "peer read only (+h, u)", n * 6.0, n * 2.0);
  }
  return 0;
}
