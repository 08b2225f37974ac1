// Diagnostic (not part of the library): the NVLink ingress ceiling of one GPU
// fed by several at once -- GPUs 1..k each push 256 MiB into GPU 0 with a plain
// SM copy kernel (local loads, peer stores), concurrently; and the same with
// the copy engines.  Build + run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/p2p_fanin.cu -o /tmp/p2p_fanin && /tmp/p2p_fanin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) push_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n16) {
  constexpr int U = 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < n16; base += stride * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; u++) { size_t i = base + (size_t)u * blockDim.x; if (i < n16) r[u] = s[i]; }
#pragma unroll
    for (int u = 0; u < U; u++) { size_t i = base + (size_t)u * blockDim.x; if (i < n16) d[i] = r[u]; }
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 3) { printf("needs >= 3 GPUs\n"); return 0; }
  const size_t bytes = 256ull << 20;
  void* dst[8] = {};
  void* src[8] = {};
  cudaSetDevice(0);
  for (int g = 1; g < n && g < 8; g++) { cudaDeviceEnablePeerAccess(g, 0); cudaMalloc(&dst[g], bytes); }
  for (int g = 1; g < n && g < 8; g++) {
    cudaSetDevice(g); cudaDeviceEnablePeerAccess(0, 0); cudaMalloc(&src[g], bytes); cudaMemset(src[g], g, bytes);
  }
  for (int ce = 0; ce < 2; ce++)
    for (int k = 1; k < n && k < 8; k++) {
      cudaStream_t st[8]; cudaEvent_t a[8], b[8];
      for (int g = 1; g <= k; g++) { cudaSetDevice(g); cudaStreamCreate(&st[g]); cudaEventCreate(&a[g]); cudaEventCreate(&b[g]); }
      float worst_best = 0;
      float best = 1e30f;
      for (int r = 0; r < 5; r++) {
        for (int g = 1; g <= k; g++) { cudaSetDevice(g); cudaDeviceSynchronize(); }
        for (int g = 1; g <= k; g++) {
          cudaSetDevice(g);
          cudaEventRecord(a[g], st[g]);
          if (ce) cudaMemcpyPeerAsync(dst[g], 0, src[g], g, bytes, st[g]);
          else push_k<<<148, 512, 0, st[g]>>>((const uint4*)src[g], (uint4*)dst[g], bytes / 16);
          cudaEventRecord(b[g], st[g]);
        }
        float worst = 0;
        for (int g = 1; g <= k; g++) {
          cudaSetDevice(g); cudaEventSynchronize(b[g]);
          float ms; cudaEventElapsedTime(&ms, a[g], b[g]); if (ms > worst) worst = ms;
        }
        if (r && worst < best) best = worst;
      }
      worst_best = best;
      printf("%s %d -> 1: %7.1f GB/s into GPU 0 (%6.1f per source)\n", ce ? "CE      " : "SM push ", k,
             k * bytes / 1e9 / (worst_best / 1e3), bytes / 1e9 / (worst_best / 1e3));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
