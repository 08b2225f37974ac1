// Throwaway hardware probe (not product code): peer-store bandwidth from SMs over
// NVLink vs CTA count, copy-engine peer bandwidth, and system-scope fence cost.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void copy_v4(const int4* __restrict__ src, int4* dst, size_t n16, int unroll_dummy) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  size_t i = tid;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int4* p = src + i + j * stride;
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(p));
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      int4* p = dst + i + j * stride;
      asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w) : "memory");
    }
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// per-CTA contiguous chunk variant
__global__ void copy_chunk(const int4* __restrict__ src, int4* dst, size_t n16) {
  size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  size_t b = blockIdx.x * per, e = b + per < n16 ? b + per : n16;
  constexpr int U = 8;
  size_t i = b + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int4* p = src + i + j * blockDim.x;
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(p));
    }
#pragma unroll
    for (int j = 0; j < U; ++j) dst[i + j * blockDim.x] = v[j];
  }
  for (; i < e; i += blockDim.x) dst[i] = src[i];
}

__global__ void fence_cost(int4* dst, int iters, unsigned long long* out) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int k = 0; k < iters; ++k) {
    dst[threadIdx.x + k * 32] = make_int4(k, k, k, k);
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

// ping-pong on flags: GPU a writes peer flag, GPU b waits and writes back
__global__ void pingpong(volatile unsigned long long* my_flag, unsigned long long* peer_flag, int iters, int initiator, unsigned long long* out) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int k = 1; k <= iters; ++k) {
    if (initiator) {
      asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((unsigned long long)k) : "memory");
      unsigned long long v; do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory"); } while (v < (unsigned long long)k);
    } else {
      unsigned long long v; do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory"); } while (v < (unsigned long long)k);
      asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((unsigned long long)k) : "memory");
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[0] = t1 - t0;
}

int main() {
  int ndev; CK(cudaGetDeviceCount(&ndev)); printf("ndev=%d\n", ndev);
  if (ndev < 2) return 0;
  int can; CK(cudaDeviceCanAccessPeer(&can, 0, 1)); printf("canAccessPeer(0,1)=%d\n", can);
  size_t bytes = 256ull << 20;
  void *s0, *d0, *d1; 
  CK(cudaSetDevice(1)); CK(cudaMalloc(&d1, bytes)); CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaSetDevice(0)); CK(cudaMalloc(&s0, bytes)); CK(cudaMalloc(&d0, bytes)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMemset(s0, 1, bytes));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;
  // copy engine
  for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); CK(cudaMemcpyPeerAsync(d1, 1, s0, 0, bytes)); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
  CK(cudaEventElapsedTime(&ms, a, b)); printf("memcpyPeer 256MiB: %.1f GB/s\n", bytes / ms / 1e6);
  size_t n16 = bytes / 16;
  int ctas[] = {4, 8, 16, 24, 32, 48, 64, 96, 132, 148, 296};
  for (int threads : {256, 512, 1024}) for (int c : ctas) {
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); copy_chunk<<<c, threads>>>((const int4*)s0, (int4*)d1, n16); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
    CK(cudaEventElapsedTime(&ms, a, b)); printf("peer chunk  ctas=%3d thr=%4d: %.1f GB/s\n", c, threads, bytes / ms / 1e6);
  }
  for (int c : ctas) {
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); copy_v4<<<c, 512>>>((const int4*)s0, (int4*)d1, n16, 0); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
    CK(cudaEventElapsedTime(&ms, a, b)); printf("peer grid-stride ctas=%3d: %.1f GB/s\n", c, bytes / ms / 1e6);
  }
  for (int c : {148, 296, 592}) {
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); copy_chunk<<<c, 512>>>((const int4*)s0, (int4*)d0, n16); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
    CK(cudaEventElapsedTime(&ms, a, b)); printf("local chunk ctas=%3d: %.1f GB/s (r+w %.1f)\n", c, bytes / ms / 1e6, 2 * bytes / ms / 1e6);
  }
  unsigned long long* out; CK(cudaMallocManaged(&out, 64));
  fence_cost<<<1, 32>>>((int4*)d1, 1000, out); CK(cudaDeviceSynchronize());
  fence_cost<<<1, 32>>>((int4*)d1, 1000, out); CK(cudaDeviceSynchronize());
  printf("peer store+fence.sys: %.1f ns/iter\n", out[0] / 1000.0);
  fence_cost<<<1, 32>>>((int4*)d0, 1000, out); CK(cudaDeviceSynchronize());
  printf("local store+fence.sys: %.1f ns/iter\n", out[0] / 1000.0);
  // ping-pong
  unsigned long long *f0, *f1, *o1; 
  CK(cudaMalloc(&f0, 128)); CK(cudaMemset(f0, 0, 128));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&f1, 128)); CK(cudaMemset(f1, 0, 128)); CK(cudaMallocManaged(&o1, 64));
  cudaStream_t st1; CK(cudaStreamCreate(&st1));
  pingpong<<<1, 1, 0, st1>>>(f1, f0, 10000, 0, o1);
  CK(cudaSetDevice(0));
  pingpong<<<1, 1>>>(f0, f1, 10000, 1, out);
  CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
  printf("flag ping-pong RTT: %.1f ns\n", out[0] / 10000.0);
  return 0;
}
