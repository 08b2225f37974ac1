// Diagnostic (not part of the library): the NVLink ceiling for the put path's
// access pattern, without the ring protocol.  GPU0 -> GPU1 (and both ways at
// once) with (1) the copy engine (cudaMemcpyPeerAsync), (2) a plain SM copy
// kernel -- local loads, peer stores -- with 16-B and 32-B vectors over a grid
// sweep, (3) SM peer stores of register data (no loads), (4) SM pull (peer loads,
// local stores), (5)-(7) both directions at once (push, pull, copy engines).  Build + run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/p2p_ceiling.cu -o /tmp/p2p_ceiling && /tmp/p2p_ceiling
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

template <int V, int U, bool LOAD>
__global__ void __launch_bounds__(512) copy_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n16) {
  // n16 = number of 16-B words; V = 16-B words per access (1 or 2)
  const size_t nacc = n16 / V;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nacc; base += stride * U) {
    uint32_t r[U][4 * V];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const size_t i = base + (size_t)u * blockDim.x;
      if (i < nacc) {
        if constexpr (LOAD) {
          if constexpr (V == 2) {
            asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]),
                           "=r"(r[u][4 % (4 * V)]), "=r"(r[u][5 % (4 * V)]), "=r"(r[u][6 % (4 * V)]), "=r"(r[u][7 % (4 * V)])
                         : "l"(s + 2 * i));
          } else {
            uint4 x = s[i];
            r[u][0] = x.x; r[u][1] = x.y; r[u][2] = x.z; r[u][3] = x.w;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4 * V; k++) r[u][k] = (uint32_t)(i * 8 + k);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const size_t i = base + (size_t)u * blockDim.x;
      if (i < nacc) {
        if constexpr (V == 2) {
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                       :: "l"(d + 2 * i), "r"(r[u][0]), "r"(r[u][1]), "r"(r[u][2]), "r"(r[u][3]),
                          "r"(r[u][4 % (4 * V)]), "r"(r[u][5 % (4 * V)]), "r"(r[u][6 % (4 * V)]), "r"(r[u][7 % (4 * V)])
                       : "memory");
        } else {
          d[i] = make_uint4(r[u][0], r[u][1], r[u][2], r[u][3]);
        }
      }
    }
  }
}

typedef void (*kfn)(const uint4*, uint4*, size_t);

static float time_kernel(int dev, kfn f, int grid, int threads, const void* s, void* d, size_t bytes, int reps) {
  cudaSetDevice(dev);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f<<<grid, threads>>>((const uint4*)s, (uint4*)d, bytes / 16);   // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a);
    f<<<grid, threads>>>((const uint4*)s, (uint4*)d, bytes / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a); cudaEventDestroy(b);
  return best;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  const size_t bytes = 256ull << 20;
  void *s0, *d0, *s1, *d1;
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&s0, bytes)); CK(cudaMalloc(&d0, bytes)); CK(cudaMemset(s0, 1, bytes));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&s1, bytes)); CK(cudaMalloc(&d1, bytes)); CK(cudaMemset(s1, 2, bytes));
  const double gb = bytes / 1e9;

  // (1) copy engine
  {
    CK(cudaSetDevice(0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 6; r++) {
      cudaEventRecord(a);
      cudaMemcpyPeerAsync(d1, 1, s0, 0, bytes);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
    }
    printf("CE  0->1 peer copy            %7.1f GB/s\n", gb / (best / 1e3));
  }
  struct K { const char* name; kfn f; };
  K ks[] = {{"SM push v4  U4 (ld local, st peer)", copy_k<1, 4, true>},
            {"SM push v4  U8", copy_k<1, 8, true>},
            {"SM push v8  U4", copy_k<2, 4, true>},
            {"SM push v8  U8", copy_k<2, 8, true>},
            {"SM store-only v4 U8 (no loads)", copy_k<1, 8, false>},
            {"SM store-only v8 U4 (no loads)", copy_k<2, 4, false>}};
  const int grids[] = {33, 66, 132, 148, 296, 592};
  for (auto& k : ks) {
    for (int g : grids) {
      for (int t : {256, 512}) {
        float ms = time_kernel(0, k.f, g, t, s0, d1, bytes, 5);
        printf("%-36s grid %4d x %3d  %7.1f GB/s\n", k.name, g, t, gb / (ms / 1e3));
      }
    }
  }
  // (4) pull: kernel on GPU1 loads GPU0's memory, stores locally
  for (int g : {66, 148, 296}) {
    float ms = time_kernel(1, copy_k<1, 8, true>, g, 512, s0, d1, bytes, 5);
    printf("SM pull v4 U8 (ld peer, st local)     grid %4d x 512  %7.1f GB/s\n", g, gb / (ms / 1e3));
  }
  // (5) both directions at once: push 0->1 and 1->0 concurrently
  for (int g : {33, 66, 148}) {
    cudaStream_t st[2];
    cudaEvent_t a[2], b[2];
    for (int dv = 0; dv < 2; dv++) {
      cudaSetDevice(dv); cudaStreamCreate(&st[dv]); cudaEventCreate(&a[dv]); cudaEventCreate(&b[dv]);
    }
    float best[2] = {1e30f, 1e30f};
    for (int r = 0; r < 5; r++) {
      for (int dv = 0; dv < 2; dv++) { cudaSetDevice(dv); cudaDeviceSynchronize(); }
      for (int dv = 0; dv < 2; dv++) {
        cudaSetDevice(dv);
        cudaEventRecord(a[dv], st[dv]);
        copy_k<1, 8, true><<<g, 512, 0, st[dv]>>>((const uint4*)(dv ? s1 : s0), (uint4*)(dv ? d0 : d1), bytes / 16);
        cudaEventRecord(b[dv], st[dv]);
      }
      for (int dv = 0; dv < 2; dv++) {
        cudaSetDevice(dv); cudaEventSynchronize(b[dv]);
        float ms; cudaEventElapsedTime(&ms, a[dv], b[dv]); if (r && ms < best[dv]) best[dv] = ms;
      }
    }
    printf("SM push v4 U8 both directions         grid %4d x 512  %7.1f + %7.1f GB/s\n", g,
           gb / (best[0] / 1e3), gb / (best[1] / 1e3));
  }
  // (6) both directions at once, pulled: GPU1 loads GPU0's memory and GPU0 loads
  // GPU1's, each storing locally (the pull placement in the pairs topology)
  for (int g : {148, 296, 444}) {
    cudaStream_t st[2];
    cudaEvent_t a[2], b[2];
    for (int dv = 0; dv < 2; dv++) {
      cudaSetDevice(dv); cudaStreamCreate(&st[dv]); cudaEventCreate(&a[dv]); cudaEventCreate(&b[dv]);
    }
    float best[2] = {1e30f, 1e30f};
    for (int r = 0; r < 5; r++) {
      for (int dv = 0; dv < 2; dv++) { cudaSetDevice(dv); cudaDeviceSynchronize(); }
      for (int dv = 0; dv < 2; dv++) {
        cudaSetDevice(dv);
        cudaEventRecord(a[dv], st[dv]);
        copy_k<1, 8, true><<<g, 512, 0, st[dv]>>>((const uint4*)(dv ? s0 : s1), (uint4*)(dv ? d1 : d0), bytes / 16);
        cudaEventRecord(b[dv], st[dv]);
      }
      for (int dv = 0; dv < 2; dv++) {
        cudaSetDevice(dv); cudaEventSynchronize(b[dv]);
        float ms; cudaEventElapsedTime(&ms, a[dv], b[dv]); if (r && ms < best[dv]) best[dv] = ms;
      }
    }
    printf("SM pull v4 U8 both directions         grid %4d x 512  %7.1f + %7.1f GB/s\n", g,
           gb / (best[0] / 1e3), gb / (best[1] / 1e3));
  }
  // (7) both directions by the copy engines
  {
    cudaStream_t st[2];
    cudaEvent_t a[2], b[2];
    for (int dv = 0; dv < 2; dv++) {
      cudaSetDevice(dv); cudaStreamCreate(&st[dv]); cudaEventCreate(&a[dv]); cudaEventCreate(&b[dv]);
    }
    float best[2] = {1e30f, 1e30f};
    for (int r = 0; r < 6; r++) {
      for (int dv = 0; dv < 2; dv++) { cudaSetDevice(dv); cudaDeviceSynchronize(); }
      for (int dv = 0; dv < 2; dv++) {
        cudaSetDevice(dv);
        cudaEventRecord(a[dv], st[dv]);
        cudaMemcpyPeerAsync(dv ? d0 : d1, dv ? 0 : 1, dv ? s1 : s0, dv, bytes, st[dv]);
        cudaEventRecord(b[dv], st[dv]);
      }
      for (int dv = 0; dv < 2; dv++) {
        cudaSetDevice(dv); cudaEventSynchronize(b[dv]);
        float ms; cudaEventElapsedTime(&ms, a[dv], b[dv]); if (r && ms < best[dv]) best[dv] = ms;
      }
    }
    printf("CE both directions                              %7.1f + %7.1f GB/s\n", gb / (best[0] / 1e3), gb / (best[1] / 1e3));
  }
  // (8) both directions driven from ONE GPU: GPU0 pushes 0 -> 1 and pulls 1 -> 0
  //     at the same time (two kernels, two streams, g CTAs each)
  for (int g : {74, 148}) {
    cudaStream_t st2[2];
    cudaEvent_t a2[2], b2[2];
    CK(cudaSetDevice(0));
    for (int k = 0; k < 2; k++) { cudaStreamCreate(&st2[k]); cudaEventCreate(&a2[k]); cudaEventCreate(&b2[k]); }
    float best[2] = {1e30f, 1e30f};
    for (int r = 0; r < 5; r++) {
      cudaDeviceSynchronize();
      cudaEventRecord(a2[0], st2[0]);
      copy_k<1, 8, true><<<g, 512, 0, st2[0]>>>((const uint4*)s0, (uint4*)d1, bytes / 16);   // push 0 -> 1
      cudaEventRecord(b2[0], st2[0]);
      cudaEventRecord(a2[1], st2[1]);
      copy_k<1, 8, true><<<g, 512, 0, st2[1]>>>((const uint4*)s1, (uint4*)d0, bytes / 16);   // pull 1 -> 0
      cudaEventRecord(b2[1], st2[1]);
      for (int k = 0; k < 2; k++) {
        cudaEventSynchronize(b2[k]);
        float ms; cudaEventElapsedTime(&ms, a2[k], b2[k]); if (r && ms < best[k]) best[k] = ms;
      }
    }
    printf("GPU0 push 0->1 + pull 1->0 at once   grid %4d x 512  %7.1f + %7.1f GB/s\n", g,
           gb / (best[0] / 1e3), gb / (best[1] / 1e3));
  }
  printf("done\n");
  return 0;
}
