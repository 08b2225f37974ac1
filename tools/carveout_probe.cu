// carveout_probe.cu — which L1/shared split does B200 give a kernel for a
// given PreferredSharedMemoryCarveout percentage, and which kernels then start
// next to each other?  (Evidence for the ring kernels' carveout choice,
// ring_internal.h preload_kernel; results in profiles/r02_carveout_probe.txt.)
//
// Part 1: a probe kernel with 3 KB of dynamic shared memory (4 KB per CTA with
// the 1 KB the system reserves) counts how many of its CTAs are resident at
// once per SM: the split is ~4 KB x that count.
// Part 2: kernel A (one CTA per SM, S_A bytes static shared memory) spins;
// kernel B (S_B bytes) is launched after it on another stream and must run
// while A spins; both with the same carveout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }

__global__ void occupancy_probe(unsigned* cur, unsigned* maxv, uint64_t dwell_ns) {
  extern __shared__ uint8_t dyn[];
  dyn[threadIdx.x] = 1;
  if (threadIdx.x == 0) {
    const uint32_t sm = smid();
    const unsigned c = atomicAdd(&cur[sm], 1u) + 1;
    atomicMax(&maxv[sm], c);
    const uint64_t t0 = gt();
    while (gt() - t0 < dwell_ns) {}
    atomicSub(&cur[sm], 1u);
  }
}

template <int S>
__global__ void spinner(volatile int* flag, uint64_t* out, uint64_t budget) {
  __shared__ uint8_t pad[S];
  pad[threadIdx.x % S] = 1;
  __syncthreads();
  const uint64_t t0 = gt();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t0;
  while (*flag == 0 && gt() - t0 < budget) {}
  if (pad[0] == 7) out[3] = 1;
}

template <int S>
__global__ void setter(int* flag, uint64_t* out) {
  __shared__ uint8_t pad[S];
  pad[threadIdx.x % S] = 1;
  __syncwarp();
  out[1] = gt() + (pad[0] == 7);
  *flag = 1;
}

template <int SA, int SB>
void coresident(int pct, int nsm, int gridA = 0, int thrA = 224, int gridB = 1, int thrB = 32) {
  if (!gridA) gridA = nsm;
  int* flag; uint64_t* out;
  cudaMalloc(&flag, 4); cudaMalloc(&out, 64);
  cudaMemset(flag, 0, 4); cudaMemset(out, 0, 64);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, spinner<SA>);
  cudaFuncGetAttributes(&fa, setter<SB>);
  if (pct >= 0) {
    cudaFuncSetAttribute(spinner<SA>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(setter<SB>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  }
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaDeviceSynchronize();
  spinner<SA><<<gridA, thrA, 0, s1>>>(flag, out, 300000);   // 300 us budget
  setter<SB><<<gridB, thrB, 0, s2>>>(flag, out);
  cudaDeviceSynchronize();
  uint64_t h[4];
  cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
  const double dt = (double)(int64_t)(h[1] - h[0]) / 1e3;
  printf("  carveout %3d%%: A=%dx%d (%5d B static) then B=%dx%d (%5d B static): B starts %+8.1f us after A -> %s\n",
         pct, gridA, thrA, SA, gridB, thrB, SB, dt, dt < 100 ? "co-resident" : "BLOCKED until A ends");
  cudaStreamDestroy(s1); cudaStreamDestroy(s2);
  cudaFree(flag); cudaFree(out);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned *cur, *maxv;
  cudaMalloc(&cur, 4 * 256); cudaMalloc(&maxv, 4 * 256);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, occupancy_probe);
  printf("Part 1: resident 4-KB CTAs per SM (3 KB dynamic + 1 KB reserved) by carveout\n");
  const int pcts[] = {-1, 0, 4, 7, 8, 13, 14, 15, 20, 28, 29, 30, 43, 44, 50, 57, 58, 72, 86, 100};
  for (int p : pcts) {
    if (p >= 0) cudaFuncSetAttribute(occupancy_probe, cudaFuncAttributePreferredSharedMemoryCarveout, p);
    cudaMemset(cur, 0, 4 * 256); cudaMemset(maxv, 0, 4 * 256);
    occupancy_probe<<<nsm * 40, 32, 3072>>>(cur, maxv, 200000);
    cudaDeviceSynchronize();
    unsigned h[256];
    cudaMemcpy(h, maxv, 4 * 256, cudaMemcpyDeviceToHost);
    unsigned lo = 1000, hi = 0;
    for (int i = 0; i < nsm; ++i) { lo = h[i] < lo ? h[i] : lo; hi = h[i] > hi ? h[i] : hi; }
    printf("  carveout %3d%%: %u-%u CTAs/SM -> split ~%u KB shared\n", p, lo, hi, 4 * hi);
  }
  printf("Part 2: co-residency (A spins on every SM, B launched after it)\n");
  const int tests[] = {-1, 0, 7, 8, 14, 15, 29, 100};
  for (int p : tests) {
    coresident<11392, 4112>(p, nsm);
    coresident<5120, 4112>(p, nsm);
    coresident<4112, 11392>(p, nsm, nsm, 224, 140, 224);   // copy-out get first, then a put grid
  }
  if (cudaError_t e = cudaGetLastError()) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
