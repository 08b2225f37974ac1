// Does a small kernel launched after two spinning kernels (other streams) get scheduled?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template <int REGS, int SMEM>
__global__ void spin(volatile int* flag, uint64_t* out, int which, uint64_t budget) {
  __shared__ float pad[SMEM / 4 + 1];
  pad[threadIdx.x % (SMEM / 4 + 1)] = 1.f;
  __syncthreads();
  // keep REGS live values to set the register footprint
  float acc[REGS];
#pragma unroll
  for (int i = 0; i < REGS; ++i) acc[i] = threadIdx.x * (i + 1);
  const uint64_t t0 = gt();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[which * 4] = t0;
  while (*flag == 0 && gt() - t0 < budget) {
#pragma unroll
    for (int i = 0; i < REGS; ++i) acc[i] = acc[i] * 1.0001f + 0.5f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < REGS; ++i) s += acc[i];
  if (s == 12345.f + pad[threadIdx.x % (SMEM / 4 + 1)]) out[3] = 1;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[which * 4 + 1] = gt();
}

template <int SMEM>
__global__ void setter(int* flag, uint64_t* out) {
  __shared__ float pad[SMEM / 4 + 1];
  pad[threadIdx.x % (SMEM / 4 + 1)] = 1.f;
  __syncwarp();
  out[8] = gt() + (pad[0] == 3.f);
  *flag = 1;
  __threadfence_system();
}

template <int REGS, int SS = 0, int SSET = 0>
void run(int gA, int tA, int gB, int tB, int smem, uint64_t budgetA = 1000000000ull, int carveA = -2, int carveS = -2) {
  if (carveA != -2) cudaFuncSetAttribute(spin<REGS, SS>, cudaFuncAttributePreferredSharedMemoryCarveout, carveA);
  if (carveS != -2) cudaFuncSetAttribute(setter<SSET>, cudaFuncAttributePreferredSharedMemoryCarveout, carveS);
  printf("carveA=%d carveS=%d ", carveA, carveS);
  int* flag; uint64_t* out;
  cudaMalloc(&flag, 4); cudaMalloc(&out, 128);
  cudaMemset(flag, 0, 4); cudaMemset(out, 0, 128);
  cudaFuncSetAttribute(spin<REGS, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, setter<SSET>); cudaFuncGetAttributes(&fa, spin<REGS, SS>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spin<REGS, SS>, tA, smem);
  cudaStream_t s1, s2, s3;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
  cudaDeviceSynchronize();
  spin<REGS, SS><<<gA, tA, smem, s1>>>(flag, out, 0, budgetA);
  if (gB) spin<REGS, SS><<<gB, tB, smem, s2>>>(flag, out, 1, 1000000000ull);
  setter<SSET><<<1, 32, 0, s3>>>(flag, out);
  cudaFuncGetAttributes(&fa, setter<SSET>);
  cudaDeviceSynchronize();
  uint64_t h[16];
  cudaMemcpy(h, out, 128, cudaMemcpyDeviceToHost);
  printf("SS=%d SSET=%d budgetA=%llu ", SS, SSET, (unsigned long long)budgetA);
  printf("regs=%d(%d) occ/SM=%d A=%dx%d B=%dx%d smem=%d: setter at %+.1f us after A start; A ran %.1f us, B start %+.1f us\n",
         fa.numRegs, REGS, occ, gA, tA, gB, tB, smem, (double)((int64_t)(h[8] - h[0])) / 1e3,
         (double)(h[1] - h[0]) / 1e3, gB ? (double)((int64_t)(h[4] - h[0])) / 1e3 : 0.0);
  cudaFree(flag); cudaFree(out);
  cudaStreamDestroy(s1); cudaStreamDestroy(s2); cudaStreamDestroy(s3);
  if (cudaError_t e = cudaGetLastError()) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  run<80, 11392, 4112>(148, 224, 0, 0, 0, 200000);
  run<80, 11392, 0>(148, 224, 0, 0, 0, 200000);
  run<80, 11392, 4112>(148, 224, 0, 0, 0, 200000, 100, 100);
  run<80, 11392, 4112>(148, 224, 0, 0, 0, 200000, 50, 50);
  run<80, 11392, 4112>(148, 224, 0, 0, 0, 200000, 100, -1);
  run<80, 11392, 4112>(148, 224, 148, 224, 0, 200000, 100, 100);
  run<80, 11392, 4112>(148, 512, 0, 0, 0, 200000, 100, 100);
  return 0;
}
