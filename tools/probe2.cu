// Throwaway hardware probe #2 (not product code): TMA bulk peer stores, 256-bit
// stores, fence / flag costs, bidirectional peer traffic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk: one elected thread per CTA streams chunks local->smem->peer, STAGES deep.
template <int STAGES>
__global__ void tma_copy(const char* __restrict__ src, char* dst, size_t bytes, int chunk) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  size_t per = (bytes + gridDim.x - 1) / gridDim.x; per = (per + 15) & ~size_t(15);
  size_t b = blockIdx.x * per, e = min(bytes, b + per);
  if (threadIdx.x != 0 || b >= e) return;
  for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[STAGES] = {};
  int nchunks = (int)((e - b + chunk - 1) / chunk);
  for (int i = 0; i < nchunks + STAGES; ++i) {
    // issue load for chunk i
    if (i < nchunks) {
      int s = i % STAGES;
      if (i >= STAGES) {
        // make sure store of chunk i-STAGES has finished reading smem
        asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(STAGES - 1) : "memory");
      }
      size_t off = b + (size_t)i * chunk; int n = (int)min((size_t)chunk, e - off);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(n) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(smem + s * chunk)), "l"(src + off), "r"(n), "r"(smem_u32(&bar[s])) : "memory");
    }
    int j = i - (STAGES - 1);
    if (j >= 0 && j < nchunks) {
      int s = j % STAGES;
      uint32_t ok = 0;
      while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(phase[s]) : "memory");
      phase[s] ^= 1;
      size_t off = b + (size_t)j * chunk; int n = (int)min((size_t)chunk, e - off);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + off), "r"(smem_u32(smem + s * chunk)), "r"(n) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

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

// 256-bit per thread: two v4 adjacent
__global__ void copy_chunk32(const int4* __restrict__ src, int4* dst, size_t n16) {
  size_t n32 = n16 / 2;
  size_t per = (n32 + gridDim.x - 1) / gridDim.x;
  size_t b = blockIdx.x * per, e = b + per < n32 ? b + per : n32;
  constexpr int U = 4;
  size_t i = b + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
    int4 v[U][2];
#pragma unroll
    for (int j = 0; j < U; ++j) { v[j][0] = src[2 * (i + j * blockDim.x)]; v[j][1] = src[2 * (i + j * blockDim.x) + 1]; }
#pragma unroll
    for (int j = 0; j < U; ++j) { dst[2 * (i + j * blockDim.x)] = v[j][0]; dst[2 * (i + j * blockDim.x) + 1] = v[j][1]; }
  }
}

// pull: read peer, write local
__global__ void pull_chunk(const int4* src_peer, int4* dst, size_t n16) {
  size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  size_t b = blockIdx.x * per, e = b + per < n16 ? b + per : n16;
  constexpr int U = 8;
  size_t i = b + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = src_peer[i + j * blockDim.x];
#pragma unroll
    for (int j = 0; j < U; ++j) dst[i + j * blockDim.x] = v[j];
  }
}

__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void lat_probe(uint64_t* peer, uint64_t* local, int iters, uint64_t* out) {
  uint64_t t0, t1, v = 0;
  // 0: fence.acq_rel.gpu after peer store
  t0 = gtime(); for (int k = 0; k < iters; ++k) { peer[k & 15] = k; asm volatile("fence.acq_rel.gpu;" ::: "memory"); } t1 = gtime(); out[0] = (t1 - t0) / iters;
  // 1: fence.acq_rel.sys after peer store
  t0 = gtime(); for (int k = 0; k < iters; ++k) { peer[k & 15] = k; asm volatile("fence.acq_rel.sys;" ::: "memory"); } t1 = gtime(); out[1] = (t1 - t0) / iters;
  // 2: st.release.sys to peer back to back
  t0 = gtime(); for (int k = 0; k < iters; ++k) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer + (k & 15)), "l"((uint64_t)k) : "memory"); t1 = gtime(); out[2] = (t1 - t0) / iters;
  // 3: ld.acquire.sys peer (round trip)
  t0 = gtime(); for (int k = 0; k < iters; ++k) { uint64_t x; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(peer + (k & 15)) : "memory"); v += x; } t1 = gtime(); out[3] = (t1 - t0) / iters;
  // 4: atom.cas.sys peer
  t0 = gtime(); for (int k = 0; k < iters; ++k) { uint64_t x; asm volatile("atom.acq_rel.sys.global.cas.b64 %0, [%1], %2, %3;" : "=l"(x) : "l"(peer + 32), "l"((uint64_t)0), "l"((uint64_t)0) : "memory"); v += x; } t1 = gtime(); out[4] = (t1 - t0) / iters;
  // 5: ld.acquire.sys local
  t0 = gtime(); for (int k = 0; k < iters; ++k) { uint64_t x; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(local + (k & 15)) : "memory"); v += x; } t1 = gtime(); out[5] = (t1 - t0) / iters;
  // 6: fence.acq_rel.sys with no prior stores
  t0 = gtime(); for (int k = 0; k < iters; ++k) { asm volatile("fence.acq_rel.sys;" ::: "memory"); } t1 = gtime(); out[6] = (t1 - t0) / iters;
  // 7: local store + fence.acq_rel.gpu
  t0 = gtime(); for (int k = 0; k < iters; ++k) { local[k & 15] = k; asm volatile("fence.acq_rel.gpu;" ::: "memory"); } t1 = gtime(); out[7] = (t1 - t0) / iters;
  // 8: st.release.gpu local
  t0 = gtime(); for (int k = 0; k < iters; ++k) asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(local + (k & 15)), "l"((uint64_t)k) : "memory"); t1 = gtime(); out[8] = (t1 - t0) / iters;
  // 9: ld.relaxed.sys peer (volatile) round trip
  t0 = gtime(); for (int k = 0; k < iters; ++k) { uint64_t x; asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(peer + (k & 15)) : "memory"); v += x; } t1 = gtime(); out[9] = (t1 - t0) / iters;
  // 10: peer store + fence.sc.sys
  t0 = gtime(); for (int k = 0; k < iters; ++k) { peer[k & 15] = k; asm volatile("fence.sc.sys;" ::: "memory"); } t1 = gtime(); out[10] = (t1 - t0) / iters;
  out[15] = v;
}

// one-way latency with a relaxed store publisher + consumer spinning (relaxed vs release)
__global__ void pingpong(uint64_t* my_flag, uint64_t* peer_flag, int iters, int initiator, int rel, uint64_t* out) {
  uint64_t t0 = gtime();
  for (int k = 1; k <= iters; ++k) {
    if (initiator) {
      if (rel) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((uint64_t)k) : "memory");
      else asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((uint64_t)k) : "memory");
      uint64_t v; do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory"); } while (v < (uint64_t)k);
    } else {
      uint64_t v; do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory"); } while (v < (uint64_t)k);
      if (rel) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((uint64_t)k) : "memory");
      else asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((uint64_t)k) : "memory");
    }
  }
  out[0] = (gtime() - t0) / iters;
}

int main() {
  size_t bytes = 256ull << 20;
  void *s0, *d0, *d1, *s1;
  CK(cudaSetDevice(1)); CK(cudaMalloc(&d1, bytes)); CK(cudaMalloc(&s1, bytes)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMemset(s1, 2, bytes));
  CK(cudaSetDevice(0)); CK(cudaMalloc(&s0, bytes)); CK(cudaMalloc(&d0, bytes)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMemset(s0, 1, bytes));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;
  auto smem4 = [](int chunk) { return 4 * chunk; };
  for (int chunk : {8192, 16384, 32768, 49152}) {
    CK(cudaFuncSetAttribute(tma_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4(chunk)));
    for (int c : {4, 8, 16, 24, 32, 48, 64, 148}) {
      for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); tma_copy<4><<<c, 32, smem4(chunk)>>>((const char*)s0, (char*)d1, bytes, chunk); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
      CK(cudaGetLastError());
      CK(cudaEventElapsedTime(&ms, a, b)); printf("tma peer chunk=%5d ctas=%3d: %.1f GB/s\n", chunk, c, bytes / ms / 1e6);
    }
  }
  // TMA with 2 CTAs per SM
  for (int c : {148, 296}) {
    int chunk = 16384;
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); tma_copy<4><<<c, 32, smem4(chunk)>>>((const char*)s0, (char*)d1, bytes, chunk); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
    CK(cudaEventElapsedTime(&ms, a, b)); printf("tma peer chunk=%5d ctas=%3d: %.1f GB/s\n", chunk, c, bytes / ms / 1e6);
  }
  // TMA local
  for (int c : {148, 296}) {
    int chunk = 32768;
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); tma_copy<4><<<c, 32, smem4(chunk)>>>((const char*)s0, (char*)d0, bytes, chunk); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
    CK(cudaEventElapsedTime(&ms, a, b)); printf("tma local chunk=%5d ctas=%3d: %.1f GB/s payload\n", chunk, c, bytes / ms / 1e6);
  }
  size_t n16 = bytes / 16;
  for (int c : {32, 64, 148, 296}) {
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a)); copy_chunk32<<<c, 512>>>((const int4*)s0, (int4*)d1, n16); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); }
    CK(cudaEventElapsedTime(&ms, a, b)); printf("lsu32 peer ctas=%3d: %.1f GB/s\n", c, bytes / ms / 1e6);
  }
  // pull: device 1 reads device 0 memory
  CK(cudaSetDevice(1));
  cudaEvent_t a1, b1; CK(cudaEventCreate(&a1)); CK(cudaEventCreate(&b1));
  for (int c : {32, 64, 148, 296}) {
    for (int r = 0; r < 3; ++r) { CK(cudaEventRecord(a1)); pull_chunk<<<c, 512>>>((const int4*)s0, (int4*)d1, n16); CK(cudaEventRecord(b1)); CK(cudaEventSynchronize(b1)); }
    CK(cudaEventElapsedTime(&ms, a1, b1)); printf("pull peer->local ctas=%3d: %.1f GB/s\n", c, bytes / ms / 1e6);
  }
  // bidirectional push: dev0 -> d1 and dev1 -> d0 concurrently
  cudaStream_t st1; CK(cudaStreamCreateWithFlags(&st1, cudaStreamNonBlocking));
  CK(cudaSetDevice(0));
  cudaStream_t st0; CK(cudaStreamCreateWithFlags(&st0, cudaStreamNonBlocking));
  for (int c : {32, 64, 148}) {
    float ms0 = 0, ms1 = 0;
    for (int r = 0; r < 3; ++r) {
      CK(cudaSetDevice(0)); CK(cudaEventRecord(a, st0)); copy_chunk<<<c, 512, 0, st0>>>((const int4*)s0, (int4*)d1, n16); CK(cudaEventRecord(b, st0));
      CK(cudaSetDevice(1)); CK(cudaEventRecord(a1, st1)); copy_chunk<<<c, 512, 0, st1>>>((const int4*)s1, (int4*)d0, n16); CK(cudaEventRecord(b1, st1));
      CK(cudaEventSynchronize(b)); CK(cudaEventSynchronize(b1));
    }
    CK(cudaEventElapsedTime(&ms0, a, b)); CK(cudaEventElapsedTime(&ms1, a1, b1));
    printf("bidir push ctas=%3d: %.1f / %.1f GB/s per direction\n", c, bytes / ms0 / 1e6, bytes / ms1 / 1e6);
  }
  CK(cudaSetDevice(0));
  uint64_t* out; CK(cudaMallocManaged(&out, 16 * 8));
  lat_probe<<<1, 1>>>((uint64_t*)d1, (uint64_t*)d0, 2000, out); CK(cudaDeviceSynchronize());
  lat_probe<<<1, 1>>>((uint64_t*)d1, (uint64_t*)d0, 2000, out); CK(cudaDeviceSynchronize());
  const char* names[] = {"peer st + fence.acq_rel.gpu", "peer st + fence.acq_rel.sys", "st.release.sys peer", "ld.acquire.sys peer", "atom.cas.acq_rel.sys peer", "ld.acquire.sys local", "fence.acq_rel.sys alone", "local st + fence.acq_rel.gpu", "st.release.gpu local", "ld.relaxed.sys peer", "peer st + fence.sc.sys"};
  for (int i = 0; i < 11; ++i) printf("%-32s %llu ns\n", names[i], (unsigned long long)out[i]);
  // ping-pong relaxed vs release
  uint64_t *f0, *f1, *o1;
  CK(cudaMalloc(&f0, 128));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&f1, 128)); CK(cudaMallocManaged(&o1, 64));
  for (int rel = 0; rel < 2; ++rel) {
    CK(cudaSetDevice(1)); CK(cudaMemset(f1, 0, 128)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0)); CK(cudaMemset(f0, 0, 128)); CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1)); pingpong<<<1, 1, 0, st1>>>(f1, f0, 5000, 0, rel, o1);
    CK(cudaSetDevice(0)); pingpong<<<1, 1>>>(f0, f1, 5000, 1, rel, out);
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    printf("ping-pong RTT (%s stores): %llu ns\n", rel ? "release" : "relaxed", (unsigned long long)out[0]);
  }
  return 0;
}
