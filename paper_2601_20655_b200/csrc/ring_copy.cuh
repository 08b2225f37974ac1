// ring_copy.cuh — the copy CTAs shared by the put and get kernels.
//
// A launch is a pipeline of "items" (planned entries) written by a control
// warp into LaunchCtx::plan[] and consumed in order by every copy CTA.  Item i
// is copied by the first `cnt` copy CTAs, each taking one contiguous 16-byte
// aligned share, through 16-byte integer vector loads/stores (R17: bit-exact)
// with 8 loads in flight per thread.  When a CTA's share is done it arrives on
// arrive[i % kPlanRing] with a gpu-scope release after a CTA barrier: the
// finisher warp that observes the full count and then performs a system-scope
// release (the tail store) makes every CTA's NVLink stores visible to the
// consumer before the tail (PTX causality order is transitive across scopes).
#pragma once
#include "ring_internal.h"

namespace b200ring {

__device__ __forceinline__ void copy_span(const uint8_t* __restrict__ src, uint8_t* dst, uint64_t nb, int tid, int T) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    const uint64_t n16 = nb >> 4;
    uint64_t i = tid;
    constexpr int U = 8;
    for (; i + (U - 1) * (uint64_t)T < n16; i += U * (uint64_t)T) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = ld_stream16(s + i + (uint64_t)j * T);
#pragma unroll
      for (int j = 0; j < U; ++j) st16(d + i + (uint64_t)j * T, v[j]);
    }
    for (; i < n16; i += T) st16(d + i, ld_stream16(s + i));
    for (uint64_t j = (n16 << 4) + tid; j < nb; j += T) dst[j] = src[j];
  } else if ((((uintptr_t)src | (uintptr_t)dst) & 3) == 0) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    const uint64_t n4 = nb >> 2;
    for (uint64_t i = tid; i < n4; i += T) d[i] = s[i];
    for (uint64_t j = (n4 << 2) + tid; j < nb; j += T) dst[j] = src[j];
  } else {
    for (uint64_t j = tid; j < nb; j += T) dst[j] = src[j];
  }
}

struct SharedItem {
  uint64_t src, dst, len, hdr_dst;
  uint32_t cnt, abort, cta_base;
  uint32_t hdr[16];
};

// Copy CTA `cta` (0-based among `n_ctas` copy CTAs) processes items
// [first, first+count); item i is shared by the cnt CTAs that follow
// cta_base cyclically, so consecutive small entries land on different CTAs.
// Waits for each plan with a no-progress budget of `timeout_ns`; on expiry it
// leaves (the control warp reports RING_ETIMEDOUT for the affected messages).
__device__ __forceinline__ void copy_worker(LaunchCtx* ctx, uint64_t first, uint64_t count, uint32_t cta,
                                            uint32_t n_ctas, uint64_t timeout_ns) {
  __shared__ SharedItem si;
  const int tid = threadIdx.x, T = blockDim.x;
  for (uint64_t i = first; i < first + count; ++i) {
    if (tid == 0) {
      uint32_t ab = 0;
      if (ld_acquire_gpu64(&ctx->plan_seq) <= i) {
        const uint64_t end = globaltimer() + 2 * timeout_ns;
        while (ld_acquire_gpu64(&ctx->plan_seq) <= i) {
          if (globaltimer() > end) { ab = 1; break; }
        }
      }
      si.abort = ab;
      if (!ab) {
        const Plan& p = ctx->plan[i % kPlanRing];
        si.src = p.src; si.dst = p.dst; si.len = p.len; si.hdr_dst = p.hdr_dst; si.cnt = p.cnt;
        si.cta_base = p.cta_base;
        if (p.hdr_dst) {
#pragma unroll
          for (int w = 0; w < 16; ++w) si.hdr[w] = p.hdr[w];
        }
      }
    }
    __syncthreads();
    if (si.abort) return;
    const uint32_t share = (cta + n_ctas - si.cta_base % n_ctas) % n_ctas;
    if (share < si.cnt) {
      const uint64_t per = ((si.len + si.cnt - 1) / si.cnt + 15) & ~15ull;
      const uint64_t lo = min(si.len, (uint64_t)share * per);
      const uint64_t hi = min(si.len, lo + per);
      if (share == 0 && si.hdr_dst && tid < 4) {
        int4 v = make_int4((int)si.hdr[4 * tid], (int)si.hdr[4 * tid + 1], (int)si.hdr[4 * tid + 2], (int)si.hdr[4 * tid + 3]);
        st16(reinterpret_cast<uint8_t*>(si.hdr_dst) + 16 * tid, v);
      }
      copy_span(reinterpret_cast<const uint8_t*>(si.src) + lo, reinterpret_cast<uint8_t*>(si.dst) + lo, hi - lo, tid, T);
      __syncthreads();
      if (tid == 0) red_release_gpu_add(&ctx->arrive[i % kPlanRing], 1u);
    }
    __syncthreads();
  }
}

// Number of copy CTAs for a payload: one per `chunk_min` bytes, at least 1.
__device__ __forceinline__ uint32_t ctas_for(uint64_t len, uint32_t copy_ctas, uint32_t chunk_min) {
  uint64_t c = (len + chunk_min - 1) / chunk_min;
  if (c < 1) c = 1;
  if (c > copy_ctas) c = copy_ctas;
  return (uint32_t)c;
}

}  // namespace b200ring
