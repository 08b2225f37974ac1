// ring_copy.cuh — copy warps shared by the put and get kernels, and the
// per-launch bookkeeping helpers.
//
// A launch is a pipeline of items (entries) planned in order by one control
// warp into LaunchCtx::plan[].  The payload of each item is cut into fixed
// `chunk`-byte work units numbered consecutively across items
// (first_unit .. first_unit + nunits - 1).  Every copy warp of the grid grabs
// the next unit with one atomicAdd (dynamic, warp-granular scheduling: small
// and large entries mix without idle CTAs), waits until the control warp has
// published a plan covering that unit, copies it through 16-byte integer
// vector registers (R17: bit-exact, NaN payloads preserved; 8 loads in flight
// per lane), and arrives on arrive[item] with a gpu-scope release.  The
// publisher / finisher warp that observes the full count then performs one
// system-scope release (the tail store, or the head store for a consumer):
// PTX causality order is transitive across scopes, so every copy warp's NVLink
// stores are visible to the other GPU before that release.
#pragma once
#include "ring_internal.h"

namespace b200ring {

__device__ __forceinline__ uint32_t ld_cg32(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint64_t ld_cg64(const uint64_t* p) { return __ldcg(reinterpret_cast<const unsigned long long*>(p)); }

// Warp copy of `nb` bytes, lanes striding 16 B.
__device__ __forceinline__ void warp_copy(const uint8_t* __restrict__ src, uint8_t* dst, uint64_t nb, int lane) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    const uint32_t n16 = (uint32_t)(nb >> 4);
    uint32_t i = lane;
    constexpr int U = 16;   // 8 KiB in flight per warp
    for (; i + (U - 1) * 32 < n16; i += U * 32) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = ld_stream16(s + i + j * 32);
#pragma unroll
      for (int j = 0; j < U; ++j) st16(d + i + j * 32, v[j]);
    }
    for (; i < n16; i += 32) st16(d + i, ld_stream16(s + i));
    for (uint64_t j = ((uint64_t)n16 << 4) + lane; j < nb; j += 32) dst[j] = src[j];
  } else if ((((uintptr_t)src | (uintptr_t)dst) & 3) == 0) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    const uint64_t n4 = nb >> 2;
    for (uint64_t i = lane; i < n4; i += 32) d[i] = s[i];
    for (uint64_t j = (n4 << 2) + lane; j < nb; j += 32) dst[j] = src[j];
  } else {
    for (uint64_t j = lane; j < nb; j += 32) dst[j] = src[j];
  }
}

// Zero the counter set a launch will hand to its successor.
__device__ __forceinline__ void reset_set(LaunchSet* s, int lane) {
  for (int i = lane; i < kPlanRing; i += 32) s->arrive[i] = 0;
  if (lane == 0) {
    s->planned = 0;
    s->pub_seq = 0;
    s->next_unit = 0;
    s->done = 0;
  }
}

// Copy warp main loop: take the next unit with one atomicAdd (dynamic,
// warp-granular scheduling).  Only warps that are resident take units, so the
// launch makes progress even if some of its CTAs cannot be scheduled (other
// kernels occupying SMs): the kernel never needs all its CTAs co-resident.
// Returns when the control warp is done and every unit has been handed out, or
// after `2 * timeout_ns` without progress.
__device__ __forceinline__ void copy_warp(LaunchCtx* ctx, LaunchSet* S, uint32_t chunk, uint64_t timeout_ns) {
  const int lane = threadIdx.x & 31;
  uint32_t cur = 0;   // items before `cur` hold no unit this warp can still take
  while (true) {
    uint32_t u = 0, quit = 0, ps = 0;
    if (lane == 0) {
      u = atomicAdd(&S->next_unit, 1u);
      uint64_t end = 0;
      // Poll with relaxed loads (no L1 invalidation per poll; thousands of
      // warps may wait here), then one acquire once the unit is planned.
      while (true) {
        if (planned_units(ld_relaxed<false>(&S->planned)) > u) break;
        if (ld_relaxed_gpu32(&S->done)) {
          (void)ld_acquire_gpu32(&S->done);     // `planned` is final once done is seen
          if (planned_units(ld_acquire<false>(&S->planned)) > u) break;
          quit = 1;
          break;
        }
        const uint64_t t = globaltimer();
        if (!end) end = t + 2 * timeout_ns;
        else if (t > end) { quit = 1; break; }
        __nanosleep(64);
      }
      // one acquire of the word that covered u: its items include u's item
      ps = planned_items(ld_acquire<false>(&S->planned));
    }
    __syncwarp();
    quit = __shfl_sync(0xffffffffu, quit, 0);
    if (quit) return;
    u = __shfl_sync(0xffffffffu, u, 0);
    ps = __shfl_sync(0xffffffffu, ps, 0);
    // find the item holding unit u (plans are read through L2: ring slots are reused)
    uint32_t item = 0xffffffffu;
    for (uint32_t b = cur; b < ps && item == 0xffffffffu; b += 32) {
      const uint32_t i = b + lane;
      bool hit = false;
      if (i < ps) {
        const Plan& p = ctx->plan[i % kPlanRing];
        const uint32_t nu = ld_cg32(&p.nunits);
        const uint32_t fu = ld_cg32(&p.first_unit);
        hit = nu && u >= fu && u - fu < nu;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      if (m) item = b + __ffs(m) - 1;
    }
    if (item == 0xffffffffu) return;   // cannot happen with a consistent plan
    cur = item;
    const Plan& p = ctx->plan[item % kPlanRing];
    const uint64_t src = ld_cg64(&p.src), dst = ld_cg64(&p.dst), len = ld_cg64(&p.len);
    const uint64_t hdr_dst = ld_cg64(&p.hdr_dst);
    const uint32_t c = u - ld_cg32(&p.first_unit);
    const uint64_t lo = (uint64_t)c * chunk;
    const uint64_t hi = min(len, lo + chunk);
    if (c == 0 && hdr_dst && lane < 4) {
      const int4 h = __ldcg(reinterpret_cast<const int4*>(p.hdr) + lane);
      st16(reinterpret_cast<uint8_t*>(hdr_dst) + 16 * lane, h);
    }
    if (hi > lo) warp_copy(reinterpret_cast<const uint8_t*>(src) + lo, reinterpret_cast<uint8_t*>(dst) + lo, hi - lo, lane);
    __syncwarp();
    if (lane == 0) red_release_gpu_add(&S->arrive[item % kPlanRing], 1u);
  }
}

// `chunk` is a power of two (host-enforced): a shift, not a 64-bit division
// (the division subroutine cost ~0.3 us per message in the serial leader path).
__device__ __forceinline__ uint32_t units_for(uint64_t len, uint32_t chunk) {
  const uint64_t u = (len + chunk - 1) >> (__ffs(chunk) - 1);
  return u ? (uint32_t)u : 1u;   // at least one: it also writes the header
}

// Load the CRC slicing tables into shared memory (whole CTA participates).
__device__ __forceinline__ void load_crc_table(uint32_t* s_tab, const uint32_t* g_tab) {
  for (int i = threadIdx.x; i < kCrcTableWords; i += blockDim.x) s_tab[i] = g_tab[i];
  __syncthreads();
}

}  // namespace b200ring
