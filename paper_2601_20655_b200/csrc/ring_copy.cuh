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
// vector registers (R17: bit-exact, NaN payloads preserved; 16 loads in flight
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
// V = 3: coherent 16-B loads (ld.global.cg) -- the consumer's copy-out reads
// ring entries that producers write while it runs (the non-coherent .nc path
// is only for data read-only during the kernel: the put's sources).
// V = 2: 32-B accesses (LDG/STG.256) when both sides are 32-B aligned
// (payloads start 64 B into a 128-B aligned entry, so whenever the source is):
// +1.5 % over NVLink, but -12 % for HBM -> HBM (C2), so only the put kernel
// instance for NVLink destinations uses it (profiles/r01_nvlink_sweep.txt).
#ifndef B200RING_COPY_U
#define B200RING_COPY_U 16
#endif
#ifndef B200RING_TAIL_U
#define B200RING_TAIL_U 4
#endif
template <int V = 1>
__device__ __forceinline__ void warp_copy(const uint8_t* __restrict__ src, uint8_t* dst, uint64_t nb, int lane,
                                          bool align_src = false) {
  // Copy-out loads on 128-B lines.  A payload starts 64 B into its 128-B
  // aligned entry (kHdr), so a warp's 512-B load would touch five lines, four
  // of them partially; pulled over NVLink (placements ring_open /
  // ring_create_split) that costs ~1/7 of the link (profiles/r02_pull_align.txt).
  // The loop starts at the line boundary below `src` instead: the lanes before
  // `src` load bytes of the same line (the header or the previous unit, never
  // outside the ring's data region) and store nothing; the stores then sit off
  // their lines locally, which L2 takes at 32-B sector granularity.  Peeling
  // the first bytes instead would cost each unit one dependent round trip.
  // With align_src the units after an entry's first also start on lines
  // (copy_warp), so only the first unit of each entry takes this path.  Local
  // copy-out (the ring in this GPU's HBM) keeps its stores aligned instead
  // (~1 % faster in C2, same-box A/B).
  if (V == 3 && align_src && (((uintptr_t)src | (uintptr_t)dst) & 15) == 0 && ((uintptr_t)src & 127) &&
      nb >= 1024) {
    const uint32_t off16 = (uint32_t)(((uintptr_t)src & 127) >> 4);
    const int4* s = reinterpret_cast<const int4*>(src) - off16;
    int4* d = reinterpret_cast<int4*>(dst) - off16;
    const uint32_t n16 = (uint32_t)(nb >> 4) + off16;
    constexpr int U = B200RING_COPY_U;
    uint32_t i = lane;
    for (; i + (U - 1) * 32 < n16; i += U * 32) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = ld_cg16(s + i + j * 32);
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (i + j * 32 >= off16) st16(d + i + j * 32, v[j]);
    }
    constexpr int T = B200RING_TAIL_U;   // the ragged rest: T loads in flight per lane, not one round trip per 512 B
    for (; i < n16; i += T * 32) {
      int4 v[T];
#pragma unroll
      for (int j = 0; j < T; ++j)
        if (i + j * 32 < n16) v[j] = ld_cg16(s + i + j * 32);
#pragma unroll
      for (int j = 0; j < T; ++j)
        if (i + j * 32 < n16 && i + j * 32 >= off16) st16(d + i + j * 32, v[j]);
    }
    const uint64_t done = (uint64_t)(n16 - off16) << 4;
    for (uint64_t j = done + lane; j < nb; j += 32) dst[j] = __ldcg(src + j);
    return;
  }
  if (V == 2 && (((uintptr_t)src | (uintptr_t)dst) & 31) == 0) {
    const uint32_t n32 = (uint32_t)(nb >> 5);
    constexpr int U = B200RING_COPY_U / 2;   // same 8 KiB in flight per warp
    uint32_t i = lane;
    for (; i + (U - 1) * 32 < n32; i += U * 32) {
      v8u32 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = ld_stream32(src + 32ull * (i + j * 32));
#pragma unroll
      for (int j = 0; j < U; ++j) st32(dst + 32ull * (i + j * 32), v[j]);
    }
    for (; i < n32; i += 32) st32(dst + 32ull * i, ld_stream32(src + 32ull * i));
    for (uint64_t j = ((uint64_t)n32 << 5) + lane; j < nb; j += 32) dst[j] = V == 3 ? __ldcg(src + j) : src[j];
  } else if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    const uint32_t n16 = (uint32_t)(nb >> 4);
    constexpr int U = B200RING_COPY_U;   // 16: 8 KiB in flight per warp
    uint32_t i = lane;
    for (; i + (U - 1) * 32 < n16; i += U * 32) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = V == 3 ? ld_cg16(s + i + j * 32) : ld_stream16(s + i + j * 32);
#pragma unroll
      for (int j = 0; j < U; ++j) st16(d + i + j * 32, v[j]);
    }
    constexpr int T = B200RING_TAIL_U;
    for (; i < n16; i += T * 32) {
      int4 v[T];
#pragma unroll
      for (int j = 0; j < T; ++j)
        if (i + j * 32 < n16) v[j] = V == 3 ? ld_cg16(s + i + j * 32) : ld_stream16(s + i + j * 32);
#pragma unroll
      for (int j = 0; j < T; ++j)
        if (i + j * 32 < n16) st16(d + i + j * 32, v[j]);
    }
    for (uint64_t j = ((uint64_t)n16 << 4) + lane; j < nb; j += 32) dst[j] = V == 3 ? __ldcg(src + j) : src[j];
  } else if ((((uintptr_t)src | (uintptr_t)dst) & 3) == 0) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    const uint64_t n4 = nb >> 2;
    for (uint64_t i = lane; i < n4; i += 32) d[i] = V == 3 ? __ldcg(s + i) : s[i];
    for (uint64_t j = (n4 << 2) + lane; j < nb; j += 32) dst[j] = V == 3 ? __ldcg(src + j) : src[j];
  } else {
    for (uint64_t j = lane; j < nb; j += 32) dst[j] = V == 3 ? __ldcg(src + j) : src[j];
  }
}

__device__ __forceinline__ uint32_t units_for(uint64_t len, uint32_t chunk) {
  // an empty payload has no unit: entry headers are written by the put's publisher
  return (uint32_t)((len + chunk - 1) >> (__ffs(chunk) - 1));
}

// Zero the counter set a launch will hand to its successor.
__device__ __forceinline__ void reset_set(LaunchSet* s, int lane) {
  for (int i = lane; i < kPlanRing; i += 32) s->arrive[i] = 0;
  if (lane == 0) {
    s->planned = 0;
    s->pub_seq = 0;
    s->next_unit = 0;
  }
}

__device__ __forceinline__ uint64_t ld_acquire_cta_shared64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "l"(v) : "memory");
}

// Lane 0: wait until unit u is planned (returns the `planned` word that covers
// it) or the launch has no unit u (returns a done word with fewer units).
// Causality: control warp release -> (gpu acquire) poller -> (cta release /
// acquire through shared memory) this warp; the plan loads that follow are
// ordered after it (PTX causality order is transitive across scopes).
__device__ __forceinline__ uint64_t wait_planned(LaunchSet* S, CopyShared* cs, uint32_t u, uint64_t timeout_ns,
                                                 bool& timed_out) {
  uint64_t end = 0;
  while (true) {
    const uint64_t v = ld_acquire_cta_shared64(&cs->pl);
    if (planned_units(v) > u || planned_done(v)) return v;
    if (atomicCAS_block(&cs->owner, 0u, 1u) == 0u) {
      // relaxed polls, one acquire fence when the word has moved: an
      // ld.acquire invalidates the SM's L1 (CCTL.IVALL) on every poll, and
      // the L1 stages the in-flight loads of the copy warps still working
      uint64_t g = ld_relaxed<false>(&S->planned);
      if (g != v) {
        fence_acq_rel<false>();
        st_release_cta_shared64(&cs->pl, g);              // monotonic: one poller at a time
      }
      atomicExch_block(&cs->owner, 0u);
      if (planned_units(g) > u || planned_done(g)) return g;
    }
    const uint64_t t = globaltimer();
    if (!end) end = t + 2 * timeout_ns;
    else if (t > end) { timed_out = true; return v; }
    __nanosleep(64);
  }
}

// Copy warp main loop: take the next unit with one atomicAdd (dynamic,
// warp-granular scheduling).  Only warps that are resident take units, so the
// launch makes progress even if some of its CTAs cannot be scheduled (other
// kernels occupying SMs): the kernel never needs all its CTAs co-resident.
// Returns when the control warp is done and every unit has been handed out, or
// after `2 * timeout_ns` without progress.  `cs` must be zeroed (and the CTA
// synchronised) before the first call.
//
// After the control warp's release: one poller per CTA acquires it, then the
// lanes read 32 candidate plans' copy sectors (unit range AND copy fields) in
// one round trip; the hit lane broadcasts its fields.
template <int V = 1>
__device__ __forceinline__ void copy_warp(LaunchCtx* ctx, LaunchSet* S, CopyShared* cs, uint32_t chunk,
                                          uint64_t timeout_ns, uint64_t* trace = nullptr,
                                          const SpecRound* spec = nullptr, bool align_src = false) {
  const int lane = threadIdx.x & 31;
  uint32_t cur = 0;   // items before `cur` hold no unit this warp can still take
  // First unit: the CTA took a block of units for all its copy warps with ONE
  // atomicAdd when it started (~1,000 warps each taking their first unit with
  // an atomicAdd on one word serialise for microseconds); only a running CTA
  // takes units, so a launch still never needs all its CTAs resident.  Later
  // units: one atomicAdd each.
  uint32_t first = cs->first + (threadIdx.x >> 5) - (blockIdx.x == 0 ? 2u : 0u);
  bool have_first = true;
  // debug timeline: the first unit of the first copy warp of each CTA
  uint64_t* tr = (trace && (threadIdx.x >> 5) == (blockIdx.x == 0 ? 2 : 0)) ? trace + 1280 + 4 * blockIdx.x : nullptr;
  // The item of the last unit, cached: consecutive units usually belong to the
  // same entry, and its plan cannot change while this warp still holds one of
  // its units (the slot is reused only after the item is published).
  uint32_t c_item = 0xffffffffu, c_fu = 0, c_nu = 0;
  uint64_t c_src = 0, c_dst = 0, c_len = 0;
  while (true) {
    uint32_t u = 0, quit = 0, ps = 0;
    if (lane == 0) {
      if (tr) tr[0] = globaltimer();
      u = have_first ? first : atomicAdd(&S->next_unit, 1u);
      if (!(spec && u < spec->n_units)) {      // not covered by the CTA's speculative first round
        bool to = false;
        const uint64_t pl = wait_planned(S, cs, u, timeout_ns, to);
        if (to || planned_units(pl) <= u) {
          quit = 1;
          if (trace) atomicMax(reinterpret_cast<unsigned long long*>(trace + 254), (unsigned long long)globaltimer());
        }
        ps = planned_items(pl);
      }
      if (tr) tr[1] = globaltimer();
    }
    __syncwarp();
    have_first = false;
    quit = __shfl_sync(0xffffffffu, quit, 0);
    if (quit) return;
    u = __shfl_sync(0xffffffffu, u, 0);
    ps = __shfl_sync(0xffffffffu, ps, 0);
    uint32_t item = 0xffffffffu, fu = 0, nu_hit = 0;
    uint64_t src = 0, dst = 0, len = 0;
    if (c_nu && u - c_fu < c_nu) {             // same entry as the previous unit: no plan read
      item = c_item; fu = c_fu; nu_hit = c_nu; src = c_src; dst = c_dst; len = c_len;
    }
    if (item == 0xffffffffu && spec && u < spec->n_units) {   // the CTA's own evaluation of the first rounds
      for (uint32_t b = 0; b < spec->n; b += 32) {
        const uint32_t i = b + lane;
        const bool in = i < spec->n;
        const SpecItem& si = spec->it[in ? i : 0];
        const bool hit = in && si.nunits && u >= si.first_unit && u - si.first_unit < si.nunits;
        const uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (m) {
          const SpecItem& sh = spec->it[b + __ffs(m) - 1];
          item = sh.item;
          fu = sh.first_unit;
          nu_hit = sh.nunits;
          src = sh.src;
          dst = sh.dst;
          len = sh.len;
          break;
        }
      }
    }
    // find the item holding unit u (plans are read through L2: ring slots are reused)
    for (uint32_t b = cur; item == 0xffffffffu && b < ps; b += 32) {
      const uint32_t i = b + lane;
      bool hit = false;
      ulonglong2 q0 = make_ulonglong2(0, 0), q1 = make_ulonglong2(0, 0);
      if (i < ps) {
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(&ctx->plan[i % kPlanRing]);
        q0 = __ldcg(p);        // src, dst
        q1 = __ldcg(p + 1);    // len, first_unit | nunits << 32
        const uint32_t f0 = (uint32_t)q1.y, nu = (uint32_t)(q1.y >> 32);
        hit = nu && u >= f0 && u - f0 < nu;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      if (m) {
        const int h = __ffs(m) - 1;
        item = b + h;
        src = __shfl_sync(0xffffffffu, q0.x, h);
        dst = __shfl_sync(0xffffffffu, q0.y, h);
        len = __shfl_sync(0xffffffffu, q1.x, h);
        fu = (uint32_t)__shfl_sync(0xffffffffu, q1.y, h);
        nu_hit = (uint32_t)(__shfl_sync(0xffffffffu, q1.y, h) >> 32);
        break;
      }
    }
    if (item == 0xffffffffu) return;   // cannot happen with a consistent plan
    cur = item;
    c_item = item; c_fu = fu; c_nu = nu_hit; c_src = src; c_dst = dst; c_len = len;
    const uint32_t c = u - fu;
    // align_src: units after the first start on the source's 128-B lines (the
    // first is `sh` bytes short; the control warp planned units_for(len + sh))
    const uint32_t sh = align_src ? (uint32_t)(src & 127u) : 0u;
    uint64_t lo = c ? (uint64_t)c * chunk - sh : 0;
    uint64_t hi = min(len, (uint64_t)(c + 1) * chunk - sh);
#ifndef B200RING_RAGGED_FIRST
#define B200RING_RAGGED_FIRST 1
#endif
    if (B200RING_RAGGED_FIRST && !align_src && nu_hit > 1) {
      // the ragged part of an item is its FIRST unit, so the units a launch
      // hands out last are whole ones
      const uint64_t rag = len - (uint64_t)(nu_hit - 1) * chunk;
      lo = c ? rag + (uint64_t)(c - 1) * chunk : 0;
      hi = c ? rag + (uint64_t)c * chunk : rag;
    }
    if (tr && lane == 0) tr[2] = globaltimer();
    RING_CHECK(c < (uint32_t)((len + sh + chunk - 1) / chunk) || len == 0, "unit inside its item", u, item);
    if (hi > lo)
      warp_copy<V>(reinterpret_cast<const uint8_t*>(src) + lo, reinterpret_cast<uint8_t*>(dst) + lo, hi - lo, lane,
                   align_src);
    __syncwarp();
    if (lane == 0) red_release_gpu_add(&S->arrive[item % kPlanRing], 1u);
    if (tr && lane == 0) tr[3] = globaltimer();
    tr = nullptr;
  }
}

// `chunk` is a power of two (host-enforced): a shift, not a 64-bit division
// (the division subroutine cost ~0.3 us per message in the serial leader path).
// ---------------------------------------------------------------------------
// TMA copy engine (copy_mode 1): each engine warp (up to kMaxEngineWarps per
// CTA, put.cu) drives its own ring of `stages`
// shared-memory buffers of `chunk` bytes with bulk asynchronous copies
// (cp.async.bulk global -> shared, completion on an mbarrier; then
// shared -> global, completion by bulk group).  One elected lane issues; the
// warp helps to find the entry of a unit and writes headers and ragged tails.
// The SM's LSU and registers stay free (the paper's L3 concern about GPU
// interference), and each SM keeps stages*chunk bytes in flight.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct EngineStage {
  uint64_t dst;
  uint32_t n, item;
};

// Finds the item holding unit u among planned items [cur, ps); warp-uniform.
__device__ __forceinline__ uint32_t find_item(LaunchCtx* ctx, uint32_t u, uint32_t cur, uint32_t ps, int lane) {
  for (uint32_t b = cur; b < ps; b += 32) {
    const uint32_t i = b + lane;
    bool hit = false;
    if (i < ps) {
      const Plan& p = ctx->plan[i % kPlanRing];
      const uint32_t nu = ld_cg32(&p.nunits);
      const uint32_t fu = ld_cg32(&p.first_unit);
      hit = nu && u >= fu && u - fu < nu;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, hit);
    if (m) return b + __ffs(m) - 1;
  }
  return 0xffffffffu;
}

// Unit u's (item, first unit, src, dst, len) from a CTA's speculative first
// round, or item = 0xffffffff if not covered.
__device__ __forceinline__ void spec_lookup(const SpecRound* spec, uint32_t u, int lane, uint32_t& item, uint32_t& fu,
                                            uint64_t& src, uint64_t& dst, uint64_t& len) {
  item = 0xffffffffu;
  if (!spec || u >= spec->n_units) return;
  for (uint32_t b = 0; b < spec->n; b += 32) {
    const uint32_t i = b + lane;
    const bool in = i < spec->n;
    const SpecItem& si = spec->it[in ? i : 0];
    const bool hit = in && si.nunits && u >= si.first_unit && u - si.first_unit < si.nunits;
    const uint32_t m = __ballot_sync(0xffffffffu, hit);
    if (m) {
      const SpecItem& sh = spec->it[b + __ffs(m) - 1];
      item = sh.item; fu = sh.first_unit; src = sh.src; dst = sh.dst; len = sh.len;
      return;
    }
  }
}

template <int N>
__device__ __forceinline__ void bulk_wait_group(uint32_t allow) {   // all but the `allow` newest groups complete
  switch (allow) {
    case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 7;" ::: "memory"); break;
  }
}
template <int N>
__device__ __forceinline__ void bulk_wait_group_read(uint32_t allow) {   // their smem reads done
  switch (allow) {
    case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory"); break;
  }
}

// Pipelined TMA engine.  Counters over the engine's units in issue order:
//   k_issue  loads issued (global -> shared, mbarrier complete_tx)
//   k_store  stores issued (shared -> global, one bulk group each)
//   k_free   stores whose shared-memory reads are done: the stage is reusable
//   k_done   stores complete (global writes done): the unit is counted (arrive)
// The next unit's control (take, planned check, find) is resolved while the
// previous ones are in flight; stages are reused as soon as their store has
// READ shared memory; arrives follow full completion, lazily (at most STAGES
// stores outstanding).
template <int STAGES>
__device__ void copy_engine(LaunchCtx* ctx, LaunchSet* S, uint32_t chunk, uint64_t timeout_ns, uint8_t* bufs,
                            const SpecRound* spec = nullptr, int ew = 0) {
  const int lane = threadIdx.x & 31;
  // per engine warp `ew` of the CTA: its own stages, barriers and bookkeeping
  __shared__ __align__(8) uint64_t bar_all[kMaxEngineWarps][STAGES];
  __shared__ EngineStage st_all[kMaxEngineWarps][STAGES];
  __shared__ uint32_t items_all[kMaxEngineWarps][2 * STAGES];   // item of unit k (k_issue - k_done <= 2 STAGES)
  uint64_t* bar = bar_all[ew];
  EngineStage* st = st_all[ew];
  uint32_t* items = items_all[ew];
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;                       // parity bit per stage
  uint32_t k_issue = 0, k_store = 0, k_free = 0, k_done = 0, cur = 0;
  uint32_t pending_u = 0xffffffffu;         // unit taken, not resolved yet
  bool exhausted = false;
  uint64_t wait_end = 0;
  // Control kept off the per-unit path (one warp drives all of a CTA's
  // copies): units are taken kTake at a time (one atomicAdd), the `planned`
  // word is re-read only when a unit is past the cached one, and the entry of
  // the last unit is cached (consecutive units usually share it).
  constexpr uint32_t kTake = 2 * STAGES;
  uint32_t q_next = 0, q_end = 0;
  uint64_t pl_cache = 0;
  uint32_t c_item = 0xffffffffu, c_fu = 0, c_nu = 0;
  uint64_t c_src = 0, c_dst = 0, c_len = 0;
  if (lane == 0) {
    q_next = atomicAdd(&S->next_unit, kTake);
    q_end = q_next + kTake;
  }
  while (true) {
    bool progress = false;
    // ---- 1. resolve the next unit and load it into a free stage
    if (!exhausted && k_issue - k_free < (uint32_t)STAGES) {
      uint32_t u = 0, state = 0, ps = 0;    // 0 = planned, 1 = not yet, 2 = none left
      if (lane == 0) {
        if (pending_u == 0xffffffffu) {
          if (q_next == q_end) {
            q_next = atomicAdd(&S->next_unit, kTake);
            q_end = q_next + kTake;
          }
          pending_u = q_next++;
        }
        u = pending_u;
        if (!(spec && u < spec->n_units)) {
          if (planned_units(pl_cache) <= u && !planned_done(pl_cache)) {
            const uint64_t pl = ld_relaxed<false>(&S->planned);
            if (pl != pl_cache) {
              fence_acq_rel<false>();       // acquire the plans behind the new word
              pl_cache = pl;
            }
          }
          if (planned_units(pl_cache) <= u) state = planned_done(pl_cache) ? 2 : 1;
          else ps = planned_items(pl_cache);
        }
      }
      state = __shfl_sync(0xffffffffu, state, 0);
      if (state == 2) {
        exhausted = true;
      } else if (state == 1) {
        if (k_done == k_issue) {            // nothing in flight: wait politely (bounded)
          const uint64_t t = globaltimer();
          if (!wait_end) wait_end = t + 2 * timeout_ns;
          else if (t > wait_end) exhausted = true;
          __nanosleep(64);
        }
      } else {
        wait_end = 0;
        u = __shfl_sync(0xffffffffu, u, 0);
        ps = __shfl_sync(0xffffffffu, ps, 0);
        pending_u = 0xffffffffu;
        uint32_t item = 0xffffffffu, fu = 0;
        uint64_t src = 0, dst = 0, len = 0;
        if (c_nu && u - c_fu < c_nu) {      // same entry as the previous unit
          item = c_item; fu = c_fu; src = c_src; dst = c_dst; len = c_len;
        } else {
          spec_lookup(spec, u, lane, item, fu, src, dst, len);
          uint32_t nu = 0;
          if (item != 0xffffffffu) {
            nu = units_for(len, chunk);
          } else {
            item = find_item(ctx, u, cur, ps, lane);
            if (item != 0xffffffffu) {
              const Plan& p = ctx->plan[item % kPlanRing];
              src = ld_cg64(&p.src); dst = ld_cg64(&p.dst); len = ld_cg64(&p.len);
              fu = ld_cg32(&p.first_unit);
              nu = ld_cg32(&p.nunits);
              cur = item;
            }
          }
          if (item != 0xffffffffu) { c_item = item; c_fu = fu; c_nu = nu; c_src = src; c_dst = dst; c_len = len; }
        }
        if (item == 0xffffffffu) {
          exhausted = true;
        } else {
          const uint32_t c = u - fu;
          const uint64_t lo = (uint64_t)c * chunk;
          const uint64_t hi = min(len, lo + chunk);
          const uint8_t* s8 = reinterpret_cast<const uint8_t*>(src) + lo;
          uint8_t* d8 = reinterpret_cast<uint8_t*>(dst) + lo;
          const uint64_t n = hi > lo ? hi - lo : 0;
          const bool aligned = ((((uintptr_t)s8) | ((uintptr_t)d8)) & 15) == 0;
          const uint32_t n16 = aligned ? (uint32_t)(n & ~15ull) : 0u;
          if (n16 < n) warp_copy(s8 + n16, d8 + n16, n - n16, lane);   // ragged tail / unaligned: LSU
          __syncwarp();                     // lanes' stores precede the arrive issued later by lane 0
          if (n16 == 0) {
            if (lane == 0) red_release_gpu_add(&S->arrive[item % kPlanRing], 1u);
          } else {
            if (lane == 0) {
              const int s = (int)(k_issue % STAGES);
              st[s].dst = reinterpret_cast<uint64_t>(d8);
              st[s].n = n16;
              st[s].item = item;
              items[k_issue % (2 * STAGES)] = item;
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[s])), "r"(n16)
                           : "memory");
              asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                           ::"r"(smem_addr(bufs + (size_t)s * chunk)), "l"(s8), "r"(n16), "r"(smem_addr(&bar[s]))
                           : "memory");
            }
            ++k_issue;
          }
          progress = true;
        }
      }
    }
    // ---- 2. the oldest loaded stage -> its store (non-blocking check)
    if (k_store < k_issue) {
      uint32_t ok = 0;
      if (lane == 0) {
        const int s = (int)(k_store % STAGES);
        const uint32_t par = (phase >> s) & 1u;
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(smem_addr(&bar[s])), "r"(par) : "memory");
        if (ok) {
          phase ^= 1u << s;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(st[s].dst), "r"(smem_addr(bufs + (size_t)s * chunk)), "r"(st[s].n) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok) { ++k_store; progress = true; }
    }
    // ---- 3. free a stage once its store has read shared memory (when needed)
    if (k_free < k_store && (k_issue - k_free == (uint32_t)STAGES || !progress)) {
      if (lane == 0) bulk_wait_group_read<STAGES>(k_store - k_free - 1);
      ++k_free;
      progress = true;
    }
    // ---- 4. count completed stores (lazily: keep at most STAGES outstanding)
    if (k_done < k_free && (k_store - k_done > (uint32_t)STAGES || !progress || exhausted)) {
      if (lane == 0) {
        bulk_wait_group<STAGES>(k_store - k_done - 1);
        asm volatile("fence.proxy.async.global;" ::: "memory");   // async-proxy writes before the generic release
        red_release_gpu_add(&S->arrive[items[k_done % (2 * STAGES)] % kPlanRing], 1u);
      }
      ++k_done;
      progress = true;
    }
    __syncwarp();
    if (exhausted && k_done == k_issue) break;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Load the CRC slicing tables into shared memory (whole CTA participates).
__device__ __forceinline__ void load_crc_table(uint32_t* s_tab, const uint32_t* g_tab) {
  for (int i = threadIdx.x; i < kCrcTableWords; i += blockDim.x) s_tab[i] = g_tab[i];
  __syncthreads();
}

}  // namespace b200ring
