// get.cu — the receiver side of the double ring (receiver
// steps 1-5) and the in-order release (R13).
//
// get_kernel: CTA 0 warp 0 is the control warp; with copy-out, CTA 0 warp 1 is
// the finisher and every other warp of the grid a copy warp (ring_copy.cuh).
//   control warp, one batch of up to 32 entries per round, one entry per lane:
//     lane 0 polls the tail until its sequence differs from the read cursor G
//     (steps 1-2, R7; "wait-free" for the producers); lanes read
//     the size slots of all entries already published, a warp prefix sum of
//     the footprints gives every entry's start (the pointer formula of
//     PAPER.md:731-739 is addition mod R once PAD entries fill every wrap,
//     R3); each lane reads its 64-B header, verifies the CRC-32 (step 3 +
//     PAPER.md:768-769) and writes its view record.  Consuming without
//     copy-out, the lanes also clear the busy bits and the head moves past the
//     whole batch (steps 4-5) with ONE fence, then is pushed to every
//     producer's mirror (credit, R1).
//   finisher (copy-out): releases entries in order once their copies are done.
#include "ring_copy.cuh"

namespace b200ring {

__device__ __forceinline__ uint64_t* g_tail(uint8_t* ring) { return reinterpret_cast<uint64_t*>(ring + kTailOff); }
__device__ __forceinline__ uint64_t* g_head(uint8_t* ring) { return reinterpret_cast<uint64_t*>(ring + kHeadOff); }
__device__ __forceinline__ uint64_t* g_cursor(uint8_t* ring) { return reinterpret_cast<uint64_t*>(ring + kCursorOff); }
__device__ __forceinline__ uint64_t* g_slot(uint8_t* ring, uint32_t N, uint32_t q) {
  return reinterpret_cast<uint64_t*>(ring + kSlotsOff) + (q & (N - 1));
}

// Step 5 made visible: one fence orders the slot clears (and every read of the
// released entries) before the head store and the mirror stores.
template <bool SYS>
__device__ __forceinline__ void publish_head(uint8_t* ring, uint64_t** mirrors, uint32_t n_mirrors, uint64_t H) {
  fence_acq_rel<SYS>();
  st_relaxed<SYS>(g_head(ring), H);
  for (uint32_t i = 0; i < n_mirrors; ++i) {
    uint64_t* m = mirrors[i];
    if (m) st_relaxed<SYS>(m, H | kMirrorValid);
  }
}

__device__ __forceinline__ void st_u32_relaxed_gpu_g(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool SYS>
__device__ void get_control(const GetArgs& a, LaunchCtx* ctx, LaunchSet* S, const uint32_t* crc_tab) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const bool copy = a.dst != nullptr;
  const bool inline_release = a.consume && !copy;
  uint64_t G = ld_cg64(g_cursor(a.ring));
  uint64_t H = ld_cg64(g_head(a.ring));
  uint32_t k = 0, items = 0, units = 0, pending = 0;
  uint32_t fail = RING_OK;
  while (k < a.n) {
    // ---- steps 1-2: wait until the tail passes the read cursor
    uint64_t T = 0, tvis = 0;
    uint32_t st = RING_OK;
    if (lane == 0) {
      T = ld_acquire<SYS>(g_tail(a.ring));
      if (ptr_seq(T) == ptr_seq(G)) {
        if (pending) { publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H); pending = 0; }
        if (a.flags & RING_TRY) {
          st = RING_EMPTY;
        } else {
          // relaxed polls, one acquire fence once the tail moved (an acquire
          // per poll invalidates this SM's L1 under the copy warps' loads)
          const uint64_t end = globaltimer() + a.timeout_ns;
          do {
            T = ld_relaxed<SYS>(g_tail(a.ring));
            if (globaltimer() > end) break;
          } while (ptr_seq(T) == ptr_seq(G));
          if (ptr_seq(T) == ptr_seq(G)) st = RING_ETIMEDOUT;
          else fence_acq_rel<SYS>();
        }
      }
      tvis = (a.flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
    }
    __syncwarp();
    st = __shfl_sync(0xffffffffu, st, 0);
    pending = __shfl_sync(0xffffffffu, pending, 0);
    if (st != RING_OK) { fail = st; break; }
    T = __shfl_sync(0xffffffffu, T, 0);
    tvis = __shfl_sync(0xffffffffu, tvis, 0);
    const uint32_t avail = seq_dist(ptr_seq(T), ptr_seq(G));
    const uint32_t e = min(avail, 32u);
    // ---- slots of every published entry (one per lane)
    uint64_t w = 0;
    if ((uint32_t)lane < e) w = ld_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(G) + lane));
    // footprint: bits 0-39 (fault-tolerant rings keep a sequence tag in 40-61, R21; R < 2^40)
    const uint64_t f = (uint32_t)lane < e ? (w & kFLow) : 0;
    const bool pad = (w & kPad) != 0;
    const bool ismsg = (uint32_t)lane < e && !pad;
    const uint64_t incl = warp_incl_scan64(f, lane);
    uint64_t start = ptr_off(G) + (incl - f);
    if (start >= a.R) start -= a.R;
    // ---- cut the batch after the last message still wanted (trailing PAD
    // entries stay for the next call, as the oracle's receiver leaves them)
    const uint32_t msgmask = __ballot_sync(0xffffffffu, ismsg);
    const uint32_t need = a.n - k;
    uint32_t e2 = e;
    if ((uint32_t)__popc(msgmask) >= need) {
      uint32_t mm = msgmask;
      for (uint32_t q = 1; q < need; ++q) mm &= mm - 1;   // keep the need-th set bit lowest
      e2 = __ffs(mm);                                    // lanes [0, e2) up to and including it
    }
    const bool in = (uint32_t)lane < e2;
    const uint32_t mi = k + __popc(msgmask & lt_mask);
    // ---- step 3: header + checksum, view record
    uint64_t len = 0;
    uint32_t status = RING_OK;
    bool deliver = false;
    uint32_t hw[16] = {};
    if (in && ismsg) {
      const int4* hp = reinterpret_cast<const int4*>(
          a.hdrs ? a.hdrs + 64ull * ((ptr_seq(G) + lane) & (a.N - 1)) : a.data + start);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 v = __ldcg(hp + q);
        hw[4 * q] = (uint32_t)v.x; hw[4 * q + 1] = (uint32_t)v.y; hw[4 * q + 2] = (uint32_t)v.z; hw[4 * q + 3] = (uint32_t)v.w;
      }
      const uint32_t crc = crc52(hw, crc_tab);
      len = (hw[8] >> 16) | ((uint64_t)(hw[9] & 0xffffu) << 16);
      if (crc != hw[0] || kHdr + len > f) { status = RING_ECORRUPT; len = 0; }   // discarded, still consumed
      else if (copy && len > a.dst_stride) status = RING_EMSGSIZE;
      else deliver = true;
    }
    // payload checksum (header flags bit 0, fault-tolerant rings, Q10): one warp per entry
    uint32_t pmask = __ballot_sync(0xffffffffu, in && ismsg && status != RING_ECORRUPT && ((hw[13] >> 16) & 1u));
    while (pmask) {
      const int j = __ffs(pmask) - 1;
      pmask &= pmask - 1;
      const uint64_t sj = __shfl_sync(0xffffffffu, start, j);
      const uint64_t lj = __shfl_sync(0xffffffffu, len, j);
      const uint32_t c = warp_crc32(a.data + sj + kHdr, lj, crc_tab, a.crc_table + kCrcTableWords, lane);
      if (lane == j && c != hw[10]) { status = RING_ECORRUPT; len = 0; deliver = false; }
    }
    if (in && ismsg) {
      ring_view_t* v = a.views + mi;
      RING_CHECK(mi < a.n && start % kAlign == 0 && start + f <= a.R && f >= kHdr, "received entry inside R", start, f);
      v->offset = start + kHdr;
      v->len = len;
      v->footprint = f;
      v->start = start;
      v->slot_seq = (ptr_seq(G) + lane) & kSeqMask;
      v->status = status;
      v->t_visible = tvis;
      v->reserved[0] = 0;
      v->reserved[1] = 0;
      int4* vh = reinterpret_cast<int4*>(v->header);
#pragma unroll
      for (int q = 0; q < 4; ++q) vh[q] = make_int4((int)hw[4 * q], (int)hw[4 * q + 1], (int)hw[4 * q + 2], (int)hw[4 * q + 3]);
    }
    const uint64_t fsum = warp_sum64(in ? f : 0);
    uint64_t G2b = ptr_off(G) + fsum;
    if (G2b >= a.R) G2b -= a.R;
    const uint64_t G2 = pack_ptr(G2b, ptr_seq(G) + e2);
    if (copy) {
      // ---- one item per entry; the copy warps move the payloads
      const uint32_t inmask = __ballot_sync(0xffffffffu, in);
      uint32_t flow_to = 0;
      if (lane == 0 && items + e2 - ld_acquire_gpu32(&S->pub_seq) > (uint32_t)kPlanRing) {
        const uint64_t end = globaltimer() + 2 * a.timeout_ns;
        while (items + e2 - ld_acquire_gpu32(&S->pub_seq) > (uint32_t)kPlanRing)
          if (globaltimer() > end) { flow_to = 1; break; }
      }
      // Plan slots still in use by the copy warps / finisher are never
      // overwritten: on a flow-control timeout the batch is left unread.
      if (__shfl_sync(0xffffffffu, flow_to, 0)) { fail = RING_ETIMEDOUT; break; }
      // remote buffer region: units on the payload's 128-B lines (copy_warp align_src)
      const uint32_t sh = a.remote_data ? (uint32_t)(reinterpret_cast<uintptr_t>(a.data + start + kHdr) & 127u) : 0u;
      uint32_t nu = (in && deliver && len) ? units_for(len + sh, a.chunk) : 0;
      uint32_t nu_incl = nu;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, nu_incl, o);
        if (lane >= o) nu_incl += y;
      }
      if (in) {
        const uint32_t item = items + __popc(inmask & lt_mask);
        Plan& p = ctx->plan[item % kPlanRing];
        p.src = reinterpret_cast<uint64_t>(a.data + start + kHdr);
        p.dst = reinterpret_cast<uint64_t>(a.dst + (uint64_t)mi * a.dst_stride);
        RING_CHECK(mi < a.n && (!deliver || len <= a.dst_stride), "copy-out inside dst", mi, len);
        p.len = deliver ? len : 0;
        p.nunits = nu;
        p.first_unit = units + nu_incl - nu;
        p.f = f;
        p.slot = (ptr_seq(G) + lane) & kSeqMask;
        p.flags = a.consume ? kRelease : 0u;
      }
      items += e2;
      units += __shfl_sync(0xffffffffu, nu_incl, 31);
      __syncwarp();
      if (lane == 0) {
        st_release<false>(&S->planned, make_planned(items, units));
        if (a.trace) {
          const uint32_t k = atomicAdd(reinterpret_cast<unsigned int*>(a.trace + 1023), 1u) % 255;
          a.trace[2 * k] = globaltimer();
          a.trace[2 * k + 1] = items;
        }
      }
    }
    // ---- steps 4-5 (no copy-out): clear busy bits, move the head past the batch
    const uint32_t first_msg = msgmask ? (uint32_t)__ffs(msgmask) - 1 : 32u;
    if (inline_release) {
      if (in) st_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(G) + lane), 0ull);
      H = G2;
      pending = 1;
    } else if (!a.consume && G == H) {
      // nothing held: PAD entries in front of the first message are released at
      // once so that a producer waiting for their space can proceed (R3)
      const bool lead_pad = in && (uint32_t)lane < first_msg;
      const uint32_t nlead = min(first_msg, e2);
      if (nlead) {
        if (lead_pad) st_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(G) + lane), 0ull);
        const uint64_t padsum = warp_sum64(lead_pad ? f : 0);
        uint64_t hb = ptr_off(H) + padsum;
        if (hb >= a.R) hb -= a.R;
        H = pack_ptr(hb, ptr_seq(H) + nlead);
        pending = 1;
      }
    }
    __syncwarp();
    if (inline_release && lane == 0 && pending) {
      publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H);
      pending = 0;
    }
    pending = __shfl_sync(0xffffffffu, pending, 0);
    G = G2;
    k += __popc(msgmask & ((e2 >= 32) ? 0xffffffffu : ((1u << e2) - 1u)));
  }
  // views of messages not received (RING_TRY: EMPTY; timeout)
  for (uint32_t q = k + lane; q < a.n; q += 32) {
    ring_view_t* v = a.views + q;
    v->offset = 0; v->len = 0; v->footprint = 0; v->start = 0; v->slot_seq = 0;
    v->status = fail; v->t_visible = 0;
  }
  __syncwarp();
  if (lane == 0) {
    *g_cursor(a.ring) = G;
    if (pending) publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H);
    if (copy) st_release<false>(&S->planned, make_planned(items, units) | kPlannedDone);
  }
}

// Copy-out mode: releases entries (consume) in order once their copies are done.
template <bool SYS>
__device__ void get_finisher(const GetArgs& a, LaunchCtx* ctx, LaunchSet* S) {
  const int lane = threadIdx.x & 31;
  uint64_t H = ld_cg64(g_head(a.ring));
  uint32_t i = 0;
  uint64_t idle_since = 0;
  while (true) {
    uint32_t ps = 0, done = 0;
    if (lane == 0) {
      const uint64_t pl = ld_acquire<false>(&S->planned);
      ps = planned_items(pl);
      done = planned_done(pl);
    }
    __syncwarp();
    ps = __shfl_sync(0xffffffffu, ps, 0);
    done = __shfl_sync(0xffffffffu, done, 0);
    if (i >= ps && done) break;
    const uint32_t j = i + lane;
    bool ready = false;
    uint32_t flags = 0, nunits = 0, slot = 0;
    uint64_t f = 0;
    if (j < ps) {
      const Plan& p = ctx->plan[j % kPlanRing];
      flags = ld_cg32(&p.flags);
      nunits = ld_cg32(&p.nunits);
      slot = ld_cg32(&p.slot);
      f = ld_cg64(&p.f);
      ready = nunits == 0 || ld_acquire_gpu32(&S->arrive[j % kPlanRing]) == nunits;
    }
    const uint32_t notready = __ballot_sync(0xffffffffu, !ready);
    const uint32_t run = notready ? __ffs(notready) - 1 : 32;
    if (run == 0) {
      const uint64_t t = globaltimer();
      if (!idle_since) idle_since = t;
      else if (t - idle_since > 2 * a.timeout_ns) break;
      continue;
    }
    idle_since = 0;
    const bool rel = (uint32_t)lane < run && (flags & kRelease);
    if ((uint32_t)lane < run && nunits) S->arrive[j % kPlanRing] = 0;
    if (rel) st_relaxed<SYS>(g_slot(a.ring, a.N, slot), 0ull);
    const uint32_t nrel = __popc(__ballot_sync(0xffffffffu, rel));
    const uint64_t fsum = warp_sum64(rel ? f : 0);
    __syncwarp();
    if (nrel) {
      uint64_t hb = ptr_off(H) + fsum;
      if (hb >= a.R) hb -= a.R;
      H = pack_ptr(hb, ptr_seq(H) + nrel);
      if (lane == 0) {
        publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H);
        if (a.trace) {
          const uint32_t k = atomicAdd(reinterpret_cast<unsigned int*>(a.trace + 1022), 1u) % 255;
          a.trace[512 + 2 * k] = globaltimer();
          a.trace[512 + 2 * k + 1] = i + run;
        }
      }
    }
    i += run;
    if (lane == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&S->pub_seq), "r"(i) : "memory");
  }
}

template <bool SYS>
__device__ void release_held(uint8_t* ring, uint64_t** mirrors, uint32_t n_mirrors, uint64_t R, uint32_t N,
                             uint32_t count);

template <bool SYS>
__global__ void __maxnreg__(120) get_kernel(const GetArgs a) {
  LaunchCtx* ctx = a.ctx;
  LaunchSet* S = &ctx->set[a.launch & 1];
  const int warp = threadIdx.x >> 5;
  __shared__ uint32_t s_crc[kCrcTableWords];
  __shared__ CopyShared cs;
  if (threadIdx.x == 0) {
    // ring_consume after a ring_get that left entries held: release them
    // first (in order), so the head stays on entry boundaries; the control
    // and finisher warps read the head after the CTA barrier below.
    if (blockIdx.x == 0 && a.consume && *g_cursor(a.ring) != *g_head(a.ring))
      release_held<SYS>(a.ring, a.mirrors, a.n_mirrors, a.R, a.N, 0xffffffffu);
    cs.pl = 0;
    cs.owner = 0;
    if (a.dst) cs.first = atomicAdd(&S->next_unit, (blockDim.x >> 5) - (blockIdx.x == 0 ? 2u : 0u));
  }
  if (blockIdx.x == 0) {
    load_crc_table(s_crc, a.crc_table);   // (its __syncthreads also covers cs)
    if (warp == 0) {
      reset_set(&ctx->set[(a.launch + 1) & 1], threadIdx.x & 31);
      get_control<SYS>(a, ctx, S, s_crc);
      return;
    }
    if (warp == 1) {
      if (a.dst) get_finisher<SYS>(a, ctx, S);
      return;
    }
  }
  if (blockIdx.x != 0) __syncthreads();
  if (a.dst) copy_warp<3>(ctx, S, &cs, a.chunk, a.timeout_ns, nullptr, nullptr, a.remote_data != 0);
}

// In-order release of `count` received entries plus the PAD entries the read
// cursor has passed (R13): receiver steps 4-5.  One thread.
template <bool SYS>
__device__ void release_held(uint8_t* ring, uint64_t** mirrors, uint32_t n_mirrors, uint64_t R, uint32_t N,
                             uint32_t count) {
  uint64_t H = *g_head(ring);
  const uint64_t G = *g_cursor(ring);
  bool moved = false;
  while (ptr_seq(H) != ptr_seq(G)) {
    const uint64_t w = ld_relaxed<SYS>(g_slot(ring, N, ptr_seq(H)));
    if (!(w & kPad)) {
      if (count == 0) break;
      --count;
    }
    st_relaxed<SYS>(g_slot(ring, N, ptr_seq(H)), 0ull);
    // footprint bits 0-39: a fault-tolerant ring's slots carry a tag above (R21)
    H = pack_ptr(advance(ptr_off(H), w & kFLow, R), seq_inc(ptr_seq(H)));
    moved = true;
  }
  if (moved) publish_head<SYS>(ring, mirrors, n_mirrors, H);
}

template <bool SYS>
__global__ void release_kernel(const ReleaseArgs a) {
  if (threadIdx.x != 0) return;
  release_held<SYS>(a.ring, a.mirrors, a.n_mirrors, a.R, a.N, a.count);
}

cudaError_t preload_get() {   // see preload_put (put.cu)
  cudaError_t e = preload_kernel(get_kernel<true>);
  if (e == cudaSuccess) e = preload_kernel(get_kernel<false>);
  if (e == cudaSuccess) e = preload_kernel(release_kernel<true>);
  if (e == cudaSuccess) e = preload_kernel(release_kernel<false>);
  return e;
}

cudaError_t launch_get(const GetArgs& a, uint32_t ctas, uint32_t threads, cudaStream_t s) {
  const uint32_t grid = a.dst ? ctas : 1;
  const uint32_t thr = a.dst ? threads : 32;
  if (a.sys) get_kernel<true><<<grid, thr, 0, s>>>(a);
  else get_kernel<false><<<grid, thr, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_release(const ReleaseArgs& a, cudaStream_t s) {
  if (a.sys) release_kernel<true><<<1, 32, 0, s>>>(a);
  else release_kernel<false><<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace b200ring
