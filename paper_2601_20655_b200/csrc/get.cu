// get.cu — the receiver side of the double ring (receiver
// steps 1-5) and the in-order release (R13).
//
// get_kernel grid = 1 control CTA (+ copy CTAs when copying out).
//   control CTA warp 0: for each entry, in order: poll the tail until its
//     sequence differs from the read cursor G (steps 1-2, R7; wait-free for
//     the producers), read the size slot (a PAD entry is stepped
//     over with its size metadata, R3), read the 64-B header and verify its
//     CRC-32 (step 3 + PAPER.md:768-769), write the view record.  When
//     consuming without copy-out it also clears the busy bit and moves the head
//     (steps 4-5) and pushes the head to the producers' mirrors (credit, R1),
//     one system-scope fence per batch of releases.
//   copy CTAs + control CTA warp 1 ("finisher"), copy-out only: copy payloads
//     to the user buffer; the finisher releases each entry (consume) once its
//     copy is complete, in order.
#include "ring_copy.cuh"

namespace b200ring {

__device__ __forceinline__ uint64_t* g_tail(const GetArgs& a) { return reinterpret_cast<uint64_t*>(a.ring + kTailOff); }
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
  for (uint32_t i = 0; i < n_mirrors; ++i)
    if (mirrors[i]) st_relaxed<SYS>(mirrors[i], H | kMirrorValid);
}

struct CtlOut {
  uint64_t start, f, t_vis;
  uint32_t status, slot_seq, pad_item;  // pad_item: a PAD item was emitted for this entry
};

template <bool SYS>
__device__ void get_control(const GetArgs& a) {
  const int lane = threadIdx.x & 31;
  __shared__ CtlOut co;
  const bool copy = a.dst != nullptr;
  const bool inline_release = a.consume && !copy;
  LaunchCtx* ctx = a.ctx;
  uint64_t G = 0, H = 0;
  uint32_t pending = 0, cta_rot = 0;
  bool aborted = false, empty = false;
  if (lane == 0) {
    G = *g_cursor(a.ring);
    H = *g_head(a.ring);
    if (copy) {            // resynchronise the plan ring
      for (int i = 0; i < kPlanRing; ++i) ctx->arrive[i] = 0;
      ctx->pub_seq = 2 * a.base;
      st_release_gpu64(&ctx->plan_seq, 2 * a.base);
    }
  }
  __syncwarp();
  for (uint32_t k = 0; k < a.n; ++k) {
    const uint64_t item0 = 2 * (a.base + k), item1 = item0 + 1;
    if (lane == 0) {
      CtlOut o = {};
      o.status = RING_OK;
      if (copy && item1 - ld_acquire_gpu64(&ctx->pub_seq) >= (uint64_t)kPlanRing) {
        const uint64_t end = globaltimer() + 2 * a.timeout_ns;
        while (item1 - ld_acquire_gpu64(&ctx->pub_seq) >= (uint64_t)kPlanRing)
          if (globaltimer() > end) { aborted = true; break; }
      }
      while (true) {
        if (aborted) { o.status = RING_ETIMEDOUT; break; }
        if (empty) { o.status = RING_EMPTY; break; }
        // Steps 1-2: "Read the current head position ... If no new data is
        // available, wait ... and retry" -- new data = tail seq != G seq (R7).
        uint64_t T = ld_acquire<SYS>(g_tail(a));
        if (ptr_seq(T) == ptr_seq(G)) {
          if (pending) { publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H); pending = 0; }
          if (a.flags & RING_TRY) { empty = true; continue; }
          const uint64_t end = globaltimer() + a.timeout_ns;
          do {
            T = ld_acquire<SYS>(g_tail(a));
            if (globaltimer() > end) break;
          } while (ptr_seq(T) == ptr_seq(G));
          if (ptr_seq(T) == ptr_seq(G)) { aborted = true; continue; }
        }
        o.t_vis = (a.flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
        const uint64_t w = ld_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(G)));
        const uint64_t f = w & kFMask;
        if (w & kPad) {
          // Step over a PAD entry using its size (R3).
          const uint64_t G2 = pack_ptr(advance(ptr_off(G), f, a.R), seq_inc(ptr_seq(G)));
          if (inline_release || (!a.consume && G == H)) {
            // nothing held: release it at once so a producer waiting for this
            // space can proceed
            st_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(G)), 0ull);
            H = G2;
            pending++;
          } else if (a.consume) {
            Plan& pp = ctx->plan[item0 % kPlanRing];     // the finisher frees it in order
            pp.cnt = 0; pp.len = 0; pp.hdr_dst = 0; pp.f = f; pp.flags = kRelease;
            st_release_gpu64(&ctx->plan_seq, item0 + 1);
            o.pad_item = 1;
          }
          G = G2;
          continue;
        }
        o.start = ptr_off(G);
        o.f = f;
        o.slot_seq = ptr_seq(G);
        break;
      }
      co = o;
    }
    __syncwarp();
    const CtlOut o = co;
    __syncwarp();
    ring_view_t* v = a.views + k;
    // Step 3: read the entry header and verify the checksum.
    uint32_t hw = 0;
    if (o.status == RING_OK && lane < 16) hw = __ldcg(reinterpret_cast<const uint32_t*>(a.data + o.start) + lane);
    const uint32_t hw_next = __shfl_down_sync(0xffffffffu, hw, 1);
    const uint32_t crc = warp_crc52(hw_next, lane, a.crc_table);
    const uint32_t w0 = __shfl_sync(0xffffffffu, hw, 0);
    const uint32_t w8 = __shfl_sync(0xffffffffu, hw, 8);
    const uint32_t w9 = __shfl_sync(0xffffffffu, hw, 9);
    const uint64_t len = (w8 >> 16) | ((w9 & 0xffffu) << 16);
    uint32_t status = o.status;
    bool deliver = false;
    if (status == RING_OK) {
      if (crc != w0 || kHdr + len > o.f) status = RING_ECORRUPT;   // discarded, still consumed
      else if (copy && len > a.dst_stride) status = RING_EMSGSIZE;
      else deliver = true;
    }
    if (lane < 16) reinterpret_cast<uint32_t*>(v->header)[lane] = hw;
    if (lane == 0) {
      v->offset = o.start + kHdr;
      v->len = (deliver || status == RING_EMSGSIZE) ? len : 0;
      v->footprint = o.f;
      v->start = o.start;
      v->slot_seq = o.slot_seq;
      v->status = status;
      v->t_visible = o.t_vis;
      v->reserved[0] = 0;
      v->reserved[1] = 0;
      const bool have_entry = o.status == RING_OK;
      if (copy) {
        if (!o.pad_item) {
          Plan& pp = ctx->plan[item0 % kPlanRing];
          pp.cnt = 0; pp.len = 0; pp.hdr_dst = 0; pp.f = 0; pp.flags = 0;
          st_release_gpu64(&ctx->plan_seq, item0 + 1);
        }
        Plan& p = ctx->plan[item1 % kPlanRing];
        p.src = reinterpret_cast<uint64_t>(a.data + o.start + kHdr);
        p.dst = reinterpret_cast<uint64_t>(a.dst + (uint64_t)k * a.dst_stride);
        p.len = deliver ? len : 0;
        p.hdr_dst = 0;
        p.cnt = deliver ? ctas_for(len, a.copy_ctas, a.chunk_min) : 0;
        p.cta_base = cta_rot;
        cta_rot = (cta_rot + p.cnt) % a.copy_ctas;
        p.f = o.f;
        p.flags = (a.consume && have_entry) ? kRelease : 0;
        st_release_gpu64(&ctx->plan_seq, item1 + 1);
      }
      if (have_entry) {
        G = pack_ptr(advance(o.start, o.f, a.R), seq_inc(o.slot_seq));
        if (inline_release) {
          // Steps 4-5: "Reset the busy bit", "Update the head position".
          st_relaxed<SYS>(g_slot(a.ring, a.N, o.slot_seq), 0ull);
          H = G;
          if (++pending >= 8) { publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H); pending = 0; }
        }
      }
    }
  }
  if (lane == 0) {
    *g_cursor(a.ring) = G;
    if (pending) publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H);
  }
}

// Copy-out mode: waits for each item's copy CTAs, then (consume) releases the
// entry in order: clear the busy bit, advance the head (steps 4-5).
template <bool SYS>
__device__ void get_finisher(const GetArgs& a) {
  if ((threadIdx.x & 31) != 0) return;
  LaunchCtx* ctx = a.ctx;
  uint64_t H = *g_head(a.ring);
  uint32_t pending = 0;
  const uint64_t first = 2 * a.base, last = 2 * (a.base + a.n);
  for (uint64_t i = first; i < last; ++i) {
    if (ld_acquire_gpu64(&ctx->plan_seq) <= i) {
      if (pending) { publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H); pending = 0; }
      const uint64_t end = globaltimer() + 2 * a.timeout_ns;
      bool ab = false;
      while (ld_acquire_gpu64(&ctx->plan_seq) <= i)
        if (globaltimer() > end) { ab = true; break; }
      if (ab) break;
    }
    Plan& p = ctx->plan[i % kPlanRing];
    const uint32_t cnt = p.cnt, flags = p.flags;
    const uint64_t f = p.f;
    if (cnt) {
      const uint64_t end = globaltimer() + 2 * a.timeout_ns;
      bool ab = false;
      while (ld_acquire_gpu32(&ctx->arrive[i % kPlanRing]) != cnt)
        if (globaltimer() > end) { ab = true; break; }
      if (ab) break;
      ctx->arrive[i % kPlanRing] = 0;
    }
    if (flags & kRelease) {
      st_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(H)), 0ull);
      H = pack_ptr(advance(ptr_off(H), f, a.R), seq_inc(ptr_seq(H)));
      if (++pending >= 8) { publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H); pending = 0; }
    }
    st_release_gpu64(&ctx->pub_seq, i + 1);
  }
  if (pending) publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H);
}

template <bool SYS>
__global__ void __launch_bounds__(1024, 1) get_kernel(const GetArgs a) {
  if (blockIdx.x == 0) {
    const int warp = threadIdx.x >> 5;
    if (warp == 0) get_control<SYS>(a);
    else if (warp == 1 && a.dst) get_finisher<SYS>(a);
    return;
  }
  copy_worker(a.ctx, 2 * a.base, 2ull * a.n, blockIdx.x - 1, a.copy_ctas, a.timeout_ns);
}

// In-order release of `count` received entries plus the PAD entries the read
// cursor has passed (R13): receiver steps 4-5.
template <bool SYS>
__global__ void release_kernel(const ReleaseArgs a) {
  if (threadIdx.x != 0) return;
  uint64_t H = *g_head(a.ring);
  const uint64_t G = *g_cursor(a.ring);
  uint32_t count = a.count;
  bool moved = false;
  while (ptr_seq(H) != ptr_seq(G)) {
    const uint64_t w = ld_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(H)));
    if (!(w & kPad)) {
      if (count == 0) break;
      --count;
    }
    st_relaxed<SYS>(g_slot(a.ring, a.N, ptr_seq(H)), 0ull);
    H = pack_ptr(advance(ptr_off(H), w & kFMask, a.R), seq_inc(ptr_seq(H)));
    moved = true;
  }
  if (moved) publish_head<SYS>(a.ring, a.mirrors, a.n_mirrors, H);
}

cudaError_t launch_get(const GetArgs& a, uint32_t threads, cudaStream_t s) {
  const uint32_t grid = a.dst ? a.copy_ctas + 1 : 1;
  const uint32_t thr = a.dst ? threads : 64;
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
