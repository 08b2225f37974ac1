// put.cu — the sender side of the double ring (sender steps
// 1-8) as one persistent kernel per batch of messages.
//
// Grid = 1 control CTA + `copy_ctas` copy CTAs.
//   control CTA warp 0 ("leader", steps 1-4 + header): for each message, in
//     order: Lock (MPSC only, R14), read the tail, GH stale-slot check (R6),
//     space check with the interval rule (R4), PAD entry at the wrap (R3),
//     wait for credit (R12), build the 64-B header and its CRC-32 (R10/R11);
//     then hand the placement to the copy CTAs through LaunchCtx::plan[].
//   copy CTAs (step 5, WB): copy header + payload into the (peer) ring.
//   control CTA warp 1 ("publisher", steps 6-8): when all copy CTAs of an
//     entry arrived, write the size slot busy|f (WL), release-store the tail
//     (UH) and, MPSC, release the lock (Unlock).
// The leader runs ahead of the publisher by up to kPlanRing items, so the copy
// of message k+1 overlaps the publish (MEMBAR.SYS, ~1.7 us) of message k.
//
// Every message k owns two items: 2k (a PAD entry, or nothing) and 2k+1 (the
// message, or only its status).  The PAD item is published before the leader
// waits for credit for the message, as the oracle's WLpad/UHpad do, so a
// consumer can free the PAD while the producer waits (R3).
#include "ring_copy.cuh"

namespace b200ring {

__device__ __forceinline__ uint64_t* lock_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kLockOff); }
__device__ __forceinline__ uint64_t* tail_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kTailOff); }
__device__ __forceinline__ uint64_t* head_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kHeadOff); }
__device__ __forceinline__ uint64_t* slot_w(const DestDesc& d, uint32_t q) {
  return reinterpret_cast<uint64_t*>(d.ring + kSlotsOff) + (q & (d.N - 1));
}

template <bool SYS>
__device__ __forceinline__ uint64_t read_head(const DestDesc& d) {
  // The credit: the consumer's head, from the local mirror it pushes to us
  // (R1) or, if no mirror is bound, from the ring header over NVLink.
  const uint64_t m = ld_acquire<SYS>(&d.st->mirror_head);
  return (m & kMirrorValid) ? (m & ~kMirrorValid) : ld_acquire<SYS>(head_w(d));
}
__device__ __forceinline__ uint64_t read_head_rt(const DestDesc& d) {
  return d.sys ? read_head<true>(d) : read_head<false>(d);
}

// Header word i (i = 0..15) of the 64-byte entry header (R11); word 0 (CRC)
// and 14/15 (t_put) are filled by the caller.
__device__ __forceinline__ uint32_t header_word(int i, const ring_msg_t& m, uint32_t producer_id, uint32_t seq,
                                                uint32_t epoch) {
  const uint32_t* uid = reinterpret_cast<const uint32_t*>(m.hdr.uid);
  const uint32_t len = (uint32_t)m.len;
  switch (i) {
    case 1: return uid[0];
    case 2: return uid[1];
    case 3: return uid[2];
    case 4: return uid[3];
    case 5: return (uint32_t)m.hdr.accepted_at;
    case 6: return (uint32_t)(m.hdr.accepted_at >> 32);
    case 7: return m.hdr.app_id;
    case 8: return (uint32_t)m.hdr.stage | (len << 16);   // stage[32,34) payload_len[34,36)
    case 9: return len >> 16;                             // payload_len[36,38) reserved[38,40)
    case 10: return 0;                                    // reserved[40,44)
    case 11: return producer_id;
    case 12: return seq;
    case 13: return epoch & 0xffffu;                      // epoch[52,54) flags[54,56)
    default: return 0;
  }
}

struct LeaderOut {     // lane 0's decisions, broadcast to the warp through shared memory
  uint64_t start, f, pad_word, tail_after_pad, tail_after;
  uint32_t pad_slot, slot, status, has_pad, has_msg, unlock, dest, seq, epoch;
};

__device__ void put_leader(const PutArgs& a) {
  const int lane = threadIdx.x & 31;
  LaunchCtx* ctx = a.ctx;
  __shared__ LeaderOut lo;
  // lane 0 state: per destination running tail (SPSC) and channel counters
  uint64_t tails[kMaxRouterDests];
  uint64_t chans[kMaxRouterDests];
  uint32_t loaded = 0;
  uint32_t cta_rot = 0;    // rotates the copy CTAs over consecutive entries
  bool aborted = false;
  if (lane == 0) {         // resynchronise the plan ring (an aborted launch may have left it mid-way)
    for (int i = 0; i < kPlanRing; ++i) ctx->arrive[i] = 0;
    ctx->pub_seq = 2 * a.base;
    st_release_gpu64(&ctx->plan_seq, 2 * a.base);
  }
  __syncwarp();

  for (uint32_t k = 0; k < a.n; ++k) {
    const uint64_t item0 = 2 * (a.base + k), item1 = item0 + 1;
    const ring_msg_t m = a.msgs ? a.msgs[k] : a.inline_msg;
    if (lane == 0) {
      // flow control: both items of message k must fit in the plan ring
      if (item1 - ld_acquire_gpu64(&ctx->pub_seq) >= (uint64_t)kPlanRing) {
        const uint64_t end = globaltimer() + 2 * a.timeout_ns;
        while (item1 - ld_acquire_gpu64(&ctx->pub_seq) >= (uint64_t)kPlanRing)
          if (globaltimer() > end) { aborted = true; break; }
      }
      LeaderOut o = {};
      o.status = RING_OK;
      // ---- stage router: pick the destination (PAPER.md:531-532 round-robin)
      uint32_t d = 0, epoch = 0;
      if (a.routes) {
        int hit = -1;
        for (uint32_t r = 0; r < a.n_routes; ++r)
          if (a.routes[r].n && a.routes[r].app_id == m.hdr.app_id && a.routes[r].stage == m.hdr.stage) { hit = (int)r; break; }
        if (hit < 0) {
          o.status = RING_EINVAL;
        } else {
          Route& rt = a.routes[hit];
          d = rt.dests[rt.rr % rt.n];
          rt.rr = rt.rr + 1;
          epoch = rt.epoch;
        }
      }
      o.dest = d;
      o.epoch = epoch;
      const DestDesc D = a.dests[d];
      if (!(loaded & (1u << d))) {
        loaded |= 1u << d;
        tails[d] = D.st->tail_cache;
        chans[d] = D.st->chan_seq;
      }
      o.seq = (uint32_t)chans[d];
      chans[d] += 1;
      const uint64_t f = footprint(m.len);
      o.f = f;
      if (aborted) o.status = RING_ETIMEDOUT;
      else if (o.status == RING_OK && (m.len >= (1ull << 32) || f > D.R)) o.status = RING_EMSGSIZE;

      bool locked = false;
      uint64_t P = tails[d];
      if (o.status == RING_OK && D.mpsc) {
        // Step 1 "Acquire the lock using a CAS-based spinlock".
        // Our previous items (and their Unlock) must have been published first.
        const uint64_t end = globaltimer() + a.timeout_ns;
        while (ld_acquire_gpu64(&ctx->pub_seq) != item0)
          if (globaltimer() > end) { o.status = RING_ETIMEDOUT; break; }
        if (o.status == RING_OK) {
          const uint64_t me = (uint64_t)D.producer_id + 1;
          while (true) {
            const uint64_t old = D.sys ? cas_acquire<true>(lock_w(D), 0ull, me) : cas_acquire<false>(lock_w(D), 0ull, me);
            if (old == 0) { locked = true; break; }
            if (globaltimer() > end) { o.status = RING_ETIMEDOUT; break; }
          }
        }
        if (locked) {
          // Step 2: read the tail (ordered after the acquiring CAS).
          P = D.sys ? ld_relaxed<true>(tail_w(D)) : ld_relaxed<false>(tail_w(D));
          // Step 4 (R6: before the space check): a busy slot at P_seq with the
          // size ring not full means a lost sender committed WB+WL but not UH
          // (Case 7): advance the header past it before writing.
          // The head is read before the slot: a slot the consumer has released
          // is then seen cleared (it clears the slot before moving the head).
          while (true) {
            const uint64_t H = read_head_rt(D);
            if (seq_dist(ptr_seq(P), ptr_seq(H)) >= D.N) break;
            const uint64_t w = D.sys ? ld_relaxed<true>(slot_w(D, ptr_seq(P))) : ld_relaxed<false>(slot_w(D, ptr_seq(P)));
            if (!(w & kBusy)) break;
            P = pack_ptr(advance(ptr_off(P), w & kFMask, D.R), seq_inc(ptr_seq(P)));
            if (D.sys) st_release<true>(tail_w(D), P); else st_release<false>(tail_w(D), P);
          }
        }
      }
      // Step 3: space check (R4) with the PAD entry at the wrap (R3), waiting
      // for credit in BLOCK mode (R12).
      if (o.status == RING_OK) {
        uint64_t H = read_head_rt(D);
        const uint64_t end = globaltimer() + a.timeout_ns;
        bool pad_done = false;
        while (true) {
          const uint64_t pb = ptr_off(P), hb = ptr_off(H);
          const uint32_t pq = ptr_seq(P), hq = ptr_seq(H);
          bool full = seq_dist(pq, hq) >= D.N;
          if (!full && pb + f > D.R) {
            if (!pad_done && span_free(pb, pq, hb, hq, D.R - pb)) {
              o.has_pad = 1;
              o.pad_slot = pq;
              o.pad_word = kBusy | kPad | (D.R - pb);
              P = pack_ptr(0, seq_inc(pq));
              o.tail_after_pad = P;
              pad_done = true;
              // Publish the PAD now (item 0) before waiting for the message.
              Plan& pp = ctx->plan[item0 % kPlanRing];
              pp.cnt = 0; pp.len = 0; pp.hdr_dst = 0; pp.dest = d;
              pp.pad_word = o.pad_word; pp.pad_slot = o.pad_slot; pp.tail_after = P;
              pp.flags = kPublish; pp.status = RING_OK;
              st_release_gpu64(&ctx->plan_seq, item0 + 1);
              continue;
            }
            full = true;
          } else if (!full && !span_free(pb, pq, hb, hq, f)) {
            full = true;
          }
          if (!full) {
            o.start = pb;
            o.slot = pq;
            o.has_msg = 1;
            P = pack_ptr(advance(pb, f, D.R), seq_inc(pq));
            o.tail_after = P;
            break;
          }
          if (a.flags & RING_TRY) { o.status = RING_FULL; break; }   // "release the lock and abort"
          // wait until the consumer moves the head
          uint64_t H2 = read_head_rt(D);
          while (H2 == H) {
            if (globaltimer() > end) break;
            H2 = read_head_rt(D);
          }
          if (H2 == H) { o.status = RING_ETIMEDOUT; break; }
          H = H2;
        }
        if (o.has_pad == 0) {
          Plan& pp = ctx->plan[item0 % kPlanRing];
          pp.cnt = 0; pp.len = 0; pp.hdr_dst = 0; pp.dest = d; pp.pad_word = 0; pp.flags = 0; pp.status = RING_OK;
          st_release_gpu64(&ctx->plan_seq, item0 + 1);
        }
      } else {
        Plan& pp = ctx->plan[item0 % kPlanRing];
        pp.cnt = 0; pp.len = 0; pp.hdr_dst = 0; pp.dest = d; pp.pad_word = 0; pp.flags = 0; pp.status = RING_OK;
        st_release_gpu64(&ctx->plan_seq, item0 + 1);
      }
      tails[d] = P;
      if (o.status == RING_ETIMEDOUT) aborted = true;
      o.unlock = locked ? 1u : 0u;
      lo = o;
    }
    __syncwarp();
    const LeaderOut o = lo;
    __syncwarp();
    // ---- header (step 5 payload framing) + CRC-32 over bytes [4,56) (R10),
    // computed by the whole warp.
    Plan& p = ctx->plan[item1 % kPlanRing];
    if (o.has_msg) {
      const DestDesc& D = a.dests[o.dest];
      const uint32_t w_mine = header_word(lane, m, D.producer_id, o.seq, o.epoch);
      const uint32_t w_crc = header_word(lane + 1, m, D.producer_id, o.seq, o.epoch);
      const uint32_t crc = warp_crc52(w_crc, lane, a.crc_table);
      if (lane < 16) {
        uint32_t w = w_mine;
        if (lane == 0) w = crc;
        if (lane == 14 || lane == 15) {
          const uint64_t t = (a.flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
          w = lane == 14 ? (uint32_t)t : (uint32_t)(t >> 32);
        }
        p.hdr[lane] = w;
      }
      if (lane == 0) {
        p.src = m.src;
        p.dst = reinterpret_cast<uint64_t>(D.data + o.start + kHdr);
        p.len = m.len;
        p.hdr_dst = reinterpret_cast<uint64_t>(D.data + o.start);
        p.cnt = ctas_for(m.len, a.copy_ctas, a.chunk_min);
        p.cta_base = cta_rot;
        cta_rot = (cta_rot + p.cnt) % a.copy_ctas;
        p.start = o.start;
        p.f = o.f;
        p.slot = o.slot;
        p.pad_word = 0;
        p.tail_after = o.tail_after;
        p.flags = kHasMsg | kPublish | (o.unlock ? kUnlock : 0);
      }
    } else if (lane == 0) {
      p.cnt = 0; p.len = 0; p.hdr_dst = 0; p.pad_word = 0;
      p.flags = o.unlock ? kUnlock : 0;
    }
    if (lane == 0) {
      p.dest = o.dest;
      p.status = o.status;
      if (a.dest_out) a.dest_out[k] = o.dest;
    }
    __syncwarp();
    if (lane == 0) st_release_gpu64(&ctx->plan_seq, item1 + 1);
  }
  if (lane == 0) {
    for (uint32_t d = 0; d < kMaxRouterDests && d < a.n_dests; ++d)
      if (loaded & (1u << d)) {
        a.dests[d].st->chan_seq = chans[d];
        if (!a.dests[d].mpsc) a.dests[d].st->tail_cache = tails[d];
      }
  }
}

// Steps 6-8 (WL, UH, Unlock) in item order.
__device__ void put_publisher(const PutArgs& a) {
  if ((threadIdx.x & 31) != 0) return;
  LaunchCtx* ctx = a.ctx;
  const uint64_t first = 2 * a.base, last = 2 * (a.base + a.n);
  for (uint64_t i = first; i < last; ++i) {
    if (ld_acquire_gpu64(&ctx->plan_seq) <= i) {
      const uint64_t end = globaltimer() + 2 * a.timeout_ns;
      bool ab = false;
      while (ld_acquire_gpu64(&ctx->plan_seq) <= i)
        if (globaltimer() > end) { ab = true; break; }
      if (ab) return;
    }
    Plan& p = ctx->plan[i % kPlanRing];
    const uint32_t cnt = p.cnt, flags = p.flags;
    if (cnt) {
      if (ld_acquire_gpu32(&ctx->arrive[i % kPlanRing]) != cnt) {
        const uint64_t end = globaltimer() + 2 * a.timeout_ns;
        bool ab = false;
        while (ld_acquire_gpu32(&ctx->arrive[i % kPlanRing]) != cnt)
          if (globaltimer() > end) { ab = true; break; }
        if (ab) return;
      }
      ctx->arrive[i % kPlanRing] = 0;
    }
    const DestDesc& D = a.dests[p.dest];
    if (D.sys) {
      if (p.pad_word) st_relaxed<true>(slot_w(D, p.pad_slot), p.pad_word);            // WL of the PAD entry
      if (flags & kHasMsg) st_relaxed<true>(slot_w(D, p.slot), kBusy | p.f);           // WL: size + busy bit
      if (flags & kPublish) st_release<true>(tail_w(D), p.tail_after);                  // UH
      if (flags & kUnlock) st_release<true>(lock_w(D), 0ull);                           // Unlock
    } else {
      if (p.pad_word) st_relaxed<false>(slot_w(D, p.pad_slot), p.pad_word);
      if (flags & kHasMsg) st_relaxed<false>(slot_w(D, p.slot), kBusy | p.f);
      if (flags & kPublish) st_release<false>(tail_w(D), p.tail_after);
      if (flags & kUnlock) st_release<false>(lock_w(D), 0ull);
    }
    if (i & 1) a.status[(i - first) >> 1] = p.status;
    st_release_gpu64(&ctx->pub_seq, i + 1);
  }
}

__global__ void __launch_bounds__(1024, 1) put_kernel(const PutArgs a) {
  if (blockIdx.x == 0) {
    const int warp = threadIdx.x >> 5;
    if (warp == 0) put_leader(a);
    else if (warp == 1) put_publisher(a);
    return;
  }
  copy_worker(a.ctx, 2 * a.base, 2ull * a.n, blockIdx.x - 1, a.copy_ctas, a.timeout_ns);
}

cudaError_t launch_put(const PutArgs& a, uint32_t threads, cudaStream_t s) {
  put_kernel<<<a.copy_ctas + 1, threads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace b200ring
