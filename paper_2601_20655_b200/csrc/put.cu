// put.cu — the sender side of the double ring (sender steps
// 1-8) as one persistent kernel per batch of messages.
//
// Grid = `ctas` CTAs.  CTA 0 warp 0 is the leader, CTA 0 warp 1 the
// publisher; every other warp of the grid is a copy warp (ring_copy.cuh).
//   leader (steps 1-4 + framing): takes the batch 32 messages at a time, one
//     per lane.  Lane 0 places them in order: Lock (MPSC only, R14), read the
//     tail (SPSC: producer-local), GH stale-slot check (R6), space check with
//     the interval rule (R4) against the cached head, PAD entry at the wrap
//     (R3), waiting for credit only when nothing else is pending (R12).  Then
//     every lane writes its placement; one release hands the round's copies
//     out, then the lanes build the 64-B headers (R11) and CRC-32 (R10) into
//     the plans while the copies run (a second release, `hdr_seq`).
//   copy warps (step 5, WB): payload into the (peer) ring.
//   publisher (steps 5-8): lanes check 32 consecutive items at once; for the
//     leading run of complete items they write the headers (WB) and the size
//     slots busy|f (WL),
//     then lane 0 moves the tail with ONE system-scope release (UH) and, MPSC,
//     releases the lock (Unlock).  The fence (MEMBAR.SYS, ~1.7 us on B200) is
//     thus paid once per run of entries, and overlaps later copies.
// A PAD item is published before the leader waits for credit for the message
// that follows it (as the oracle's WLpad/UHpad do), so a consumer can free the
// PAD while the producer waits (R3).
#include "ring_copy.cuh"

namespace b200ring {

__device__ __forceinline__ uint64_t* lock_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kLockOff); }
__device__ __forceinline__ uint64_t* tail_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kTailOff); }
__device__ __forceinline__ uint64_t* head_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kHeadOff); }
__device__ __forceinline__ uint64_t* resv_w(const DestDesc& d) { return reinterpret_cast<uint64_t*>(d.ring + kResvOff); }
__device__ __forceinline__ uint64_t* slot_w(const DestDesc& d, uint32_t q) {
  return reinterpret_cast<uint64_t*>(d.ring + kSlotsOff) + (q & (d.N - 1));
}

// The credit: the consumer's head, from the local mirror it pushes to us (R1)
// or, while no mirror is bound, from the ring header over NVLink.
__device__ __forceinline__ uint64_t read_head(const DestDesc& d) {
  const uint64_t m = d.sys ? ld_acquire<true>(&d.st->mirror_head) : ld_acquire<false>(&d.st->mirror_head);
  if (m & kMirrorValid) return m & ~kMirrorValid;
  return d.sys ? ld_acquire<true>(head_w(d)) : ld_acquire<false>(head_w(d));
}

__device__ __forceinline__ uint64_t read_head_relaxed(const DestDesc& d) {
  const uint64_t m = d.sys ? ld_relaxed<true>(&d.st->mirror_head) : ld_relaxed<false>(&d.st->mirror_head);
  if (m & kMirrorValid) return m & ~kMirrorValid;
  return d.sys ? ld_relaxed<true>(head_w(d)) : ld_relaxed<false>(head_w(d));
}

__device__ __forceinline__ void st_u32_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_u32_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Per-message decisions of lane 0, read back by every lane.
struct GroupSlot {
  uint64_t start, tail_after;
  uint32_t item, dest, seq, epoch, status, slot, flags, first_unit, nunits, _p;
};

struct LeaderState {
  uint64_t tails[kMaxRouterDests];  // SPSC running tail per destination
  uint64_t heads[kMaxRouterDests];  // cached credit per destination
  uint64_t chans[kMaxRouterDests];  // channel counters (R18)
  uint32_t loaded;
  uint32_t items, units;
  bool aborted;
  bool dead;                        // fault injection (reserve-then-commit): the sender is lost
  bool flow_to;                     // plan-ring flow control timed out: plan slots may still be in use
  uint32_t nrounds;                 // rounds so far (debug timeline of an engine: the last 64 rounds)
  uint64_t me;                      // reserve-then-commit: this round's lock word
};

__device__ __forceinline__ void write_pad_plan(LaunchCtx* ctx, uint32_t item, uint32_t dest, uint32_t slot,
                                               uint64_t word, uint64_t tail_after) {
  Plan& p = ctx->plan[item % kPlanRing];
  p.len = 0; p.nunits = 0; p.first_unit = 0;
  p.slot_word = word; p.slot = slot; p.tail_after = tail_after; p.dest = dest;
  p.flags = kEntry; p.status = RING_OK; p.msg = 0;
}

// Lane 0: place messages [k0, k0 + gmax) of the batch; returns how many were
// decided (the rest wait for the next round).  Items are numbered in order.
struct MsgBrief {        // the fields lane 0 needs, computed in parallel by all lanes
  uint64_t len;
  uint64_t f;            // footprint (R9)
  uint32_t app_id;
  uint32_t stage;
  uint32_t nunits;       // copy work units
  uint32_t _p;
  uint64_t t_arr;        // arrival time (hdr.accepted_at): fast-reject admission
};

__device__ __forceinline__ uint64_t tagged_word(uint64_t w, uint32_t q) { return w | ((q & kTagMask) << kTagShift); }

template <bool SYS>
__device__ __forceinline__ uint64_t dcas(uint64_t* p, uint64_t cmp, uint64_t val) { return cas_acq_rel<SYS>(p, cmp, val); }
__device__ __forceinline__ uint64_t dcas(const DestDesc& D, uint64_t* p, uint64_t cmp, uint64_t val) {
  return D.sys ? dcas<true>(p, cmp, val) : dcas<false>(p, cmp, val);
}
__device__ __forceinline__ uint64_t dld(const DestDesc& D, const uint64_t* p) {
  return D.sys ? ld_acquire<true>(p) : ld_acquire<false>(p);
}

// ---- reserve-then-commit helpers (oracle/reserve.py) -------------------------
// Move the tail over the leading run of committed slots of [tail, resv)
// (serial; the publisher has a warp-parallel version).  Returns the tail.
__device__ uint64_t rc_help_advance(const DestDesc& D) {
  uint64_t T = dld(D, tail_w(D));
  while (true) {
    const uint64_t Rv = dld(D, resv_w(D)), H = read_head(D);
    const uint32_t tq = ptr_seq(T);
    if (tq == ptr_seq(Rv) || seq_dist(tq, ptr_seq(H)) >= D.N) return T;
    const uint64_t w = dld(D, slot_w(D, tq));
    if (!(w & kBusy)) return T;
    const uint64_t T2 = pack_ptr(advance(ptr_off(T), w & kFLow, D.R), seq_inc(tq));
    const uint64_t old = dcas(D, tail_w(D), T, T2);
    T = old == T ? T2 : old;
  }
}
// A reservation stuck at the tail: after it has been observed unchanged for
// the hole timeout (longer than any live sender's claim-to-commit time: a
// copy of the largest message) its sender is presumed lost and the slot becomes a PAD (reserved ->
// busy|pad, CAS) that the receiver skips.  `seen`/`since` carry the watch.
__device__ void rc_hole_watch(const PutArgs& a, const DestDesc& D, uint64_t& seen, uint64_t& since) {
  const uint64_t T = dld(D, tail_w(D));
  const uint64_t w = dld(D, slot_w(D, ptr_seq(T)));
  const uint64_t key = (w & kResvBit) ? (T ^ (w << 1)) | 1ull : 0ull;
  const uint64_t now = globaltimer();
  if (!key) { seen = 0; return; }
  if (key != seen) { seen = key; since = now; return; }
  if (now - since > a.hole_timeout_ns) {
    dcas(D, slot_w(D, ptr_seq(T)), w, kBusy | kPad | (w & kFLow));
    if (a.trace) atomicAdd(reinterpret_cast<unsigned long long*>(a.trace + 1891), 1ull);
    seen = 0;
  }
}
// The ring lock with take-over of a lost holder (same word for the hole
// timeout: a live holder's claims can take tens of microseconds when NVLink
// is saturated by copies, so the short TL would take over live holders).
__device__ bool rc_lock(const PutArgs& a, const DestDesc& D, uint64_t me, uint64_t t_start) {
  uint64_t seen = 0, seen_at = 0;
  while (true) {
    const uint64_t old = dcas(D, lock_w(D), 0ull, me);
    if (old == 0) return true;
    const uint64_t now = globaltimer();
    if (old != seen) { seen = old; seen_at = now; }
    else if (now - seen_at > a.hole_timeout_ns && dcas(D, lock_w(D), old, me) == old) {
      if (a.trace) atomicAdd(reinterpret_cast<unsigned long long*>(a.trace + 1890), 1ull);
      return true;
    }
    if (now - t_start > a.timeout_ns) return false;
  }
}

__device__ uint32_t leader_place(const PutArgs& a, uint32_t flags, LaunchCtx* ctx, LaunchSet* S, LeaderState& L, uint32_t k0,
                                 uint32_t gmax, GroupSlot* gs, const MsgBrief* brief, const DestDesc* dests) {
  (void)k0;
  // MPSC: the lock taken for the round's first message is kept for the
  // following messages to the same ring and released after the round's last
  // item (lock coarsening).  Equivalent to the oracle schedule in which the
  // producer re-acquires the lock right after each Unlock.
  int held = -1;
  uint32_t done_l = gmax;
  uint32_t last_pad = 0xffffffffu;
  for (uint32_t l = 0; l < gmax; ++l) {
    if (a.trace && k0 == 0 && l < 32) a.trace[128 + l] = globaltimer();
    const MsgBrief& m = brief[l];
    GroupSlot o = {};
    o.status = RING_OK;
    // ---- stage router (PAPER.md:531-532 round-robin; epoch = reassignment)
    uint32_t d = 0;
    int hit = -1;
    uint64_t adm_next = 0;   // admission state to commit with the message
    if (a.routes) {
      for (uint32_t r = 0; r < a.n_routes; ++r)
        if (a.routes[r].n && a.routes[r].app_id == m.app_id && a.routes[r].stage == m.stage) { hit = (int)r; break; }
      if (hit < 0) {
        o.status = RING_EINVAL;
      } else {
        Route& rt = a.routes[hit];
        d = rt.dests[rt.rr % rt.n];
        o.epoch = rt.epoch;
        // Request Monitor / fast reject: admitted iff the
        // arrival is not earlier than the next admissible time (rate K/T_X,
        // burst 1, the oracle's pipeline.fast_reject); rejected requests are
        // never sent and leave the round robin where it was.
        adm_next = rt.adm_next;
        if (rt.adm_k) {
          const uint64_t t = m.t_arr * rt.adm_k;
          if (t >= rt.adm_next) adm_next = max(rt.adm_next, t) + rt.adm_tx;
          else o.status = RING_EREJECTED;
        }
      }
    }
    const DestDesc D = dests[d];
    if (l > 0 && ((D.mpsc && held != (int)d) || (!D.mpsc && held >= 0))) { done_l = l; break; }
    o.dest = d;
    if (!(L.loaded & (1u << d))) {
      L.loaded |= 1u << d;
      L.tails[d] = D.st->tail_cache;
      L.chans[d] = D.st->chan_seq;
      L.heads[d] = read_head(D);
    }
    const uint64_t f = m.f;
    if (L.aborted) o.status = RING_ETIMEDOUT;
    else if (o.status == RING_OK && (m.len >= (1ull << 32) || f > D.R)) o.status = RING_EMSGSIZE;

    bool locked = held == (int)d;
    uint64_t P = L.tails[d];
    // %globaltimer is read only when a wait starts (keeps the serial path lean).
    uint64_t t_start = (o.status == RING_OK && D.mpsc && !locked) ? globaltimer() : 0;
    if (o.status == RING_OK && D.mpsc && !locked) {
      // Step 1 "Acquire the lock using a CAS-based spinlock",
      // after our own previous items (and their Unlock) are published.
      while (!D.rc && ld_acquire_gpu32(&S->pub_seq) != L.items)   // RC: the leader unlocks itself
        if (globaltimer() - t_start > a.timeout_ns) { o.status = RING_ETIMEDOUT; break; }
      if (a.trace) { a.trace[1900] = globaltimer(); a.trace[1901] = L.items; a.trace[1902] = ld_acquire_gpu32(&S->pub_seq); }
      if (o.status == RING_OK && D.rc) {
        // reserve-then-commit: a lock word with an acquisition count, taken
        // over from a lost holder after TL (the lock is held only for claims)
        L.me = ((uint64_t)(++D.st->lock_acq) << 16) | (uint64_t)(D.producer_id + 1);
        locked = rc_lock(a, D, L.me, t_start);
        if (!locked) o.status = RING_ETIMEDOUT;
      } else if (o.status == RING_OK) {
        const uint64_t me = (uint64_t)D.producer_id + 1;
        while (true) {
          const uint64_t old = D.sys ? cas_acquire<true>(lock_w(D), 0ull, me) : cas_acquire<false>(lock_w(D), 0ull, me);
          if (old == 0) { locked = true; break; }
          if (a.trace) a.trace[1903] = old;
          if (globaltimer() - t_start > a.timeout_ns) { o.status = RING_ETIMEDOUT; break; }
        }
      }
      if (locked && D.rc) {
        // reserve-then-commit: claim from the reservation frontier (entries
        // between the tail and it are reserved or committed).  Nothing slow
        // under the lock: a holder past TL would be taken over (publishing
        // committed entries left behind is done without it, below and by the
        // publishers)
        P = dld(D, resv_w(D));
        L.heads[d] = read_head(D);
        held = (int)d;
      } else if (locked) {
        // Step 2: read the tail (ordered after the acquiring CAS).
        P = D.sys ? ld_relaxed<true>(tail_w(D)) : ld_relaxed<false>(tail_w(D));
        if (a.trace) { a.trace[1904] = globaltimer(); a.trace[1905] = P; }
        // Step 4 (R6, before the space check): a busy slot at P_seq with the
        // size ring not full means a lost sender committed WB+WL but not UH
        // (Case 7): advance the header past it first.  The head is read
        // before the slot: a released slot is then seen cleared.
        while (true) {
          const uint64_t H = read_head(D);
          L.heads[d] = H;
          if (seq_dist(ptr_seq(P), ptr_seq(H)) >= D.N) break;
          const uint64_t w = D.sys ? ld_relaxed<true>(slot_w(D, ptr_seq(P))) : ld_relaxed<false>(slot_w(D, ptr_seq(P)));
          if (!(w & kBusy)) break;
          P = pack_ptr(advance(ptr_off(P), w & kFLow, D.R), seq_inc(ptr_seq(P)));
          if (D.sys) st_release<true>(tail_w(D), P); else st_release<false>(tail_w(D), P);
        }
        held = (int)d;
      }
    }
    bool defer = false;
    // a PAD planned for this message is withdrawn if the message is deferred
    // (below): PAD and message are placed under one lock hold, as the
    // sender's steps 1-8 place them (R3), so no other sender's entry can land
    // between them
    const uint32_t items_in = L.items;
    const uint64_t P_in = P;
    const auto last_pad_in = last_pad;
    // Step 3: space check (R4), PAD entry at the wrap (R3), credit wait (R12).
    if (o.status == RING_OK) {
      while (true) {
        const uint64_t H = L.heads[d];
        const uint64_t pb = ptr_off(P), hb = ptr_off(H);
        const uint32_t pq = ptr_seq(P), hq = ptr_seq(H);
        bool full = seq_dist(pq, hq) >= D.N;
        if (!full && pb + f > D.R) {
          if (span_free(pb, pq, hb, hq, D.R - pb)) {
            const uint64_t P2 = pack_ptr(0, seq_inc(pq));
            if (D.rc) {   // a PAD is claimed and committed at once (nothing to copy)
              if (D.sys) { st_relaxed<true>(slot_w(D, pq), kBusy | kPad | (D.R - pb)); st_relaxed<true>(resv_w(D), P2); }
              else { st_relaxed<false>(slot_w(D, pq), kBusy | kPad | (D.R - pb)); st_relaxed<false>(resv_w(D), P2); }
            }
            write_pad_plan(ctx, L.items, d, pq, kBusy | kPad | (D.R - pb), P2);
            last_pad = L.items;
            L.items++;
            P = P2;
            L.tails[d] = P;
            continue;
          }
          full = true;
        } else if (!full && !span_free(pb, pq, hb, hq, f)) {
          full = true;
        }
        if (!full) {
          o.start = pb;
          o.slot = pq;
          P = pack_ptr(advance(pb, f, D.R), seq_inc(pq));
          o.tail_after = P;
          if (D.rc) {   // claim: reserved slot + frontier, under the lock
            if (D.sys) { st_relaxed<true>(slot_w(D, pq), kResvBit | f); st_relaxed<true>(resv_w(D), P); }
            else { st_relaxed<false>(slot_w(D, pq), kResvBit | f); st_relaxed<false>(resv_w(D), P); }
          }
          break;
        }
        // Not enough credit with the cached head: re-read it once.
        const uint64_t H2 = read_head(D);
        if (H2 != H) { L.heads[d] = H2; continue; }
        if (flags & RING_TRY) { o.status = RING_FULL; break; }   // "release the lock and abort"
        if (D.rc && l == 0) {
          // reserve-then-commit: wait for credit WITHOUT the lock (it is only
          // for claims; a holder waiting past TL would be taken over), helping
          // to publish committed entries and turning a lost sender's
          // reservation at the tail into a PAD; then claim again
          st_release<false>(&S->planned, make_planned(L.items, L.units));   // our PADs to the publisher
          dcas(D, lock_w(D), L.me, 0ull);
          held = -1;
          if (!t_start) t_start = globaltimer();
          uint64_t seen = 0, since = 0;
          bool moved = false;
          while (!moved) {
            if (globaltimer() - t_start > a.timeout_ns) break;
            rc_help_advance(D);
            rc_hole_watch(a, D, seen, since);
            moved = read_head(D) != H2;
          }
          if (!moved) { o.status = RING_ETIMEDOUT; break; }
          L.me = ((uint64_t)(++D.st->lock_acq) << 16) | (uint64_t)(D.producer_id + 1);
          if (!rc_lock(a, D, L.me, t_start)) { o.status = RING_ETIMEDOUT; break; }
          held = (int)d;
          P = dld(D, resv_w(D));
          L.heads[d] = read_head(D);
          continue;
        }
        if (l > 0) {
          // Hand what is decided to the copy warps and the publisher (and
          // release the lock) before waiting; this message, with its PAD, is
          // placed again in the next round.
          if (!D.rc && L.items != items_in) { L.items = items_in; P = P_in; last_pad = last_pad_in; }
          defer = true;
          break;
        }
        // A PAD planned in this round must be published before waiting: the
        // consumer may have to free it for this message to fit (R3).
        st_release<false>(&S->planned, make_planned(L.items, L.units));
        if (!t_start) t_start = globaltimer();
        if (a.trace) { a.trace[1906] = globaltimer(); a.trace[1907] = P; a.trace[1908] = H2; a.trace[1909] = f; a.trace[1910]++; }
        // relaxed polls (an acquire per poll invalidates the SM's L1, where the
        // copy warps' loads are staged), one acquire fence once the head moved
        uint64_t H3 = H2;
        while (H3 == H2) {
          if (globaltimer() - t_start > a.timeout_ns) break;
          H3 = read_head_relaxed(D);
        }
        if (H3 != H2) { if (D.sys) fence_acq_rel<true>(); else fence_acq_rel<false>(); }
        if (H3 == H2) { o.status = RING_ETIMEDOUT; break; }
        L.heads[d] = H3;
      }
    }
    L.tails[d] = P;
    if (defer) { done_l = l; break; }
    if (o.status == RING_ETIMEDOUT) L.aborted = true;
    if (hit >= 0 && o.status != RING_EREJECTED) {   // committed: advance the round robin and the admission
      a.routes[hit].rr = a.routes[hit].rr + 1;
      a.routes[hit].adm_next = adm_next;
    }
    if (o.status != RING_EREJECTED) {   // a rejected request never reaches the channel
      o.seq = (uint32_t)L.chans[d];
      L.chans[d] += 1;
    }
    o.item = L.items++;
    o.flags = kStatus | (o.status == RING_OK ? kEntry : 0u);
    if (o.status == RING_OK) {
      o.nunits = m.nunits;
      o.first_unit = L.units;
      L.units += o.nunits;
    }
    gs[l] = o;
  }
  if (held >= 0 && dests[held].rc) {
    // reserve-then-commit: the claims are done -- unlock now (acq_rel CAS:
    // orders the reserved slots and the frontier before it; fails harmlessly
    // if the lock was taken over); copies and commits happen outside the lock.
    // Fault injection (tests): a sender lost holding the lock, or after its
    // claims before any commit.
    const DestDesc& D = dests[held];
    const bool hit = a.fault.die_after && k0 <= a.fault.msg && a.fault.msg < k0 + done_l;
    if (!(hit && a.fault.die_after == RING_AT_LOCK)) dcas(D, lock_w(D), L.me, 0ull);
    if (hit) L.dead = true;
  } else if (held >= 0) {
    // Step 8 "Release the lock" after the round's LAST item (a PAD planned
    // for a deferred message comes after the last message item).
    if (last_pad == L.items - 1) ctx->plan[last_pad % kPlanRing].flags |= kUnlock;
    else gs[done_l - 1].flags |= kUnlock;
  }
  return done_l;
}

// Warp-parallel placement of one round for a single SPSC destination (no
// router, no lock): the serial rule of leader_place evaluated for all lanes at
// once.  Without a wrap, message l starts at P_b + (footprints of the messages
// before it); at the first message that would cross R a PAD entry fills the
// rest of the buffer region and the following messages start again from 0
// (R3; an exact fit wraps to 0 without a PAD).  Every lane then
// checks exactly the serial space rule (R4) and slot count (R5) at its own
// position against the cached head; the leading run of lanes that fit is
// placed.  Returns the run length; 0 leaves the round to the serial path
// (credit wait, second wrap, EMSGSIZE).
// The placement rule of one round, per lane (also evaluated by every CTA at
// launch start to start copies before the leader's plans arrive, see
// SpecRound): a pure function of the tail P, the head H and the lengths.
struct RoundPlace {
  uint64_t start, tail_after, pad_start;
  uint32_t seq, item_off, fu_off, nu, run, w, pad_seq, nu_total;
  bool pad_used, c;
};
__device__ __forceinline__ RoundPlace place_round(uint64_t P, uint64_t H, bool act, uint64_t f, uint32_t nu_in,
                                                  const DestDesc& D) {
  const int lane = threadIdx.x & 31;
  RoundPlace r;
  const uint64_t pb = ptr_off(P), hb = ptr_off(H);
  const uint32_t pq = ptr_seq(P), hq = ptr_seq(H);
  const uint64_t incl = warp_incl_scan64(f, lane);
  const uint64_t excl = incl - f;
  const uint32_t wmask = __ballot_sync(0xffffffffu, act && pb + incl > D.R);
  const uint32_t w = wmask ? (uint32_t)__ffs(wmask) - 1 : 32u;
  const uint64_t excl_w = __shfl_sync(0xffffffffu, excl, w & 31);
  const uint64_t pad_start = pb + excl_w;
  const bool has_pad = w < 32 && pad_start < D.R;      // exact fit before w: no PAD
  const uint32_t pad_seq = (pq + w) & kSeqMask;
  uint64_t start;
  uint32_t seq;
  if ((uint32_t)lane < w) {
    start = pb + excl;
    seq = pq + lane;
  } else {
    start = excl - excl_w;
    seq = pq + lane + (has_pad ? 1 : 0);
  }
  seq &= kSeqMask;
  bool ok = act && start + f <= D.R && seq_dist(seq, hq) < D.N && span_free(start, seq, hb, hq, f);
  if (has_pad && (uint32_t)lane >= w)
    ok = ok && seq_dist(pad_seq, hq) < D.N && span_free(pad_start, pad_seq, hb, hq, D.R - pad_start);
  const uint32_t notok = __ballot_sync(0xffffffffu, !ok);
  const uint32_t run = notok ? (uint32_t)__ffs(notok) - 1 : 32u;
  r.run = run;
  r.pad_used = has_pad && w < run;
  r.c = (uint32_t)lane < run;
  r.nu = r.c ? nu_in : 0;
  const uint32_t nu_incl = warp_incl_scan32(r.nu, lane);
  r.fu_off = nu_incl - r.nu;
  r.nu_total = __shfl_sync(0xffffffffu, nu_incl, 31);
  r.start = start;
  r.seq = seq;
  r.item_off = lane + ((r.pad_used && (uint32_t)lane >= w) ? 1 : 0);
  r.tail_after = pack_ptr(advance(start, f, D.R), seq_inc(seq));
  r.w = w;
  r.pad_start = pad_start;
  r.pad_seq = pad_seq;
  return r;
}

__device__ uint32_t fast_place(const PutArgs& a, LaunchCtx* ctx, LeaderState& L, uint32_t gmax, GroupSlot* gs,
                               const MsgBrief* brief, const DestDesc& D) {
  const int lane = threadIdx.x & 31;
  const bool act = (uint32_t)lane < gmax;
  const uint64_t f = act ? brief[lane].f : 0;
  const uint64_t len = act ? brief[lane].len : 0;
  if (__ballot_sync(0xffffffffu, act && (len >= (1ull << 32) || f > D.R))) return 0;
  const RoundPlace r = place_round(L.tails[0], L.heads[0], act, f, act ? brief[lane].nunits : 0, D);
  const uint32_t run = r.run;
  if (run == 0) return 0;
  const bool pad_used = r.pad_used;
  const bool c = r.c;
  const uint32_t nu = r.nu;
  const uint32_t items0 = L.items, units0 = L.units;
  const uint64_t chan0 = L.chans[0];
  const uint64_t tail_after = r.tail_after;
  const uint64_t start = r.start;
  const uint32_t seq = r.seq, w = r.w, pad_seq = r.pad_seq;
  const uint64_t pad_start = r.pad_start;
  if (c) {
    GroupSlot o = {};
    o.start = start;
    o.slot = seq;
    o.tail_after = tail_after;
    o.item = items0 + r.item_off;
    o.dest = 0;
    o.seq = (uint32_t)(chan0 + lane);
    o.status = RING_OK;
    o.flags = kStatus | kEntry;
    o.nunits = nu;
    o.first_unit = units0 + r.fu_off;
    gs[lane] = o;
  }
  if (pad_used && (uint32_t)lane == w)
    write_pad_plan(ctx, items0 + w, 0, pad_seq, kBusy | kPad | (D.R - pad_start), pack_ptr(0, seq_inc(pad_seq)));
  const uint64_t last_tail = __shfl_sync(0xffffffffu, tail_after, run - 1);
  const uint32_t nu_total = r.nu_total;
  __syncwarp();
  if (lane == 0) {
    L.items = items0 + run + (pad_used ? 1 : 0);
    L.units = units0 + nu_total;
    L.chans[0] = chan0 + run;
    L.tails[0] = last_tail;
  }
  __syncwarp();
  return run;
}

// ---------------------------------------------------------------------------
// Fault-tolerant sender (RING_CREATE_FAULT_TOLERANT, the
// oracle's FaultSim step for step).  One message at a time, every action by
// lane 0 of the leader warp except WB's payload, which the copy warps move
// (one plan item per message; the publisher only counts it).  Tagged slot
// words: busy | pad | (seq mod 2^22) << 40 | f (reading R21).
// ---------------------------------------------------------------------------
// Fault injection point `at` for message k (lane 0).  Returns true if the
// sender must stop for good here.
__device__ bool ft_point(const PutArgs& a, uint32_t at, uint32_t k, uint64_t timeout_ns) {
  const FaultSpec& F = a.fault;
  if (k != F.msg) return false;
  if (F.pause_mask & (1u << at)) {
    volatile uint32_t* arr = F.arrived;
    volatile uint32_t* go = F.go;
    __threadfence_system();
    arr[at] = 1u;
    __threadfence_system();
    const uint64_t t0 = globaltimer();
    while (go[at] == 0u)
      if (globaltimer() - t0 > timeout_ns) break;
    __threadfence_system();
  }
  return F.die_after == at;
}

__device__ void ft_put(const PutArgs& a, LaunchCtx* ctx, LaunchSet* S, uint32_t* s_crc) {
  const int lane = threadIdx.x & 31;
  const DestDesc& D = a.dest0;
  for (int i = lane; i < kCrcTableWords; i += 32) s_crc[i] = a.crc_table[i];
  __syncwarp();
  const uint32_t* pw = a.crc_table + kCrcTableWords;
  uint64_t chan = 0, acq = 0;
  if (lane == 0) { chan = D.st->chan_seq; acq = D.st->lock_acq; }
  chan = __shfl_sync(0xffffffffu, chan, 0);
  uint32_t items = 0, units = 0;
  bool dead = false;
  const uint64_t t_begin = globaltimer();
  for (uint32_t k = 0; k < a.n && !dead; ++k) {
    const ring_msg_t* mp = a.msgs ? a.msgs + k : &a.inline_msg;
    const uint64_t len = mp->len;
    const uint64_t f = footprint(len);
    uint32_t status = RING_OK;
    if (len >= (1ull << 32) || f > D.R) status = RING_EMSGSIZE;
    // payload checksum first: it goes into the header (bytes [40,44))
    const uint32_t pcrc = status == RING_OK ? warp_crc32(reinterpret_cast<const uint8_t*>(mp->src), len, s_crc, pw, lane) : 0u;
    uint64_t P = 0, me = 0;
    uint32_t st = status, die = 0;
    if (lane == 0 && st == RING_OK) {
      const uint64_t t_msg = globaltimer();
      bool have_lock = false;
      uint64_t seen = 0, seen_at = 0;
      while (st == RING_OK) {                                   // ---- step 1: Lock (+ TL take-over)
        if (!have_lock) {
          me = (++acq << 16) | (uint64_t)(D.producer_id + 1);
          while (true) {
            const uint64_t old = dcas(D, lock_w(D), 0ull, me);
            if (old == 0) break;
            const uint64_t now = globaltimer();
            if (old != seen) { seen = old; seen_at = now; }
            else if (now - seen_at > a.lock_timeout_ns) {     // TL: the holder is presumed lost
              if (dcas(D, lock_w(D), old, me) == old) break;
            }
            if (now - t_msg > a.timeout_ns) { st = RING_ETIMEDOUT; break; }
          }
          if (st != RING_OK) break;
          have_lock = true;
          if (ft_point(a, RING_AT_LOCK, k, a.timeout_ns)) { die = 1; break; }
        }
        // ---- steps 2-4: GH (tail, head, next slot: repair a lost sender's entry / clear a stale write)
        P = dld(D, tail_w(D));
        const uint64_t H = read_head(D);
        const uint32_t pq = ptr_seq(P), hq = ptr_seq(H);
        const uint64_t pb = ptr_off(P), hb = ptr_off(H);
        if (seq_dist(pq, hq) < D.N) {
          const uint64_t w = dld(D, slot_w(D, pq));
          if (w & kBusy) {
            if (((w >> kTagShift) & kTagMask) == (pq & kTagMask))      // Case 7: publish it
              dcas(D, tail_w(D), P, pack_ptr(advance(pb, w & kFLow, D.R), seq_inc(pq)));
            else                                                        // R21: stale write
              dcas(D, slot_w(D, pq), w, 0ull);
            continue;
          }
        }
        // ---- step 3: space (R4), PAD at the wrap (R3)
        bool full = seq_dist(pq, hq) >= D.N;
        if (!full && pb + f > D.R) {
          if (span_free(pb, pq, hb, hq, D.R - pb)) {
            if (dcas(D, slot_w(D, pq), 0ull, tagged_word(kBusy | kPad | (D.R - pb), pq)) == 0ull)
              dcas(D, tail_w(D), P, pack_ptr(0, seq_inc(pq)));
            continue;                                           // re-read (GH) after the PAD
          }
          full = true;
        } else if (!full && !span_free(pb, pq, hb, hq, f)) {
          full = true;
        }
        if (full) {                                             // unlock, wait for the head, start over
          if (a.flags & RING_TRY) { dcas(D, lock_w(D), me, 0ull); st = RING_FULL; break; }
          dcas(D, lock_w(D), me, 0ull);
          have_lock = false;
          while (read_head(D) == H)
            if (globaltimer() - t_msg > a.timeout_ns) { st = RING_ETIMEDOUT; break; }
          continue;
        }
        if (ft_point(a, RING_AT_GH, k, a.timeout_ns)) { die = 1; break; }
        break;                                                  // placement decided: P
      }
      if (st != RING_OK && !die) {
        // nothing written (FULL / timeout); the lock is ours only if still held
        if (me) dcas(D, lock_w(D), me, 0ull);
      }
    }
    st = __shfl_sync(0xffffffffu, st, 0);
    die = __shfl_sync(0xffffffffu, die, 0);
    P = __shfl_sync(0xffffffffu, P, 0);
    me = __shfl_sync(0xffffffffu, me, 0);
    if (die) { dead = true; break; }
    if (st == RING_OK) {
      // ---- step 5: WB -- header (lanes 0-3) and payload (copy warps)
      const uint64_t start = ptr_off(P);
      if (lane < 4) {
        uint32_t w[16];
        const uint32_t* uid = reinterpret_cast<const uint32_t*>(mp->hdr.uid);
        const uint32_t len32 = (uint32_t)len;
        w[1] = uid[0]; w[2] = uid[1]; w[3] = uid[2]; w[4] = uid[3];
        w[5] = (uint32_t)mp->hdr.accepted_at;
        w[6] = (uint32_t)(mp->hdr.accepted_at >> 32);
        w[7] = mp->hdr.app_id;
        w[8] = (uint32_t)mp->hdr.stage | (len32 << 16);
        w[9] = len32 >> 16;
        w[10] = pcrc;                                  // reserved[40,44): payload CRC
        w[11] = D.producer_id;
        w[12] = (uint32_t)(chan + k);
        w[13] = 1u << 16;                              // epoch 0, flags bit 0: payload CRC present
        w[0] = crc52(w, s_crc);
        const uint64_t t = (a.flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
        w[14] = (uint32_t)t;
        w[15] = (uint32_t)(t >> 32);
        st16(D.data + start + 16 * lane, make_int4((int)w[4 * lane], (int)w[4 * lane + 1], (int)w[4 * lane + 2],
                                                   (int)w[4 * lane + 3]));
      }
      const uint32_t nu = units_for(len, a.chunk);
      if (lane == 0) {
        Plan& p = ctx->plan[items % kPlanRing];
        p.src = mp->src;
        p.dst = reinterpret_cast<uint64_t>(D.data + start + kHdr);
        p.len = len;
        p.first_unit = units;
        p.nunits = nu;
        p.flags = 0;                                   // the publisher only counts it
        p.msg = k;
        S->arrive[items % kPlanRing] = 0;
        st_release<false>(&S->planned, make_planned(items + 1, units + nu));
        const uint64_t t0 = globaltimer();
        while (nu && ld_acquire_gpu32(&S->arrive[items % kPlanRing]) != nu)
          if (globaltimer() - t0 > a.timeout_ns) break;
      }
      ++items;
      units += nu;
      __syncwarp();
      if (lane == 0) {
        if (ft_point(a, RING_AT_WB, k, a.timeout_ns)) die = 1;
        // ---- step 6: WL = CAS(slot, 0 -> busy|tag|f); release: WB before WL (a GH repair may publish it)
        if (!die) {
          const uint32_t pq = ptr_seq(P);
          if (dcas(D, slot_w(D, pq), 0ull, tagged_word(kBusy | f, pq)) != 0ull) {
            st = RING_EDROPPED;
            dcas(D, lock_w(D), me, 0ull);                          // Unlock (may fail: taken over)
          } else {
            if (ft_point(a, RING_AT_WL, k, a.timeout_ns)) die = 1;
            // ---- step 7: UH = CAS(tail, P -> new); failing = committed, a later GH publishes it
            if (!die) {
              dcas(D, tail_w(D), P, pack_ptr(advance(ptr_off(P), f, D.R), seq_inc(pq)));
              if (ft_point(a, RING_AT_UH, k, a.timeout_ns)) die = 1;
            }
            if (!die) dcas(D, lock_w(D), me, 0ull);                // ---- step 8: Unlock = CAS(me -> 0)
          }
        }
      }
      st = __shfl_sync(0xffffffffu, st, 0);
      die = __shfl_sync(0xffffffffu, die, 0);
      if (die) { dead = true; break; }
    }
    if (lane == 0) a.status[k] = st;
  }
  (void)t_begin;
  if (lane == 0) {
    st_release<false>(&S->planned, make_planned(items, units) | kPlannedDone);
    if (!dead) {
      D.st->chan_seq = chan + a.n;
      D.st->lock_acq = acq;
    }
  }
}

// The messages of one batch: a launch's (kernel parameters), or an engine batch's.
struct BatchRef {
  const ring_msg_t* msgs;
  uint32_t* status;
  uint32_t n, flags;
};

// One batch of messages (a launch's, or an engine batch's): rounds of up to
// 32 messages placed by the leader warp, each handed out with one release.
__device__ __forceinline__ void leader_batch(const PutArgs& a, const BatchRef& B, LaunchCtx* ctx, LaunchSet* S,
                                             LeaderState& L, GroupSlot* gs, MsgBrief* brief, uint32_t& s_g,
                                             const DestDesc* s_dests, bool fast) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k0 = 0; k0 < B.n;) {
    const uint32_t gmax = min((uint32_t)kGroup, B.n - k0);
    if ((uint32_t)lane < gmax) {   // stage the round's lengths / routing keys in parallel
      const ring_msg_t* mp = B.msgs ? B.msgs + k0 + lane : &a.inline_msg;
      const uint64_t len = mp->len;
      brief[lane].len = len;
      brief[lane].f = footprint(len);
      brief[lane].app_id = mp->hdr.app_id;
      brief[lane].stage = mp->hdr.stage;
      brief[lane].nunits = units_for(len, a.chunk);
      brief[lane].t_arr = mp->hdr.accepted_at;
    }
    // t_put of the round's messages: the leader takes them up now, before any claim
    const uint64_t t_in = __shfl_sync(0xffffffffu, (B.flags & RING_NO_TIMESTAMP) ? 0ull : globaltimer(), 0);
    uint64_t tc = 0, cq = 0;   // issued together with the brief loads (first round)
    if (lane == 0 && fast && !(L.loaded & 1u)) {
      tc = a.dest0.st->tail_cache;
      cq = a.dest0.st->chan_seq;
    }
    __syncwarp();
    if (lane == 0) {
      // Flow control: the round adds at most 2 items per message.
      if (L.items + 2 * gmax > (uint32_t)kPlanRing &&
          L.items + 2 * gmax - ld_acquire_gpu32(&S->pub_seq) > (uint32_t)kPlanRing) {
        const uint64_t end = globaltimer() + 2 * a.timeout_ns;
        while (L.items + 2 * gmax - ld_acquire_gpu32(&S->pub_seq) > (uint32_t)kPlanRing)
          if (globaltimer() > end) { L.aborted = true; L.flow_to = true; break; }
      }
      const uint32_t rnd = a.engine ? L.nrounds % 64 : k0 / kGroup;
      if (a.trace && rnd < 64) a.trace[rnd * 4] = globaltimer();
      // the fast path needs destination 0's state and a fresh credit
      if (fast) {
        if (!(L.loaded & 1u)) {
          L.loaded |= 1u;
          L.tails[0] = tc;
          L.chans[0] = cq;
        }
        L.heads[0] = read_head(a.dest0);
      }
    }
    __syncwarp();
    if (L.flow_to) {
      // Plan slots the copy warps / publisher may still read are never
      // overwritten: the remaining messages time out without a plan item.
      for (uint32_t k = k0 + lane; k < B.n; k += 32) B.status[k] = RING_ETIMEDOUT;
      break;
    }
    uint32_t g = 0;
    if (fast && !L.aborted) g = fast_place(a, ctx, L, gmax, gs, brief, a.dest0);
    if (g == 0) {
      const uint32_t it0 = L.items, un0 = L.units;
      if (lane == 0) s_g = leader_place(a, B.flags, ctx, S, L, k0, gmax, gs, brief, s_dests);
      __syncwarp();
      g = s_g;
      if (L.dead) {              // fault injection: the sender is lost, this round is never planned
        if (lane == 0) { L.items = it0; L.units = un0; }
        __syncwarp();
        break;
      }
    }
    // placements: one release hands the round's copies (and headers) out
    const uint32_t k = k0 + lane;
    const GroupSlot o = gs[lane & 31];
    if ((uint32_t)lane < g) {
      Plan& p = ctx->plan[o.item % kPlanRing];
      p.msg = k;
      p.status = o.status;
      p.dest = o.dest;
      p.flags = o.flags;
      p.nunits = o.nunits;
      p.first_unit = o.first_unit;
      p.len = 0;
      p.t_in = t_in;
      if (o.status == RING_OK) {
        const ring_msg_t* mp = B.msgs ? B.msgs + k : &a.inline_msg;
        const DestDesc& D = s_dests[o.dest];
        const uint64_t len = brief[lane].len;
        const uint64_t f = brief[lane].f;
        p.src = mp->src;
        p.dst = reinterpret_cast<uint64_t>(D.data + o.start + kHdr);
        RING_CHECK(o.start % kAlign == 0 && o.start + f <= D.R && kHdr + len <= f, "put entry inside R", o.start, f);
        RING_CHECK(o.item - ld_acquire_gpu32(&S->pub_seq) < (uint32_t)kPlanRing, "plan slot free", o.item,
                   ld_acquire_gpu32(&S->pub_seq));
        p.len = len;
        p.start = o.start;
        p.slot = o.slot;
        p.slot_word = kBusy | f;
        p.tail_after = o.tail_after;
        p.f = f;
        p.seq = o.seq;
        p.epoch = o.epoch;
        if (a.engine) p.msgp = reinterpret_cast<uint64_t>(mp);
      }
      if (a.engine) p.statusp = reinterpret_cast<uint64_t>(B.status + k);
      // An arrive counter is reused by item + kPlanRing, planned only once
      // pub_seq has passed the item (flow control); the first kPlanRing items
      // start from the zeroed set, and the speculative first round only ever
      // counts into those.  (No reset in the publisher: its flush fence then
      // has nothing left to wait for.)
      if (o.item >= (uint32_t)kPlanRing) S->arrive[o.item % kPlanRing] = 0;
      if (a.dest_out) a.dest_out[k] = o.dest;
    }
    __syncwarp();
    if (lane == 0) {
      st_release<false>(&S->planned, make_planned(L.items, L.units));
      const uint32_t rnd = a.engine ? L.nrounds++ % 64 : k0 / kGroup;
      if (a.trace && rnd < 64) {
        a.trace[rnd * 4 + 1] = globaltimer();
        a.trace[rnd * 4 + 2] = L.items;
        a.trace[rnd * 4 + 3] = g;
      }
    }
    k0 += g;
  }
}


__device__ void put_leader(const PutArgs& a, LaunchCtx* ctx, LaunchSet* S) {
  const int lane = threadIdx.x & 31;
  __shared__ GroupSlot gs[kGroup];
  __shared__ MsgBrief brief[kGroup];
  __shared__ uint32_t s_g;
  __shared__ LeaderState L;
  __shared__ DestDesc s_dests[kMaxRouterDests];   // destination descriptors, read every message
  if (a.n_dests == 1) {
    if (lane == 0) s_dests[0] = a.dest0;
  } else {
    for (uint32_t d = lane; d < a.n_dests && d < (uint32_t)kMaxRouterDests; d += 32) s_dests[d] = a.dests[d];
  }
  // the fast path (one SPSC destination, no router) reads its state from the kernel parameters
  const bool fast = !a.routes && a.n_dests == 1 && !a.dest0.mpsc;
  if (lane == 0) {
    L.loaded = 0;
    L.items = 0;
    L.units = 0;
    L.aborted = false;
    L.dead = false;
    L.flow_to = false;
    L.nrounds = 0;
  }
  __syncwarp();
  if (!a.engine) {
    leader_batch(a, BatchRef{a.msgs, a.status, a.n, a.flags}, ctx, S, L, gs, brief, s_g, s_dests, fast);
  } else {
    // Persistent engine: batches from the queue until the host's stop.  Each
    // batch is independent (a timed-out message aborts the rest of ITS batch).
    EngineQueue* q = a.engine;
    uint64_t lease = 0, since = 0;
    for (uint64_t b = 0;; ++b) {
      uint32_t go = 0;
      if (lane == 0) {
        while (true) {
          const uint64_t c = ld_acquire<false>(&q->ctl);
          if ((c & ~kEngineClosed) > b) { go = 1; break; }
          if (c & kEngineClosed) break;                   // stopped: every posted batch is planned
          // idle: close the queue once nothing is in flight and the host has
          // made no call on the attachment for the idle time
          const uint64_t now = globaltimer();
          const uint64_t ls = a.engine_host->lease;
          if (ls != lease || !since || ld_acquire<false>(&q->done) != b) { lease = ls; since = now; }
          else if (now - since > a.engine_idle_ns && atomicCAS(reinterpret_cast<unsigned long long*>(&q->ctl), c,
                                                               c | kEngineClosed) == c)
            break;
          __nanosleep(256);
        }
      }
      go = __shfl_sync(0xffffffffu, go, 0);
      if (!go) break;
      const EngineBatch& eb = q->batch[b % kEngineQueue];
      const BatchRef B{eb.msgs, eb.status, eb.n, eb.flags};
      if (lane == 0) { L.aborted = false; L.flow_to = false; }
      __syncwarp();
      leader_batch(a, B, ctx, S, L, gs, brief, s_g, s_dests, fast);
      if (lane == 0) {
        q->batch[b % kEngineQueue].item_end = L.items;
        st_release<false>(&q->planned_batches, b + 1);
      }
      __syncwarp();
    }
  }
  if (lane == 0) {
    st_release<false>(&S->planned, make_planned(L.items, L.units) | kPlannedDone);
    for (uint32_t d = 0; d < kMaxRouterDests && d < a.n_dests && !L.dead; ++d)
      if (L.loaded & (1u << d)) {
        a.dests[d].st->chan_seq = L.chans[d];
        if (!a.dests[d].mpsc) a.dests[d].st->tail_cache = L.tails[d];
      }
    // the next launch's starting tail, in ITS counter set (spec_first_round)
    if (fast && (L.loaded & 1u) && !L.dead) ctx->set[(a.launch + 1) & 1].start_tail = L.tails[0];
  }
  if (lane == 0 && a.engine) {   // the host restarts a closed engine at its next submission
    __threadfence_system();
    a.engine_host->alive = 0u;
  }
}

// Entry header (R11) + CRC-32 over bytes [4, 56) (R10) of plan item j,
// written to the ring together with the item's status and, for an SPSC ring,
// its size slot (WL).  SPSC: no reader looks at a slot past the tail (the
// stale-slot check GH runs under the MPSC lock only, R6), so the slot can be
// written before the payload is complete; the fence before the tail store
// still orders it, and nothing is left for that fence to wait for.
__device__ __forceinline__ void write_header(const PutArgs& a, LaunchCtx* ctx, uint32_t j, const uint32_t* crc_tab) {
  const Plan& p = ctx->plan[j % kPlanRing];
  const uint32_t flags = ld_cg32(&p.flags), status = ld_cg32(&p.status), msg = ld_cg32(&p.msg);
  if (flags & kStatus) {
    if (a.engine) *reinterpret_cast<uint32_t*>(ld_cg64(&p.statusp)) = status;
    else a.status[msg] = status;
  }
  if (!(flags & kEntry)) return;
  const DestDesc& D = a.dests[ld_cg32(&p.dest)];
  if ((flags & kStatus) && status == RING_OK) {
    const ring_msg_t* mp = a.engine ? reinterpret_cast<const ring_msg_t*>(ld_cg64(&p.msgp))
                                    : (a.msgs ? a.msgs + msg : &a.inline_msg);
    const uint32_t* uid = reinterpret_cast<const uint32_t*>(mp->hdr.uid);   // (4-B aligned in kernel params)
    const uint4 u0 = make_uint4(uid[0], uid[1], uid[2], uid[3]);
    const uint64_t acc = mp->hdr.accepted_at;
    const uint32_t app = mp->hdr.app_id, stage = mp->hdr.stage;
    const uint32_t len32 = (uint32_t)ld_cg64(&p.len);
    uint32_t w[16];
    w[1] = u0.x; w[2] = u0.y; w[3] = u0.z; w[4] = u0.w;
    w[5] = (uint32_t)acc;
    w[6] = (uint32_t)(acc >> 32);
    w[7] = app;
    w[8] = stage | (len32 << 16);          // stage[32,34) payload_len[34,36)
    w[9] = len32 >> 16;                    // payload_len[36,38) reserved[38,40)
    w[10] = 0;                             // reserved[40,44)
    w[11] = D.producer_id;
    w[12] = ld_cg32(&p.seq);
    w[13] = ld_cg32(&p.epoch) & 0xffffu;   // epoch[52,54) flags[54,56)
    w[0] = crc52(w, crc_tab);
    const uint64_t t = ld_cg64(&p.t_in);    // t_put: when the leader took the message up (0: RING_NO_TIMESTAMP)
    w[14] = (uint32_t)t;
    w[15] = (uint32_t)(t >> 32);
    uint8_t* hd = D.data + ld_cg64(&p.start);
    RING_CHECK(ld_cg64(&p.start) + kHdr <= D.R, "header inside R", ld_cg64(&p.start), D.R);
#pragma unroll
    for (int q = 0; q < 4; ++q) st16(hd + 16 * q, make_int4((int)w[4 * q], (int)w[4 * q + 1], (int)w[4 * q + 2], (int)w[4 * q + 3]));
    if (D.hdrs) {   // split placement: the consumer reads the header from its own memory
      uint8_t* hm = D.hdrs + 64ull * (ld_cg32(&p.slot) & (D.N - 1));
#pragma unroll
      for (int q = 0; q < 4; ++q) st16(hm + 16 * q, make_int4((int)w[4 * q], (int)w[4 * q + 1], (int)w[4 * q + 2], (int)w[4 * q + 3]));
    }
  }
  if (!D.mpsc) {   // WL (SPSC, early; PAD entries carry the pad bit)
    if (D.sys) st_relaxed<true>(slot_w(D, ld_cg32(&p.slot)), ld_cg64(&p.slot_word));
    else st_relaxed<false>(slot_w(D, ld_cg32(&p.slot)), ld_cg64(&p.slot_word));
  }
}

// Reserve-then-commit: move the tail over the leading run of committed slots,
// warp-parallel (the lanes read up to 32 slots from the tail; entries tile the
// ring and PADs fill every wrap, so offsets add mod R; ONE CAS per run).  With
// `wait`, keep going until the tail has passed seq `last` (our last committed
// entry), turning a reservation stuck at the tail for the hole timeout into a
// PAD (a lost sender, reading R23).
__device__ void rc_advance(const PutArgs& a, const DestDesc& D, int lane, bool wait, uint32_t last) {
  uint64_t T = 0, Rv = 0, H = 0;
  if (lane == 0) { T = dld(D, tail_w(D)); Rv = dld(D, resv_w(D)); H = read_head(D); }
  T = __shfl_sync(0xffffffffu, T, 0);
  Rv = __shfl_sync(0xffffffffu, Rv, 0);
  H = __shfl_sync(0xffffffffu, H, 0);
  uint64_t seen = 0, since = 0;
  const uint64_t t0 = globaltimer();
  while (true) {
    const uint32_t tq = ptr_seq(T);
    const uint32_t room = D.N - min(D.N, seq_dist(tq, ptr_seq(H)));
    const uint32_t k = min(min(seq_dist(ptr_seq(Rv), tq), room), 32u);
    uint64_t w = 0;
    if ((uint32_t)lane < k) w = dld(D, slot_w(D, (tq + lane) & kSeqMask));
    const uint32_t notbusy = __ballot_sync(0xffffffffu, !((uint32_t)lane < k && (w & kBusy)));
    const uint32_t nrun = notbusy ? __ffs(notbusy) - 1 : 32u;
    if (nrun == 0) {
      if (!wait || seq_dist(tq, last) - 1u < (1u << 23) || globaltimer() - t0 > a.timeout_ns) return;
      if (lane == 0) {
        rc_hole_watch(a, D, seen, since);
        T = dld(D, tail_w(D)); Rv = dld(D, resv_w(D)); H = read_head(D);
      }
      T = __shfl_sync(0xffffffffu, T, 0);
      Rv = __shfl_sync(0xffffffffu, Rv, 0);
      H = __shfl_sync(0xffffffffu, H, 0);
      continue;
    }
    const uint64_t fsum = warp_sum64((uint32_t)lane < nrun ? (w & kFLow) : 0);
    const uint64_t T2 = pack_ptr((ptr_off(T) + fsum) % D.R, tq + nrun);
    uint64_t old = 0;
    if (lane == 0) old = dcas(D, tail_w(D), T, T2);
    old = __shfl_sync(0xffffffffu, old, 0);
    T = old == T ? T2 : old;                           // moved (look further) or somebody else did
  }
}

// Engine: batches [done, ..) whose every item is below `published` are done;
// returns the new count (released to the doorbell / wait kernels).
__device__ __forceinline__ uint64_t engine_advance_done(EngineQueue* q, uint64_t done, uint32_t published) {
  const uint64_t pb = ld_acquire<false>(&q->planned_batches);
  const uint64_t d0 = done;
  while (done < pb && (int32_t)(published - ld_cg32(&q->batch[done % kEngineQueue].item_end)) >= 0) ++done;
  if (done != d0) st_release<false>(&q->done, done);
  return done;
}

// Steps 5-8 (WB header, WL, UH, Unlock), in item order.  As soon as items are
// planned the lanes write their headers (write_header), off the copy critical
// path.  For publication lane l caches the plan of item i + l (read once);
// each look only polls the arrive counters.  For the leading run of complete
// items the lanes write the size slots (WL, MPSC rings).  Runs accumulate
// while whole windows keep completing; then ONE fence orders the payload
// copies (observed through the arrive counters), headers and slots before the
// tail store (UH), the Unlock and pub_seq.  A flush happens at a partial
// window, at an Unlock, at a change of destination and whenever nothing more
// is complete.
__device__ void put_publisher(const PutArgs& a, LaunchCtx* ctx, LaunchSet* S, const uint32_t* crc_tab) {
  const int lane = threadIdx.x & 31;
  uint32_t i = 0, trace_n = 0, ps = 0, hq = 0;
  bool done = false;
  uint64_t idle_since = 0;
  bool have = false;
  uint32_t flags = 0, dest = 0, nunits = 0, slot = 0;
  uint64_t slot_word = 0, tail_after = 0;
  // accumulated, not yet fenced: destination, tail, Unlock
  bool pend = false, pend_entries = false, pend_unlock = false;
  uint32_t pend_dest = 0, pend_n = 0;
  uint64_t pend_tail = 0;
  bool rc_any = false;       // reserve-then-commit: committed entries to see published
  uint32_t rc_last = 0, rc_dest = 0;
  if (a.trace && lane == 0) a.trace[255] = globaltimer();
  uint64_t bdone = 0;   // engine: batches whose every item is published (lane 0)
  auto flush = [&]() {
    const DestDesc& D = a.dests[pend_dest];
    // acquire for the arrive counters read before, release for the copies, headers and slots
    if (D.sys) fence_acq_rel<true>(); else fence_acq_rel<false>();
    if (lane == 0) {
      if (pend_entries) {   // UH
        if (D.sys) st_relaxed<true>(tail_w(D), pend_tail); else st_relaxed<false>(tail_w(D), pend_tail);
      }
      if (pend_unlock) {    // Unlock after the tail
        if (D.sys) st_release<true>(lock_w(D), 0ull); else st_release<false>(lock_w(D), 0ull);
      }
      st_u32_relaxed_gpu(&S->pub_seq, i);   // ordered by the fence
      if (a.engine) bdone = engine_advance_done(a.engine, bdone, i);
      if (a.trace && (trace_n < 512 || a.engine)) {
        a.trace[256 + 2 * (trace_n % 512)] = globaltimer();
        a.trace[257 + 2 * (trace_n % 512)] = i;
      }
    }
    trace_n++;
    pend = pend_entries = pend_unlock = false;
    pend_n = 0;
  };
  while (true) {
    const uint32_t j = i + lane;
    // Independent loads in one pass: lane 0 looks for newly planned items
    // (relaxed), every lane with a cached item polls its arrive counter.
    uint64_t pl = 0;
    uint32_t arr = 0;
    if (lane == 0 && !done) pl = ld_relaxed<false>(&S->planned);
    if (have && nunits) arr = ld_relaxed_gpu32(&S->arrive[j % kPlanRing]);
    pl = __shfl_sync(0xffffffffu, pl, 0);
    if (!done && (planned_done(pl) || planned_items(pl) != ps)) {
      uint64_t p = 0;
      if (lane == 0) p = ld_acquire<false>(&S->planned);   // acquire the newer plans
      p = __shfl_sync(0xffffffffu, p, 0);
      ps = planned_items(p);
      done = planned_done(p);
      // headers of the newly planned items
      for (; hq < ps; hq += 32)
        if (hq + lane < ps) write_header(a, ctx, hq + lane, crc_tab);
      hq = ps;
    }
    if (i >= ps && done) break;
    if (!have && j < ps) {
      const Plan& p = ctx->plan[j % kPlanRing];
      flags = ld_cg32(&p.flags);
      dest = ld_cg32(&p.dest);
      nunits = ld_cg32(&p.nunits);
      slot = ld_cg32(&p.slot);
      slot_word = ld_cg64(&p.slot_word);
      tail_after = ld_cg64(&p.tail_after);
      have = true;
      if (nunits) arr = ld_relaxed_gpu32(&S->arrive[j % kPlanRing]);
    }
    const bool ready = have && (nunits == 0 || arr == nunits);
    const uint32_t notready = __ballot_sync(0xffffffffu, !ready);
    uint32_t run = notready ? __ffs(notready) - 1 : 32;
    const bool full = run == 32;
    // a run stays on one destination and ends at an Unlock
    const uint32_t dest0 = __shfl_sync(0xffffffffu, dest, 0);
    const uint32_t other = __ballot_sync(0xffffffffu, (uint32_t)lane < run && dest != dest0);
    if (other) run = min(run, (uint32_t)(__ffs(other) - 1));
    const uint32_t unl = __ballot_sync(0xffffffffu, (uint32_t)lane < run && (flags & kUnlock));
    if (unl) run = min(run, (uint32_t)__ffs(unl));
    if (run == 0) {
      if (pend) { flush(); continue; }
      const uint64_t t = globaltimer();
      if (a.engine) {            // batches planned after their items were published
        if (lane == 0) bdone = engine_advance_done(a.engine, bdone, i);
        __nanosleep(64);
      }
      if (!idle_since) idle_since = t;
      else if (t - idle_since > 2 * (a.engine ? kForeverNs : a.timeout_ns)) break;
      continue;
    }
    idle_since = 0;
    if (pend && dest0 != pend_dest) flush();
    const DestDesc& D = a.dests[dest0];
    const bool mine = (uint32_t)lane < run;
    if (D.rc) {
      // Reserve-then-commit (oracle/reserve.py): WL commits each reserved slot
      // (reserved -> busy, after the copies: fence), then the tail moves over
      // the leading run of committed slots -- ours or another sender's.
      if (pend) flush();
      if (D.sys) fence_acq_rel<true>(); else fence_acq_rel<false>();
      bool committed = false;
      if (mine && (flags & kEntry) && !(slot_word & kPad)) {
        const uint64_t want = kResvBit | (slot_word & kFLow);
        committed = dcas(D, slot_w(D, slot), want, slot_word) == want;
        if (!committed) {
          a.status[ld_cg32(&ctx->plan[j % kPlanRing].msg)] = RING_EDROPPED;   // reservation taken (TL)
          if (a.trace) {
            atomicAdd(reinterpret_cast<unsigned long long*>(a.trace + 1892), 1ull);
            a.trace[1893] = dld(D, slot_w(D, slot));
            a.trace[1894] = want;
          }
        }
      }
      const uint32_t cm = __ballot_sync(0xffffffffu, committed);
      if (cm) { rc_any = true; rc_last = __shfl_sync(0xffffffffu, slot, 31 - __clz(cm)); rc_dest = dest0; }
      __syncwarp();
      {
        rc_advance(a, D, lane, false, 0u);
        if (lane == 0) st_u32_relaxed_gpu(&S->pub_seq, i + run);
      }
      i += run;
      const uint32_t srcl = min((uint32_t)lane + run, 31u);
      const bool hv = __shfl_sync(0xffffffffu, have, srcl) && (uint32_t)lane + run < 32;
      flags = __shfl_sync(0xffffffffu, flags, srcl);
      dest = __shfl_sync(0xffffffffu, dest, srcl);
      nunits = __shfl_sync(0xffffffffu, nunits, srcl);
      slot = __shfl_sync(0xffffffffu, slot, srcl);
      slot_word = __shfl_sync(0xffffffffu, slot_word, srcl);
      tail_after = __shfl_sync(0xffffffffu, tail_after, srcl);
      have = hv;
      continue;
    }
    if (mine && (flags & kEntry) && D.mpsc) {   // WL: size + busy bit (PAD entries carry the pad bit)
      if (D.sys) st_relaxed<true>(slot_w(D, slot), slot_word);
      else st_relaxed<false>(slot_w(D, slot), slot_word);
    }
    const uint32_t entries = __ballot_sync(0xffffffffu, mine && (flags & kEntry));
    if (entries) {
      pend_tail = __shfl_sync(0xffffffffu, tail_after, 31 - __clz(entries));
      pend_entries = true;
    }
    pend = true;
    pend_dest = dest0;
    pend_n += run;
    const bool unlock_now = unl && (uint32_t)__ffs(unl) == run;
    pend_unlock = unlock_now;
    i += run;
    // slide the window by `run`
    const uint32_t src = min((uint32_t)lane + run, 31u);
    const bool h2 = __shfl_sync(0xffffffffu, have, src) && (uint32_t)lane + run < 32;
    flags = __shfl_sync(0xffffffffu, flags, src);
    dest = __shfl_sync(0xffffffffu, dest, src);
    nunits = __shfl_sync(0xffffffffu, nunits, src);
    slot = __shfl_sync(0xffffffffu, slot, src);
    slot_word = __shfl_sync(0xffffffffu, slot_word, src);
    tail_after = __shfl_sync(0xffffffffu, tail_after, src);
    have = h2;
    // keep accumulating only while whole windows complete
    if (!full || unlock_now || run < 32 || pend_n >= 96) flush();
  }
  if (pend) flush();
  if (a.engine && lane == 0) bdone = engine_advance_done(a.engine, bdone, i);
  // reserve-then-commit: the put returns once its entries are published --
  // waited for only here, after every commit of the launch (waiting per run
  // would hold back our later commits that other senders' entries wait on)
  if (rc_any) rc_advance(a, a.dests[rc_dest], lane, true, rc_last);
}

// One warp per CTA: the first kSpecRounds rounds' placement as the leader will
// decide it (place_round on the producer-local tail and a fresh head; round r
// starts from round r-1's last tail, as the leader's does), into shared memory
// for the CTA's copy warps.  n_units = 0 when not applicable.
__device__ void spec_first_round(const PutArgs& a, SpecRound* sp) {
  const int lane = threadIdx.x & 31;
  const DestDesc& D = a.dest0;
  // not under RING_TRY: an aborted message would shift every later placement
  const bool fast = !a.routes && a.n_dests == 1 && !D.mpsc && !D.ft && a.msgs && !(a.flags & RING_TRY);
  if (!fast) {
    if (lane == 0) { sp->n_units = 0; sp->n = 0; }
    return;
  }
  uint64_t P = 0, H = 0, P0 = 0;
  if (lane == 0) {
    P = __ldcg(reinterpret_cast<const unsigned long long*>(&D.st->tail_cache));
    // The tail is this launch's starting tail only until the leader finishes
    // and writes the new one; a CTA dispatched after that -- e.g. its SM was
    // held by another kernel -- would speculate into the NEXT launch's entries
    // and count the unit as done (a unit of this launch never copied).  The
    // previous launch's leader left this launch's starting tail in this
    // launch's counter set, which no one writes during the launch: speculate
    // only when the two agree (any other writer of the tail -- a routed
    // launch, the fused device put -- also makes them differ: no speculation).
    P0 = __ldcg(reinterpret_cast<const unsigned long long*>(&a.ctx->set[a.launch & 1].start_tail));
    H = read_head(D);
  }
  P = __shfl_sync(0xffffffffu, P, 0);
  P0 = __shfl_sync(0xffffffffu, P0, 0);
  H = __shfl_sync(0xffffffffu, H, 0);
  if (P != P0) {
    if (lane == 0) { sp->n_units = 0; sp->n = 0; }
    return;
  }
  uint32_t n_msgs = 0, units = 0, items = 0;
  for (int rnd = 0; rnd < kSpecRounds; ++rnd) {
    const uint32_t k0 = rnd * kGroup;
    if (k0 >= a.n) break;
    const uint32_t gmax = min((uint32_t)kGroup, a.n - k0);
    const bool act = (uint32_t)lane < gmax;
    uint64_t len = 0, src = 0;
    if (act) { len = a.msgs[k0 + lane].len; src = a.msgs[k0 + lane].src; }
    const uint64_t f = act ? footprint(len) : 0;
    if (__ballot_sync(0xffffffffu, act && (len >= (1ull << 32) || f > D.R))) break;   // the leader goes serial
    const RoundPlace r = place_round(P, H, act, f, act ? units_for(len, a.chunk) : 0, D);
    if (r.c) {
      SpecItem& it = sp->it[k0 + lane];
      it.src = src;
      it.dst = reinterpret_cast<uint64_t>(D.data + r.start + kHdr);
      RING_CHECK(r.start + footprint(len) <= D.R, "speculative entry inside R", r.start, len);
      it.len = len;
      it.first_unit = units + r.fu_off;
      it.nunits = r.nu;
      it.item = items + r.item_off;
    }
    n_msgs = k0 + r.run;
    units += r.nu_total;
    items += r.run + (r.pad_used ? 1u : 0u);
    if (r.run < (uint32_t)kGroup) break;                 // the next round starts elsewhere (credit)
    P = __shfl_sync(0xffffffffu, r.tail_after, 31);
  }
  if (lane == 0) { sp->n = n_msgs; sp->n_units = n_msgs ? units : 0; }
  if (a.trace && lane == 0 && blockIdx.x == 1) {
    a.trace[1880] = sp->n_units; a.trace[1881] = n_msgs; a.trace[1882] = H; a.trace[1883] = P;
    a.trace[1884] = globaltimer();
  }
}

// MODE 0: LSU copy warps; MODE 1: TMA engine warps; MODE 2: LSU
// copy warps with 32-B accesses (NVLink destinations).  Separate kernels, so
// one path's registers never change another's copy loop.
template <int MODE>
__global__ void __maxnreg__(96) put_kernel(const __grid_constant__ PutArgs a) {
  LaunchCtx* ctx = a.ctx;
  LaunchSet* S = &ctx->set[a.launch & 1];
  const int warp = threadIdx.x >> 5;
  __shared__ uint32_t s_crc[kCrcTableWords];
  __shared__ CopyShared cs;
  const int lane = threadIdx.x & 31;
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 120) a.trace[1920 + blockIdx.x] = globaltimer();
  if (threadIdx.x == 0) {
    cs.pl = 0;
    cs.owner = 0;
    // the block of first units of this CTA's copy warps (copy_mode 0)
    const uint32_t ncw = (blockDim.x >> 5) - (blockIdx.x == 0 ? 2u : 0u);
    if (MODE != 1) cs.first = atomicAdd(&S->next_unit, ncw);
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    if (a.trace && threadIdx.x == 0) a.trace[252] = globaltimer();
    if (warp == 0) {
      reset_set(&ctx->set[(a.launch + 1) & 1], lane);
      if (a.dest0.ft && !a.routes) ft_put(a, ctx, S, s_crc);
      else put_leader(a, ctx, S);
      return;
    }
    if (warp == 1) {   // the publisher writes the headers: it holds the CRC tables
      for (int i = lane; i < kCrcTableWords; i += 32) s_crc[i] = a.crc_table[i];
      __syncwarp();
      put_publisher(a, ctx, S, s_crc);
      if (a.trace && lane == 0) a.trace[253] = globaltimer();
      return;
    }
  }
  __shared__ SpecRound spec;
  if (MODE == 1) {
    // TMA engines: every warp of the CTA but CTA 0's two control warps drives
    // its own ring of kEngineStages shared-memory stages (a warp blocks while
    // it waits for a store to complete before its arrive; the others keep
    // their copies in flight).  The first engine warp evaluates the first round.
    extern __shared__ __align__(128) uint8_t dyn_smem[];
    const int ew = warp - (blockIdx.x == 0 ? 2 : 0);
    const int n_ew = min((int)(blockDim.x >> 5) - (blockIdx.x == 0 ? 2 : 0), kMaxEngineWarps);
    if (ew < 0 || ew >= n_ew) return;
    if (ew == 0) spec_first_round(a, &spec);
    asm volatile("bar.sync 3, %0;" ::"r"(n_ew * 32) : "memory");
    copy_engine<kEngineStages>(ctx, S, a.chunk, a.timeout_ns, dyn_smem + (size_t)ew * kEngineStages * a.chunk, &spec,
                               ew);
    return;
  }
  // the CTA's first copy warp evaluates the first round; the copy warps meet
  // on named barrier 2 (CTA 0's control warps never wait for it)
  const uint32_t ncopy = blockDim.x - (blockIdx.x == 0 ? 64u : 0u);
  if (warp == (blockIdx.x == 0 ? 2 : 0)) spec_first_round(a, &spec);
  asm volatile("bar.sync 2, %0;" ::"r"(ncopy) : "memory");
  copy_warp<MODE == 2 ? 2 : 1>(ctx, S, &cs, a.chunk, a.engine ? kForeverNs : a.timeout_ns, a.trace, &spec);
}

// With CUDA's lazy module loading, the first launch of a kernel loads it, and
// loading waits for kernels already running on the device.  A consumer kernel
// spinning for data would then block the producer's first launch until it
// times out; so every kernel is loaded when a device is first used.

// ---- persistent engine: doorbell / stop (one thread, on the submitting stream) ----
// Batch b goes to slot b % kEngineQueue once the engine is done with batch
// b - kEngineQueue and batch b - 1 is posted (doorbells on several streams
// still post in submission order); then `posted` = b + 1 is released.  With
// `wait`, the kernel returns once the batch is published (stream semantics of
// a put launch); on a timeout the remaining statuses are left to the engine.
__global__ void engine_doorbell_kernel(EngineQueue* q, uint64_t b, const ring_msg_t* msgs, uint32_t* status,
                                       uint32_t n, uint32_t flags, uint32_t wait, uint64_t timeout_ns) {
  __shared__ uint32_t rejected;
  if (threadIdx.x == 0) {
    rejected = 1;
    const uint64_t t0 = globaltimer();
    while (true) {
      const uint64_t c = ld_acquire<false>(&q->ctl);
      if (c & kEngineClosed) break;                      // closed: the batch is not taken
      if (c == b && ld_acquire<false>(&q->done) + kEngineQueue > b) {
        EngineBatch& e = q->batch[b % kEngineQueue];
        e.msgs = msgs;
        e.status = status;
        e.n = n;
        e.flags = flags;
        __threadfence();                                 // the slot before the count
        if (atomicCAS(reinterpret_cast<unsigned long long*>(&q->ctl), b, b + 1) == b) rejected = 0;
        break;
      }
      if (globaltimer() - t0 > timeout_ns) break;
    }
    if (!rejected && wait)
      while (ld_acquire<false>(&q->done) <= b)
        if (globaltimer() - t0 > 2 * timeout_ns) break;
  }
  __syncwarp();
  if (rejected)
    for (uint32_t k = threadIdx.x; k < n; k += 32) status[k] = RING_ECLOSED;
}
__global__ void engine_stop_kernel(EngineQueue* q) {
  if (threadIdx.x == 0) {
    unsigned long long c = ld_acquire<false>(&q->ctl);
    while (!(c & kEngineClosed)) {
      const unsigned long long o = atomicCAS(reinterpret_cast<unsigned long long*>(&q->ctl), c, c | kEngineClosed);
      if (o == c) break;
      c = o;
    }
  }
}
__global__ void engine_wait_kernel(EngineQueue* q, uint64_t upto, uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = globaltimer();
  while (true) {
    const uint64_t c = ld_acquire<false>(&q->ctl), d = ld_acquire<false>(&q->done);
    if (d >= upto || ((c & kEngineClosed) && d >= (c & ~kEngineClosed))) return;
    if (globaltimer() - t0 > timeout_ns) return;
  }
}

// NodeManager reassignment (router_set_route), stream-ordered
// and without a host round trip: the new route (and a new destination's
// descriptor) travel in the kernel parameters; the destinations, the set size
// and the app / stage are written first, the epoch last with a release -- the
// device-side epoch flip a reader acquiring the epoch sees whole.  The
// round-robin counter and the admission state stay device-owned.
__global__ void route_update_kernel(Route* d, const Route nr, DestDesc* desc_slot, const DestDesc desc,
                                    uint32_t new_dest) {
  if (threadIdx.x != 0) return;
  if (new_dest) *desc_slot = desc;
  for (int i = 0; i < kMaxDests; ++i) d->dests[i] = nr.dests[i];
  d->app_id = nr.app_id;
  d->stage = nr.stage;
  d->n = nr.n;
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&d->epoch), "r"(nr.epoch) : "memory");
}
cudaError_t launch_route_update(Route* d, const Route& nr, DestDesc* desc_slot, const DestDesc* desc, cudaStream_t s) {
  route_update_kernel<<<1, 32, 0, s>>>(d, nr, desc_slot, desc ? *desc : DestDesc{}, desc ? 1u : 0u);
  return cudaGetLastError();
}

cudaError_t launch_engine_doorbell(EngineQueue* q, uint64_t b, const ring_msg_t* msgs, uint32_t* status, uint32_t n,
                                   uint32_t flags, bool wait, uint64_t timeout_ns, cudaStream_t s) {
  engine_doorbell_kernel<<<1, 32, 0, s>>>(q, b, msgs, status, n, flags, wait ? 1u : 0u, timeout_ns);
  return cudaGetLastError();
}
cudaError_t launch_engine_stop(EngineQueue* q, cudaStream_t s) {
  engine_stop_kernel<<<1, 32, 0, s>>>(q);
  return cudaGetLastError();
}
cudaError_t launch_engine_wait(EngineQueue* q, uint64_t upto, uint64_t timeout_ns, cudaStream_t s) {
  engine_wait_kernel<<<1, 32, 0, s>>>(q, upto, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_put(const PutArgs& a, uint32_t ctas, uint32_t threads, cudaStream_t s) {
  const size_t dyn = a.copy_mode == 1 ? (size_t)kMaxEngineWarps * kEngineStages * a.chunk : 0;
  if (a.copy_mode == 1) put_kernel<1><<<ctas, 32u * (kMaxEngineWarps < 3 ? 3 : kMaxEngineWarps), dyn, s>>>(a);
  else if (a.dest0.sys && !a.routes) put_kernel<2><<<ctas, threads, 0, s>>>(a);
  else put_kernel<0><<<ctas, threads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t preload_put() {
  cudaError_t e = preload_kernel(put_kernel<0>);
  if (e == cudaSuccess) e = preload_kernel(engine_doorbell_kernel);
  if (e == cudaSuccess) e = preload_kernel(route_update_kernel);
  if (e == cudaSuccess) e = preload_kernel(engine_stop_kernel);
  if (e == cudaSuccess) e = preload_kernel(engine_wait_kernel);
  if (e == cudaSuccess) e = preload_kernel(put_kernel<1>, (int)cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) e = preload_kernel(put_kernel<2>);
  if (e == cudaSuccess)   // TMA engine stages (up to kEngineStages x 48 KiB)
    e = cudaFuncSetAttribute(put_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEngineSmem);
  return e;
}

}  // namespace b200ring
