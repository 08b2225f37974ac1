/*
 * b200ring_device.cuh — device-side put for producer kernels.
 *
 * A stage kernel that produces a tensor for the next stage can write it
 * straight into the peer ring and publish it itself (the
 * TaskWorker's result goes to the ResultDeliver; here without an intermediate
 * buffer or a separate put launch).  Host side: ring_peer_device_view() fills
 * a ring_dev_peer_t (b200ring.h) for a single-producer attachment; pass it to
 * the kernel by value.  Device side, ONE message per launch, every thread of
 * every CTA calls:
 *
 *   using namespace b200ring::stage;
 *   StageCtl* ctl = reinterpret_cast<StageCtl*>(peer.ctl);
 *   uint64_t P = grid_reserve<SYS>(peer, ctl, len, timeout_ns); // steps 2-4 (CTA 0), broadcast
 *   if (P) { uint8_t* out = payload_ptr(peer, P); ... write len bytes ... }   // step 5 (WB)
 *   grid_commit<SYS>(peer, ctl, P, len, hdr, flags, d_status);  // header, WL, UH (last CTA)
 *
 * SYS = (peer.sys != 0): system-scope ordering when the ring lives on another
 * GPU.  CTA 0 must be able to make progress while the others wait for the
 * placement (it is scheduled first); the consumer must run concurrently if the
 * ring can be full.  Self-contained (b200ring.h + b200ring_layout.cuh); the
 * library's own fused stage (ring_stage_scale_bf16_put) is built on it.
 */
// Implementation notes: a device-side put for producer kernels that write
// their output into the peer ring ("ring_put_dev as the epilogue
// of the producing stage's last kernel ... saving a HBM read + a launch";
// the TaskWorker hands its result to the ResultDeliver).
//
// The sender steps split around the stage's own stores:
//   reserve  (one thread, CTA 0): steps 2-4 on an SPSC attachment -- tail
//            from the producer-local cache, credit from the head mirror, PAD
//            at the wrap (published at once, R3), wait for credit (R12);
//            the placement is broadcast to the grid through `ctl`;
//   (the stage's threads write the payload at data + start + 64: step 5, WB)
//   commit   (the last CTA to finish): header + CRC-32 (R10/R11), WL, one
//            fence, UH; producer-local tail / channel counter advanced.
// Single-producer attachments only (the lock is elided, R14); a fused put
// must not run concurrently with ring_put* on the same attachment.
#pragma once
#include "b200ring.h"
#include "b200ring_layout.cuh"

namespace b200ring {
namespace stage {

// Grid coordination words of one attachment (device memory, 128 B).  Reset
// by the committing CTA, so consecutive stream-ordered launches start clean.
struct alignas(128) StageCtl {
  uint64_t P;          // tail word at the entry (placement)
  uint32_t ready;      // 1 once P is valid (release)
  uint32_t status;     // RING_OK / RING_EMSGSIZE / RING_ETIMEDOUT
  uint32_t done;       // CTAs finished writing
  uint32_t _p[27];
};
static_assert(sizeof(StageCtl) == 128, "StageCtl");

template <bool SYS>
__device__ __forceinline__ uint64_t head_of(const ring_dev_peer_t& p) {
  const DestState* st = reinterpret_cast<const DestState*>(p.state);
  const uint64_t m = ld_acquire<SYS>(&st->mirror_head);
  if (m & kMirrorValid) return m & ~kMirrorValid;
  return ld_acquire<SYS>(reinterpret_cast<const uint64_t*>(p.ring + kHeadOff));
}

// Steps 2-4 for one entry of `len` payload bytes (called by one thread).
template <bool SYS>
__device__ uint32_t reserve_one(const ring_dev_peer_t& p, uint64_t len, uint64_t timeout_ns, uint64_t* P_out) {
  DestState* st = reinterpret_cast<DestState*>(p.state);
  uint8_t* ring = reinterpret_cast<uint8_t*>(p.ring);
  const uint64_t f = footprint(len);
  if (len >= (1ull << 32) || f > p.R) return RING_EMSGSIZE;
  uint64_t P = st->tail_cache;
  uint64_t H = head_of<SYS>(p);
  const uint64_t t0 = globaltimer();
  while (true) {
    const uint64_t pb = ptr_off(P), hb = ptr_off(H);
    const uint32_t pq = ptr_seq(P), hq = ptr_seq(H);
    bool full = seq_dist(pq, hq) >= p.N;
    if (!full && pb + f > p.R) {
      if (span_free(pb, pq, hb, hq, p.R - pb)) {          // PAD [pb, R) (R3), published at once
        uint64_t* slot = reinterpret_cast<uint64_t*>(ring + kSlotsOff) + (pq & (p.N - 1));
        st_relaxed<SYS>(slot, kBusy | kPad | (p.R - pb));
        P = pack_ptr(0, seq_inc(pq));
        st_release<SYS>(reinterpret_cast<uint64_t*>(ring + kTailOff), P);
        st->tail_cache = P;
        continue;
      }
      full = true;
    } else if (!full && !span_free(pb, pq, hb, hq, f)) {
      full = true;
    }
    if (!full) break;
    const uint64_t H2 = head_of<SYS>(p);                  // wait for credit (R12)
    if (H2 == H && globaltimer() - t0 > timeout_ns) return RING_ETIMEDOUT;
    H = H2;
  }
  *P_out = P;
  return RING_OK;
}

// WL + UH for the reserved entry, after its payload is complete (one thread;
// the caller has ordered the grid's payload stores before this call).
template <bool SYS>
__device__ void commit_one(const ring_dev_peer_t& p, uint64_t P, uint64_t len, const ring_hdr_t& h, uint32_t flags) {
  DestState* st = reinterpret_cast<DestState*>(p.state);
  uint8_t* ring = reinterpret_cast<uint8_t*>(p.ring);
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(p.crc_table);
  const uint64_t f = footprint(len);
  const uint64_t start = ptr_off(P);
  const uint32_t pq = ptr_seq(P);
  // header (R11) + CRC over [4, 56) (R10)
  uint32_t w[16];
  const uint32_t* uid = reinterpret_cast<const uint32_t*>(h.uid);
  const uint32_t len32 = (uint32_t)len;
  w[1] = uid[0]; w[2] = uid[1]; w[3] = uid[2]; w[4] = uid[3];
  w[5] = (uint32_t)h.accepted_at;
  w[6] = (uint32_t)(h.accepted_at >> 32);
  w[7] = h.app_id;
  w[8] = (uint32_t)h.stage | (len32 << 16);
  w[9] = len32 >> 16;
  w[10] = 0;
  w[11] = p.producer_id;
  w[12] = (uint32_t)st->chan_seq;
  w[13] = 0;
  w[0] = crc52(w, tab);
  const uint64_t t = (flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
  w[14] = (uint32_t)t;
  w[15] = (uint32_t)(t >> 32);
  uint8_t* hd = reinterpret_cast<uint8_t*>(p.data) + start;
#pragma unroll
  for (int q = 0; q < 4; ++q) st16(hd + 16 * q, make_int4((int)w[4 * q], (int)w[4 * q + 1], (int)w[4 * q + 2], (int)w[4 * q + 3]));
  uint64_t* slot = reinterpret_cast<uint64_t*>(ring + kSlotsOff) + (pq & (p.N - 1));
  st_relaxed<SYS>(slot, kBusy | f);                                  // WL (step 6)
  const uint64_t T = pack_ptr(advance(start, f, p.R), seq_inc(pq));
  st_release<SYS>(reinterpret_cast<uint64_t*>(ring + kTailOff), T);   // UH (step 7): fence + store
  st->tail_cache = T;
  st->chan_seq = st->chan_seq + 1;
}

// A reservation as returned to the stage's threads: the tail word at the
// entry with bit 63 set (tail offsets are < 2^39, so bit 63 is free); 0 = none.
constexpr uint64_t kReserved = 1ull << 63;

// Grid-wide protocol for a fused stage kernel writing ONE message:
//   const uint64_t P = grid_reserve(p, ctl, len, timeout);   // every thread
//   ... write payload bytes at payload_ptr(p, P) ...
//   grid_commit(p, ctl, len, hdr, flags, status);            // every thread
// Returns the placement to every thread of every CTA (0 on failure; then the
// status is in ctl->status and nothing must be written).
template <bool SYS>
__device__ uint64_t grid_reserve(const ring_dev_peer_t& p, StageCtl* ctl, uint64_t len, uint64_t timeout_ns) {
  __shared__ uint64_t s_P;
  if (threadIdx.x == 0) {
    uint64_t P = 0;
    if (blockIdx.x == 0) {
      const uint32_t s = reserve_one<SYS>(p, len, timeout_ns, &P);
      P = s == RING_OK ? (P | kReserved) : 0;
      ctl->P = P;
      ctl->status = s;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&ctl->ready), "r"(1u) : "memory");
    } else {
      const uint64_t t0 = globaltimer();
      while (ld_acquire_gpu32(&ctl->ready) == 0u)
        if (globaltimer() - t0 > 2 * timeout_ns) break;
      P = ctl->status == RING_OK ? ctl->P : 0;
    }
    s_P = P;
  }
  __syncthreads();
  return s_P;
}

__device__ __forceinline__ uint8_t* payload_ptr(const ring_dev_peer_t& p, uint64_t P) {
  return reinterpret_cast<uint8_t*>(p.data) + ptr_off(P & ~kReserved) + kHdr;
}

template <bool SYS>
__device__ void grid_commit(const ring_dev_peer_t& p, StageCtl* ctl, uint64_t P, uint64_t len, const ring_hdr_t& h,
                            uint32_t flags, uint32_t* status) {
  __syncthreads();                          // this CTA's payload stores precede its arrival
  if (threadIdx.x == 0) {
    if (SYS) __threadfence_system(); else __threadfence();
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&ctl->done) : "memory");
    if (prev + 1 == gridDim.x) {            // last CTA: every payload store is ordered before this point
      const uint32_t s = ctl->status;
      if (s == RING_OK && P) commit_one<SYS>(p, P & ~kReserved, len, h, flags);
      if (status) *status = s;
      ctl->ready = 0;                       // reset for the next stream-ordered launch
      ctl->done = 0;
      ctl->P = 0;
    }
  }
}

}  // namespace stage
}  // namespace b200ring
