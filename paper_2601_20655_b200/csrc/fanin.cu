// fanin.cu — lock-free fan-in: instead of one MPSC ring
// whose producers serialise on the paper's lock, every
// producer gets its own single-producer ring (lock elided, R14) on the
// consumer GPU and ONE consumer warp serves all of them: lane i owns ring i,
// polls its tail (R7) and, when data is there, runs the receiver steps 1-5
// on it -- slot, header, CRC, view,
// busy bit, head, credit mirror -- all rings in parallel, one entry per ring
// per round.  Rounds start at a rotating lane so no producer is starved.
// Per-channel order is each ring's FIFO order; the merged order is the
// consumer's round order (reported through d_ring_idx).
#include "ring_copy.cuh"

namespace b200ring {

struct SetRing {
  uint8_t* ring;
  uint8_t* data;
  uint64_t** mirrors;    // the ring's device array of producer mirror pointers (slot 0: the producer)
  uint64_t R;
  uint32_t N;
  uint32_t _p;
};

struct SetArgs {
  const SetRing* rings;
  ring_view_t* views;
  uint32_t* ring_idx;
  const uint32_t* crc_table;
  uint64_t timeout_ns;
  uint32_t k;            // rings (<= 32)
  uint32_t n;            // messages to consume
  uint32_t flags;
  uint32_t rr;           // first lane of the first round (rotates across launches)
};

// Round structure: lane i < k polls ring i's tail; the round's 32 lanes are
// then dealt out over the rings that have entries, one at a time in rotated
// ring order (so each ring gets a fair share and a ring with a backlog gets
// several lanes), each lane taking the next entry of its ring.  A ring's lanes
// are contiguous: a segmented prefix sum of their footprints gives every
// entry's start (PAD entries fill every wrap, R3), the last lane of a ring
// moves its head and pushes the credit.
template <bool SYS>
__global__ void __launch_bounds__(32) set_consume_kernel(const SetArgs a) {
  __shared__ uint32_t s_crc[kCrcTableWords];
  __shared__ uint32_t s_ring[32], s_idx[32];
  const int lane = threadIdx.x;
  for (int i = lane; i < kCrcTableWords; i += 32) s_crc[i] = a.crc_table[i];
  __syncwarp();
  const bool mine = (uint32_t)lane < a.k;
  SetRing own{};
  uint64_t G = 0;                        // cursor of ring `lane` (lanes < k)
  if (mine) {
    own = a.rings[lane];
    G = ld_cg64(reinterpret_cast<const uint64_t*>(own.ring + kCursorOff));
  }
  uint32_t got = 0, rot = a.rr % max(a.k, 1u);
  uint64_t idle_since = 0;
  while (got < a.n) {
    // ---- steps 1-2 on every ring: entries published past the cursor
    uint32_t avail = 0;
    if (mine) {
      const uint64_t T = ld_acquire<SYS>(reinterpret_cast<const uint64_t*>(own.ring + kTailOff));
      avail = seq_dist(ptr_seq(T), ptr_seq(G));
    }
    if (!__ballot_sync(0xffffffffu, avail)) {
      if (a.flags & RING_TRY) break;
      const uint64_t t = globaltimer();
      if (!idle_since) idle_since = t;
      else if (t - idle_since > a.timeout_ns) break;
      continue;
    }
    idle_since = 0;
    // ---- deal lanes over rings (lane 0): at most n - got entries this round
    uint32_t av[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) av[r] = __shfl_sync(0xffffffffu, avail, r);
    if (lane == 0) {
      uint32_t take[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) take[r] = 0;
      uint32_t used = 0, budget = min(32u, a.n - got);
      bool progress = true;
      while (used < budget && progress) {
        progress = false;
        for (uint32_t j = 0; j < a.k && used < budget; ++j) {
          const uint32_t r = (rot + j) % a.k;
          if (take[r] < av[r]) { ++take[r]; ++used; progress = true; }
        }
      }
      uint32_t l = 0;
      for (uint32_t j = 0; j < a.k; ++j) {            // contiguous lanes per ring, rotated ring order
        const uint32_t r = (rot + j) % a.k;
        for (uint32_t e = 0; e < take[r]; ++e, ++l) { s_ring[l] = r; s_idx[l] = e; }
      }
      for (; l < 32; ++l) { s_ring[l] = 0xffffffffu; s_idx[l] = 0; }
    }
    __syncwarp();
    const uint32_t r = s_ring[lane], e = s_idx[lane];
    const bool act = r != 0xffffffffu;
    // this lane's ring: cursor from the owning lane, ring fields
    const uint64_t Gr = __shfl_sync(0xffffffffu, G, act ? r : 0);
    SetRing rg{};
    if (act) rg = a.rings[r];
    const uint32_t q = (ptr_seq(Gr) + e) & kSeqMask;
    uint64_t w = 0;
    if (act) w = ld_relaxed<SYS>(reinterpret_cast<const uint64_t*>(rg.ring + kSlotsOff) + (q & (rg.N - 1)));
    const uint64_t f = act ? (w & kFLow) : 0;
    const bool pad = act && (w & kPad);
    // segmented prefix sum of footprints within each ring's lanes
    uint64_t incl = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      const uint32_t ry = __shfl_up_sync(0xffffffffu, r, o);
      if (lane >= o && ry == r && e >= (uint32_t)o) incl += y;
    }
    uint64_t start = ptr_off(Gr) + (incl - f);
    if (act && start >= rg.R) start -= rg.R;
    // ---- step 3: header + checksum, view (in lane order: ring-major, FIFO within a ring)
    const bool msg = act && !pad;
    const uint32_t msgs_before = __popc(__ballot_sync(0xffffffffu, msg) & ((1u << lane) - 1u));
    if (msg) {
      const int4* hp = reinterpret_cast<const int4*>(rg.data + start);
      uint32_t hw[16];
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const int4 v = __ldcg(hp + qq);
        hw[4 * qq] = (uint32_t)v.x; hw[4 * qq + 1] = (uint32_t)v.y; hw[4 * qq + 2] = (uint32_t)v.z; hw[4 * qq + 3] = (uint32_t)v.w;
      }
      uint64_t len = (hw[8] >> 16) | ((uint64_t)(hw[9] & 0xffffu) << 16);
      uint32_t status = RING_OK;
      if (crc52(hw, s_crc) != hw[0] || kHdr + len > f) { status = RING_ECORRUPT; len = 0; }
      const uint32_t slot_out = got + msgs_before;
      ring_view_t* v = a.views + slot_out;
      v->offset = start + kHdr;
      v->len = len;
      v->footprint = f;
      v->start = start;
      v->slot_seq = q;
      v->status = status;
      v->t_visible = (a.flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
      v->reserved[0] = r;
      v->reserved[1] = 0;
      int4* vh = reinterpret_cast<int4*>(v->header);
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) vh[qq] = make_int4((int)hw[4 * qq], (int)hw[4 * qq + 1], (int)hw[4 * qq + 2], (int)hw[4 * qq + 3]);
      if (a.ring_idx) a.ring_idx[slot_out] = r;
    }
    // ---- steps 4-5: busy bits, then each ring's last lane moves its head and pushes the credit
    if (act) st_relaxed<SYS>(reinterpret_cast<uint64_t*>(rg.ring + kSlotsOff) + (q & (rg.N - 1)), 0ull);
    const uint32_t r_next = __shfl_down_sync(0xffffffffu, r, 1);
    const bool last_of_ring = act && (lane == 31 || r_next != r);
    __syncwarp();
    uint64_t newG = 0;
    if (last_of_ring) {
      uint64_t hb = start + f;
      if (hb >= rg.R) hb -= rg.R;
      newG = pack_ptr(hb, q + 1);
      fence_acq_rel<SYS>();
      st_relaxed<SYS>(reinterpret_cast<uint64_t*>(rg.ring + kHeadOff), newG);
      uint64_t* m = rg.mirrors[0];
      if (m) st_relaxed<SYS>(m, newG | kMirrorValid);
    }
    // the owning lane of each ring takes the new cursor
    const uint32_t lastmask = __ballot_sync(0xffffffffu, last_of_ring);
    for (uint32_t mm = lastmask; mm; mm &= mm - 1) {
      const int src = __ffs(mm) - 1;
      const uint32_t rr = __shfl_sync(0xffffffffu, r, src);
      const uint64_t ng = __shfl_sync(0xffffffffu, newG, src);
      if ((uint32_t)lane == rr) G = ng;
    }
    got += __popc(__ballot_sync(0xffffffffu, msg));
    rot = (rot + 1) % max(a.k, 1u);
  }
  // views of messages not received (RING_TRY: EMPTY; timeout)
  const uint32_t fail = (a.flags & RING_TRY) ? RING_EMPTY : RING_ETIMEDOUT;
  for (uint32_t q = got + lane; q < a.n; q += 32) {
    ring_view_t* v = a.views + q;
    v->offset = 0; v->len = 0; v->footprint = 0; v->start = 0; v->slot_seq = 0;
    v->status = fail; v->t_visible = 0;
    if (a.ring_idx) a.ring_idx[q] = 0xffffffffu;
  }
  if (mine) *reinterpret_cast<uint64_t*>(own.ring + kCursorOff) = G;
}

cudaError_t preload_fanin() {
  cudaError_t e = preload_kernel(set_consume_kernel<true>);
  if (e == cudaSuccess) e = preload_kernel(set_consume_kernel<false>);
  return e;
}

cudaError_t launch_set_consume(const SetRing* rings, uint32_t k, ring_view_t* views, uint32_t* ring_idx, uint32_t n,
                               const uint32_t* crc, uint32_t flags, uint64_t timeout_ns, uint32_t rr, bool sys,
                               cudaStream_t s) {
  SetArgs a{};
  a.rings = rings;
  a.views = views;
  a.ring_idx = ring_idx;
  a.crc_table = crc;
  a.timeout_ns = timeout_ns;
  a.k = k;
  a.n = n;
  a.flags = flags;
  a.rr = rr;
  if (sys) set_consume_kernel<true><<<1, 32, 0, s>>>(a);
  else set_consume_kernel<false><<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace b200ring
