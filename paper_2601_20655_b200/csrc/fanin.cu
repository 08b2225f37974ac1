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

template <bool SYS>
__global__ void __launch_bounds__(32) set_consume_kernel(const SetArgs a) {
  __shared__ uint32_t s_crc[kCrcTableWords];
  const int lane = threadIdx.x;
  for (int i = lane; i < kCrcTableWords; i += 32) s_crc[i] = a.crc_table[i];
  __syncwarp();
  const bool mine = (uint32_t)lane < a.k;
  SetRing rg{};
  uint64_t G = 0, H = 0;
  if (mine) {
    rg = a.rings[lane];
    G = ld_cg64(reinterpret_cast<const uint64_t*>(rg.ring + kCursorOff));
    H = ld_cg64(reinterpret_cast<const uint64_t*>(rg.ring + kHeadOff));
  }
  uint32_t got = 0, rot = a.rr % max(a.k, 1u);
  uint64_t idle_since = 0;
  while (got < a.n) {
    // ---- steps 1-2 on every ring at once: tail past the cursor?
    bool has = false;
    uint64_t w = 0;
    if (mine) {
      const uint64_t T = ld_acquire<SYS>(reinterpret_cast<const uint64_t*>(rg.ring + kTailOff));
      has = ptr_seq(T) != ptr_seq(G);
      if (has) w = ld_relaxed<SYS>(reinterpret_cast<const uint64_t*>(rg.ring + kSlotsOff) + (ptr_seq(G) & (rg.N - 1)));
    }
    const bool pad = has && (w & kPad);
    const uint64_t f = w & ((1ull << 40) - 1);
    // a PAD at a ring's cursor is stepped over and freed at once (R3)
    bool msg = has && !pad;
    // at most n - got messages this round, taken in rotated lane order
    const uint32_t want = __ballot_sync(0xffffffffu, msg);
    const uint32_t rotl = (want >> rot) | (rot ? (want << (32 - rot)) : 0u);   // bit j = lane (rot + j) % 32
    const uint32_t lane_r = ((uint32_t)lane + 32u - rot) & 31u;                // my position in rotated order
    const uint32_t before = __popc(rotl & ((1u << lane_r) - 1u));
    if (msg && before >= a.n - got) msg = false;
    const uint32_t take = __ballot_sync(0xffffffffu, msg);
    if (!take && !__ballot_sync(0xffffffffu, pad)) {
      if (a.flags & RING_TRY) break;
      const uint64_t t = globaltimer();
      if (!idle_since) idle_since = t;
      else if (t - idle_since > a.timeout_ns) break;
      continue;
    }
    idle_since = 0;
    const uint64_t start = ptr_off(G);
    if (msg) {
      // ---- step 3: header + checksum, view (slot in rotated order)
      const int4* hp = reinterpret_cast<const int4*>(rg.data + start);
      uint32_t hw[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 v = __ldcg(hp + q);
        hw[4 * q] = (uint32_t)v.x; hw[4 * q + 1] = (uint32_t)v.y; hw[4 * q + 2] = (uint32_t)v.z; hw[4 * q + 3] = (uint32_t)v.w;
      }
      uint64_t len = (hw[8] >> 16) | ((uint64_t)(hw[9] & 0xffffu) << 16);
      uint32_t status = RING_OK;
      if (crc52(hw, s_crc) != hw[0] || kHdr + len > f) { status = RING_ECORRUPT; len = 0; }
      const uint32_t rotk = (take >> rot) | (rot ? (take << (32 - rot)) : 0u);
      const uint32_t slot_out = got + __popc(rotk & ((1u << lane_r) - 1u));
      ring_view_t* v = a.views + slot_out;
      v->offset = start + kHdr;
      v->len = len;
      v->footprint = f;
      v->start = start;
      v->slot_seq = ptr_seq(G);
      v->status = status;
      v->t_visible = (a.flags & RING_NO_TIMESTAMP) ? 0 : globaltimer();
      v->reserved[0] = lane;
      v->reserved[1] = 0;
      int4* vh = reinterpret_cast<int4*>(v->header);
#pragma unroll
      for (int q = 0; q < 4; ++q) vh[q] = make_int4((int)hw[4 * q], (int)hw[4 * q + 1], (int)hw[4 * q + 2], (int)hw[4 * q + 3]);
      if (a.ring_idx) a.ring_idx[slot_out] = lane;
    }
    // ---- steps 4-5 per ring: busy bit, head, credit mirror
    if (msg || pad) {
      st_relaxed<SYS>(reinterpret_cast<uint64_t*>(rg.ring + kSlotsOff) + (ptr_seq(G) & (rg.N - 1)), 0ull);
      G = pack_ptr(advance(start, f, rg.R), seq_inc(ptr_seq(G)));
      H = G;
      fence_acq_rel<SYS>();
      st_relaxed<SYS>(reinterpret_cast<uint64_t*>(rg.ring + kHeadOff), H);
      uint64_t* m = rg.mirrors[0];
      if (m) st_relaxed<SYS>(m, H | kMirrorValid);
    }
    got += __popc(take);
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
  if (mine) *reinterpret_cast<uint64_t*>(rg.ring + kCursorOff) = G;
}

cudaError_t preload_fanin() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, set_consume_kernel<true>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, set_consume_kernel<false>);
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
