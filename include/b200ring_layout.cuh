// b200ring_layout.cuh — device-side layout, word packing and memory-ordering
// primitives of the B200 double ring (sm_100a), shared by the library's
// kernels and by producer kernels that put from the device (b200ring_device.cuh).
//
// Layout ("lock region, fixed-length header
// with head and tail, buffer region, size region"):
//   [0,128)   lock  u64   0 = free, producer_id+1 = held          (R14)
//   [128,256) tail  u64   (P_b << 24) | P_seq                      (R8, R5)
//   [256,384) head  u64   (H_b << 24) | H_seq
//   [384,512) read cursor G u64 (consumer private)
//   [512, 512+8N) size slots u64: busy<<63 | pad<<62 | footprint   (R9, R3)
//   [D, D+R)  buffer region, D = align_up(512 + 8N, 4096)
#pragma once
#include <cstdint>

namespace b200ring {

constexpr uint64_t kLockOff = 0;
constexpr uint64_t kTailOff = 128;
constexpr uint64_t kHeadOff = 256;
constexpr uint64_t kCursorOff = 384;
constexpr uint64_t kSlotsOff = 512;
constexpr uint64_t kAlign = 128;     // entry alignment (R11)
constexpr uint64_t kHdr = 64;        // entry header bytes (R11)
constexpr uint64_t kBusy = 1ull << 63;
constexpr uint64_t kPad = 1ull << 62;
// Footprint bits of a size slot: 0-39 (R < 2^39, R8).  Fault-tolerant rings
// keep a 22-bit sequence tag in bits 40-61 (R21), so every reader masks the
// footprint with kFLow, never with the full 62 bits.
constexpr int kTagShift = 40;
constexpr uint64_t kTagMask = (1ull << 22) - 1;
constexpr uint64_t kFLow = (1ull << kTagShift) - 1;
constexpr uint64_t kResvBit = 1ull << 61;   // reserve-then-commit: slot claimed, entry not committed yet
constexpr uint64_t kResvOff = 64;          // reservation frontier word (lock line; written under the lock)
constexpr uint32_t kSeqMask = (1u << 24) - 1;
constexpr int kPlanRing = 128;       // in-flight items (entries) per launch context
constexpr int kGroup = 32;           // messages planned per leader round (one per lane)
constexpr int kMaxDests = 8;          // destinations per route
constexpr int kMaxRouterDests = 32;   // destinations per launch (bit mask)

__host__ __device__ inline uint64_t data_offset(uint32_t n_slots) {
  return (kSlotsOff + 8ull * n_slots + 4095ull) & ~4095ull;
}
// Split placement (ring_create_split): a copy of each entry header, indexed by
// slot, follows the size region in the consumer's control allocation.
__host__ __device__ inline uint64_t hdr_mirror_offset(uint32_t n_slots) {
  return (kSlotsOff + 8ull * n_slots + 127) / 128 * 128;
}
__host__ __device__ inline uint64_t split_control_bytes(uint32_t n_slots) {
  return (hdr_mirror_offset(n_slots) + 64ull * n_slots + 4095) / 4096 * 4096;
}
// f = align_up(64 + len, 128)  (R9)
__host__ __device__ inline uint64_t footprint(uint64_t len) { return (kHdr + len + kAlign - 1) & ~(kAlign - 1); }
// P_b update, PAPER.md:731-739 (strict '<': exact fit wraps to 0)
__host__ __device__ inline uint64_t advance(uint64_t p_b, uint64_t f, uint64_t R) { return p_b + f < R ? p_b + f : 0; }
__host__ __device__ inline uint32_t seq_inc(uint32_t q) { return (q + 1) & kSeqMask; }  // PAPER.md:741-745 (R5)
__host__ __device__ inline uint64_t pack_ptr(uint64_t b, uint32_t q) { return (b << 24) | (q & kSeqMask); }
__host__ __device__ inline uint64_t ptr_off(uint64_t w) { return w >> 24; }
__host__ __device__ inline uint32_t ptr_seq(uint64_t w) { return (uint32_t)(w & kSeqMask); }
__host__ __device__ inline uint32_t seq_dist(uint32_t p, uint32_t h) { return (p - h) & kSeqMask; }

// Space rule (R4): can [p_b, p_b+f) (p_b+f <= R) be written without touching
// the live range [h_b, p_b) of unreleased entries?
__host__ __device__ inline bool span_free(uint64_t p_b, uint32_t p_q, uint64_t h_b, uint32_t h_q, uint64_t f) {
  if (p_q == h_q) return true;          // empty
  if (p_b > h_b) return true;           // live range does not wrap
  if (p_b < h_b) return p_b + f <= h_b; // live range wraps: free gap is [p_b, h_b)
  return false;                         // same offset, non-empty: full
}

// ---------------------------------------------------------------------------
// Memory-ordering primitives.  Scope is a template parameter: rings whose
// producer and consumer sit on one GPU use .gpu (MEMBAR.GPU, ~0.4 us); rings
// crossing NVLink use .sys (MEMBAR.SYS, ~1.7 us measured on B200).
// ---------------------------------------------------------------------------
template <bool SYS>
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  if (SYS) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  if (SYS) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <bool SYS>
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  if (SYS) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <bool SYS>
__device__ __forceinline__ void fence_acq_rel() {
  if (SYS) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
template <bool SYS>
__device__ __forceinline__ uint64_t cas_acquire(uint64_t* p, uint64_t cmp, uint64_t val) {
  uint64_t old;
  if (SYS) asm volatile("atom.acquire.sys.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(val) : "memory");
  else asm volatile("atom.acquire.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(val) : "memory");
  return old;
}
template <bool SYS>
__device__ __forceinline__ uint64_t cas_acq_rel(uint64_t* p, uint64_t cmp, uint64_t val) {
  uint64_t old;
  if (SYS) asm volatile("atom.acq_rel.sys.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(val) : "memory");
  else asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(val) : "memory");
  return old;
}
// Launch-local coordination (all on the producer's own GPU): gpu scope.
__device__ __forceinline__ uint64_t ld_acquire_gpu64(const uint64_t* p) { return ld_acquire<false>(p); }
__device__ __forceinline__ uint32_t ld_acquire_gpu32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu64(uint64_t* p, uint64_t v) { st_release<false>(p, v); }
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// Streaming 16-byte copies through integer registers only (R17: bit-exact,
// NaN payloads preserved).  Loads bypass L1 (read once).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int4 ld_stream16(const void* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// Coherent 16-byte load (L2, never the non-coherent path): for memory another
// agent writes while the kernel runs -- the consumer reading ring entries
// (in its own HBM, or over NVLink with pull placement).
__device__ __forceinline__ int4 ld_cg16(const void* p) {
  int4 v;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st16(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// 32-byte accesses (LDG.256 / STG.256 on sm_100): half the instructions per
// byte of the 16-byte ones; over NVLink the SM's store issue rate is what
// limits a copy on a small grid (tools/p2p_ceiling.cu).
struct alignas(32) v8u32 { uint32_t r[8]; };
__device__ __forceinline__ v8u32 ld_stream32(const void* p) {
  v8u32 v;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]), "=r"(v.r[6]),
                 "=r"(v.r[7])
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st32(void* p, const v8u32& v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.r[0]), "r"(v.r[1]), "r"(v.r[2]),
               "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]), "r"(v.r[7])
               : "memory");
}

__device__ __forceinline__ uint64_t warp_incl_scan64(uint64_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}
__device__ __forceinline__ uint32_t warp_incl_scan32(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}
__device__ __forceinline__ uint64_t warp_sum64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ uint32_t ld_relaxed_gpu32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// CRC-32/IEEE (reflected 0xEDB88320, init/xorout 0xFFFFFFFF) of the 52 header
// bytes [4,56) (R10), one header per thread, slicing-by-4: four 256-entry
// tables in shared memory (tab[k*256 + i]; built on the host by host.cu from
// its own shift-register CRC), one 32-bit header word per step.  `w[1..13]`
// are the header words 1..13 (little-endian).  A warp checksums 32 headers at
// once.
// ---------------------------------------------------------------------------
constexpr int kCrcTableWords = 4 * 256;
constexpr int kCrcPowWords = 32;   // after the tables in the global copy: x^(2^n) mod P
__device__ __forceinline__ uint32_t crc52(const uint32_t* w, const uint32_t* __restrict__ tab) {
  uint32_t c = 0xFFFFFFFFu;
#pragma unroll
  for (int i = 1; i <= 13; ++i) {
    c ^= w[i];
    c = tab[3 * 256 + (c & 0xFFu)] ^ tab[2 * 256 + ((c >> 8) & 0xFFu)] ^ tab[256 + ((c >> 16) & 0xFFu)] ^ tab[c >> 24];
  }
  return ~c;
}

// ---------------------------------------------------------------------------
// CRC-32/IEEE of a byte range (the fault-tolerant rings' payload checksum,
// SURVEY.md Q10), one warp per range: lane l takes a contiguous slice, the
// slice CRCs are combined with crc(A || B) = (crc(A) * x^(8|B|) mod P) ^ crc(B)
// (GF(2) multiply by a power of x built from the x^(2^n) table `pw`).
// The GF(2) combine follows the construction of zlib's crc32_combine
// (multmodp / x2nmodp, zlib 1.2.12+, (C) 1995-2022 Jean-loup Gailly and Mark
// Adler, zlib license: use permitted with this notice; this is an independent
// rewrite of that canonical routine, not a copy of its source).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t gf2_mulmod_dev(uint32_t a, uint32_t b) {
  uint32_t p = 0;
  for (int i = 31; i >= 0; --i) {
    if (a & (1u << i)) p ^= b;
    b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
  }
  return p;
}
// x^(8 n) mod P
__device__ __forceinline__ uint32_t x8n_mod(uint64_t n, const uint32_t* __restrict__ pw) {
  uint32_t p = 1u << 31;   // x^0
  int k = 3;
  while (n) {
    if (n & 1) p = gf2_mulmod_dev(pw[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}
__device__ __forceinline__ uint32_t crc32_combine_dev(uint32_t c1, uint32_t c2, uint64_t len2, const uint32_t* pw) {
  return len2 ? gf2_mulmod_dev(x8n_mod(len2, pw), c1) ^ c2 : c1;
}
__device__ __forceinline__ uint32_t crc32_range(const uint8_t* p, uint64_t n, const uint32_t* __restrict__ tab) {
  uint32_t c = 0xFFFFFFFFu;
  uint64_t i = 0;
  for (; i < n && ((uintptr_t)(p + i) & 3); ++i) c = tab[(c ^ __ldcg(p + i)) & 0xFFu] ^ (c >> 8);
  for (; i + 4 <= n; i += 4) {
    c ^= __ldcg(reinterpret_cast<const uint32_t*>(p + i));
    c = tab[3 * 256 + (c & 0xFFu)] ^ tab[2 * 256 + ((c >> 8) & 0xFFu)] ^ tab[256 + ((c >> 16) & 0xFFu)] ^ tab[c >> 24];
  }
  for (; i < n; ++i) c = tab[(c ^ __ldcg(p + i)) & 0xFFu] ^ (c >> 8);
  return ~c;
}
// Whole-warp CRC of [p, p + n); every lane returns the result.
__device__ __forceinline__ uint32_t warp_crc32(const uint8_t* p, uint64_t n, const uint32_t* tab, const uint32_t* pw,
                                               int lane) {
  const uint64_t slice = ((n + 31) / 32 + 15) & ~15ull;
  const uint64_t lo = min(n, (uint64_t)lane * slice), hi = min(n, lo + slice);
  uint32_t c = crc32_range(p + lo, hi - lo, tab);
  uint64_t len = hi - lo;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {     // tree: lane l (multiple of 2s) absorbs lane l + s
    const uint32_t c2 = __shfl_down_sync(0xffffffffu, c, s);
    const uint64_t l2 = __shfl_down_sync(0xffffffffu, len, s);
    if ((lane & (2 * s - 1)) == 0) {
      c = crc32_combine_dev(c, c2, l2, pw);
      len += l2;
    }
  }
  return __shfl_sync(0xffffffffu, c, 0);
}


// Mirror word: head | kMirrorValid once the consumer has bound the mirror.
constexpr uint64_t kMirrorValid = 1ull << 63;

// Producer-local state of one attachment (one producer -> one ring channel),
// allocated on the producer GPU and exported to the consumer by CUDA IPC so
// that the consumer's release can push the head into `mirror_head` (the
// credit direction of the double ring, R1).
struct alignas(128) DestState {
  uint64_t mirror_head;  // written by the consumer (NVLink store); read locally by the leader
  uint64_t _p0[15];
  uint64_t tail_cache;   // SPSC: tail after the last planned entry (leader-owned)
  uint64_t chan_seq;     // next header seq of this channel (R18)
  uint64_t lock_acq;     // fault-tolerant rings: lock acquisitions by this attachment
  uint64_t _p1[13];
};
static_assert(sizeof(DestState) == 256, "DestState layout");

}  // namespace b200ring
