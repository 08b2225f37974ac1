// ring_internal.h — structures shared by the host runtime (host.cu) and the
// kernels (put.cu, get.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/b200ring.h"
#include "ring_device.cuh"

namespace b200ring {

// Producer-local state of one attachment (one producer -> one ring channel),
// allocated on the producer GPU and exported to the consumer by CUDA IPC so
// that the consumer's release can push the head into `mirror_head` (the
// credit direction of the double ring, R1).
// Mirror word: head | kMirrorValid once the consumer has bound the mirror.
constexpr uint64_t kMirrorValid = 1ull << 63;

struct alignas(128) DestState {
  uint64_t mirror_head;  // written by the consumer (NVLink store); read locally by the leader
  uint64_t _p0[15];
  uint64_t tail_cache;   // SPSC: tail after the last planned entry (leader-owned)
  uint64_t chan_seq;     // next header seq of this channel (R18)
  uint64_t _p1[14];
};
static_assert(sizeof(DestState) == 256, "DestState layout");

// A destination ring as seen by a producer.
struct DestDesc {
  uint8_t* ring;         // ring base mapped into the producer's address space
  uint8_t* data;         // ring + data_offset
  DestState* st;         // producer-local state (same GPU as the producer)
  uint64_t R;
  uint32_t N;
  uint32_t mpsc;         // 1: take the lock; 0: lock elided (R14)
  uint32_t producer_id;
  uint32_t has_mirror;   // 1: consumer pushes the head into st->mirror_head
  uint32_t sys;          // 1: ring / consumer on another GPU -> .sys scope
  uint32_t _pad;
};
static_assert(sizeof(DestDesc) == 56 || sizeof(DestDesc) == 64, "DestDesc layout");

enum PlanFlags : uint32_t { kHasMsg = 1, kUnlock = 2, kPublish = 4, kRelease = 8 };

// One planned message: written by the leader warp, read by copy CTAs and the
// publisher warp.  256 bytes.
struct alignas(64) Plan {
  uint64_t src;         // payload source
  uint64_t dst;         // payload destination
  uint64_t len;         // payload bytes
  uint64_t start;       // entry start in the buffer region
  uint64_t f;           // footprint
  uint64_t tail_after;  // tail word after this plan's entries (put)
  uint64_t pad_word;    // slot word of a PAD entry placed first (0 = none)
  uint32_t pad_slot, slot;
  uint32_t dest, cnt;   // destination index; copy CTAs taking part (0 = nothing to copy)
  uint32_t status, flags;
  uint64_t hdr_dst;     // where the first copy CTA writes the 64-B header (0 = none)
  uint32_t cta_base;    // copy CTAs (cta_base + j) % copy_ctas, j < cnt, take part
  uint32_t _q;
  uint64_t _p[3];
  uint32_t hdr[16];     // the 64-B entry header
};
static_assert(sizeof(Plan) == 192, "Plan layout");

// Per-launch-context coordination (one per producer attachment, router or
// consumer), on the launching GPU.  Counters are monotonic across launches:
// message k of a launch has global index base + k, base tracked by the host.
struct LaunchCtx {
  uint64_t plan_seq;   // leader: plans [0, plan_seq) are written
  uint64_t _p0[15];
  uint64_t pub_seq;    // publisher / finisher: plans [0, pub_seq) are complete
  uint64_t _p1[15];
  uint64_t g_cursor;   // get: read cursor published by the control warp
  uint64_t _p2[15];
  uint32_t arrive[kPlanRing];
  Plan plan[kPlanRing];
};

struct Route {
  uint32_t app_id;
  uint16_t stage;
  uint16_t n;           // destinations (0 = unused entry)
  uint32_t epoch;
  uint32_t rr;          // round-robin counter (device-owned)
  uint32_t dests[kMaxDests];
};

struct PutArgs {
  ring_msg_t inline_msg;  // used when msgs == nullptr (ring_put of one message)
  const ring_msg_t* msgs;
  uint32_t* status;
  uint32_t* dest_out;
  LaunchCtx* ctx;
  const DestDesc* dests;
  Route* routes;
  const uint32_t* crc_table;
  uint64_t base;
  uint64_t timeout_ns;
  uint32_t n;
  uint32_t flags;
  uint32_t n_dests;
  uint32_t n_routes;
  uint32_t copy_ctas;
  uint32_t chunk_min;
  uint32_t copy_mode;
  uint32_t _pad;
};

struct GetArgs {
  uint8_t* ring;
  uint8_t* data;
  ring_view_t* views;
  uint8_t* dst;
  uint64_t** mirrors;   // device array of mirror word pointers (consumer address space)
  LaunchCtx* ctx;
  const uint32_t* crc_table;
  uint64_t R;
  uint64_t dst_stride;
  uint64_t base;
  uint64_t timeout_ns;
  uint32_t N;
  uint32_t n;
  uint32_t flags;
  uint32_t consume;     // 1: release each entry after reading (and copying)
  uint32_t sys;         // producers may be remote: .sys scope
  uint32_t n_mirrors;
  uint32_t copy_ctas;
  uint32_t chunk_min;
};

struct ReleaseArgs {
  uint8_t* ring;
  uint64_t** mirrors;
  uint64_t R;
  uint32_t N;
  uint32_t count;
  uint32_t sys;
  uint32_t n_mirrors;
};

// Launchers (defined in put.cu / get.cu).
cudaError_t launch_put(const PutArgs& a, uint32_t threads, cudaStream_t s);
cudaError_t launch_get(const GetArgs& a, uint32_t threads, cudaStream_t s);
cudaError_t launch_release(const ReleaseArgs& a, cudaStream_t s);

}  // namespace b200ring
