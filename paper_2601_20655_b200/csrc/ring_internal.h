// ring_internal.h — structures shared by the host runtime (host.cu) and the
// kernels (put.cu, get.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/b200ring.h"
#include "../../include/b200ring_layout.cuh"

namespace b200ring {

// Device-side invariant checks (compute-sanitizer is not available on this
// pool): built with B200RING_NVCC_DEFINES=-DB200RING_CHECKS, a violated bound
// prints the site and traps, which fails the launch (RING_ECUDA / a CUDA
// error at the next synchronisation).  Compiled out otherwise.
#ifdef B200RING_CHECKS
#define RING_CHECK(cond, what, x, y)                                                              \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("B200RING_CHECK failed: %s (%s:%d) %llu %llu\n", what, __FILE__, __LINE__,            \
             (unsigned long long)(x), (unsigned long long)(y));                                   \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define RING_CHECK(cond, what, x, y) \
  do {                               \
  } while (0)
#endif


// A destination ring as seen by a producer.
struct DestDesc {
  uint8_t* ring;         // ring base mapped into the producer's address space
  uint8_t* data;         // ring + data_offset
  DestState* st;         // producer-local state (same GPU as the producer)
  uint64_t R;
  uint32_t N;
  uint32_t mpsc;         // 1: take the lock; 0: lock elided (R14)
  uint32_t producer_id;
  uint32_t has_mirror;   // unused by the kernels (mirror validity is in-band)
  uint32_t sys;          // 1: ring / consumer on another GPU -> .sys scope
  uint32_t ft;           // RING_CREATE_FAULT_TOLERANT: take-over, CAS WL/UH/Unlock, tags, payload CRC
  uint32_t rc;           // RING_CREATE_RESERVE_COMMIT: claim under the lock, copy and commit outside it
  uint32_t _pad2;
  uint8_t* hdrs;         // split placement: the consumer's header copies (slot-indexed, 64 B each), else null
};

// Test-only fault injection of a put launch (ring_peer_set_fault).
struct FaultSpec {
  uint32_t die_after = 0;
  uint32_t pause_mask = 0;
  uint32_t msg = 0;
  uint32_t _r = 0;
  uint32_t* arrived = nullptr;
  uint32_t* go = nullptr;
};

enum PlanFlags : uint32_t {
  kEntry = 1,    // publish a size slot (slot_word) and move the tail to tail_after
  kStatus = 2,   // write status[msg]
  kUnlock = 4,   // release the ring lock after publishing (MPSC)
  kRelease = 8,  // consumer copy-out: release this entry once its copy is complete
};

// One item of a launch: a PAD entry, a message entry, or a status-only
// record (message not placed).  Written by the control warp, read by the copy
// warps and the publisher / finisher warp.  192 bytes.
struct alignas(64) Plan {
  // what a copy warp needs, in the first 32-B sector (one vector load pair per lane)
  uint64_t src, dst, len;           // copy: payload source / destination / bytes
  uint32_t first_unit, nunits;      // copy work units [first_unit, first_unit + nunits)
  uint64_t slot_word;               // busy | pad | f
  uint64_t tail_after;              // tail word once this entry is published (put)
  uint32_t slot, dest, msg, status; // slot seq; destination index; message index in the launch; status
  uint32_t flags, seq, epoch, _q;   // put: header seq (R18) and epoch of a message entry
  uint64_t f;
  uint64_t start;                   // put: entry offset in the data region (header goes to data + start)
  uint64_t msgp;                    // put engine: the message descriptor (header fields) of this item
  uint64_t statusp;                 // put engine: its status word
  uint64_t t_in;                    // put: %globaltimer when the leader took the message up (header t_put)
  uint64_t _p[1];
  uint32_t _h[16];
};
static_assert(sizeof(Plan) == 192, "Plan layout");
static_assert(offsetof(Plan, nunits) == 28, "copy fields in the first sector");

// Speculative first round (put, single SPSC destination): every CTA evaluates
// the leader's placement rule for the launch's first <= 32 messages from the
// producer-local tail and its own snapshot of the head, so its copy warps can
// start before the leader's plans arrive.  Placement does not depend on the
// head (only *whether* an entry fits does, and the head only moves forward):
// every entry that fits for the CTA fits identically for the leader.
struct SpecItem {
  uint64_t src, dst, len;
  uint32_t first_unit, nunits, item, _p;
};
#ifndef B200RING_SPEC_ROUNDS
#define B200RING_SPEC_ROUNDS 1
#endif
constexpr int kSpecRounds = B200RING_SPEC_ROUNDS;   // leader rounds evaluated speculatively
struct SpecRound {
  uint32_t n_units;     // units [0, n_units) are described by it[]
  uint32_t n;           // messages described
  uint32_t _p[2];
  SpecItem it[kSpecRounds * kGroup];
};

// Per-CTA cache of the launch's `planned` word for the copy warps: one warp
// at a time polls the global word (gpu-scope acquire) and republishes it in
// shared memory (cta-scope release), so ~one poller per SM instead of one per
// warp hits that L2 line.
struct CopyShared {
  uint64_t pl;
  uint32_t owner;
  uint32_t first;       // first unit of the CTA's copy warps (one atomicAdd per CTA, taken at CTA start)
};

// Per-launch counters.  A context holds two sets used by alternate launches;
// launch L uses set[L & 1] and zeroes set[(L + 1) & 1] for launch L + 1 (the
// two launches are stream-ordered, so no launch ever sees a stale counter).
struct alignas(128) LaunchSet {
  // (units << 32) | items, one word written with ONE release store by the
  // control warp: items [0, items) are written and copy work units
  // [0, units) are described by them.  (Two separate words written after one
  // fence may become visible in either order.)
  uint64_t planned;
  uint64_t _a[15];
  uint32_t pub_seq;        // items [0, pub_seq) are published / finished
  uint32_t _b[31];
  uint32_t next_unit;      // copy work units handed out (atomic)
  uint32_t _c[31];
  // the producer-local tail this launch starts from, written by the previous
  // launch's leader when it finished (put.cu, spec_first_round)
  uint64_t start_tail;
  uint32_t _d[30];
  uint32_t arrive[kPlanRing];
};
// Bit 31 of the items field: the control warp is done, the word is final.
constexpr uint64_t kPlannedDone = 1ull << 31;
__host__ __device__ inline uint32_t planned_items(uint64_t p) { return (uint32_t)p & 0x7fffffffu; }
__host__ __device__ inline bool planned_done(uint64_t p) { return (p & kPlannedDone) != 0; }
__host__ __device__ inline uint32_t planned_units(uint64_t p) { return (uint32_t)(p >> 32); }
__host__ __device__ inline uint64_t make_planned(uint32_t items, uint32_t units) {
  return ((uint64_t)units << 32) | items;
}

struct LaunchCtx {
  LaunchSet set[2];
  Plan plan[kPlanRing];
};

struct Route {
  uint32_t app_id;
  uint16_t stage;
  uint16_t n;           // destinations (0 = unused entry)
  uint32_t epoch;
  uint32_t rr;          // round-robin counter (device-owned)
  uint32_t dests[kMaxDests];
  // Fast reject: admit at rate adm_k / adm_tx (burst 1) by
  // arrival time hdr.accepted_at; adm_next = next admissible time * adm_k
  // (exact integer arithmetic).  adm_k == 0: no admission control.
  uint64_t adm_tx;
  uint32_t adm_k;
  uint32_t _ra;
  uint64_t adm_next;    // device-owned
};

// Persistent put engine (ring_peer_engine_start): one resident put grid per
// attachment takes batches from this queue instead of one launch per batch.
// A doorbell kernel on the submitting stream fills slot b % kEngineQueue and
// moves `ctl` from b to b + 1 with a CAS (stream order = batch order); the
// leader plans batch after batch (items and work units numbered across
// batches, as in one long launch); the publisher releases `done` = b + 1 once
// every item of batch b is published.  Closing: bit 63 of `ctl` -- set by the
// stop kernel (the engine drains the batches posted before it and exits) or
// by the engine itself when it has been idle, with nothing in flight and no
// host call on the attachment (the host lease), for the idle time: a
// resident kernel whose process has gone then ends by itself, and a live
// host restarts it at its next submission (EngineHost::alive).  A doorbell
// that finds the queue closed writes RING_ECLOSED into its batch's statuses.
constexpr uint32_t kEngineQueue = 64;
constexpr uint64_t kEngineClosed = 1ull << 63;
struct EngineHost {            // pinned, mapped host memory
  volatile uint64_t lease;     // host: bumped by every engine call of the attachment
  volatile uint32_t alive;     // host 1 at launch; the engine 0 when it exits
  uint32_t _p;
};
struct EngineBatch {
  const ring_msg_t* msgs;
  uint32_t* status;
  uint32_t n, flags;
  uint32_t item_end;     // leader: items [.., item_end) hold this batch (valid once planned_batches > b)
  uint32_t _p;
};
struct alignas(128) EngineQueue {
  uint64_t ctl;               // doorbells: batches posted | kEngineClosed
  uint64_t _a[15];
  uint64_t planned_batches;   // leader: batches fully planned
  uint64_t _b[15];
  uint64_t done;              // publisher: batches fully published
  uint64_t _c[15];
  uint64_t _d[16];
  EngineBatch batch[kEngineQueue];
};
static_assert(offsetof(EngineQueue, planned_batches) == 128 && offsetof(EngineQueue, done) == 256,
              "EngineQueue layout (ring_peer_engine_state)");
constexpr uint64_t kForeverNs = 1ull << 60;   // engine copy warps / publisher never give up while idle

struct PutArgs {
  ring_msg_t inline_msg;  // used when msgs == nullptr (ring_put of one message)
  DestDesc dest0;         // dests[0] by value (a peer's only destination: no load before placement)
  const ring_msg_t* msgs;
  uint32_t* status;
  uint32_t* dest_out;
  LaunchCtx* ctx;
  const DestDesc* dests;
  Route* routes;
  const uint32_t* crc_table;  // CRC-32 slicing tables
  uint64_t* trace;            // debug timeline (B200RING_TRACE=1), else null
  uint64_t timeout_ns;
  uint32_t launch;
  uint32_t n;
  uint32_t flags;
  uint32_t n_dests;
  uint32_t n_routes;
  uint32_t chunk;             // bytes per copy work unit
  uint32_t copy_mode;         // 0: LSU copy warps, 1: TMA engine per CTA
  uint32_t _pad;
  uint64_t lock_timeout_ns;   // TL (fault-tolerant and reserve-then-commit rings)
  uint64_t hole_timeout_ns;   // reserve-then-commit: a reservation this old at the tail is a lost sender's
  FaultSpec fault;            // test-only fault injection
  EngineQueue* engine;        // persistent put engine: batches come from here (msgs / n / status unused)
  EngineHost* engine_host;    // its lease / alive words (device address of the mapped host memory)
  uint64_t engine_idle_ns;    // idle time after which it closes itself
};

#ifndef B200RING_ENGINE_STAGES
#define B200RING_ENGINE_STAGES 2
#endif
constexpr int kEngineStages = B200RING_ENGINE_STAGES;   // TMA engine: shared-memory stages of `chunk` bytes
constexpr uint32_t kEngineSmem = 200u << 10;             // dynamic shared memory the stages may use
#ifndef B200RING_ENGINE_WARPS
#define B200RING_ENGINE_WARPS 6
#endif
constexpr int kMaxEngineWarps = B200RING_ENGINE_WARPS;    // TMA engine warps per CTA (CTA 0: one)

struct GetArgs {
  uint8_t* ring;
  uint8_t* data;
  const uint8_t* hdrs;  // split placement: local header copies (slot-indexed), else null: headers at data + start
  ring_view_t* views;
  uint8_t* dst;
  uint64_t** mirrors;   // device array of mirror word pointers (consumer address space)
  LaunchCtx* ctx;
  const uint32_t* crc_table;
  uint64_t R;
  uint64_t dst_stride;
  uint64_t timeout_ns;
  uint32_t launch;
  uint32_t N;
  uint32_t n;
  uint32_t flags;
  uint32_t consume;     // 1: release each entry after reading (and copying)
  uint32_t sys;         // producers may be remote: .sys scope
  uint32_t remote_data;  // the buffer region is on another GPU (pull / split): copy-out loads on 128-B lines
  uint32_t n_mirrors;
  uint32_t chunk;
  uint64_t* trace;      // debug timeline (B200RING_TRACE=1): [0,512) control rounds, [512,1024) releases
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
cudaError_t launch_put(const PutArgs& a, uint32_t ctas, uint32_t threads, cudaStream_t s);
cudaError_t launch_get(const GetArgs& a, uint32_t ctas, uint32_t threads, cudaStream_t s);
cudaError_t launch_release(const ReleaseArgs& a, cudaStream_t s);
cudaError_t launch_engine_doorbell(EngineQueue* q, uint64_t b, const ring_msg_t* msgs, uint32_t* status, uint32_t n,
                                   uint32_t flags, bool wait, uint64_t timeout_ns, cudaStream_t s);
cudaError_t launch_engine_stop(EngineQueue* q, cudaStream_t s);
cudaError_t launch_route_update(Route* d, const Route& nr, DestDesc* desc_slot, const DestDesc* desc, cudaStream_t s);
cudaError_t launch_probe_ping(uint64_t* remote, const uint64_t* local, uint32_t iters, uint64_t* t_send,
                              uint64_t* rtt, uint64_t timeout_ns, cudaStream_t s);
cudaError_t launch_probe_pong(uint64_t* remote, const uint64_t* local, uint32_t iters, uint64_t* t_seen,
                              uint64_t timeout_ns, cudaStream_t s);
cudaError_t launch_engine_wait(EngineQueue* q, uint64_t upto, uint64_t timeout_ns, cudaStream_t s);
// Load a kernel on the current device now and give it the ring's shared-memory
// carveout.  Lazy loading: a module loaded at first launch waits for the
// kernels already running, and a consumer may be spinning for that launch's
// data.  Carveout: on B200 a CTA is only placed on an SM whose L1/shared split
// matches its kernel's, and without a preference every kernel gets the
// smallest split its static shared memory fits -- a 148-CTA put (11 KB static)
// then leaves no SM on which a 1-CTA get (4 KB) can start, and a put spinning
// for the get's credit only ends by timing out (profiles/r02_sched_carveout.txt).
// Every ring kernel therefore asks for the same split: 8 % (a 32 KB shared
// split: room for two put CTAs and a get CTA on one SM), so L1 keeps ~224 KB --
// the copy loops' outstanding loads are staged in L1, and an all-shared split
// (28 KB of L1) costs the C2 put ~10-20 %.  Measured (tools/carveout_probe.cu,
// profiles/r02_carveout_probe.txt): 8 % lets a put grid start next to a
// copy-out get grid and vice versa; 0-7 % and, oddly, 14 % do not.  The TMA
// engine (put_kernel<1>, up to 200 KB of stages) takes its own split and starts
// only on SMs free of other ring kernels.  B200RING_CARVEOUT (percent)
// overrides the split (experiments).
int ring_carveout_percent();
template <class K>
cudaError_t preload_kernel(K* k, int carveout = -1) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, k);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                             carveout >= 0 ? carveout : ring_carveout_percent());
  return e;
}
cudaError_t preload_put();
cudaError_t preload_get();
cudaError_t preload_clock();
cudaError_t preload_stage();
cudaError_t preload_fanin();
struct SetRing;
cudaError_t launch_set_consume(const SetRing* rings, uint32_t k, ring_view_t* views, uint32_t* ring_idx, uint32_t n,
                               const uint32_t* crc, uint32_t flags, uint64_t timeout_ns, uint32_t rr, bool sys,
                               cudaStream_t s);
cudaError_t launch_stage_scale_put(const ring_dev_peer_t& peer, const void* in, uint64_t n, float scale,
                                   const ring_hdr_t& hdr, uint32_t flags, uint32_t* status, uint64_t timeout_ns,
                                   uint32_t ctas, cudaStream_t s);
cudaError_t launch_clock_publish(unsigned long long* mapped_host, unsigned long long duration_ns, cudaStream_t s);

}  // namespace b200ring
