/*
 * b200ring.h — C ABI of the B200-native double-ring tensor transport.
 *
 * Implements the hot path of arXiv 2601.20655 §6 "RDMA Network" / §6.1 "Ring
 * Buffer": a multi-producer / single-consumer ring of
 * variable-size messages held in the consumer's memory, written one-sidedly by
 * producers, with a size region whose busy bits only the consumer clears.
 * On one 8xB200 box the one-sided RDMA verbs become SM-issued
 * NVLink 5 peer stores and system-scope atomics into a ring in the consumer
 * GPU's HBM.  Readings of the paper are cited as R<n>.
 *
 * Conventions for every entry point
 *   - Plain C types only; device pointers are `void*` / `uint64_t`; CUDA streams
 *     are passed as `void*` (a cudaStream_t; NULL = the legacy default stream).
 *   - Synchronous errors (bad arguments, CUDA/IPC failures) are the return
 *     value.  Data-path outcomes (RING_FULL, RING_EMPTY, RING_ETIMEDOUT,
 *     RING_ECORRUPT, RING_EMSGSIZE on copy-out) are written by the kernels to
 *     device status words / view records in stream order: no host
 *     synchronisation happens on the data path ("no CPU
 *     intervention").
 *   - Every device-side spin (lock, credit, new data) is bounded by the
 *     timeout set with ring_set_timeout_ns (default 2 s) and then reports
 *     RING_ETIMEDOUT instead of hanging (R12).
 *   - Not thread-safe per handle: one host thread / one stream per ring_t
 *     (the single consumer) and per ring_peer_t (one
 *     producer stream).
 */
#ifndef B200RING_H
#define B200RING_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RING_OK = 0,
  RING_EINVAL = 1,     /* bad argument (zero sizes, N not a power of two, R not a multiple of 128, ...) */
  RING_ENOMEM = 2,     /* device allocation failed */
  RING_EMSGSIZE = 3,   /* entry footprint align_up(64+len,128) > R (R15), or copy-out buffer too small */
  RING_FULL = 4,       /* RING_TRY put found insufficient space: "release the lock and abort" */
  RING_EMPTY = 5,      /* RING_TRY get found no new data */
  RING_ETIMEDOUT = 6,  /* a device spin exceeded its budget */
  RING_ECORRUPT = 7,   /* header checksum mismatch: entry discarded and consumed */
  RING_ECUDA = 8,      /* a CUDA runtime call failed (see ring_last_cuda_error) */
  RING_EPEER = 9,      /* no peer access between the two devices / IPC open failed */
  RING_EPENDING = 10,  /* initial value of a device status word not yet written */
  RING_EDROPPED = 11,  /* fault-tolerant ring: WL found the size slot taken -- the lock was taken over
                          while this sender was delayed ("WL(X) fails due to the busy bit",
                          PAPER.md:797); the message is dropped, no retransmission */
  RING_EREJECTED = 12, /* routed put: refused by the route's admission control (fast reject) */
  RING_ECLOSED = 13    /* put engine: the queue was closed (stopped, or idle-closed) before this batch reached it;
                          nothing of the batch was written -- submit it again */
} ring_status_t;

/* flags for ring_put* / ring_get* */
#define RING_BLOCK 0u        /* wait for credit / data (default, R12) */
#define RING_TRY 1u          /* do not wait: RING_FULL / RING_EMPTY */
#define RING_NO_TIMESTAMP 2u /* leave t_put / t_visible zero */
#define RING_ASYNC 4u        /* ring_put_batch to a running put engine: return on the stream as soon as the
                                batch is queued (see ring_peer_engine_start) */

/* flags for ring_create */
#define RING_CREATE_DEFAULT 0u
#define RING_CREATE_LOCAL 1u /* every producer runs on the ring's own device: gpu-scope ordering (cheaper fences) */
/* The paper's liveness machinery, for senders that may be
 * lost or delayed: the lock word is {acquisition count:48, owner+1:16}; a sender
 * spinning on the lock takes it over (CAS old -> self) once it has observed
 * the same word for the lock timeout (TL; local
 * observation, no cross-GPU clock); GH publishes a committed entry a lost
 * sender left behind (Case 7) or clears a stale write (R21); WL = CAS(slot,
 * 0 -> busy|seq tag|f) (fails -> RING_EDROPPED); UH = CAS(tail, value read at
 * GH -> new) (a taken-over sender cannot move the tail back, Q22); Unlock =
 * CAS(self -> 0); every entry carries a payload CRC-32 in header bytes
 * [40,44) (flags bit 0), checked by the consumer (torn payloads, Q10).
 * Slot words gain a 22-bit sequence tag in bits 40-61 (R21).  Each message is
 * appended with the sender's steps one at a time (no batching of publishes). */
#define RING_CREATE_FAULT_TOLERANT 2u
/* Reserve-then-commit MPSC: the lock guards only the
 * claim -- under it a sender reads the reservation frontier and the head,
 * applies the space rule, marks the size slot reserved (bit 61) with its
 * footprint and advances the frontier -- and the payload is copied outside the
 * lock, so producers of one ring copy concurrently; WL commits the slot
 * (reserved -> busy) and any sender moves the tail over the leading run of
 * committed slots (CAS), so entries are published in claim order; a put
 * returns once its entries are published.  The receiver is unchanged.  Lost
 * senders: a lock held past the hole timeout is taken over (acquisition-
 * counted lock word), a reservation stuck at the tail for the hole timeout
 * (ring_set_hole_timeout_ns) becomes a PAD the
 * receiver skips (its sender's commit then fails: RING_EDROPPED), and claims
 * first publish committed entries left behind.  Not combinable with
 * RING_CREATE_FAULT_TOLERANT. */
#define RING_CREATE_RESERVE_COMMIT 4u

/* Geometry limits (R5, R8) */
#define RING_ENTRY_ALIGN 128u
#define RING_HDR_BYTES 64u
#define RING_MAX_SLOTS (1u << 23)
#define RING_MAX_PRODUCERS 64u

typedef struct ring_s* ring_t;           /* consumer side; OWNS the ring allocation in HBM */
typedef struct ring_peer_s* ring_peer_t; /* producer side; BORROWS a mapping of the ring, OWNS its local state */
typedef struct router_s* router_t;       /* stage router (NodeManager / ResultDeliver stand-in) */

/* Opaque, position-independent handle exchanged between processes (e.g. with a
 * torch.distributed all_gather of 256-byte tensors).  Carries the CUDA IPC memory
 * handle(s) plus the ring geometry. */
typedef struct { unsigned char bytes[256]; } ring_handle_t;

/* User-supplied header fields of a workflow message (UUID
 * assigned by the proxy, proxy timestamp, application ID, stage). 32 bytes. */
typedef struct {
  uint8_t uid[16];
  uint64_t accepted_at;
  uint32_t app_id;
  uint16_t stage;
  uint16_t reserved; /* must be 0 */
} ring_hdr_t;

/* One message of a put batch, in DEVICE memory of the producer GPU. 48 bytes. */
typedef struct {
  uint64_t src;      /* device pointer to the payload (readable by the producer GPU) */
  uint64_t len;      /* payload bytes (0 allowed, R19) */
  ring_hdr_t hdr;
} ring_msg_t;

/* Result of one get, written by the get kernel to DEVICE memory. 128 bytes.
 * `header` is the entry header exactly as read from the ring (64 bytes,
 * layout R11: crc32[0,4) uid[4,20) accepted_at[20,28) app_id[28,32)
 * stage[32,34) payload_len[34,38) reserved[38,44) producer_id[44,48)
 * seq[48,52) epoch[52,54) flags[54,56) t_put[56,64)). */
typedef struct {
  uint64_t offset;     /* payload byte offset inside the buffer region (entry start + 64) */
  uint64_t len;        /* payload bytes (from the header; 0 if corrupt) */
  uint64_t footprint;  /* f from the size slot */
  uint64_t start;      /* entry start offset inside the buffer region */
  uint32_t slot_seq;   /* size-region sequence number (24 bit) */
  uint32_t status;     /* RING_OK / RING_ECORRUPT / RING_EMPTY / RING_ETIMEDOUT / RING_EMSGSIZE */
  uint64_t t_visible;  /* %globaltimer (ns) when the consumer saw the entry */
  uint64_t reserved[2];
  uint8_t header[64];
} ring_view_t;

/* Geometry / addresses of a ring (host-side query). */
typedef struct {
  int device;
  uint32_t n_slots;        /* N */
  uint32_t max_producers;
  uint64_t data_bytes;     /* R */
  uint64_t base;           /* device pointer of the ring allocation (consumer GPU) */
  uint64_t data;           /* device pointer of the buffer region = base + data_offset */
  uint64_t data_offset;
  uint64_t alloc_bytes;
} ring_info_t;

/* ---- lifetime -------------------------------------------------------------
 * ring_create: allocate and zero one ring on `device` (lock
 * region, header with head/tail, buffer region of `data_bytes` = R bytes, size
 * region of `n_slots` = N slots).  R must be a positive multiple of 128 below
 * 2^39 (R8: packed pointer words; bit 63 of a mirror word marks it bound);
 * N a power of two <= 2^23; 1 <= max_producers <= 64.  With
 * max_producers == 1 the lock is elided (R14).  Layout: DESIGN.md §3. */
ring_status_t ring_create(int device, uint64_t data_bytes, uint32_t n_slots, uint32_t max_producers,
                          uint32_t flags, ring_t* out);
/* Free the ring.  All peers must be detached first (their mappings are borrowed). */
ring_status_t ring_destroy(ring_t ring);
/* ring_create_split: split placement (reading R28).  The control
 * words, the size slots and a copy of every entry header stay on the
 * consumer's `device` (polled and read locally, as in the paper's layout); the
 * buffer region of R bytes is allocated on `data_device` -- the producer's GPU.
 * The producer writes each entry (header + payload) into its local HBM and
 * the header, size slot and tail into the consumer's control region; the
 * consumer's copy-out get pulls the payload over NVLink (the paper's one-sided
 * READ).  Same protocol, placements and oracle as ring_create; only the
 * memory the buffer region lives in changes.  Producers attach with
 * ring_attach_peer as usual (from any process; the handle carries both
 * allocations).  RING_EINVAL with RING_CREATE_LOCAL, FAULT_TOLERANT or
 * RESERVE_COMMIT; fused device puts (ring_peer_device_view) are refused. */
ring_status_t ring_create_split(int device, int data_device, uint64_t data_bytes, uint32_t n_slots,
                                uint32_t max_producers, uint32_t flags, ring_t* out);
/* ring_open: the consumer side of a ring that lives in ANOTHER GPU's memory
 * (pull placement).  The ring is created (and destroyed, after every ring_open
 * of it) on the producer's GPU, its producers attach there as usual; the
 * consumer on `device` opens its handle (same process: peer access; other
 * process: CUDA IPC) and gets / consumes / releases through the returned
 * ring_t, whose kernels run on `device` and read the ring over NVLink -- with
 * copy-out, the payload is pulled into `d_dst` on `device`.  Same protocol and
 * placements as a ring at the consumer (the oracle does not see the
 * difference); the paper's one-sided READ carries the
 * payload instead of the one-sided WRITE (reading R24).  Bind the
 * producers' mirrors on this ring_t (ring_bind_mirror).  RING_EINVAL for
 * RING_CREATE_LOCAL / fault-tolerant / reserve-then-commit rings.
 * ring_destroy of an opened ring releases the mapping only. */
ring_status_t ring_open(const ring_handle_t* handle, int device, ring_t* out);
ring_status_t ring_get_info(ring_t ring, ring_info_t* out);
/* Export a handle for producers in other processes (CUDA IPC) or this process. */
ring_status_t ring_export(ring_t ring, ring_handle_t* out);

/* ring_attach_peer: map the ring of `h` for a producer running on
 * `producer_device` with id `producer_id` (< max_producers, unique per ring).
 * Same process: direct pointer + cudaDeviceEnablePeerAccess; other process:
 * cudaIpcOpenMemHandle.  Allocates the producer-local state (head mirror,
 * message counters) on `producer_device` and returns its handle in
 * `mirror_out`, which the consumer passes to ring_bind_mirror so that releases
 * push the head to this producer (credit ring, R1).  RING_EPEER if the devices
 * cannot access each other. */
ring_status_t ring_attach_peer(const ring_handle_t* h, int producer_device, uint32_t producer_id,
                               ring_peer_t* out, ring_handle_t* mirror_out);
/* Consumer side: register producer `producer_id`'s head mirror.  Until bound,
 * that producer reads the head word over NVLink instead (correct, slower). */
ring_status_t ring_bind_mirror(ring_t ring, uint32_t producer_id, const ring_handle_t* mirror);
ring_status_t ring_detach(ring_peer_t peer);

/* ---- producer ----------------------------------------------------------------
 * ring_put_batch: append `n` messages (device array `d_msgs` on the producer
 * GPU) in order, as the sender's 8 steps each: lock (MPSC
 * only), read tail, GH stale-slot check, space check (PAD entry at the wrap,
 * R3/R4), write the 64-B header + payload into the peer ring (WB), set the
 * size slot busy|f (WL), advance the tail (UH, release at system scope),
 * unlock.  One kernel launch; copies of message k+1 overlap the publish of k.
 * `d_status` (device, n words) receives one ring_status_t per message
 * (RING_OK / RING_FULL under RING_TRY / RING_ETIMEDOUT / RING_EMSGSIZE).
 * The payloads must stay valid until the launch completes in stream order.
 * Header seq (R18) = this attachment's running message count.
 * While the attachment's put engine runs (below), the batch goes to the
 * engine instead of a launch: same steps, same placements and statuses. */
ring_status_t ring_put_batch(ring_peer_t peer, const ring_msg_t* d_msgs, uint32_t n, uint32_t flags,
                             uint32_t* d_status, void* stream);
/* Persistent put engine of one attachment: ONE resident put grid (the same
 * leader / publisher / copy warps as a put launch) that takes batch after
 * batch from a device queue, so that consecutive batches run back to back
 * with no launch, ramp-up or drain between them (items and copy work units
 * are numbered across batches, as in one long launch).
 *   ring_peer_engine_start: launch the engine (on a stream of its own, after
 *     the work already queued on `stream`).  RING_EINVAL for fault-tolerant or
 *     reserve-then-commit rings, the TMA copy mode, or an engine already on.
 *   ring_put_batch while it runs: a one-thread doorbell kernel on `stream`
 *     queues the batch (stream order = batch order; at most 64 batches in
 *     flight).  Without RING_ASYNC the doorbell returns once the batch is
 *     published (the stream semantics of a put launch); with RING_ASYNC it
 *     returns at once, and the payloads, descriptors and status words must
 *     stay untouched until ring_peer_engine_wait / _stop has run on a stream.
 *     ring_put (host header) and routed / fused puts to the attachment are
 *     RING_EINVAL while the engine runs.
 *   ring_peer_engine_wait: the stream waits until every queued batch is published.
 *   ring_peer_engine_stop: the engine drains the queued batches and exits;
 *     `stream` waits for its exit; ring_put_batch launches again afterwards.
 *   Idle close: an engine with nothing in flight and no engine call on its
 *     attachment for the idle time (max(1 s, ring_set_timeout_ns)) closes its
 *     queue and exits -- so an engine whose process has died ends by itself,
 *     and a host call that synchronises the whole device (cudaMalloc may)
 *     waits at most that long; the next ring_put_batch restarts it.  A batch
 *     whose doorbell finds the queue closed gets RING_ECLOSED statuses (only
 *     possible if its stream was held back for longer than the idle time).
 *   While an engine runs, the library's host calls that would synchronise the
 *   device synchronise the legacy default stream instead.
 * Limit: 2^31 items / 2^32 work units per engine session (restart to reset). */
ring_status_t ring_peer_engine_start(ring_peer_t peer, void* stream);
ring_status_t ring_peer_engine_wait(ring_peer_t peer, void* stream);
ring_status_t ring_peer_engine_stop(ring_peer_t peer, void* stream);
/* Engine counters now (host, synchronous, never waits for a stream): batches
 * posted, fully planned, fully published, and whether the queue is closed. */
ring_status_t ring_peer_engine_state(ring_peer_t peer, uint64_t* out4);
/* Single message convenience form: `d_payload` device pointer, `hdr` host
 * pointer (copied into the launch), one status word. */
ring_status_t ring_put(ring_peer_t peer, const void* d_payload, uint64_t len, const ring_hdr_t* hdr,
                       uint32_t flags, uint32_t* d_status, void* stream);
/* Tuning: copy CTAs and threads per CTA of this attachment's put kernel
 * (0 = default: 148 x 256 with 32 KiB work units for a same-GPU ring,
 * 33 x 512 with 16 KiB units across NVLink; threads <= 512), copy engine
 * (0 = vector LSU -- 16-B accesses same-GPU, 32-B across NVLink -- or
 * 1 = TMA bulk).  RING_EINVAL for values out of range. */
ring_status_t ring_peer_config(ring_peer_t peer, uint32_t copy_ctas, uint32_t threads, uint32_t copy_mode);
/* Host-side count of messages this attachment has submitted (= next header seq). */
uint64_t ring_peer_submitted(ring_peer_t peer);

/* ---- lock-free fan-in ----------
 * Instead of one MPSC ring whose producers serialise on the lock (PAPER.md:697,
 * 706), give every producer its own single-producer ring (max_producers = 1,
 * lock elided, R14) on the consumer GPU and serve them all with ONE consumer
 * warp: lane i polls ring i's tail and runs the receiver steps 1-5 on it, all
 * rings in parallel, one entry per ring per round, rounds starting at a
 * rotating ring (no producer starves).  Per-channel order = each ring's FIFO;
 * the merged order is the consumer's round order. */
typedef struct ring_set_s* ring_set_t;
/* 1 <= n <= 32 rings, all on one device; their producers must be bound
 * (ring_bind_mirror) before consuming.  The rings must only be read through
 * the set afterwards (its consume releases every entry it reads). */
ring_status_t ring_set_create(const ring_t* rings, uint32_t n, ring_set_t* out);
ring_status_t ring_set_destroy(ring_set_t set);
/* Receive and release the next `n` messages from any ring of the set: view
 * records as ring_consume (reserved[0] = ring index) and, if not NULL, the ring
 * index of each in d_ring_idx (device, n words).  RING_TRY: stop at the first
 * round with nothing to read (remaining views RING_EMPTY). */
ring_status_t ring_set_consume(ring_set_t set, uint32_t n, ring_view_t* d_views, uint32_t* d_ring_idx, uint32_t flags,
                               void* stream);

/* ---- fused device-side put -------------------
 * A producer kernel can write its output straight into the peer ring slot and
 * publish it itself (include/b200ring_device.cuh: grid_reserve / payload_ptr /
 * grid_commit), saving the output's HBM round trip and the put launch.  This
 * is the device-side view of a single-producer attachment it needs.  The
 * attachment must not be used by ring_put* concurrently. */
typedef struct {
  uint64_t ring;         /* ring base in the producer's address space */
  uint64_t data;         /* buffer region */
  uint64_t state;        /* producer-local state: head mirror, tail cache, channel counter */
  uint64_t ctl;          /* 128-B grid-coordination block of this attachment */
  uint64_t crc_table;    /* CRC-32 tables on the producer device */
  uint64_t R;
  uint32_t N;
  uint32_t producer_id;
  uint32_t sys;          /* 1: system-scope ordering (ring on another GPU) */
  uint32_t reserved;
} ring_dev_peer_t;
/* RING_EINVAL for a multi-producer (locked) ring. */
ring_status_t ring_peer_device_view(ring_peer_t peer, ring_dev_peer_t* out);
/* A synthetic stage with a fused put epilogue: out = bf16(in * scale) for
 * `n_elems` bf16 elements of `d_in`, written by the computing threads directly
 * into the next entry of the peer ring (one message of 2 * n_elems bytes,
 * header from `hdr`), in ONE launch.  Status word as ring_put. */
ring_status_t ring_stage_scale_bf16_put(ring_peer_t peer, const void* d_in, uint64_t n_elems, float scale,
                                        const ring_hdr_t* hdr, uint32_t flags, uint32_t* d_status, void* stream);

/* ---- fault injection (tests of the fault-tolerant path) --------
 * The labelled sender actions of PAPER.md:778-789 at which a put can be made to
 * stop for good (a lost sender) or to pause (a delayed sender) while another
 * sender takes the lock over.  Applies to message `msg` of every later launch
 * of this attachment on a RING_CREATE_FAULT_TOLERANT ring.  On a
 * RING_CREATE_RESERVE_COMMIT ring only die_after is used: RING_AT_LOCK = lost
 * holding the lock right after its round's claims, RING_AT_WB = lost after the
 * claims and the unlock, before any copy or commit (a hole). */
#define RING_AT_LOCK 1u  /* after Lock (step 1) */
#define RING_AT_GH 2u    /* after GH (steps 2-4: tail, head, stale-slot check) */
#define RING_AT_WB 3u    /* after WB (step 5: header + payload written) */
#define RING_AT_WL 4u    /* after WL (step 6) */
#define RING_AT_UH 5u    /* after UH (step 7) */
typedef struct {
  uint32_t die_after;   /* RING_AT_*: stop right after this action (0 = never) */
  uint32_t pause_mask;  /* bit (1 << RING_AT_*): after that action set arrived[l] = 1, then wait for go[l] != 0 */
  uint32_t msg;         /* index of the message in the launch */
  uint32_t reserved;
  uint32_t* arrived;    /* pinned host memory (mapped), >= 8 words, written by the kernel */
  uint32_t* go;         /* pinned host memory (mapped), >= 8 words, written by the host */
} ring_fault_t;
/* NULL clears.  RING_EINVAL unless the ring is fault tolerant. */
ring_status_t ring_peer_set_fault(ring_peer_t peer, const ring_fault_t* fault);
/* Lock timeout TL of fault-tolerant and reserve-then-commit rings (default 200 us). */
ring_status_t ring_set_lock_timeout_ns(uint64_t ns);
/* Reserve-then-commit rings: a reservation left uncommitted at the tail this
 * long is a lost sender's and becomes a PAD, and a lock word unchanged this
 * long is taken over (default 50 ms; must exceed the longest claim-to-commit
 * time of a live sender, i.e. its largest copy, and a claim round under a
 * saturated NVLink). */
ring_status_t ring_set_hole_timeout_ns(uint64_t ns);

/* ---- consumer ------------------------------------------------------------------
 * ring_get: receive the next `n` entries (receiver steps 1-3, PAPER.md:711-715,
 * plus the checksum check): poll the tail (R7), read the
 * size slot (stepping over PAD entries, R3), read the header, verify the CRC,
 * and write one view record per entry to `d_views` (device, n records).  If
 * `d_dst` is not NULL the payload of entry i is also copied to
 * d_dst + i*dst_stride (RING_EMSGSIZE in the view if len > dst_stride); else
 * the view points into the ring (zero copy, valid until released).  Does not
 * release.  RING_TRY: entries with nothing to read get status RING_EMPTY. */
ring_status_t ring_get(ring_t ring, uint32_t n, ring_view_t* d_views, void* d_dst, uint64_t dst_stride,
                       uint32_t flags, void* stream);
/* ring_release: receiver steps 4-5 for the `count` oldest
 * received entries, in order (R13): clear the busy bits, advance the head with
 * the pointer formulas, free PAD slots already passed, then
 * push the head to every bound producer mirror (credit).  `count` larger than
 * the number held is clamped. */
ring_status_t ring_release(ring_t ring, uint32_t count, void* stream);
/* ring_consume: ring_get + ring_release of each entry as soon as it has been
 * read (and copied, if d_dst != NULL): the paper's receiver loop as one launch.
 * Entries still held from an earlier ring_get are released first (in order). */
ring_status_t ring_consume(ring_t ring, uint32_t n, ring_view_t* d_views, void* d_dst, uint64_t dst_stride,
                           uint32_t flags, void* stream);
/* Tuning: CTAs / threads of the copy-out get (0 = default).  A copy-out get
 * and a put on the SAME GPU spin on each other: one CTA of each must fit on an
 * SM together (the defaults do: ~23 K + ~27 K registers); a get grid of 512
 * threads per CTA does not, and the pair then only ends by timing out.
 * RING_EINVAL: threads > 512 (the kernel's launch bound), not a multiple of 32,
 * or a one-CTA grid with fewer than 96 threads (no copy warp). */
ring_status_t ring_config(ring_t ring, uint32_t copy_ctas, uint32_t threads);

/* ---- inspection (tests, debugging; synchronous) ---------------------------------
 * Copy the control words and size slots to host memory: lock, tail, head,
 * read cursor, and `n_slots` slot words (host array of N u64). */
ring_status_t ring_read_image(ring_t ring, uint64_t* lock, uint64_t* tail, uint64_t* head, uint64_t* cursor,
                              uint64_t* slots);
/* Copy `len` bytes at `offset` of the buffer region to / from host memory
 * (synchronous; tests: ring-image comparison and corruption injection). */
ring_status_t ring_read_data(ring_t ring, uint64_t offset, uint64_t len, void* host_dst);
/* Debug: with B200RING_TRACE=1 in the environment, each put launch records a
 * %globaltimer timeline of its leader rounds and publisher runs; copy the last
 * one (up to n words) to host memory.  RING_EINVAL if tracing is off. */
ring_status_t ring_peer_trace(ring_peer_t peer, uint64_t* host_out, uint32_t n);
/* Debug timeline of the copy-out gets of a ring (B200RING_TRACE=1 at the first
 * get): words [0,510) = (%globaltimer, items planned) per control round,
 * [512,1022) = (%globaltimer, entries released) per finisher release, both
 * rings of 255 pairs; n <= 1024 words. */
ring_status_t ring_get_trace(ring_t ring, uint64_t* host_out, uint32_t n);
ring_status_t ring_write_data(ring_t ring, uint64_t offset, uint64_t len, const void* host_src);

/* ---- environment knobs (read by the host at each launch; for experiments and tests)
 *   B200RING_TRACE=1          debug timelines (ring_peer_trace, ring_get_trace)
 *   B200RING_CHUNK=<bytes>    copy unit size, power of two 4 KiB .. 1 MiB (default
 *                             16 KiB for NVLink destinations, 32 KiB otherwise)
 *   B200RING_CARVEOUT=<pct>   shared-memory carveout of every ring kernel (default 8:
 *                             kernels of one carveout co-reside on an SM)
 *   B200RING_COPYOUT_ALIGN=0|1  force the copy-out loads on the source's 128-B lines
 *                             off / on (default: on iff the buffer region is on another
 *                             GPU -- ring_open, ring_create_split) */

/* ---- stage router (PAPER.md:524-532 round-robin ResultDeliver; PAPER.md:914-924
 * NodeManager reassignment, mechanism only) ------------------------------------------
 * A device-resident route table on the producer GPU: for each (app_id, stage)
 * a list of up to 8 destination attachments, a round-robin counter and an epoch.
 * router_set_route replaces the list and flips the epoch; puts already launched
 * finish to their old destination.  The update is a one-thread
 * kernel on `stream` (the route travels in its parameters): destinations
 * first, the epoch last with a release -- no host synchronisation.  Attachments
 * of fault-tolerant rings or with a running put engine are refused. */
ring_status_t router_create(int device, uint32_t max_routes, router_t* out);
ring_status_t router_destroy(router_t r);
ring_status_t router_set_route(router_t r, uint32_t app_id, uint16_t stage, const ring_peer_t* dests, uint32_t n,
                               void* stream);
/* Routed put: each message of the batch picks dests[rr++ % n] of the route for
 * its (hdr.app_id, hdr.stage), then runs the sender steps on that ring.
 * The chosen destination index is written to d_dest (device, n words) if not NULL. */
ring_status_t ring_put_routed(router_t r, const ring_msg_t* d_msgs, uint32_t n, uint32_t flags, uint32_t* d_status,
                              uint32_t* d_dest, void* stream);
/* Fast reject ("whenever the incoming request rate exceeds
 * K/T_X, the proxy rejects additional requests"): routed puts to (app_id,
 * stage) are admitted at rate k / t_x with burst 1, by arrival time =
 * hdr.accepted_at (the proxy's timestamp), in the units
 * t_x is given in: a message arriving at t is admitted iff t >= next, then
 * next = max(next, t) + t_x / k (exact integer arithmetic on t * k).
 * Rejected messages get RING_EREJECTED and are never sent.  k = 0 disables.
 * The route must exist (router_set_route). */
ring_status_t router_set_admission(router_t r, uint32_t app_id, uint16_t stage, uint64_t t_x, uint32_t k,
                                   void* stream);
/* Theorem 1: M = ceil(K * T_Y / T_X) instances of stage Y
 * give it the output rate K / T_X of stage X.  0 on bad input (t_x or t_y 0, k 0). */
uint64_t ring_required_instances(uint64_t t_x, uint64_t t_y, uint32_t k);
/* Size a route by Theorem 1 and drive it: route (app_id, stage) to the first
 * M = ring_required_instances(t_x, t_y, k) attachments of `pool` (round robin,
 * epoch flip) and admit requests at k / t_x (router_set_admission).  Writes M
 * to *m_out.  RING_EINVAL if the pool has fewer than M (or more than 8 are needed). */
ring_status_t router_size_route(router_t r, uint32_t app_id, uint16_t stage, uint64_t t_x, uint64_t t_y, uint32_t k,
                                const ring_peer_t* pool, uint32_t n_pool, uint32_t* m_out, void* stream);

/* ---- misc ------------------------------------------------------------------------ */
ring_status_t ring_set_timeout_ns(uint64_t ns);
const char* ring_strerror(ring_status_t s);
const char* ring_last_cuda_error(void);
/* Number of kernels this library has launched in this process (for bench accounting). */
uint64_t ring_launch_count(void);
/* Measurement support (not on the data path): offset in ns between `device`'s
 * %globaltimer (the clock of t_put / t_visible) and the host CLOCK_MONOTONIC,
 * offset = gpu - host, within about one PCIe write latency.  Lets latencies
 * between two GPUs of one host be computed on one time base.  Synchronous,
 * ~3 ms. */
ring_status_t ring_clock_offset_ns(int device, int64_t* offset_ns);
/* Measurement support: `iters` flag round trips
 * between one thread on `dev_a` and one on `dev_b` (dev_a == dev_b: two kernels
 * on one GPU), each polling a word in its own memory that the other stores to
 * with system-scope release / acquire -- the ring's signalling pattern.  First
 * 10 % dropped.  Returns the minimum and median round trip, and (if not NULL)
 * the NTP-style offset of dev_b's %globaltimer minus dev_a's from the
 * minimum-RTT round (pong's stamp - (ping's send + RTT/2)), a cross-check of
 * ring_clock_offset_ns.  Synchronous.  RING_ETIMEDOUT if a side stalled (2 s). */
ring_status_t ring_probe_rtt(int dev_a, int dev_b, uint32_t iters, uint64_t* rtt_min_ns, uint64_t* rtt_p50_ns,
                            int64_t* offset_b_minus_a_ns);
/* Footprint of a payload: align_up(64 + len, 128) (R9, R11). */
uint64_t ring_footprint(uint64_t len);

#ifdef __cplusplus
}
#endif
#endif /* B200RING_H */
