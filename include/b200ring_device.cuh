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
 * ring can be full.  Implementation: paper_2601_20655_b200/csrc/ring_stage.cuh
 * (compiled for sm_100a).
 */
#pragma once
#include "../paper_2601_20655_b200/csrc/ring_stage.cuh"
