"""GPU: release bookkeeping against the oracle.

* A fault-tolerant ring (slot words carry a sequence tag in bits 40-61, R21)
  streamed through many laps with get + release of one entry at a time: every
  placement and the head word after every release equal the oracle's
  (PAPER.md:716-717 receiver steps 4-5; the footprint is bits 0-39 only).
* ring_consume after a ring_get that left entries held releases the held
  entries first, in order (R13): the head stays on entry boundaries and later
  placements still equal the oracle's.
* Argument checks of the routing / tuning calls that have no data path.
"""
import numpy as np
import pytest
import torch

import synth
from gpu_util import upload, msg_tensor, views_host
from oracle.ring import Layout, spsc_image, pack, adv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(2_000_000_000)
    return ring


def _entries(L, stream):
    img = spsc_image(L, [m.length for m in stream])
    return [e for e in img["entries"] if not e[3]], img


def test_fault_tolerant_release_keeps_head_on_entries(R):
    L = Layout(1024, 4)
    stream = synth.random_stream(synth.SEED_BASE + 50, 0, 60, 0, 300)
    ents, img = _entries(L, stream)
    ring = R.ring_create(0, L.R, L.N, 2, R.RING_CREATE_FAULT_TOLERANT)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    R.ring_peer_config(peer, 2, 256, 0)
    buf, srcs = upload(stream, "cuda")
    msgs = msg_tensor(stream, srcs, "cuda")
    st = torch.full((1,), 10, dtype=torch.int32, device="cuda")
    vt = torch.zeros(128, dtype=torch.uint8, device="cuda")
    try:
        for k, m in enumerate(stream):
            R.ring_put_batch(peer, msgs[k * 48:(k + 1) * 48], 1, 0, st)
            R.ring_get(ring, 1, vt)
            torch.cuda.synchronize()
            assert int(st[0]) == 0, k
            v = views_host(vt)[0]
            q, start, f, _ = ents[k]
            assert int(v["status"]) == 0, (k, int(v["status"]))
            assert (int(v["start"]), int(v["footprint"]), int(v["slot_seq"])) == (start, f, q), k
            assert R.ring_read_data(ring, int(v["offset"]), int(v["len"])) == m.payload.tobytes()
            R.ring_release(ring, 1)
            im = R.ring_read_image(ring)
            assert im["head"] == pack(adv(L, start, f), (q + 1) & 0xFFFFFF), (k, hex(im["head"]))
        assert im["tail"] == img["tail"]
        assert im["slots"] == [0] * L.N
    finally:
        R.ring_detach(peer)
        R.ring_destroy(ring)


def test_consume_releases_entries_held_by_get(R):
    L = Layout(4096, 8)
    stream = synth.random_stream(synth.SEED_BASE + 51, 0, 40, 1, 700)
    ents, img = _entries(L, stream)
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, "cuda")
    msgs = msg_tensor(stream, srcs, "cuda")
    st = torch.full((8,), 10, dtype=torch.int32, device="cuda")
    vt = torch.zeros(8 * 128, dtype=torch.uint8, device="cuda")
    k = 0
    try:
        while k < len(stream):
            nb = min(4, len(stream) - k)   # 4 entries (+ a PAD) always fit in an emptied ring
            R.ring_put_batch(peer, msgs[k * 48:(k + nb) * 48], nb, 0, st)
            held = min(2, nb)
            R.ring_get(ring, held, vt)                      # entries k, k+1 held
            if nb > held:
                R.ring_consume(ring, nb - held, vt[held * 128:], None)   # releases the held ones first
            else:
                R.ring_release(ring, held)
            torch.cuda.synchronize()
            assert (st[:nb] == 0).all().item()
            v = views_host(vt)
            for j in range(nb):
                q, start, f, _ = ents[k + j]
                assert int(v[j]["status"]) == 0
                assert (int(v[j]["start"]), int(v[j]["footprint"]), int(v[j]["slot_seq"])) == (start, f, q), k + j
            im = R.ring_read_image(ring)
            q, start, f, _ = ents[k + nb - 1]
            assert im["cursor"] == pack(adv(L, start, f), (q + 1) & 0xFFFFFF)
            assert im["head"] == im["cursor"], (k, hex(im["head"]), hex(im["cursor"]))
            k += nb
        assert im["tail"] == img["tail"] and im["slots"] == [0] * L.N
    finally:
        R.ring_detach(peer)
        R.ring_destroy(ring)


def test_argument_checks(R):
    ring = R.ring_create(0, 1 << 20, 8, 2, R.RING_CREATE_FAULT_TOLERANT)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    router = R.router_create(0)
    try:
        with pytest.raises(R.RingError):     # routed puts run the batched sender: no fault-tolerant rings
            R.router_set_route(router, 7, 1, [peer])
        with pytest.raises(R.RingError):     # get_kernel's launch bound
            R.ring_config(ring, 0, 1024)
        with pytest.raises(R.RingError):     # one CTA of 64 threads: no copy warp
            R.ring_config(ring, 1, 64)
        with pytest.raises(R.RingError):
            R.ring_peer_config(peer, 1, 64, 0)
        R.ring_config(ring, 1, 96)
        R.ring_peer_config(peer, 1, 96, 0)
    finally:
        R.router_destroy(router)
        R.ring_detach(peer)
        R.ring_destroy(ring)
