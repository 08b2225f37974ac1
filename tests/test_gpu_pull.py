"""GPU: pull placement (ring_open) against the oracle.

The ring lives in the PRODUCER's GPU memory; its producer writes entries
locally and the consumer on another GPU opens the ring, polls it and pulls
every payload over NVLink with its copy-out get (the paper's one-sided READ,
PAPER.md:181-188, carrying the data instead of the one-sided WRITE; DESIGN.md
reading R24).  The protocol is the same, so the placements, headers and bytes
must be exactly the oracle's.
"""
import numpy as np
import pytest
import torch

import synth
from gpu_util import upload, msg_tensor, views_host, oracle_spsc, to_oracle_msgs, check_views_against_oracle, \
    devices, replay_mpsc
from oracle.ring import Layout, decode_header

pytestmark = pytest.mark.gpu
CROSS = pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(10_000_000_000)
    return ring


def _pull_stream(R, L, stream, prod, cons, cap):
    owner = R.ring_create(prod, L.R, L.N, 1, 0)               # the ring at the producer
    h = R.ring_export(owner)
    peer, mh = R.ring_attach_peer(h, prod, 0)
    ring = R.ring_open(h, cons)                               # the consumer pulls from it
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, f"cuda:{prod}")
    msgs = msg_tensor(stream, srcs, f"cuda:{prod}")
    n = len(stream)
    vt = torch.zeros(n * 128, dtype=torch.uint8, device=f"cuda:{cons}")
    dst = torch.zeros(n * cap, dtype=torch.uint8, device=f"cuda:{cons}")
    st = torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{prod}")
    sc, sp = torch.cuda.Stream(cons), torch.cuda.Stream(prod)
    R.ring_consume(ring, n, vt, dst, cap, 0, sc)              # consumer first: it waits for data
    R.ring_put_batch(peer, msgs, n, 0, st, sp)
    torch.cuda.synchronize(prod)
    torch.cuda.synchronize(cons)
    v = views_host(vt)
    d = dst.cpu().numpy()
    pl = [d[j * cap: j * cap + int(v[j]["len"])].tobytes() for j in range(n)]
    img = R.ring_read_image(ring)
    status = st.cpu().tolist()
    R.ring_destroy(ring)
    R.ring_detach(peer)
    R.ring_destroy(owner)
    return v, pl, status, img


@CROSS
def test_pull_c3_wan_tensors(R, cross):
    """BASELINE.json configs[2] with the ring at the producer: 48 Wan2.1-shaped
    tensors (4,194,304 / 4,193,280 B), one streaming put launch and one
    copy-out consume that pulls every payload."""
    prod, cons = devices(2, cross)
    L = Layout(64 << 20, 64)
    stream = synth.wan_stream(synth.SEED_BASE + 3, 0, 48)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _pull_stream(R, L, stream, prod, cons, 4194304)
    assert st == [0] * 48, st
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail == img["head"]


@CROSS
def test_pull_small_ring_many_laps(R, cross):
    """C1's stream (1,000 messages of U[1, 4096] B) through an 8-slot 32-KiB
    ring at the producer: ~130 laps, PAD entries at the wraps, credit through
    the mirror, every payload pulled."""
    prod, cons = devices(2, cross)
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 1000, 1, 4096)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _pull_stream(R, L, stream, prod, cons, 4096)
    assert st == [0] * 1000
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]


@CROSS
def test_pull_mpsc_three_producers(R, cross):
    """Three producers into one MPSC ring (paper lock) that lives on the first
    producer's GPU; the consumer pulls from another GPU.  Per-channel order
    exact, the observed merge replayed by the oracle, every payload pulled."""
    devs = devices(4, cross)          # consumer devs[0], producers devs[1..3], ring at devs[1]
    L = Layout(1 << 20, 32)
    n = 120
    streams = {pid: synth.random_stream(synth.SEED_BASE + 6, pid, n, 1, 40000) for pid in range(3)}
    owner = R.ring_create(devs[1], L.R, L.N, 3, 0)
    h = R.ring_export(owner)
    ring = R.ring_open(h, devs[0])
    peers, bufs, tens, sts, strs = [], [], [], [], []
    for pid in range(3):
        dev = devs[pid + 1]
        pe, mh = R.ring_attach_peer(h, dev, pid)
        R.ring_bind_mirror(ring, pid, mh)
        peers.append(pe)
        b, srcs = upload(streams[pid], f"cuda:{dev}")
        bufs.append(b)
        tens.append(msg_tensor(streams[pid], srcs, f"cuda:{dev}"))
        sts.append(torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{dev}"))
        strs.append(torch.cuda.Stream(dev))
    cap = 40000
    vt = torch.zeros(3 * n * 128, dtype=torch.uint8, device=f"cuda:{devs[0]}")
    dst = torch.zeros(3 * n * cap, dtype=torch.uint8, device=f"cuda:{devs[0]}")
    sc = torch.cuda.Stream(devs[0])
    try:
        R.ring_consume(ring, 3 * n, vt, dst, cap, 0, sc)
        for pid in range(3):
            R.ring_put_batch(peers[pid], tens[pid], n, 0, sts[pid], strs[pid])
        for d in set(devs):
            torch.cuda.synchronize(d)
        for pid in range(3):
            assert sts[pid].cpu().tolist() == [0] * n, pid
        v = views_host(vt)
        d = dst.cpu().numpy()
        hdrs = [decode_header(bytes(x["header"])) for x in v]
        order = [hh["producer_id"] for hh in hdrs]
        for pid in range(3):
            assert [hh["seq"] for hh in hdrs if hh["producer_id"] == pid] == list(range(n))
        for j, hh in enumerate(hdrs):
            m = streams[hh["producer_id"]][hh["seq"]]
            assert d[j * cap: j * cap + int(v[j]["len"])].tobytes() == m.payload.tobytes()
        sim = replay_mpsc(L, {pid: to_oracle_msgs(streams[pid]) for pid in range(3)}, order)
        for x, dd in zip(v, sim.cons.delivered):
            assert (int(x["start"]), int(x["footprint"]), int(x["slot_seq"])) == (dd.start, dd.f, dd.seq_slot)
        img = R.ring_read_image(ring)
        assert img["lock"] == 0 and img["tail"] == sim.mem.tail == img["head"]
    finally:
        for d in set(devs):
            torch.cuda.synchronize(d)
        R.ring_destroy(ring)
        for pe in peers:
            R.ring_detach(pe)
        R.ring_destroy(owner)


def test_open_rejects_local_rings(R):
    owner = R.ring_create(0, 1 << 20, 8, 1, R.RING_CREATE_LOCAL)
    try:
        with pytest.raises(R.RingError):
            R.ring_open(R.ring_export(owner), 0)
    finally:
        R.ring_destroy(owner)


# ---------------------------------------------------------------------------------------
# split placement (ring_create_split): control words + header copies at the
# consumer, the buffer region at the producer
# ---------------------------------------------------------------------------------------
def _split_stream(R, L, stream, prod, cons, cap):
    ring = R.ring_create_split(cons, prod, L.R, L.N, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), prod, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, f"cuda:{prod}")
    msgs = msg_tensor(stream, srcs, f"cuda:{prod}")
    n = len(stream)
    vt = torch.zeros(n * 128, dtype=torch.uint8, device=f"cuda:{cons}")
    dst = torch.zeros(n * cap, dtype=torch.uint8, device=f"cuda:{cons}")
    st = torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{prod}")
    sc, sp = torch.cuda.Stream(cons), torch.cuda.Stream(prod)
    R.ring_consume(ring, n, vt, dst, cap, 0, sc)
    R.ring_put_batch(peer, msgs, n, 0, st, sp)
    torch.cuda.synchronize(prod)
    torch.cuda.synchronize(cons)
    v = views_host(vt)
    d = dst.cpu().numpy()
    pl = [d[j * cap: j * cap + int(v[j]["len"])].tobytes() for j in range(n)]
    img = R.ring_read_image(ring)
    status = st.cpu().tolist()
    R.ring_detach(peer)
    R.ring_destroy(ring)
    return v, pl, status, img


@CROSS
def test_split_c3_wan_tensors(R, cross):
    prod, cons = devices(2, cross)
    L = Layout(64 << 20, 64)
    stream = synth.wan_stream(synth.SEED_BASE + 3, 0, 48)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _split_stream(R, L, stream, prod, cons, 4194304)
    assert st == [0] * 48, st
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail == img["head"]


@CROSS
def test_split_small_ring_many_laps(R, cross):
    prod, cons = devices(2, cross)
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 1000, 1, 4096)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _split_stream(R, L, stream, prod, cons, 4096)
    assert st == [0] * 1000
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]


def test_split_rejects(R):
    with pytest.raises(R.RingError):
        R.ring_create_split(0, 0, 1 << 20, 8, 1, R.RING_CREATE_FAULT_TOLERANT)
    ring = R.ring_create_split(0, 0, 1 << 20, 8, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    try:
        with pytest.raises(R.RingError):
            R.ring_peer_device_view(peer)        # a fused put would not write the header copies
        with pytest.raises(R.RingError):
            R.ring_open(R.ring_export(ring), 0)  # consumed where its control words live
    finally:
        R.ring_detach(peer)
        R.ring_destroy(ring)
