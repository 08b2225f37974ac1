"""Reserve-then-commit MPSC rings (oracle/reserve.py):
producers on concurrent streams (and across GPUs when available) claim under
the lock and copy outside it, with a consumer running concurrently.  Every
channel is delivered exactly once, in order, byte-exact; the entries tile the
ring by the pointer formulas (R3) -- as one producer's
stream with the merged lengths would, except that a PAD reserved by a sender
that then waits for credit without the lock (R23) may precede another
sender's smaller message."""
import numpy as np
import pytest

import synth
from gpu_util import msg_tensor, upload, views_host
from oracle.ring import Layout, decode_header, footprint, seq_next, spsc_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(5_000_000_000)
    return ring


@pytest.mark.parametrize("cross", [False, True])
def test_reserve_commit_concurrent_producers(R, cross):
    if cross and torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    L = Layout(1 << 20, 32)
    devs = [0, 1, 1] if cross else [0, 0, 0]
    n = 60
    ring = R.ring_create(0, L.R, L.N, 3, R.RING_CREATE_RESERVE_COMMIT | (0 if cross else R.RING_CREATE_LOCAL))
    h = R.ring_export(ring)
    peers, keep, sts, strs, streams = [], [], [], [], {}
    for pid, d in enumerate(devs):
        pe, mh = R.ring_attach_peer(h, d, pid)
        R.ring_bind_mirror(ring, pid, mh)
        peers.append(pe)
        streams[pid] = synth.random_stream(synth.SEED_BASE + 80, pid, n, 1, 40000)
        b, s = upload(streams[pid], f"cuda:{d}")
        m = msg_tensor(streams[pid], s, f"cuda:{d}")
        keep += [b, m]
        sts.append(torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{d}"))
        strs.append(torch.cuda.Stream(d))
    total = 3 * n
    vt = torch.zeros(total * 128, dtype=torch.uint8, device="cuda:0")
    cap = 40064
    dst = torch.zeros(total * cap, dtype=torch.uint8, device="cuda:0")
    sc = torch.cuda.Stream(0)
    R.ring_consume(ring, total, vt, dst, cap, 0, sc)          # consumer first; copies out before release
    for b in range(6):                                         # producers interleave launches of 10
        for pid, d in enumerate(devs):
            m = keep[2 * pid + 1]
            R.ring_put_batch(peers[pid], m[b * 10 * 48:(b + 1) * 10 * 48], 10, 0, sts[pid][b * 10:(b + 1) * 10],
                             strs[pid])
    for d in set(devs):
        torch.cuda.synchronize(d)
    assert all((s == 0).all().item() for s in sts)
    v = views_host(vt)
    assert (v["status"] == 0).all()
    out = dst.cpu().numpy()
    hs = [decode_header(bytes(x["header"])) for x in v]
    for pid in range(3):
        assert [h["seq"] for h in hs if h["producer_id"] == pid] == list(range(n))
    for j, (x, hd) in enumerate(zip(v, hs)):
        m = streams[hd["producer_id"]][hd["seq"]]
        assert out[j * cap: j * cap + int(x["len"])].tobytes() == m.payload.tobytes()
    # Placement: the pointer formulas over the observed entries.
    # A PAD here may belong to a sender that reserved it and then waited for
    # credit WITHOUT the lock (reserve-then-commit, R23; oracle/reserve.py:
    # ClaimPad, then UnlockFull -> AdvW / RH) while another sender's smaller
    # message went in after it, so the PADs are where the GPU put them:
    # each one fills [end of the previous entry, R) and is needed by a message
    # of a waiting sender: the next message of one of the producers after it
    # does not fit in [pos, R) (the others may place many messages first).
    ent = [(int(x["slot_seq"]), int(x["start"]), int(x["footprint"])) for x in v]
    pids = [h["producer_id"] for h in hs]
    assert [e[2] for e in ent] == [footprint(L, int(x["len"])) for x in v]
    pos = 0
    for q, (sq, st, f) in enumerate(ent):
        if q and sq == seq_next(seq_next(ent[q - 1][0])):   # one PAD slot in between: [pos, R), then 0
            assert pos < L.R and st == 0, (q, pos, st)
            nxt = [next((j for j in range(q, len(ent)) if pids[j] == p), None) for p in set(pids)]
            assert any(j is not None and ent[j][2] > L.R - pos for j in nxt), (q, pos)
        else:
            assert q == 0 or sq == seq_next(ent[q - 1][0]), (q, sq, ent[q - 1][0])
            assert st == (pos if pos < L.R else 0), (q, st, pos)
        pos = st + f
    # unless such a PAD went in ahead of a message that fits, the placement is
    # exactly the SPSC rule over the merged order
    early_pad = any(ent[q][0] == seq_next(seq_next(ent[q - 1][0])) and
                    ent[q][2] <= L.R - (ent[q - 1][1] + ent[q - 1][2]) for q in range(1, len(ent)))
    merged = [streams[hd["producer_id"]][hd["seq"]].length for hd in hs]
    img = [e for e in spsc_image(L, merged)["entries"] if not e[3]]
    if not early_pad:
        assert ent == [tuple(e[:3]) for e in img]
    im = R.ring_read_image(ring)
    assert im["lock"] == 0 and im["tail"] == im["head"]
    for pe in peers:
        R.ring_detach(pe)
    R.ring_destroy(ring)


@pytest.mark.parametrize("die_at", ["lock", "wb"])
def test_reserve_commit_lost_sender(R, die_at):
    """A sender lost with its reservation made -- holding the lock (RING_AT_LOCK)
    or after unlocking, before its copy and commit (RING_AT_WB): the next sender
    takes the lock over, its entries wait behind the hole until the hole
    becomes a PAD the receiver skips (both after the hole timeout) (oracle/reserve.py crash
    mode); the live sender's messages arrive complete, in order, at the places
    the oracle's placement rule gives when the lost entry is kept as padding."""
    R.ring_set_hole_timeout_ns(1_000_000)
    L = Layout(1 << 16, 16)
    ring = R.ring_create(0, L.R, L.N, 2, R.RING_CREATE_RESERVE_COMMIT | R.RING_CREATE_LOCAL)
    h = R.ring_export(ring)
    peers = []
    for pid in range(2):
        pe, mh = R.ring_attach_peer(h, 0, pid)
        R.ring_bind_mirror(ring, pid, mh)
        peers.append(pe)
    xs = synth.random_stream(synth.SEED_BASE + 81, 0, 1, 100, 3000)
    ys = synth.random_stream(synth.SEED_BASE + 81, 1, 3, 100, 3000)
    keep = []
    for pid, stream in ((0, xs), (1, ys)):
        b, s = upload(stream, "cuda:0")
        keep += [b, msg_tensor(stream, s, "cuda:0")]
    arrived = torch.zeros(8, dtype=torch.int32).pin_memory()
    go = torch.zeros(8, dtype=torch.int32).pin_memory()
    R.ring_peer_set_fault(peers[0], R.RING_AT_LOCK if die_at == "lock" else R.RING_AT_WB, 0, 0, arrived, go)
    stx = torch.full((1,), 10, dtype=torch.int32, device="cuda:0")
    sty = torch.full((3,), 10, dtype=torch.int32, device="cuda:0")
    R.ring_put_batch(peers[0], keep[1], 1, 0, stx)
    torch.cuda.synchronize()
    R.ring_put_batch(peers[1], keep[3], 3, 0, sty)
    torch.cuda.synchronize()
    assert stx.cpu().tolist() == [R.RING_EPENDING] and sty.cpu().tolist() == [0, 0, 0]
    vt = torch.zeros(4 * 128, dtype=torch.uint8, device="cuda:0")
    R.ring_consume(ring, 4, vt, None, 0, R.RING_TRY)
    torch.cuda.synchronize()
    v = views_host(vt)
    assert [int(x["status"]) for x in v] == [0, 0, 0, R.RING_EMPTY]
    hs = [decode_header(bytes(x["header"])) for x in v[:3]]
    assert [(h["producer_id"], h["seq"]) for h in hs] == [(1, 0), (1, 1), (1, 2)]
    img = [e for e in spsc_image(L, [xs[0].length] + [m.length for m in ys])["entries"] if not e[3]]
    assert [(int(x["slot_seq"]), int(x["start"]), int(x["footprint"])) for x in v[:3]] == [tuple(e[:3]) for e in img[1:]]
    for x, m in zip(v[:3], ys):
        assert R.ring_read_data(ring, int(x["offset"]), int(x["len"])) == m.payload.tobytes()
    R.ring_set_hole_timeout_ns(50_000_000)
    for pe in peers:
        R.ring_detach(pe)
    R.ring_destroy(ring)
