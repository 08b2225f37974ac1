"""Lock-free fan-in: per-producer single-producer rings on
the consumer GPU served by one consumer warp (ring_set_consume).  Producers
stream concurrently with the consumer; every channel must arrive exactly once,
in order, byte-exact, with each ring's placement as the fault-free oracle
predicts for that producer's length sequence, and no
producer may be starved while others have data (rounds rotate)."""
import numpy as np
import pytest

import synth
from gpu_util import msg_tensor, upload, views_host
from oracle.ring import Layout, decode_header, spsc_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(5_000_000_000)
    return ring


@pytest.mark.parametrize("remote", [False, True])
def test_set_consume_three_producers(R, remote):
    if remote and torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    L = Layout(256 << 10, 64)
    devs = [0, 1, 1] if remote else [0, 0, 0]
    rings, peers, streams, data = [], [], [], []
    for i, d in enumerate(devs):
        r = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_DEFAULT if d != 0 else R.RING_CREATE_LOCAL)
        pe, mh = R.ring_attach_peer(R.ring_export(r), d, 0)
        R.ring_bind_mirror(r, 0, mh)
        rings.append(r)
        peers.append(pe)
        stream = synth.random_stream(synth.SEED_BASE + 70, i, 40, 1, 4096)
        buf, srcs = upload(stream, f"cuda:{d}")
        data.append((stream, buf, msg_tensor(stream, srcs, f"cuda:{d}")))
        streams.append(torch.cuda.Stream(d))
    s = R.ring_set_create(rings)
    total = sum(len(x[0]) for x in data)
    views = torch.zeros(total * 128, dtype=torch.uint8, device="cuda:0")
    idx = torch.full((total,), 99, dtype=torch.int32, device="cuda:0")
    sc = torch.cuda.Stream(0)
    R.ring_set_consume(s, total, views, idx, 0, sc)            # the consumer runs first and waits
    sts = []
    for i, d in enumerate(devs):                                # producers: 4 launches of 10 each
        st = torch.full((40,), 10, dtype=torch.int32, device=f"cuda:{d}")
        sts.append(st)
        for b in range(4):
            R.ring_put_batch(peers[i], data[i][2][b * 10 * 48:(b + 1) * 10 * 48], 10, 0, st[b * 10:(b + 1) * 10],
                             streams[i])
    for d in set(devs):
        torch.cuda.synchronize(d)
    assert all((st == 0).all().item() for st in sts)
    v = views_host(views)
    ix = [int(x) for x in idx.cpu().tolist()]
    assert all(x["status"] == 0 for x in v)
    assert sorted(ix) == sorted([i for i in range(3) for _ in range(40)])
    for i in range(3):
        mine = [x for x, j in zip(v, ix) if j == i]
        assert all(int(x["reserved"][0]) == i for x in mine)
        stream = data[i][0]
        img = [e for e in spsc_image(L, [m.length for m in stream])["entries"] if not e[3]]
        for k, x in enumerate(mine):
            h = decode_header(bytes(x["header"]))
            assert (h["seq"], h["uid"], h["payload_len"], h["crc_ok"]) == (k, stream[k].uid, stream[k].length, True)
            assert (int(x["slot_seq"]), int(x["start"]), int(x["footprint"])) == tuple(img[k][:3])
            assert R.ring_read_data(rings[i], int(x["offset"]), int(x["len"])) == stream[k].payload.tobytes()
    R.ring_set_destroy(s)
    for pe in peers:
        R.ring_detach(pe)
    for r in rings:
        R.ring_destroy(r)


def test_set_consume_try_and_rotation(R):
    """RING_TRY on empty rings reports EMPTY; with every ring holding data, one
    call of k messages takes one from each ring (the round serves all lanes)."""
    L = Layout(64 << 10, 16)
    rings, peers = [], []
    for i in range(4):
        r = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
        pe, mh = R.ring_attach_peer(R.ring_export(r), 0, 0)
        R.ring_bind_mirror(r, 0, mh)
        rings.append(r)
        peers.append(pe)
    s = R.ring_set_create(rings)
    views = torch.zeros(8 * 128, dtype=torch.uint8, device="cuda:0")
    R.ring_set_consume(s, 2, views, None, R.RING_TRY)
    torch.cuda.synchronize()
    assert [int(x["status"]) for x in views_host(views)[:2]] == [R.RING_EMPTY] * 2
    keep = []
    for i in range(4):
        stream = synth.fixed_stream(synth.SEED_BASE + 71, i, 3, 500)
        buf, srcs = upload(stream, "cuda:0")
        m = msg_tensor(stream, srcs, "cuda:0")
        st = torch.zeros(3, dtype=torch.int32, device="cuda:0")
        R.ring_put_batch(peers[i], m, 3, 0, st)
        keep += [buf, m, st]
    torch.cuda.synchronize()
    idx = torch.zeros(8, dtype=torch.int32, device="cuda:0")
    R.ring_set_consume(s, 4, views, idx, R.RING_TRY)
    torch.cuda.synchronize()
    assert sorted(int(x) for x in idx[:4].cpu().tolist()) == [0, 1, 2, 3]
    R.ring_set_consume(s, 8, views, idx, R.RING_TRY)
    torch.cuda.synchronize()
    st8 = [int(x["status"]) for x in views_host(views)[:8]]
    assert st8 == [0] * 8
    R.ring_set_destroy(s)
    for pe in peers:
        R.ring_detach(pe)
    for r in rings:
        R.ring_destroy(r)
