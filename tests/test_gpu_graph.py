"""CUDA-graph capture of the data path (per-launch counter sets
alternate by launch parity, so a graph holding an even number of launches per
context can be replayed): puts and copy-out consumes captured on two streams,
replayed several times; every replay delivers the batch byte-exact, and the
entries' placement continues lap after lap exactly as the oracle predicts for
the concatenated length sequence."""
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
    ring.ring_set_timeout_ns(2_000_000_000)
    return ring


def test_graph_replay_put_consume(R):
    L = Layout(1 << 20, 16)
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    m, G, replays = 6, 2, 3                       # 6 messages per step, 2 steps per graph (even)
    streams = [synth.random_stream(synth.SEED_BASE + 90, 0, m, 1, 60000) for _ in range(1)]
    stream = streams[0]
    buf, srcs = upload(stream, "cuda:0")
    msgs = msg_tensor(stream, srcs, "cuda:0")
    cap = 60032
    st = torch.full((G, m), 10, dtype=torch.int32, device="cuda:0")
    vts = [torch.zeros(m * 128, dtype=torch.uint8, device="cuda:0") for _ in range(G)]
    dsts = [torch.zeros(m * cap, dtype=torch.uint8, device="cuda:0") for _ in range(G)]
    sp, sc, capst = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    # warm-up (loads kernels, allocates), then capture
    R.ring_put_batch(peer, msgs, m, 0, st[0], sp)
    R.ring_consume(ring, m, vts[0], dsts[0], cap, 0, sc)
    R.ring_put_batch(peer, msgs, m, 0, st[1], sp)
    R.ring_consume(ring, m, vts[1], dsts[1], cap, 0, sc)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    capst.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=capst, capture_error_mode="relaxed"):
        sp.wait_stream(capst)
        sc.wait_stream(capst)
        for s in range(G):
            R.ring_put_batch(peer, msgs, m, 0, st[s], sp)
            R.ring_consume(ring, m, vts[s], dsts[s], cap, 0, sc)
        capst.wait_stream(sp)
        capst.wait_stream(sc)
    lengths = [x.length for x in stream]
    img = [e for e in spsc_image(L, lengths * (2 + G * replays))["entries"] if not e[3]]
    for r in range(replays):
        g.replay()
        torch.cuda.synchronize()
        assert (st == 0).all().item()
        for s in range(G):
            v = views_host(vts[s])
            out = dsts[s].cpu().numpy()
            for j, x in enumerate(v):
                assert x["status"] == 0
                h = decode_header(bytes(x["header"]))
                step = 2 + r * G + s
                assert h["seq"] == step * m + j
                assert out[j * cap: j * cap + int(x["len"])].tobytes() == stream[j].payload.tobytes()
                e = img[step * m + j]
                assert (int(x["slot_seq"]), int(x["start"]), int(x["footprint"])) == tuple(e[:3])
    R.ring_detach(peer)
    R.ring_destroy(ring)
