"""Multi-launch streaming stress: producer and consumer on two GPUs (one
process, peer access), or on one GPU with a system-scope ring and two streams.

Many put / consume launch pairs are queued back to back on two streams (no
host synchronisation between launches), as the benchmark does, with the ring
wrapping many times and the producer waiting for credit.  Every delivered
entry's placement (start, footprint, size-region sequence) and header is
compared with the oracle's prediction for the same stream; the first mismatch
is reported.  Payloads are compared byte for byte in copy-out mode.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu]
CROSS = pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])

import synth  # noqa: E402
from oracle.ring import Layout, Sim, Msg, run, decode_header  # noqa: E402
from gpu_util import upload, msg_tensor, views_host, expected_header, devices  # noqa: E402


def _need(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPU(s)")


@pytest.fixture(scope="module")
def R():
    _need(1)
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(5_000_000_000)
    return ring


def _first_mismatch(views, sim, stream):
    for j, v in enumerate(views):
        d = sim.cons.delivered[j]
        got = (int(v["status"]), int(v["start"]), int(v["footprint"]), int(v["slot_seq"]))
        exp = (0, d.start, d.f, d.seq_slot)
        if got != exp:
            return j, got, exp
        if bytes(v["header"])[:56] != d.header[:56]:
            return j, "header", decode_header(bytes(v["header"]))
    return None


@CROSS
@pytest.mark.parametrize("copy", [False, True])
def test_pipelined_launches_p2p_c3(R, copy, cross):
    prod, cons = devices(2, cross)
    L = Layout(64 << 20, 64)
    m, steps = 32, 24
    base = synth.wan_stream(synth.SEED_BASE + 3, 0, 2 * m)            # two distinct source sets
    stream = [base[(s % 2) * m + q] for s in range(steps) for q in range(m)]
    msgs = [Msg(x.length, x.payload.tobytes(), x.uid, x.accepted_at, x.app_id, x.stage) for x in stream]
    sim = Sim(L, {0: msgs}, mpsc=False, block=True, depth=1, check=False)
    run(sim, policy="drain")
    ring = R.ring_create(cons, L.R, L.N, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), prod, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(base, f"cuda:{prod}")
    d_msgs = [msg_tensor(base[s * m:(s + 1) * m], srcs[s * m:(s + 1) * m], f"cuda:{prod}") for s in range(2)]
    sts = [torch.full((m,), 10, dtype=torch.int32, device=f"cuda:{prod}") for _ in range(steps)]
    vws = [torch.zeros(m * 128, dtype=torch.uint8, device=f"cuda:{cons}") for _ in range(steps)]
    cap = 4194304
    dsts = [torch.zeros(m * cap, dtype=torch.uint8, device=f"cuda:{cons}") for _ in range(2)] if copy else None
    sc, sp = torch.cuda.Stream(cons), torch.cuda.Stream(prod)
    for s in range(steps):
        if copy:
            R.ring_consume(ring, m, vws[s], dsts[s % 2], cap, 0, sc)
            if s % 2 == 1:      # keep the two copy-out buffers from being overwritten unchecked
                pass
        else:
            R.ring_consume(ring, m, vws[s], None, 0, 0, sc)
        R.ring_put_batch(peer, d_msgs[s % 2], m, 0, sts[s], sp)
    torch.cuda.synchronize(prod)
    torch.cuda.synchronize(cons)
    assert all((st == 0).all().item() for st in sts), [np.unique(st.cpu().numpy()).tolist() for st in sts]
    views = np.concatenate([views_host(v) for v in vws])
    mm = _first_mismatch(views, sim, stream)
    assert mm is None, mm
    if copy:       # the last two steps' payloads are still in the copy-out buffers
        for s in (steps - 2, steps - 1):
            d = dsts[s % 2].cpu().numpy()
            for q in range(m):
                x = stream[s * m + q]
                assert d[q * cap: q * cap + x.length].tobytes() == x.payload.tobytes(), (s, q)
    img = R.ring_read_image(ring)
    assert img["tail"] == sim.mem.tail == img["head"]
    R.ring_detach(peer)
    R.ring_destroy(ring)


@CROSS
def test_pipelined_launches_small_ring_many_laps(R, cross):
    """C1-sized ring (32 KiB, 8 slots), 100 launches x 20 messages of U[1,4096] B:
    hundreds of laps, a PAD at nearly every wrap, the producer waiting for
    credit inside every launch."""
    prod, cons = devices(2, cross)
    L = Layout(32768, 8)
    m, steps = 20, 100
    stream = synth.random_stream(synth.SEED_BASE + 11, 0, m * steps, 1, 4096)
    msgs = [Msg(x.length, x.payload.tobytes(), x.uid, x.accepted_at, x.app_id, x.stage) for x in stream]
    sim = Sim(L, {0: msgs}, mpsc=False, block=True, depth=1, check=False)
    run(sim, policy="drain")
    ring = R.ring_create(cons, L.R, L.N, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), prod, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, f"cuda:{prod}")
    d_msgs = msg_tensor(stream, srcs, f"cuda:{prod}")
    sts = torch.full((m * steps,), 10, dtype=torch.int32, device=f"cuda:{prod}")
    vws = torch.zeros(m * steps * 128, dtype=torch.uint8, device=f"cuda:{cons}")
    dst = torch.zeros(m * steps * 4096, dtype=torch.uint8, device=f"cuda:{cons}")
    sc, sp = torch.cuda.Stream(cons), torch.cuda.Stream(prod)
    for s in range(steps):
        R.ring_consume(ring, m, vws[s * m * 128:(s + 1) * m * 128], dst[s * m * 4096:(s + 1) * m * 4096], 4096, 0, sc)
        R.ring_put_batch(peer, d_msgs[s * m * 48:(s + 1) * m * 48], m, 0, sts[s * m:(s + 1) * m], sp)
    torch.cuda.synchronize(prod)
    torch.cuda.synchronize(cons)
    assert (sts == 0).all().item(), np.unique(sts.cpu().numpy()).tolist()
    views = views_host(vws)
    mm = _first_mismatch(views, sim, stream)
    assert mm is None, mm
    d = dst.cpu().numpy()
    for j, x in enumerate(stream):
        assert d[j * 4096: j * 4096 + x.length].tobytes() == x.payload.tobytes(), j
    R.ring_detach(peer)
    R.ring_destroy(ring)
