"""GPU fault path: the paper's liveness Cases 1-8
 replayed on a RING_CREATE_FAULT_TOLERANT ring with two
senders on one B200, each case forced into the paper's order by fault
injection (a sender stops for good after an action, or pauses after it until
the host releases it) and lock take-over after the timeout TL.  The receiver's
views, the ring bytes and each sender's statuses are compared with the fault
oracle's replay of the same schedule (oracle/fault.py), which the CPU tests pin
to the outcomes the paper states.  Plus: a torn payload under a valid header is
rejected by the payload checksum (Q10), and fault-free MPSC traffic on a
fault-tolerant ring matches the fault-free oracle's replay."""
import time

import numpy as np
import pytest
import torch

import synth
from gpu_util import views_host
from oracle.fault import replay_case
from oracle.ring import Layout, Msg, decode_header

pytestmark = pytest.mark.gpu

L = Layout(1024, 4)
X, Y = 0, 1
STATUS = {"OK": 0, "COMMITTED": 0, "DROPPED": 11}


@pytest.fixture(scope="module")
def R():
    from paper_2601_20655_b200 import ring
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ring.ring_set_timeout_ns(2_000_000_000)
    ring.ring_set_lock_timeout_ns(50_000)
    return ring


def _payload(pid, n):
    return synth.payload_bytes(synth.SEED_BASE + 40, pid, 0, n).tobytes()


class Sender:
    def __init__(self, R, ring, pid, length):
        self.R = R
        self.peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, pid)
        R.ring_bind_mirror(ring, pid, mh)
        R.ring_peer_config(self.peer, 2, 256, 0)
        self.payload = _payload(pid, length)
        self.src = torch.frombuffer(bytearray(self.payload), dtype=torch.uint8).cuda() if length else \
            torch.zeros(256, dtype=torch.uint8, device="cuda")
        a = R.make_msgs([self.src.data_ptr()], [length], [bytes(16)], [0], [0], [0])
        self.msgs = torch.from_numpy(a.view(np.uint8).copy()).cuda()
        self.status = torch.full((1,), 10, dtype=torch.int32, device="cuda")
        self.arrived = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.go = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.stream = torch.cuda.Stream()

    def fault(self, die_after=0, pause=()):
        mask = 0
        for l in pause:
            mask |= 1 << l
        self.R.ring_peer_set_fault(self.peer, die_after, mask, 0, self.arrived, self.go)

    def launch(self):
        self.R.ring_put_batch(self.peer, self.msgs, 1, 0, self.status, self.stream)

    def wait_at(self, l, timeout=10.0):
        t0 = time.time()
        while int(self.arrived[l]) == 0:
            assert time.time() - t0 < timeout, f"sender never paused at {l}"
            time.sleep(1e-4)

    def release(self, l):
        self.go[l] = 1

    def sync(self):
        self.stream.synchronize()


def _run_case(R, n, xl, yl, script):
    ring = R.ring_create(0, L.R, L.N, 2, R.RING_CREATE_FAULT_TOLERANT)
    xs, ys = Sender(R, ring, X, xl), Sender(R, ring, Y, yl)
    who = {"X": xs, "Y": ys}
    for op, *arg in script:
        if op == "fault":
            who[arg[0]].fault(**arg[1])
        elif op == "launch":
            who[arg[0]].launch()
        elif op == "wait":
            who[arg[0]].wait_at(arg[1])
        elif op == "go":
            who[arg[0]].release(arg[1])
        elif op == "sync":
            who[arg[0]].sync()
    torch.cuda.synchronize()
    progs = {X: [Msg(xl, xs.payload)], Y: [Msg(yl, ys.payload)]}
    sim = replay_case(n, L, xl, yl, progs=progs, payload_crc=True)
    expect = [(g.status, g.ident, g.f, g.start) for g in sim.got]
    views = torch.zeros(8 * 128, dtype=torch.uint8, device="cuda")
    R.ring_consume(ring, len(expect), views, None, 0, R.RING_TRY)
    torch.cuda.synchronize()
    v = views_host(views)[: len(expect)]
    got = []
    for rec in v:
        if rec["status"] == 0:
            h = decode_header(bytes(rec["header"]))
            got.append(("OK", (h["producer_id"], h["seq"]), int(rec["footprint"]), int(rec["start"])))
            data = R.ring_read_data(ring, int(rec["offset"]), int(rec["len"]))
            assert bytes(data) == bytes(progs[h["producer_id"]][h["seq"]].payload)
            assert h["payload_crc"] is not None           # fault-tolerant entries carry the payload CRC
        else:
            assert rec["status"] == R.RING_ECORRUPT, rec["status"]
            got.append(("CORRUPT", None, int(rec["footprint"]), int(rec["start"])))
    assert got == expect, (n, got, expect, sim.log)
    for s, p in ((xs, X), (ys, Y)):
        want = [STATUS[o] for o in sim.prods[p].outcomes] or [R.RING_EPENDING]
        assert s.status.cpu().tolist() == want, (n, p, s.status.cpu().tolist(), sim.prods[p].outcomes)
    return ring


# Scripts forcing the paper's order (X = producer 0, Y = producer 1).  "wait"
# blocks until the sender has paused after that action; "go" releases it.
LOCK, GH, WB, WL, UH = 1, 2, 3, 4, 5
SCRIPTS = {
    1: [("fault", "X", dict(die_after=LOCK)), ("launch", "X"), ("sync", "X"), ("launch", "Y"), ("sync", "Y")],
    2: [("fault", "X", dict(pause=(GH,))), ("launch", "X"), ("wait", "X", GH), ("launch", "Y"), ("sync", "Y"),
        ("go", "X", GH), ("sync", "X")],
    3: [("fault", "X", dict(pause=(GH, WB))), ("fault", "Y", dict(pause=(WB,))), ("launch", "X"), ("wait", "X", GH),
        ("launch", "Y"), ("wait", "Y", WB), ("go", "X", GH), ("wait", "X", WB), ("go", "Y", WB), ("sync", "Y"),
        ("go", "X", WB), ("sync", "X")],
    4: [("fault", "X", dict(pause=(GH, WL))), ("fault", "Y", dict(pause=(WB,))), ("launch", "X"), ("wait", "X", GH),
        ("launch", "Y"), ("wait", "Y", WB), ("go", "X", GH), ("wait", "X", WL), ("go", "Y", WB), ("sync", "Y"),
        ("go", "X", WL), ("sync", "X")],
    5: [("fault", "X", dict(pause=(GH, WB))), ("fault", "Y", dict(pause=(GH, WL))), ("launch", "X"),
        ("wait", "X", GH), ("launch", "Y"), ("wait", "Y", GH), ("go", "X", GH), ("wait", "X", WB), ("go", "Y", GH),
        ("wait", "Y", WL), ("go", "X", WB), ("sync", "X"), ("go", "Y", WL), ("sync", "Y")],
    6: [("fault", "X", dict(pause=(GH, WB, WL))), ("fault", "Y", dict(pause=(GH, WB))), ("launch", "X"),
        ("wait", "X", GH), ("launch", "Y"), ("wait", "Y", GH), ("go", "X", GH), ("wait", "X", WB), ("go", "Y", GH),
        ("wait", "Y", WB), ("go", "X", WB), ("wait", "X", WL), ("go", "Y", WB), ("sync", "Y"), ("go", "X", WL),
        ("sync", "X")],
    7: [("fault", "X", dict(die_after=WL)), ("launch", "X"), ("sync", "X"), ("launch", "Y"), ("sync", "Y")],
    8: [("fault", "X", dict(pause=(UH,))), ("launch", "X"), ("wait", "X", UH), ("launch", "Y"), ("sync", "Y"),
        ("go", "X", UH), ("sync", "X")],
}


@pytest.mark.parametrize("sizes", [(100, 100), (300, 100), (100, 300)])
@pytest.mark.parametrize("case", list(range(1, 9)))
def test_liveness_case_on_gpu(R, case, sizes):
    _run_case(R, case, *sizes, SCRIPTS[case])


def test_torn_payload_rejected_by_payload_crc(R):
    """A payload overwritten after its header was written (the torn entry a
    delayed sender can leave, Q10) is discarded although the header checksum is
    valid."""
    ring = R.ring_create(0, L.R, L.N, 2, R.RING_CREATE_FAULT_TOLERANT)
    s = Sender(R, ring, X, 300)
    s.launch()
    s.sync()
    R.ring_write_data(ring, 64 + 100, b"\xde\xad\xbe\xef")     # tear the payload only
    views = torch.zeros(128, dtype=torch.uint8, device="cuda")
    R.ring_consume(ring, 1, views, None, 0, R.RING_TRY)
    v = views_host(views)[0]
    assert v["status"] == R.RING_ECORRUPT and v["footprint"] == 384


@pytest.mark.parametrize("cross", [False, True])
def test_fault_free_traffic_on_fault_tolerant_ring(R, cross):
    """No faults: two senders alternating on a fault-tolerant ring deliver every
    message exactly once, in per-channel order, byte-exact; slot words carry
    the sequence tag (R21) and footprints as the fault-free oracle predicts.
    `cross`: both senders on GPU 1, the ring on GPU 0 (NVLink)."""
    if cross and torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    sdev = 1 if cross else 0
    ring = R.ring_create(0, 1 << 16, 16, 2, R.RING_CREATE_FAULT_TOLERANT)
    lens = [[100, 4000, 0, 1000, 7000], [300, 64, 2000, 5000, 10]]
    senders = []
    for pid in (X, Y):
        peer, mh = R.ring_attach_peer(R.ring_export(ring), sdev, pid)
        R.ring_bind_mirror(ring, pid, mh)
        R.ring_peer_config(peer, 2, 256, 0)
        pays = [synth.payload_bytes(synth.SEED_BASE + 41, pid, k, n).tobytes() for k, n in enumerate(lens[pid])]
        buf = torch.zeros(sum((n + 255) // 256 * 256 for n in lens[pid]) + 256, dtype=torch.uint8,
                          device=f"cuda:{sdev}")
        srcs, o = [], 0
        for p in pays:
            buf[o:o + len(p)] = torch.frombuffer(bytearray(p), dtype=torch.uint8) if p else buf[o:o]
            srcs.append(buf.data_ptr() + o)
            o += (len(p) + 255) // 256 * 256
        a = R.make_msgs(srcs, lens[pid], [bytes(16)] * 5, [0] * 5, [0] * 5, [0] * 5)
        senders.append((peer, torch.from_numpy(a.view(np.uint8).copy()).cuda(sdev), pays, buf))
    st = [torch.full((5,), 10, dtype=torch.int32, device=f"cuda:{sdev}") for _ in range(2)]
    streams = [torch.cuda.Stream(sdev), torch.cuda.Stream(sdev)]
    for pid in (X, Y):
        R.ring_put_batch(senders[pid][0], senders[pid][1], 5, 0, st[pid], streams[pid])
    torch.cuda.synchronize(sdev)
    torch.cuda.synchronize(0)
    assert all((s == 0).all().item() for s in st)
    views = torch.zeros(10 * 128, dtype=torch.uint8, device="cuda")
    R.ring_get(ring, 10, views, None, 0, R.RING_TRY)
    torch.cuda.synchronize()
    v = views_host(views)
    slots = R.ring_read_image(ring)["slots"]
    last = {X: -1, Y: -1}
    for rec in v:
        assert rec["status"] == 0
        h = decode_header(bytes(rec["header"]))
        pid, k = h["producer_id"], h["seq"]
        assert k == last[pid] + 1
        last[pid] = k
        assert bytes(R.ring_read_data(ring, int(rec["offset"]), int(rec["len"]))) == senders[pid][2][k]
        w = int(slots[int(rec["slot_seq"]) % 16])
        assert (w >> 40) & ((1 << 22) - 1) == int(rec["slot_seq"]) & ((1 << 22) - 1)
        assert w & ((1 << 40) - 1) == int(rec["footprint"]) == ((64 + lens[pid][k] + 127) // 128) * 128
    assert last == {X: 4, Y: 4}
    R.ring_release(ring, 10)
    torch.cuda.synchronize()
