"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Compared element by element on the same seeded inputs (synth/): delivered
payload bytes, the 56 checksummed header bytes (incl. producer id and channel
seq), entry placement (start offset, footprint, size-region sequence number),
statuses, and the ring image (tail, head, read cursor, size slots) at quiescent
points.  Several results are timing-dependent only under MPSC fan-in (the lock
order, R16): there the per-channel sequences are compared exactly and the
observed merge is replayed through the oracle, which must then predict every
placement.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle.ring import Layout, Sim, Msg, run, decode_header  # noqa: E402
from gpu_util import (to_oracle_msgs, oracle_spsc, upload, msg_tensor, batches, views_host,  # noqa: E402
                      check_views_against_oracle, expected_header, replay_mpsc, devices)


def _need(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPU(s)")


@pytest.fixture(scope="module")
def R():
    _need(1)
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(5_000_000_000)
    return ring


def _status(t):
    return [int(x) for x in t.cpu().tolist()]


def _run_spsc(R, L, stream, flags=0, mode="consume_copy", local=True, dev=0, max_batch=10**9, copy_mode=0):
    """Feed `stream` through one ring on `dev` in host-planned batches (put then
    get in stream order on one GPU; no two kernels ever wait on each other)."""
    ring = R.ring_create(dev, L.R, L.N, 1, R.RING_CREATE_LOCAL if local else 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), dev, 0)
    R.ring_bind_mirror(ring, 0, mh)
    R.ring_peer_config(peer, 0, 0, copy_mode)
    buf, srcs = upload(stream, f"cuda:{dev}")
    msgs = msg_tensor(stream, srcs, f"cuda:{dev}")
    views_all, payloads, put_status = [], [], []
    cap = max(m.length for m in stream) if stream else 1
    cap = max(16, (cap + 15) // 16 * 16)
    s = torch.cuda.current_stream(dev)
    for b in batches(stream, L, max_batch):
        k = len(b)
        st = torch.full((k,), 10, dtype=torch.int32, device=f"cuda:{dev}")
        R.ring_put_batch(peer, msgs[b[0] * 48:(b[-1] + 1) * 48], k, flags, st, s)
        vt = torch.zeros(k * 128, dtype=torch.uint8, device=f"cuda:{dev}")
        if mode == "consume_copy":
            dst = torch.zeros(k * cap, dtype=torch.uint8, device=f"cuda:{dev}")
            R.ring_consume(ring, k, vt, dst, cap, 0, s)
            torch.cuda.synchronize(dev)
            v = views_host(vt)
            d = dst.cpu().numpy()
            payloads += [d[j * cap: j * cap + int(v[j]["len"])].tobytes() for j in range(k)]
        elif mode == "consume_view":
            R.ring_consume(ring, k, vt, None, 0, 0, s)
            torch.cuda.synchronize(dev)
            v = views_host(vt)
        else:  # get (view) + read through the inspection ABI + in-order release
            R.ring_get(ring, k, vt, None, 0, 0, s)
            torch.cuda.synchronize(dev)
            v = views_host(vt)
            payloads += [R.ring_read_data(ring, int(x["offset"]), int(x["len"])) for x in v]
            R.ring_release(ring, k, s)
            torch.cuda.synchronize(dev)
        views_all.append(v)
        put_status += _status(st)
    img = R.ring_read_image(ring)
    R.ring_detach(peer)
    R.ring_destroy(ring)
    return np.concatenate(views_all) if views_all else None, payloads, put_status, img


@pytest.mark.parametrize("mode,copy_mode", [("consume_copy", 0), ("get_view_release", 0), ("consume_view", 0),
                                            ("consume_copy", 1), ("get_view_release", 1)])
def test_c1_stream_bit_exact(R, mode, copy_mode):
    """BASELINE.json configs[0] on the GPU: 1 -> 1, 8 slots x 4 KB (R = 32 KiB),
    1,000 messages of U[1, 4096] B."""
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 1000, 1, 4096)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    views, payloads, st, img = _run_spsc(R, L, stream, mode=mode, copy_mode=copy_mode)
    assert st == [0] * 1000
    check_views_against_oracle(views, sim, 0, stream)
    if payloads:
        assert payloads == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail and img["head"] == sim.mem.head and img["cursor"] == sim.mem.tail
    assert img["slots"] == [0] * L.N and img["lock"] == 0
    assert all(int(v["t_visible"]) > 0 for v in views)


@pytest.mark.parametrize("shape", ["c1", "wide", "c3"])
def test_copyout_line_aligned_loads(R, monkeypatch, shape):
    """The copy-out path for a buffer region on another GPU (split / pull),
    forced on one GPU: units after an entry's first start on the source's
    128-B lines, the first unit's lanes in front of the payload load the
    header's line and store nothing, ragged last units keep 4 loads in flight
    (DESIGN.md §6.2).  Sizes below 1 KiB, every ragged tail length class,
    multi-unit entries and the C3 tensors; bit-exact against the oracle."""
    monkeypatch.setenv("B200RING_COPYOUT_ALIGN", "1")
    if shape == "c1":
        L, stream = Layout(32768, 8), synth.random_stream(synth.SEED_BASE + 1, 0, 1000, 1, 4096)
    elif shape == "wide":
        L, stream = Layout(4 << 20, 32), synth.random_stream(synth.SEED_BASE + 11, 0, 300, 1000, 300000)
    else:
        L, stream = Layout(64 << 20, 64), synth.wan_stream(synth.SEED_BASE + 3, 0, 24)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    views, payloads, st, img = _run_spsc(R, L, stream, local=False)
    assert st == [0] * len(stream)
    check_views_against_oracle(views, sim, 0, stream)
    assert payloads == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail == img["head"]


def test_c1_system_scope_same_device(R):
    """The same stream through a ring created without RING_CREATE_LOCAL (sys-scope fences)."""
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 200, 1, 4096)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    views, payloads, st, img = _run_spsc(R, L, stream, local=False)
    check_views_against_oracle(views, sim, 0, stream)
    assert payloads == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail == img["head"]


@pytest.mark.parametrize("copy_mode,local", [(0, True), (1, True), (0, False)])
def test_edge_sizes_and_unaligned_sources(R, copy_mode, local):
    """Empty payload, sub-vector tails, exact fit f == R, and sources aligned to
    1, 4, 16 and 32 B (the TMA engine falls back to the LSU for unaligned ones;
    a ring without RING_CREATE_LOCAL takes the NVLink put kernel, whose 32-B
    loop falls back to 16-B, 4-B and byte copies)."""
    L = Layout(4096, 8)
    # f == R (4096 - 64 B payload) only fits an empty ring at P_b = 0 without
    # waiting for the consumer (one GPU runs put, then get), so it goes first.
    # Later entries keep f <= R/2 so that each fits after any wrap.
    lens = [4096 - 64, 0, 1, 15, 16, 17, 63, 64, 65, 127, 128, 129, 1000, 1900, 3]
    stream = [synth.Message(0, q, n, *synth.header_fields(7, 0, q), payload=synth.payload_bytes(7, 0, q, n))
              for q, n in enumerate(lens)]
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL if local else 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    R.ring_peer_config(peer, 0, 0, copy_mode)
    host = np.zeros(sum(n + 64 for n in lens), dtype=np.uint8)
    srcs_off, o = [], 0
    for q, m in enumerate(stream):
        o += (1, 4, 16, 0)[q % 4]                   # aligned to 1, 4, 16, 32 B
        srcs_off.append(o)
        host[o:o + m.length] = m.payload
        o += m.length + 16
        o = (o + 31) // 32 * 32
    buf = torch.from_numpy(host).cuda()
    msgs = msg_tensor(stream, [buf.data_ptr() + x for x in srcs_off], "cuda:0")
    got = []
    for j in range(len(stream)):                      # one message per launch
        st = torch.full((1,), 10, dtype=torch.int32, device="cuda:0")
        R.ring_put_batch(peer, msgs[j * 48:(j + 1) * 48], 1, 0, st)
        vt = torch.zeros(128, dtype=torch.uint8, device="cuda:0")
        dst = torch.zeros(4096, dtype=torch.uint8, device="cuda:0")
        R.ring_consume(ring, 1, vt, dst, 4096, 0)
        torch.cuda.synchronize()
        assert _status(st) == [0]
        v = views_host(vt)
        check_views_against_oracle(v, sim, j, stream)
        got.append(dst.cpu().numpy()[: int(v[0]["len"])].tobytes())
    assert got == [m.payload.tobytes() for m in stream]
    R.ring_detach(peer)
    R.ring_destroy(ring)


def test_emsgsize_and_try_full_w1(R, golden):
    """RING_TRY puts follow the oracle's outcomes on the W1 sequence (PAD, FULL
    by bytes, PAD skip); a message with f > R is EMSGSIZE and publishes nothing."""
    ex = golden["W1"]
    lay = ex["layout"]
    L = Layout(lay["R"], lay["N"], lay["align"], lay["hdr"])
    puts = [op["len"] for op in ex["ops"] if op["op"] == "put"]
    stream = [synth.Message(0, q, n, *synth.header_fields(9, 0, q), payload=synth.payload_bytes(9, 0, q, n))
              for q, n in enumerate(puts)]
    # oracle run of the same op sequence
    sim = Sim(L, {0: to_oracle_msgs(stream)}, mpsc=False, block=False, depth=1)
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, "cuda:0")
    msgs = msg_tensor(stream, srcs, "cuda:0")
    k = 0
    p = sim.producers[0]
    for op in ex["ops"]:
        if op["op"] == "put":
            before = len(p.outcomes)
            while len(p.outcomes) == before:
                sim.step(0)
            st = torch.full((1,), 10, dtype=torch.int32, device="cuda:0")
            R.ring_put_batch(peer, msgs[k * 48:(k + 1) * 48], 1, R.RING_TRY, st)
            torch.cuda.synchronize()
            assert R.STATUS_NAMES[_status(st)[0]] == p.outcomes[-1] == op["outcome"]
            k += 1
        else:
            nd = len(sim.cons.delivered)
            while len(sim.cons.delivered) == nd:
                sim.step("Z")
            sim.step("Zrel")
            vt = torch.zeros(128, dtype=torch.uint8, device="cuda:0")
            R.ring_consume(ring, 1, vt)
            torch.cuda.synchronize()
            v = views_host(vt)[0]
            assert int(v["start"]) == sim.cons.delivered[-1].start == op["start"]
            assert bytes(v["header"])[:56] == sim.cons.delivered[-1].header[:56]
        img = R.ring_read_image(ring)
        assert img["tail"] == sim.mem.tail and img["head"] == sim.mem.head
        assert img["slots"] == sim.mem.slots
    # EMSGSIZE: f = align_up(64 + 961, 128) = 1152 > R = 1024
    big = torch.zeros(2048, dtype=torch.uint8, device="cuda:0")
    hdr = R.ring_hdr_t()
    st = torch.full((1,), 10, dtype=torch.int32, device="cuda:0")
    before = R.ring_read_image(ring)
    R.ring_put(peer, big, 961, hdr, 0, st)
    torch.cuda.synchronize()
    assert R.STATUS_NAMES[_status(st)[0]] == "EMSGSIZE"
    assert R.ring_read_image(ring) == before
    R.ring_detach(peer)
    R.ring_destroy(ring)


def test_corrupt_header_discarded_and_consumed(R):
    """a checksum mismatch discards the entry; the consumer
    still advances using the size metadata."""
    L = Layout(8192, 8)
    stream = synth.random_stream(synth.SEED_BASE + 3, 0, 3, 100, 900)
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, "cuda:0")
    msgs = msg_tensor(stream, srcs, "cuda:0")
    st = torch.full((3,), 10, dtype=torch.int32, device="cuda:0")
    R.ring_put_batch(peer, msgs, 3, 0, st)
    torch.cuda.synchronize()
    f0 = R.ring_footprint(stream[0].length)
    h = bytearray(R.ring_read_data(ring, f0, 64))    # header of message 1
    h[30] ^= 0x10                                      # flip a bit of app_id
    R.ring_write_data(ring, f0, bytes(h))
    vt = torch.zeros(3 * 128, dtype=torch.uint8, device="cuda:0")
    R.ring_consume(ring, 3, vt)
    torch.cuda.synchronize()
    v = views_host(vt)
    assert [R.STATUS_NAMES[int(x)] for x in v["status"]] == ["OK", "ECORRUPT", "OK"]
    img = R.ring_read_image(ring)
    assert img["head"] == img["tail"] and img["slots"] == [0] * L.N
    R.ring_detach(peer)
    R.ring_destroy(ring)


def test_try_get_empty_and_block_timeout(R):
    ring = R.ring_create(0, 4096, 4, 1, R.RING_CREATE_LOCAL)
    vt = torch.zeros(2 * 128, dtype=torch.uint8, device="cuda:0")
    R.ring_get(ring, 2, vt, None, 0, R.RING_TRY)
    torch.cuda.synchronize()
    assert [R.STATUS_NAMES[int(x)] for x in views_host(vt)["status"]] == ["EMPTY", "EMPTY"]
    R.ring_set_timeout_ns(50_000_000)
    try:
        R.ring_consume(ring, 1, vt)
        torch.cuda.synchronize()
        assert R.STATUS_NAMES[int(views_host(vt)["status"][0])] == "ETIMEDOUT"
    finally:
        R.ring_set_timeout_ns(5_000_000_000)
    R.ring_destroy(ring)


def test_mpsc_three_producers_one_device(R):
    """Three attachments (lock taken per message) put in turn;
    per-channel order exact; placements = the oracle replaying the observed order."""
    L = Layout(65536, 16)
    progs_stream = {pid: synth.random_stream(synth.SEED_BASE + 5, pid, 24, 1, 3000) for pid in range(3)}
    ring = R.ring_create(0, L.R, L.N, 3, R.RING_CREATE_LOCAL)
    h = R.ring_export(ring)
    peers = []
    for pid in range(3):
        pe, mh = R.ring_attach_peer(h, 0, pid)
        R.ring_bind_mirror(ring, pid, mh)
        peers.append(pe)
    bufs, tens = [], []
    for pid in range(3):
        b, s = upload(progs_stream[pid], "cuda:0")
        bufs.append(b)
        tens.append(msg_tensor(progs_stream[pid], s, "cuda:0"))
    views = []
    for rnd in range(6):              # 6 rounds x 3 producers x 4 messages
        for pid in range(3):
            st = torch.full((4,), 10, dtype=torch.int32, device="cuda:0")
            R.ring_put_batch(peers[pid], tens[pid][rnd * 4 * 48:(rnd + 1) * 4 * 48], 4, 0, st)
            torch.cuda.synchronize()
            assert _status(st) == [0] * 4
        vt = torch.zeros(12 * 128, dtype=torch.uint8, device="cuda:0")
        dst = torch.zeros(12 * 3008, dtype=torch.uint8, device="cuda:0")
        R.ring_consume(ring, 12, vt, dst, 3008)
        torch.cuda.synchronize()
        v = views_host(vt)
        d = dst.cpu().numpy()
        for j, x in enumerate(v):
            hd = decode_header(bytes(x["header"]))
            m = progs_stream[hd["producer_id"]][hd["seq"]]
            assert d[j * 3008: j * 3008 + int(x["len"])].tobytes() == m.payload.tobytes()
        views.append(v)
    v = np.concatenate(views)
    order = [decode_header(bytes(x["header"]))["producer_id"] for x in v]
    for pid in range(3):
        seqs = [decode_header(bytes(x["header"]))["seq"] for x in v
                if decode_header(bytes(x["header"]))["producer_id"] == pid]
        assert seqs == list(range(24))
    sim = replay_mpsc(L, {pid: to_oracle_msgs(progs_stream[pid]) for pid in range(3)}, order)
    for x, d in zip(v, sim.cons.delivered):
        assert (int(x["start"]), int(x["footprint"]), int(x["slot_seq"])) == (d.start, d.f, d.seq_slot)
        assert bytes(x["header"])[:56] == d.header[:56]
    img = R.ring_read_image(ring)
    assert img["lock"] == 0 and img["tail"] == sim.mem.tail == img["head"]
    for pe in peers:
        R.ring_detach(pe)
    R.ring_destroy(ring)


def test_router_round_robin_and_epoch_flip(R):
    """round-robin over the destinations of (app_id, stage);
    PAPER.md:920-923 reassignment: a new route flips the epoch, later puts go
    to the new destination set."""
    L = Layout(65536, 16)
    rings = [R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL) for _ in range(2)]
    peers = []
    for r in rings:
        pe, mh = R.ring_attach_peer(R.ring_export(r), 0, 0)
        R.ring_bind_mirror(r, 0, mh)
        peers.append(pe)
    router = R.router_create(0, 8)
    R.router_set_route(router, 7, 2, peers)
    stream = synth.random_stream(synth.SEED_BASE + 8, 0, 12, 10, 2000, app_id=7, stage=2)
    buf, srcs = upload(stream, "cuda:0")
    msgs = msg_tensor(stream, srcs, "cuda:0")
    st = torch.full((8,), 10, dtype=torch.int32, device="cuda:0")
    dest = torch.zeros(8, dtype=torch.int32, device="cuda:0")
    R.ring_put_routed(router, msgs[: 8 * 48], 8, 0, st, dest)
    torch.cuda.synchronize()
    assert _status(st) == [0] * 8 and _status(dest) == [0, 1] * 4
    R.router_set_route(router, 7, 2, [peers[1]])          # reassignment
    st2 = torch.full((4,), 10, dtype=torch.int32, device="cuda:0")
    dest2 = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    R.ring_put_routed(router, msgs[8 * 48:], 4, 0, st2, dest2)
    torch.cuda.synchronize()
    assert _status(st2) == [0] * 4 and _status(dest2) == [1] * 4
    got = {}
    for i, (r, n) in enumerate(zip(rings, (4, 8))):
        vt = torch.zeros(n * 128, dtype=torch.uint8, device="cuda:0")
        R.ring_consume(r, n, vt)
        torch.cuda.synchronize()
        got[i] = [decode_header(bytes(x["header"])) for x in views_host(vt)]
    assert [h["uid"] for h in got[0]] == [stream[k].uid for k in (0, 2, 4, 6)]
    assert [h["uid"] for h in got[1]] == [stream[k].uid for k in (1, 3, 5, 7, 8, 9, 10, 11)]
    assert [h["epoch"] for h in got[1]] == [1, 1, 1, 1, 2, 2, 2, 2]
    assert [h["seq"] for h in got[1]] == list(range(8))          # per-channel seq
    R.router_destroy(router)
    for pe in peers:
        R.ring_detach(pe)
    for r in rings:
        R.ring_destroy(r)


@pytest.mark.parametrize("copy_mode", [0, 1])
def test_c2_full_size_same_gpu(R, copy_mode):
    """BASELINE.json configs[1] at full size: 64 slots x 1 MiB (R = 64 MiB),
    1,048,512-B payloads (footprint exactly 1 MiB), the bench's launch
    configuration (all SMs copying), two laps of the ring."""
    L = Layout(64 << 20, 64)
    stream = synth.fixed_stream(synth.SEED_BASE + 2, 0, 126, 1048512)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    views, payloads, st, img = _run_spsc(R, L, stream, mode="consume_copy", copy_mode=copy_mode)
    assert st == [0] * 126
    check_views_against_oracle(views, sim, 0, stream)
    assert payloads == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail == img["head"]


# ---------------------------------------------------------------------------------------
# Two or more GPUs, one process (peer access): producer and consumer kernels run
# concurrently on different GPUs, so credit and data flow while both spin.
# ---------------------------------------------------------------------------------------
def _p2p_stream(R, L, stream, prod_dev, cons_dev, cap, copy=True, copy_mode=0):
    ring = R.ring_create(cons_dev, L.R, L.N, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), prod_dev, 0)
    R.ring_peer_config(peer, 0, 0, copy_mode)
    if copy_mode == 1 and prod_dev == cons_dev:
        # the TMA engine takes its own shared-memory split: it starts only on SMs
        # free of other ring kernels, so the consumer's copy grid leaves half free
        R.ring_config(ring, 74, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, srcs = upload(stream, f"cuda:{prod_dev}")
    msgs = msg_tensor(stream, srcs, f"cuda:{prod_dev}")
    n = len(stream)
    vt = torch.zeros(n * 128, dtype=torch.uint8, device=f"cuda:{cons_dev}")
    dst = torch.zeros(n * cap, dtype=torch.uint8, device=f"cuda:{cons_dev}") if copy else None
    st = torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{prod_dev}")
    sc = torch.cuda.Stream(cons_dev)
    sp = torch.cuda.Stream(prod_dev)
    R.ring_consume(ring, n, vt, dst, cap if copy else 0, 0, sc)     # consumer first: it waits for data
    R.ring_put_batch(peer, msgs, n, 0, st, sp)
    torch.cuda.synchronize(prod_dev)
    torch.cuda.synchronize(cons_dev)
    v = views_host(vt)
    pl = []
    if copy:
        d = dst.cpu().numpy()
        pl = [d[j * cap: j * cap + int(v[j]["len"])].tobytes() for j in range(n)]
    img = R.ring_read_image(ring)
    R.ring_detach(peer)
    R.ring_destroy(ring)
    return v, pl, _status(st), img


@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])
def test_p2p_small_ring_streaming_wraps(R, cross):
    """C1's stream over NVLink with producer and consumer concurrently spinning:
    1,000 messages through an 8-slot 32-KiB ring (~130 laps, credit via the
    mirror, PAD entries at every wrap) in ONE put launch and ONE consume launch.
    cross=False: the same system-scope kernels on one GPU, two streams."""
    prod, cons = devices(2, cross)
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 1000, 1, 4096)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _p2p_stream(R, L, stream, prod, cons, 4096)
    assert st == [0] * 1000
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]
    assert img["tail"] == sim.mem.tail == img["head"]


@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])
@pytest.mark.parametrize("copy_mode", [0, 1])
def test_p2p_c3_wan_tensors(R, copy_mode, cross):
    """BASELINE.json configs[2]: umT5 embeddings 512x4096 bf16 (4,194,304 B)
    alternating with 480p latents 16x21x60x104 bf16 (4,193,280 B), GPU0 -> ring
    on GPU1 (R = 64 MiB, N = 64), 48 messages in one streaming launch pair."""
    prod, cons = devices(2, cross)
    L = Layout(64 << 20, 64)
    stream = synth.wan_stream(synth.SEED_BASE + 3, 0, 48)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _p2p_stream(R, L, stream, prod, cons, 4194304, copy_mode=copy_mode)
    assert st == [0] * 48, (st, [int(x["status"]) for x in v])
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]


@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])
def test_p2p_reverse_direction(R, cross):
    cons, prod = devices(2, cross)
    L = Layout(1 << 20, 16)
    stream = synth.random_stream(synth.SEED_BASE + 4, 0, 200, 1, 70000)
    sim = oracle_spsc(L, to_oracle_msgs(stream))
    v, pl, st, img = _p2p_stream(R, L, stream, prod, cons, 70016)
    check_views_against_oracle(v, sim, 0, stream)
    assert pl == [m.payload.tobytes() for m in stream]


@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])
def test_mpsc_fan_in_three_gpus(R, cross):
    """C5 shape at small scale: producers on GPUs 1..3 -> one shared MPSC ring on
    GPU0 (paper lock), all concurrent; per-channel order exact, observed merge
    replayed by the oracle.  cross=False: three producer streams and the
    consumer stream on one GPU, system-scope ring."""
    devs = devices(4, cross)
    L = Layout(1 << 20, 32)
    n = 150
    streams = {pid: synth.random_stream(synth.SEED_BASE + 6, pid, n, 1, 40000) for pid in range(3)}
    ring = R.ring_create(0, L.R, L.N, 3, 0)
    h = R.ring_export(ring)
    peers, bufs, tens, sts, strs = [], [], [], [], []
    for pid in range(3):
        dev = devs[pid + 1]
        pe, mh = R.ring_attach_peer(h, dev, pid)
        R.ring_bind_mirror(ring, pid, mh)
        peers.append(pe)
        b, s = upload(streams[pid], f"cuda:{dev}")
        bufs.append(b)
        tens.append(msg_tensor(streams[pid], s, f"cuda:{dev}"))
        sts.append(torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{dev}"))
        strs.append(torch.cuda.Stream(dev))
    cap = 40000
    vt = torch.zeros(3 * n * 128, dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros(3 * n * cap, dtype=torch.uint8, device="cuda:0")
    sc = torch.cuda.Stream(0)
    R.ring_consume(ring, 3 * n, vt, dst, cap, 0, sc)
    for pid in range(3):
        R.ring_put_batch(peers[pid], tens[pid], n, 0, sts[pid], strs[pid])
    for dev in set(devs):
        torch.cuda.synchronize(dev)
    for pid in range(3):
        assert _status(sts[pid]) == [0] * n
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
    for pe in peers:
        R.ring_detach(pe)
    R.ring_destroy(ring)
