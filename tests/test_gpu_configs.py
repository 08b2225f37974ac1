"""Bit-exact parity at every BASELINE.json configuration, on one GPU (and on
several when the box has them).

The plain definition the ring must reach ("if a producer
writes data starting at address R, the consumer will eventually read that
same data"; DESIGN.md c-1): every channel's delivered messages equal its put
messages -- payload bytes, the 56 checksummed header bytes -- exactly once, in
put order; and every entry sits where the oracle's pointer formulas put it
(PAPER.md:731-745).  Payloads too large to move through the host are compared
on the device with the seeded generator (synth/csrc/synth_dev.cu, a library
of its own that shares nothing with libb200ring.so): each view's bytes in the
ring (view mode, before release) or in the copy-out buffer, first bad byte
reported.

  C2  the bench's streaming loop exactly: put(s) and consume(s) on two streams,
      64 x 1,048,512 B per step, put(s+1) waiting inside the kernel for the
      credit consume(s) returns.
  C4  the 4-hop Wan2.1 stage chain (text-enc -> VAE-enc -> DiT -> VAE-dec ->
      sink), system-scope rings, 4,194,304 / 13,871,104 / 9,676,800 /
      447,897,600-B hops, the last on a 1 GiB 8-slot ring; all stages
      streaming concurrently.
  C5a three producers into one MPSC ring (paper lock), size sweep 4 KiB ..
      256 MiB (x4 steps); the observed merge replayed by the oracle.
  C5b the router's epoch flip at 50 % of each producer's messages (PAPER.md:
      531-532, 920-923): one producer stops, the others round-robin over two
      rings; destinations, epochs, merges and bytes against the oracle.
"""
import numpy as np
import pytest
import torch

import synth
from synth import device as SD
from gpu_util import (views_host, expected_header, device_sources, dev_u64, verify_views, replay_mpsc, devices)
from oracle.ring import Layout, Msg, spsc_image, encode_header, decode_header

pytestmark = pytest.mark.gpu

CROSS = pytest.mark.parametrize("cross", [False, pytest.param(True, marks=pytest.mark.multigpu)])
EMB = synth.wan_bytes("umt5_emb")              # 4,194,304
LAT480 = synth.wan_bytes("latent_480p")        # 4,193,280
LAT720 = synth.wan_bytes("latent_720p")        # 9,676,800
FRAMES = synth.wan_bytes("frames_720p")        # 447,897,600


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(10_000_000_000)
    return ring


def _msgs(R, ptrs, lens, hdrs, app_id, stage, device):
    a = R.make_msgs(ptrs, lens, [h[0] for h in hdrs], [h[1] for h in hdrs], [app_id] * len(lens),
                    [stage] * len(lens))
    return torch.from_numpy(a.view(np.uint8).copy()).to(device)


def _ok(bad: torch.Tensor, what):
    b = bad.cpu().tolist()
    assert all(x == -1 for x in b), (what, [(i, x) for i, x in enumerate(b) if x != -1][:8])


def _place(v):
    return int(v["start"]), int(v["footprint"]), int(v["slot_seq"])


# ---------------------------------------------------------------------------------------
# C2: the timed bench loop, verbatim
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("mode", ["consume_view", "get_verify_release", "consume_copy"])
def test_c2_bench_streaming_loop(R, mode):
    """BASELINE.json configs[1] in bench.py's launch configuration: 64 x
    1,048,512-B payloads per step (footprint exactly 1 MiB, R = 64 MiB, N = 64:
    each step fills the whole ring), 4 rotating source sets, put on one stream
    and the consumer on another, 10 steps.  Modes: the bench's zero-copy
    consume (placement + headers of every entry, payloads of the last step);
    get -> device verify in the ring -> release (every payload, in place, while
    the producer waits for that release); the bench's copy-out consume (every
    payload in the copy-out buffer)."""
    L = Layout(64 << 20, 64)
    m, plen, sets, steps = 64, 1048512, 4, 10
    seed = synth.SEED_BASE + 2
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    buf, ptrs = device_sources([(0, k, plen) for k in range(sets * m)], seed)
    hdrs = [synth.header_fields(seed, 0, k) for k in range(sets * m)]
    d_msgs = [_msgs(R, ptrs[s * m:(s + 1) * m], [plen] * m, hdrs[s * m:(s + 1) * m], 7, 1, "cuda")
              for s in range(sets)]
    keys = [dev_u64([(s % sets) * m + q for q in range(m)]) for s in range(steps)]
    chans = torch.zeros(m, dtype=torch.int32, device="cuda")
    sts = [torch.full((m,), 10, dtype=torch.int32, device="cuda") for _ in range(steps)]
    vts = [torch.zeros(m * 128, dtype=torch.uint8, device="cuda") for _ in range(steps)]
    dsts = [torch.empty(m * plen, dtype=torch.uint8, device="cuda") for _ in range(2)] if mode == "consume_copy" else []
    dptr = [dev_u64([d.data_ptr() + q * plen for q in range(m)]) for d in dsts]
    lens = dev_u64([plen] * m)
    sp, sc = torch.cuda.Stream(), torch.cuda.Stream()
    sp.wait_stream(torch.cuda.current_stream())
    sc.wait_stream(torch.cuda.current_stream())
    bads = []
    try:
        for i in range(steps):
            R.ring_put_batch(peer, d_msgs[i % sets], m, 0, sts[i], sp)
            if mode == "consume_view":
                R.ring_consume(ring, m, vts[i], None, 0, 0, sc)
            elif mode == "consume_copy":
                R.ring_consume(ring, m, vts[i], dsts[i % 2], plen, 0, sc)
                bads.append(SD.verify(dptr[i % 2], lens, chans, keys[i], seed, sc))
            else:
                R.ring_get(ring, m, vts[i], None, 0, 0, sc)
                bads.append(verify_views(ring, vts[i], m, seed, chans, keys[i], sc))
                R.ring_release(ring, m, sc)
        torch.cuda.synchronize()
        if mode == "consume_view":      # released but not overwritten: the last step's bytes
            bads.append(verify_views(ring, vts[-1], m, seed, chans, keys[steps - 1]))
        img = spsc_image(L, [plen] * (m * steps))
        ents = [e for e in img["entries"] if not e[3]]
        assert not any(e[3] for e in img["entries"])          # exact fits: no PAD at the wrap
        for i in range(steps):
            assert sts[i].cpu().tolist() == [0] * m, (i, sts[i].cpu().tolist())
            v = views_host(vts[i])
            for q in range(m):
                k = i * m + q
                assert int(v[q]["status"]) == 0, (k, int(v[q]["status"]))
                assert _place(v[q]) == ents[k][1:3] + (ents[k][0],), k
                h = hdrs[(i % sets) * m + q]
                exp = encode_header(h[0], h[1], 7, 1, plen, 0, k, 0, 0, 0)[:56]
                assert bytes(v[q]["header"])[:56] == exp, k
                assert int(v[q]["len"]) == plen
        for j, b in enumerate(bads):
            _ok(b, j)
        im = R.ring_read_image(ring)
        assert im["tail"] == img["tail"] == im["head"] == im["cursor"]
        assert im["slots"] == [0] * L.N
    finally:
        torch.cuda.synchronize()
        R.ring_detach(peer)
        R.ring_destroy(ring)


# ---------------------------------------------------------------------------------------
# C3 one way: bench.py's c3_one_way split loop
# ---------------------------------------------------------------------------------------
@CROSS
def test_c3_split_one_way_bench_loop(R, monkeypatch, cross):
    """BASELINE.json configs[2] in bench.py's c3_one_way launch configuration
    (the north-star target's ring): split placement, 256 MiB / 64 slots, 64
    Wan2.1 tensors (4,194,304 / 4,193,280 B alternating) per put launch and per
    copy-out consume launch, producer and consumer on their own streams, 4
    launches (the ring wraps with PAD entries).  Every placement and header
    against the oracle's pointer formulas, every payload in the copy-out
    buffers compared on the device.  On one GPU the line-aligned copy-out of a
    remote buffer region is forced (B200RING_COPYOUT_ALIGN=1)."""
    prod, cons = devices(2, cross)
    if not cross:
        monkeypatch.setenv("B200RING_COPYOUT_ALIGN", "1")
    L = Layout(256 << 20, 64)
    K, launches = 64, 4
    seed = synth.SEED_BASE + 33
    lens_k = [EMB if q % 2 == 0 else LAT480 for q in range(K)]
    ring = R.ring_create_split(cons, prod, L.R, L.N, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), prod, 0)
    R.ring_bind_mirror(ring, 0, mh)
    with torch.cuda.device(prod):
        buf, ptrs = device_sources([(0, k, lens_k[k]) for k in range(K)], seed, f"cuda:{prod}")
        hdrs = [synth.header_fields(seed, 0, k) for k in range(K)]
        d_msgs = _msgs(R, ptrs, lens_k, hdrs, 7, 2, f"cuda:{prod}")
        sts = [torch.full((K,), 10, dtype=torch.int32, device=f"cuda:{prod}") for _ in range(launches)]
        sp = torch.cuda.Stream(prod)
    with torch.cuda.device(cons):
        vts = [torch.zeros(K * 128, dtype=torch.uint8, device=f"cuda:{cons}") for _ in range(launches)]
        dsts = [torch.empty(K * EMB, dtype=torch.uint8, device=f"cuda:{cons}") for _ in range(2)]
        dptr = [dev_u64([d.data_ptr() + q * EMB for q in range(K)]) for d in dsts]
        dlens = dev_u64(lens_k)
        chans = torch.zeros(K, dtype=torch.int32, device=f"cuda:{cons}")
        keys = dev_u64(list(range(K)))
        sc = torch.cuda.Stream(cons)
        # load the verifier on the consumer's GPU now: a first (lazy) load would
        # wait for the consume kernel spinning there
        SD.verify(dptr[0][:1], dlens[:1], chans[:1], keys[:1], seed)
        torch.cuda.synchronize(cons)
    bads = []
    try:
        for i in range(launches):
            R.ring_consume(ring, K, vts[i], dsts[i % 2], EMB, 0, sc)
            with torch.cuda.device(cons):
                bads.append(SD.verify(dptr[i % 2], dlens, chans, keys, seed, sc))
            R.ring_put_batch(peer, d_msgs, K, 0, sts[i], sp)
        for d in {prod, cons}:
            torch.cuda.synchronize(d)
        img = spsc_image(L, lens_k * launches)
        ents = [e for e in img["entries"] if not e[3]]
        assert any(e[3] for e in img["entries"])                  # the ring wrapped with a PAD
        for i in range(launches):
            assert sts[i].cpu().tolist() == [0] * K, (i, sts[i].cpu().tolist())
            v = views_host(vts[i])
            for q in range(K):
                k = i * K + q
                assert int(v[q]["status"]) == 0, (k, int(v[q]["status"]))
                assert _place(v[q]) == ents[k][1:3] + (ents[k][0],), k
                h = hdrs[q]
                exp = encode_header(h[0], h[1], 7, 2, lens_k[q], 0, k, 0, 0, 0)[:56]
                assert bytes(v[q]["header"])[:56] == exp, k
                assert int(v[q]["len"]) == lens_k[q]
        for j, b in enumerate(bads):
            _ok(b, j)
        im = R.ring_read_image(ring)
        assert im["tail"] == img["tail"] == im["head"] == im["cursor"]
    finally:
        for d in {prod, cons}:
            torch.cuda.synchronize(d)
        R.ring_detach(peer)
        R.ring_destroy(ring)


# ---------------------------------------------------------------------------------------
# C4: the Wan2.1 I2V stage chain
# ---------------------------------------------------------------------------------------
C4_HOPS = [  # (R, N, message bytes): text-enc -> VAE-enc -> DiT -> VAE-dec -> sink
    (256 << 20, 64, EMB),
    (256 << 20, 64, LAT720 + EMB),
    (256 << 20, 64, LAT720),
    (1 << 30, 8, FRAMES),
]


@CROSS
@pytest.mark.parametrize("frames", ["push", "split"])
def test_c4_stage_chain(R, cross, frames):
    """BASELINE.json configs[3]: every stage gets its input (view, in place),
    checks it on the device, releases it and emits its own output (a seeded
    tensor of the next shape, keyed by the request) into the next hop; hops are
    system-scope rings (NVLink kernels), stages run concurrently on their own
    streams, four requests (two laps of the 1 GiB frames ring, whose producer
    waits for the sink's credit).  frames="split": the frames hop in bench.py's
    placement -- a split ring whose buffer region is on the VAE-decode GPU, the
    sink pulling each 447,897,600-B frame tensor with its copy-out consume."""
    devs = devices(4, cross)          # stage h runs on devs[h]; hop h's ring sits at its consumer
    cons_dev = [devs[(h + 1) % 4] for h in range(4)]
    nreq, seed = 4, synth.SEED_BASE + 4
    rings, peers, srcs, msgs = [], [], [], []
    for h, (Rb, N, nb) in enumerate(C4_HOPS):
        if h == 3 and frames == "split":
            rings.append(R.ring_create_split(cons_dev[h], devs[h], Rb, N, 1, 0))
        else:
            rings.append(R.ring_create(cons_dev[h], Rb, N, 1, 0))
        pe, mh = R.ring_attach_peer(R.ring_export(rings[h]), devs[h], 0)
        R.ring_bind_mirror(rings[h], 0, mh)
        peers.append(pe)
        b = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{devs[h]}")
        srcs.append(b)
        hd = [synth.header_fields(seed, h, r) for r in range(nreq)]
        msgs.append(_msgs(R, [b.data_ptr()] * nreq, [nb] * nreq, hd, 7, h + 1, f"cuda:{devs[h]}"))
    st = [torch.full((nreq,), 10, dtype=torch.int32, device=f"cuda:{devs[h]}") for h in range(4)]
    vt = [torch.zeros(nreq * 128, dtype=torch.uint8, device=f"cuda:{cons_dev[h]}") for h in range(4)]
    streams = [torch.cuda.Stream(devs[h]) for h in range(4)] + [torch.cuda.Stream(cons_dev[3])]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream(s.device))
    bads = {h: [] for h in range(4)}
    # every argument array the loop needs is on the device before anything
    # spins (a pageable host copy inside the loop may wait for its stream)
    dv = [f"cuda:{d}" for d in devs]
    cv = [f"cuda:{d}" for d in cons_dev]
    in_ch = [torch.full((1,), h, dtype=torch.int32, device=cv[h]) for h in range(4)]
    in_sq = [[torch.full((1,), r, dtype=torch.int64, device=cv[h]) for r in range(nreq)] for h in range(4)]
    out_args = [[(dev_u64([srcs[h].data_ptr()], dv[h]), dev_u64([C4_HOPS[h][2]], dv[h]),
                  torch.full((1,), h, dtype=torch.int32, device=dv[h]), dev_u64([r], dv[h])) for r in range(nreq)]
                for h in range(4)]
    pulled = None
    if frames == "split":             # the sink's copy-out buffer for one frame tensor
        pulled = torch.empty(C4_HOPS[3][2], dtype=torch.uint8, device=cv[3])
        pulled_args = (dev_u64([pulled.data_ptr()], cv[3]), dev_u64([C4_HOPS[3][2]], cv[3]))
    try:
        for r in range(nreq):
            for h in range(5):            # stage h: input hop h-1 (h > 0), output hop h (h < 4)
                s = streams[h]
                if h > 0:
                    ring_in = rings[h - 1]
                    v = vt[h - 1][r * 128:(r + 1) * 128]
                    if h == 4 and pulled is not None:      # pulled over NVLink, then checked in place
                        R.ring_consume(ring_in, 1, v, pulled, C4_HOPS[3][2], 0, s)
                        with torch.cuda.device(cons_dev[3]):
                            bads[3].append(SD.verify(*pulled_args, in_ch[3], in_sq[3][r], seed, s))
                    else:
                        R.ring_get(ring_in, 1, v, None, 0, 0, s)
                        bads[h - 1].append(verify_views(ring_in, v, 1, seed, in_ch[h - 1], in_sq[h - 1][r], s))
                        R.ring_release(ring_in, 1, s)
                if h < 4:
                    with torch.cuda.device(devs[h]), torch.cuda.stream(s):
                        SD.fill(*out_args[h][r], seed, s)
                    R.ring_put_batch(peers[h], msgs[h][r * 48:(r + 1) * 48], 1, 0, st[h][r:r + 1], s)
        for d in set(devs):
            torch.cuda.synchronize(d)
        for h, (Rb, N, nb) in enumerate(C4_HOPS):
            assert st[h].cpu().tolist() == [0] * nreq, (h, st[h].cpu().tolist())
            img = spsc_image(Layout(Rb, N), [nb] * nreq)
            ents = [e for e in img["entries"] if not e[3]]
            v = views_host(vt[h])
            for r in range(nreq):
                assert int(v[r]["status"]) == 0, (h, r)
                assert _place(v[r]) == (ents[r][1], ents[r][2], ents[r][0]), (h, r)
                u, acc, _, _ = synth.header_fields(seed, h, r)
                assert bytes(v[r]["header"])[:56] == encode_header(u, acc, 7, h + 1, nb, 0, r, 0, 0, 0)[:56]
            for r, b in enumerate(bads[h]):
                _ok(b, (h, r))
            im = R.ring_read_image(rings[h])
            assert im["tail"] == img["tail"] == im["head"], h
    finally:
        for d in set(devs):
            torch.cuda.synchronize(d)
        for pe in peers:
            R.ring_detach(pe)
        for rg in rings:
            R.ring_destroy(rg)


# ---------------------------------------------------------------------------------------
# C5a: MPSC fan-in, size sweep
# ---------------------------------------------------------------------------------------
C5_SIZES = [4096 << (2 * i) for i in range(9)]          # 4 KiB .. 256 MiB


def _sweep_counts(size):
    return 8 if size <= (1 << 20) else (4 if size <= (16 << 20) else 2)


@CROSS
def test_c5a_mpsc_size_sweep(R, cross):
    """BASELINE.json configs[4] (fan-in part) on a 1 GiB, 256-slot MPSC ring
    with the paper's lock: three producers put their whole sweep (4 KiB ..
    256 MiB, x4 steps) concurrently, the consumer gets, checks in place on the
    device and releases one entry at a time.  Per-channel order exact; the
    oracle replays the observed lock order and must predict every placement and
    header; every payload byte equal to the generator's."""
    devs = devices(4, cross)          # consumer devs[0], producers devs[1..3]
    L = Layout(1 << 30, 256)
    seed = synth.SEED_BASE + 5
    lens = [s for s in C5_SIZES for _ in range(_sweep_counts(s))]
    n = len(lens)
    ring = R.ring_create(devs[0], L.R, L.N, 3, 0)
    h = R.ring_export(ring)
    peers, bufs, tens, sts, strs = [], [], [], [], []
    for pid in range(3):
        dev = devs[pid + 1]
        pe, mh = R.ring_attach_peer(h, dev, pid)
        R.ring_bind_mirror(ring, pid, mh)
        peers.append(pe)
        b, ptrs = device_sources([(pid, k, lens[k]) for k in range(n)], seed, f"cuda:{dev}")
        bufs.append(b)
        hd = [synth.header_fields(seed, pid, k) for k in range(n)]
        tens.append(_msgs(R, ptrs, lens, hd, 7, 3, f"cuda:{dev}"))
        sts.append(torch.full((n,), 10, dtype=torch.int32, device=f"cuda:{dev}"))
        strs.append(torch.cuda.Stream(dev))
    total = 3 * n
    vt = torch.zeros(total * 128, dtype=torch.uint8, device=f"cuda:{devs[0]}")
    sc = torch.cuda.Stream(devs[0])
    bads = []
    try:
        for pid in range(3):
            R.ring_put_batch(peers[pid], tens[pid], n, 0, sts[pid], strs[pid])
        for j in range(total):
            v = vt[j * 128:(j + 1) * 128]
            R.ring_get(ring, 1, v, None, 0, 0, sc)
            bads.append(verify_views(ring, v, 1, seed, stream=sc))
            R.ring_release(ring, 1, sc)
        for d in set(devs):
            torch.cuda.synchronize(d)
        for pid in range(3):
            assert sts[pid].cpu().tolist() == [0] * n, pid
        v = views_host(vt)
        hdrs = [decode_header(bytes(x["header"])) for x in v]
        assert all(int(x["status"]) == 0 for x in v)
        order = [hh["producer_id"] for hh in hdrs]
        for pid in range(3):
            assert [hh["seq"] for hh in hdrs if hh["producer_id"] == pid] == list(range(n)), pid
        for j, b in enumerate(bads):
            _ok(b, j)
        zeros = {s: bytes(s) for s in C5_SIZES}
        progs = {}
        for pid in range(3):
            hd = [synth.header_fields(seed, pid, k) for k in range(n)]
            progs[pid] = [Msg(lens[k], zeros[lens[k]], hd[k][0], hd[k][1], 7, 3) for k in range(n)]
        sim = replay_mpsc(L, progs, order, check=False)
        for x, d in zip(v, sim.cons.delivered):
            assert _place(x) == (d.start, d.f, d.seq_slot)
            assert bytes(x["header"])[:56] == d.header[:56]
        im = R.ring_read_image(ring)
        assert im["lock"] == 0 and im["tail"] == sim.mem.tail == im["head"]
    finally:
        for d in set(devs):
            torch.cuda.synchronize(d)
        for pe in peers:
            R.ring_detach(pe)
        R.ring_destroy(ring)


# ---------------------------------------------------------------------------------------
# C5b: reassignment through the router's epoch flip
# ---------------------------------------------------------------------------------------
@CROSS
def test_c5b_epoch_flip(R, cross):
    """BASELINE.json configs[4] (reassignment part): producers P0, P1, P2 put
    Wan-shaped messages (alternating 4,194,304 / 4,193,280 B) through their
    routers into ring A (MPSC, paper lock).  At 50 % of each producer's messages
    the NodeManager reassigns: P2 stops, and P0/P1's route
    becomes {A, B} (epoch 2), round-robin from the counter
    where it stands.  Checked: every message's destination and header epoch as
    predicted from its producer's flip point, per-channel order on both rings,
    the oracle's replay of each ring's observed merge, every payload byte."""
    devs = devices(4, cross)          # ring A on devs[0], ring B on devs[3] (P2's GPU, PAPER.md:930-933 shape), producers devs[1..3]
    L = Layout(1 << 30, 256)
    seed, M = synth.SEED_BASE + 6, 24
    half = M // 2
    lens = [(EMB, LAT480)[k % 2] for k in range(M)]
    ringA = R.ring_create(devs[0], L.R, L.N, 3, 0)
    ringB = R.ring_create(devs[3], L.R, L.N, 2, 0)
    hA, hB = R.ring_export(ringA), R.ring_export(ringB)
    prod = []
    try:
        for p in range(3):
            dev = devs[p + 1]
            pa, ma = R.ring_attach_peer(hA, dev, p)
            R.ring_bind_mirror(ringA, p, ma)
            pb = None
            if p < 2:
                pb, mb = R.ring_attach_peer(hB, dev, p)
                R.ring_bind_mirror(ringB, p, mb)
            rt = R.router_create(dev, 4)
            R.router_set_route(rt, 7, 2, [pa])                 # epoch 1
            b, ptrs = device_sources([(p, k, lens[k]) for k in range(M)], seed, f"cuda:{dev}")
            hd = [synth.header_fields(seed, p, k) for k in range(M)]
            d = _msgs(R, ptrs, lens, hd, 7, 2, f"cuda:{dev}")
            prod.append(dict(dev=dev, pa=pa, pb=pb, rt=rt, buf=b, msgs=d, hd=hd,
                             st=torch.full((M,), 10, dtype=torch.int32, device=f"cuda:{dev}"),
                             dest=torch.full((M,), -1, dtype=torch.int32, device=f"cuda:{dev}"),
                             s=torch.cuda.Stream(dev)))
        exp_dest = {p: ([0] * half + [k % 2 for k in range(half, M)]) if p < 2 else [0] * half for p in range(3)}
        # predicted (producer, channel seq on that ring) -> the producer's message index k
        ks = {(ridx, p): [k for k, d in enumerate(exp_dest[p]) if d == ridx] for ridx in (0, 1) for p in range(3)}
        luts = []
        for ridx, dev in ((0, devs[0]), (1, devs[3])):
            t = [0] * (3 * M)
            for p in range(3):
                for j, k in enumerate(ks[(ridx, p)]):
                    t[p * M + j] = k
            luts.append(torch.tensor(t, dtype=torch.int64, device=f"cuda:{dev}"))
        nA = sum(len(ks[(0, p)]) for p in range(3))
        nB = sum(len(ks[(1, p)]) for p in range(3))
        vA = torch.zeros(nA * 128, dtype=torch.uint8, device=f"cuda:{devs[0]}")
        vB = torch.zeros(nB * 128, dtype=torch.uint8, device=f"cuda:{devs[3]}")
        sA, sB = torch.cuda.Stream(devs[0]), torch.cuda.Stream(devs[3])
        bads = []
        # consumers first (they wait for data): get -> verify in place -> release, one entry at a time
        for ring, vt, n, s, lut in ((ringA, vA, nA, sA, luts[0]), (ringB, vB, nB, sB, luts[1])):
            for j in range(n):
                v = vt[j * 128:(j + 1) * 128]
                R.ring_get(ring, 1, v, None, 0, 0, s)
                bads.append(verify_views(ring, v, 1, seed, stream=s, lut=lut, lut_stride=M))
                R.ring_release(ring, 1, s)
        for p, P in enumerate(prod):
            R.ring_put_routed(P["rt"], P["msgs"][: half * 48], half, 0, P["st"][:half], P["dest"][:half], P["s"])
        for p, P in enumerate(prod[:2]):      # reassignment: a device-side epoch flip in the producer's stream
            R.router_set_route(P["rt"], 7, 2, [P["pa"], P["pb"]], P["s"])    # epoch 2
            R.ring_put_routed(P["rt"], P["msgs"][half * 48:], M - half, 0, P["st"][half:], P["dest"][half:], P["s"])
        for d in set(devs):
            torch.cuda.synchronize(d)
        for p, P in enumerate(prod):
            n = M if p < 2 else half
            assert P["st"][:n].cpu().tolist() == [0] * n, p
            assert P["dest"][:n].cpu().tolist() == exp_dest[p], (p, P["dest"].cpu().tolist())
        for j, b in enumerate(bads):
            _ok(b, j)
        uid_of = {P["hd"][k][0]: (p, k) for p, P in enumerate(prod) for k in range(M)}
        for name, vt, ring, ridx in (("A", vA, ringA, 0), ("B", vB, ringB, 1)):
            v = views_host(vt)
            hd = [decode_header(bytes(x["header"])) for x in v]
            assert all(int(x["status"]) == 0 for x in v), (name, [int(x["status"]) for x in v])
            ids = [uid_of[h["uid"]] for h in hd]
            progs = {}
            for p in range(3):
                want = ks[(ridx, p)]
                assert [k for (pp, k) in ids if pp == p] == want, (name, p)
                assert [h["seq"] for h, (pp, _) in zip(hd, ids) if pp == p] == list(range(len(want)))
                if want:
                    progs[p] = [Msg(lens[k], bytes(lens[k]), prod[p]["hd"][k][0], prod[p]["hd"][k][1], 7, 2,
                                    1 if k < half else 2) for k in want]
            for h, (p, k) in zip(hd, ids):
                assert h["epoch"] == (1 if k < half else 2), (name, p, k)
            sim = replay_mpsc(L, progs, [p for (p, _) in ids], check=False)
            for x, d in zip(v, sim.cons.delivered):
                assert _place(x) == (d.start, d.f, d.seq_slot), name
                assert bytes(x["header"])[:56] == d.header[:56], name
            im = R.ring_read_image(ring)
            assert im["lock"] == 0 and im["tail"] == sim.mem.tail == im["head"], name
    finally:
        for d in set(devs):
            torch.cuda.synchronize(d)
        for P in prod:
            R.router_destroy(P["rt"])
            R.ring_detach(P["pa"])
            if P["pb"]:
                R.ring_detach(P["pb"])
        R.ring_destroy(ringA)
        R.ring_destroy(ringB)


# ---------------------------------------------------------------------------------------
# Regression: put CTAs dispatched after their leader finished
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("copy_mode", [0, 1])
def test_put_ctas_dispatched_after_the_leader(R, copy_mode):
    """A put launch whose CTAs start one by one, well after its leader CTA has
    planned the launch and finished: every SM is held by a test kernel that
    releases them 2 us apart (synth_hold_sms).  The late CTAs must not
    speculate the first round from the tail the leader has already moved
    (before the fix they copied their units into the next launch's entries and
    counted them: units never copied).  Every payload byte of every launch
    arrives (device verifier); headers and placements are the oracle's."""
    seed = synth.SEED_BASE + 77
    L = Layout(256 << 20, 64)
    rb = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    pb, mhb = R.ring_attach_peer(R.ring_export(rb), 0, 0)
    R.ring_bind_mirror(rb, 0, mhb)
    R.ring_peer_config(pb, 0, 0, copy_mode)          # LSU copy warps / TMA engines
    launches = 6
    buf_b, ptr_b = device_sources([(0, k, EMB) for k in range(launches)], seed)
    hd_b = [synth.header_fields(seed, 0, k) for k in range(launches)]
    msgs_b = _msgs(R, ptr_b, [EMB] * launches, hd_b, 7, 1, "cuda")
    st_b = [torch.full((1,), 10, dtype=torch.int32, device="cuda") for _ in range(launches)]
    vt_b = torch.zeros(launches * 128, dtype=torch.uint8, device="cuda")
    chans = torch.zeros(1, dtype=torch.int32, device="cuda")
    keys = [dev_u64([k]) for k in range(launches)]
    s_hold, s_pb, s_cb = (torch.cuda.Stream() for _ in range(3))
    bads = []
    try:
        for k in range(launches):
            torch.cuda.synchronize()
            SD.hold_sms(5_000, 2_000, s_hold)                # every SM busy; freed one per 2 us
            R.ring_put_batch(pb, msgs_b[k * 48:(k + 1) * 48], 1, 0, st_b[k], s_pb)
            v = vt_b[k * 128:(k + 1) * 128]
            R.ring_get(rb, 1, v, None, 0, 0, s_cb)
            bads.append(verify_views(rb, v, 1, seed, chans, keys[k], s_cb))
            R.ring_release(rb, 1, s_cb)
        torch.cuda.synchronize()
        img = spsc_image(L, [EMB] * launches)
        ents = [e for e in img["entries"] if not e[3]]
        v = views_host(vt_b)
        for k in range(launches):
            assert st_b[k].cpu().tolist() == [0], k
            assert int(v[k]["status"]) == 0, k
            assert _place(v[k]) == (ents[k][1], ents[k][2], ents[k][0]), k
            h = hd_b[k]
            assert bytes(v[k]["header"])[:56] == encode_header(h[0], h[1], 7, 1, EMB, 0, k, 0, 0, 0)[:56], k
        for k, b in enumerate(bads):
            _ok(b, k)
    finally:
        torch.cuda.synchronize()
        R.ring_detach(pb)
        R.ring_destroy(rb)


def test_get_ctas_dispatched_late(R):
    """The consumer side of the same hazard: a copy-out consume whose CTAs
    start one by one (every SM held, freed 2 us apart) after its control warp
    has planned every entry; the copy warps take their units from the plans
    only, so every payload byte arrives."""
    seed = synth.SEED_BASE + 78
    L = Layout(256 << 20, 64)
    ring = R.ring_create(0, L.R, L.N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    m, launches = 8, 4
    lens = [EMB if q % 2 == 0 else LAT480 for q in range(m)]
    buf, ptrs = device_sources([(0, q, lens[q]) for q in range(m)], seed)
    msgs = _msgs(R, ptrs, lens, [synth.header_fields(seed, 0, q) for q in range(m)], 7, 1, "cuda")
    st = torch.full((m,), 10, dtype=torch.int32, device="cuda")
    vt = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
    dst = torch.empty(m * EMB, dtype=torch.uint8, device="cuda")
    dptr = dev_u64([dst.data_ptr() + q * EMB for q in range(m)])
    dlen, chans, keys = dev_u64(lens), torch.zeros(m, dtype=torch.int32, device="cuda"), dev_u64(list(range(m)))
    s_hold, s_c = torch.cuda.Stream(), torch.cuda.Stream()
    try:
        for k in range(launches):
            R.ring_put_batch(peer, msgs, m, 0, st)
            torch.cuda.synchronize()                          # published before the consume starts
            SD.hold_sms(5_000, 2_000, s_hold)
            R.ring_consume(ring, m, vt, dst, EMB, 0, s_c)
            bad = SD.verify(dptr, dlen, chans, keys, seed, s_c)
            torch.cuda.synchronize()
            assert st.cpu().tolist() == [0] * m, k
            assert (views_host(vt)["status"] == 0).all(), k
            _ok(bad, k)
    finally:
        torch.cuda.synchronize()
        R.ring_detach(peer)
        R.ring_destroy(ring)
