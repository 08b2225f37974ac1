"""Pins for the oracle's ring protocol (CPU only, `-m "not gpu"`).

What pins what:
  * worked examples hand-derived from PAPER.md:731-745 (tests/golden/) ->
    placement, PAD, wrap, FULL by bytes / by slots, head/tail/slot words;
  * closed forms for constant-size streams -> the pointer formula over many laps;
  * the plain FIFO definition (exactly once, in order, byte-exact) over C1's
    1,000-message stream and MPSC streams;
  * timing independence of single-producer placement (PAPER.md:731-745 move
    P_b by sizes alone) across consumer schedules.
"""
import random

import pytest

import synth
from oracle.ring import (Layout, Sim, Msg, run, tag_msg, footprint, adv, pack, unpack, interval_free,
                         fifo_definition, delivered_by_channel, spsc_image, BUSY, PADBIT, FMASK,
                         ProtocolViolation)


def _msg(n, k=0):
    return Msg(n, bytes([(k * 7 + i) & 0xFF for i in range(n)]))


def _drive(example):
    lay = example["layout"]
    L = Layout(lay["R"], lay["N"], lay["align"], lay["hdr"])
    puts = [op["len"] for op in example["ops"] if op["op"] == "put"]
    mk = _msg if L.hdr else (lambda n, k: tag_msg(0, k, n))
    sim = Sim(L, {0: [mk(n, k) for k, n in enumerate(puts)]}, mpsc=False, block=False, depth=1)
    p = sim.producers[0]
    for op in example["ops"]:
        if op["op"] == "put":
            before = len(p.outcomes)
            while len(p.outcomes) == before:
                sim.step(0)
            assert p.outcomes[-1] == op["outcome"], op
        else:
            nd = len(sim.cons.delivered)
            while len(sim.cons.delivered) == nd:
                assert "Z" in sim.enabled(), op
                sim.step("Z")
            assert sim.cons.delivered[-1].start == op["start"]
            sim.step("Zrel")
        if "tail" in op:
            assert sim.mem.tail == int(op["tail"], 16), (op, hex(sim.mem.tail))
        if "head" in op:
            assert sim.mem.head == int(op["head"], 16), (op, hex(sim.mem.head))
        if "slots" in op:
            assert sim.mem.slots == [int(x, 16) for x in op["slots"]], (op, [hex(x) for x in sim.mem.slots])
    return sim


@pytest.mark.parametrize("name", ["W1", "W2", "W3", "W4", "SPEC143"])
def test_worked_examples(golden, name):
    _drive(golden[name])


def test_pointer_formula_strict_less_than():
    L = Layout(256, 4, 1, 0)
    assert adv(L, 192, 64) == 0        # exact fit wraps (PAPER.md:735 '<')
    assert adv(L, 100, 100) == 200
    assert adv(L, 0, 255) == 255
    assert adv(L, 0, 256) == 0


def test_footprint_values():
    L = Layout(1 << 20, 8)
    # SURVEY.md sec 8 footprint table (align_up(64 + len, 128))
    assert footprint(L, 4096) == 4224
    assert footprint(L, 1048512) == 1048576
    assert footprint(L, 4194304) == 4194432
    assert footprint(L, 4193280) == 4193408
    assert footprint(L, 9676800) == 9676928
    assert footprint(L, 447897600) == 447897728
    assert footprint(L, 0) == 128 and footprint(L, 64) == 128 and footprint(L, 65) == 256


def test_interval_rule_cases():
    L = Layout(1000, 8, 1, 0)
    assert interval_free(L, 500, 3, 500, 3, 400)          # empty
    assert interval_free(L, 600, 3, 100, 1, 400)          # tail ahead of head
    assert interval_free(L, 100, 3, 600, 1, 500)          # wrapped, fits exactly up to head
    assert not interval_free(L, 100, 3, 600, 1, 501)      # wrapped, overlaps head
    assert not interval_free(L, 300, 3, 300, 1, 1)        # same offset, non-empty: full


@pytest.mark.parametrize("R,f", [(1024, 128), (1024, 256), (1024, 384), (1024, 640), (4096, 1280),
                                 (65536, 4224), (1 << 20, 1 << 20), (3 * 128, 256)])
def test_constant_size_closed_form(R, f):
    """Closed form for a constant footprint f: m = R // f entries per lap land at
    0, f, ..., (m-1)f; if f does not divide R a PAD of R - m*f follows each lap."""
    L = Layout(R, 8, 128, 64)
    n = f - 64
    img = spsc_image(L, [n] * 37)
    m = R // f
    expect = []
    q = 0
    for k in range(37):
        if k and k % m == 0 and R % f:
            expect.append((q, m * f, R - m * f, True))
            q += 1
        expect.append((q, (k % m) * f, f, False))
        q += 1
    assert img["entries"] == expect


def test_c1_fifo_exactly_once_in_order():
    """BASELINE.json configs[0]: 1 producer -> 1 consumer, 8 slots x 4 KB
    (R = 32 KiB), 1,000 messages of U[1, 4096] bytes."""
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 1000, 1, 4096)
    msgs = [Msg(m.length, m.payload.tobytes(), m.uid, m.accepted_at, m.app_id, m.stage) for m in stream]
    sim = Sim(L, {0: msgs}, mpsc=False, block=True, depth=1)
    run(sim, policy="random", seed=3)
    got = delivered_by_channel(sim)
    assert [s for s, _ in got[0]] == list(range(1000))
    assert [p for _, p in got[0]] == fifo_definition({0: msgs})[0]
    assert all(d.status == "OK" for d in sim.cons.delivered)
    assert not any(lab.startswith("UH") and "fix" in lab for lab in sim.log)


def test_spsc_placement_independent_of_schedule():
    L = Layout(32768, 8)
    stream = synth.random_stream(synth.SEED_BASE + 1, 0, 300, 1, 4096, with_payload=False)
    lens = [m.length for m in stream]
    ref = spsc_image(L, lens)["entries"]
    for policy, seed, depth in [("rr", 0, 1), ("random", 1, 1), ("random", 2, 3), ("random", 5, 8)]:
        msgs = [Msg(n, bytes(n)) for n in lens]
        sim = Sim(L, {0: msgs}, mpsc=False, block=True, depth=depth, check=False)
        run(sim, policy=policy, seed=seed)
        starts = [(d.seq_slot, d.start, d.f) for d in sim.cons.delivered]
        assert starts == [(q, s, f) for q, s, f, pad in ref if not pad]


def test_mpsc_fifo_per_channel():
    L = Layout(16384, 8)
    progs = {}
    for pid in range(3):
        st = synth.random_stream(synth.SEED_BASE + 5, pid, 60, 1, 3000)
        progs[pid] = [Msg(m.length, m.payload.tobytes(), m.uid, m.accepted_at, 7, 2) for m in st]
    for seed in range(3):
        sim = Sim(L, progs, mpsc=True, block=True, depth=2)
        run(sim, policy="random", seed=seed)
        got = delivered_by_channel(sim)
        for pid in progs:
            assert [p for _, p in got[pid]] == fifo_definition(progs)[pid]
        # lock held from Lock to Unlock: no two producers between Lock and Unlock
        holder = None
        for lab in sim.log:
            if lab.startswith("Lock("):
                assert holder is None
                holder = lab[5:-1]
            elif lab.startswith("Unlock("):
                assert holder == lab[7:-1]
                holder = None


def test_try_mode_reports_full_and_drops():
    L = Layout(1024, 2)
    msgs = [_msg(100, k) for k in range(5)]
    sim = Sim(L, {0: msgs}, mpsc=False, block=False, depth=1)
    p = sim.producers[0]
    while p.pc != "DONE":
        sim.step(0)
    assert p.outcomes == ["OK", "OK", "FULL", "FULL", "FULL"]     # size region full at N=2
    run(sim, policy="drain")
    assert len(sim.cons.delivered) == 2


def test_corrupt_header_is_discarded_but_consumed():
    """the consumer verifies the checksum; on mismatch the data is
    discarded, and it proceeds using size metadata."""
    L = Layout(4096, 4)
    sim = Sim(L, {0: [_msg(10, 0), _msg(20, 1)]}, mpsc=False, block=True, depth=1, check=False)
    while sim.producers[0].pc != "DONE":
        sim.step(0)
    sim.mem.data[8] ^= 0x40              # flip a bit inside message 0's header
    run(sim, policy="drain")
    assert [d.status for d in sim.cons.delivered] == ["CORRUPT", "OK"]
    assert sim.mem.head == sim.mem.tail


def test_message_larger_than_ring_rejected():
    L = Layout(1024, 4)
    sim = Sim(L, {0: [_msg(1024 - 64, 0)]}, mpsc=False, block=True)   # f = 1024 = R: fits alone
    run(sim)
    assert len(sim.cons.delivered) == 1
    assert footprint(L, 1024 - 63) > L.R                                 # would be EMSGSIZE
