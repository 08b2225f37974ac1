"""Pins for the fault-mode oracle (CPU only): the paper's eight liveness cases
 replayed as explicit schedules, each checked against the
outcome the paper states for it, and exhaustive interleavings with crashes and
lock take-overs (TL) on tiny rings, checked against Theorem 2
and the hazards the hardenings exist for (DESIGN.md
R21).  Each hazard is shown to be *reachable* without its hardening (so the
checker is not vacuous) and unreachable with it."""
import itertools

import pytest

from oracle.fault import CASES, explore_faults, replay_case
from oracle.ring import Layout, Msg

L = Layout(1024, 4)
X, Y = 0, 1


def _got(sim):
    return [(g.status, g.ident, g.f) for g in sim.got]


@pytest.mark.parametrize("pcrc", [False, True])
def test_case1_lost_sender_then_takeover(pcrc):
    """Case 1: X is lost after Lock, Y takes the lock after TL; 'the receiver Z
    will read valid data written by Y and proceed'."""
    s = replay_case(1, L, 100, 300, payload_crc=pcrc)
    assert _got(s) == [("OK", (Y, 0), 384)]
    assert s.lock == 0


@pytest.mark.parametrize("pcrc", [False, True])
@pytest.mark.parametrize("case", [2, 3])
def test_cases_2_3_delayed_writer_overwrites(case, pcrc):
    """Cases 2-3: X, delayed, overwrites Y's entry; 'WL(X) fails due to the
    busy bit'.  Same sizes: Z reads valid data (X's bytes now fill Y's entry);
    X's entry larger than Y's footprint: Z 'skips invalid entries and
    proceeds using size metadata' (CORRUPT, then the next location)."""
    s = replay_case(case, L, 100, 100, payload_crc=pcrc)
    assert s.prods[X].outcomes == ["DROPPED"] and s.prods[Y].outcomes == ["OK"]
    assert _got(s) == [("OK", (X, 0), 256)]
    s = replay_case(case, L, 300, 100, payload_crc=pcrc)
    assert s.prods[X].outcomes == ["DROPPED"]
    assert _got(s) == [("CORRUPT", None, 256)]          # Y's size decides where Z goes next


@pytest.mark.parametrize("pcrc", [False, True])
def test_case4_late_writer_wins_size_slot(pcrc):
    """Case 4: 'X updates the size before Y; WL(Y) fails.  Z reads X's data'."""
    for xl, yl in ((100, 100), (100, 300), (300, 100)):
        s = replay_case(4, L, xl, yl, payload_crc=pcrc)
        assert s.prods[Y].outcomes == ["DROPPED"] and s.prods[X].outcomes == ["OK"]
        assert _got(s) == [("OK", (X, 0), 256 if xl == 100 else 384)]


@pytest.mark.parametrize("pcrc", [False, True])
def test_case5_later_writer_finalizes(pcrc):
    """Case 5: 'X writes before Y, but Y overwrites and finalizes the entry.
    Z reads valid data from Y'."""
    for xl, yl in ((100, 100), (100, 300), (300, 100)):
        s = replay_case(5, L, xl, yl, payload_crc=pcrc)
        assert s.prods[X].outcomes == ["DROPPED"]
        assert _got(s) == [("OK", (Y, 0), 256 if yl == 100 else 384)]


@pytest.mark.parametrize("pcrc", [False, True])
def test_case6_size_from_x_data_from_y(pcrc):
    """Case 6: 'X updates the size, but Y overwrites the data.  Z skips invalid
    data and proceeds' -- invalid when Y's entry does not fit X's footprint;
    when it fits, the bytes are Y's complete message."""
    s = replay_case(6, L, 100, 300, payload_crc=pcrc)
    assert s.prods[Y].outcomes == ["DROPPED"]
    assert _got(s) == [("CORRUPT", None, 256)]
    s = replay_case(6, L, 100, 100, payload_crc=pcrc)
    assert _got(s) == [("OK", (Y, 0), 256)]


@pytest.mark.parametrize("pcrc", [False, True])
@pytest.mark.parametrize("case", [7, 8])
def test_cases_7_8_both_entries_read(case, pcrc):
    """Case 7: X is lost after WL; 'Y detects this, updates the header, and
    writes new data.  Z reads both X's and Y's data'.  Case 8: X keeps the
    lock past TL; Z still reads X's entry and then Y's."""
    s = replay_case(case, L, 300, 100, payload_crc=pcrc)
    assert _got(s) == [("OK", (X, 0), 384), ("OK", (Y, 0), 256)]
    assert [g.start for g in s.got] == [0, 384]
    if case == 8:
        assert "Unlock(0)!" in s.log                  # X's late Unlock is a failing CAS (Q22)
        assert s.lock == 0


def test_case7_without_repair_would_hide_x():
    """Without Y's GH/UH repair Z could not pass X's committed slot: the
    schedule's UH(Y) right after GH(Y) is exactly the repair."""
    assert CASES[7][6:8] == ["GH(Y)", "UH(Y)"]


# -- exhaustive interleavings with crash + TL ------------------------------------------
def _msg(pid, k, units):
    n = units * 128 - 64 - 8 * (pid + 1)
    return Msg(n, bytes([(0x10 * (pid + 1) + k + i) & 0xFF for i in range(n)]))


def _progs(a, b, c):
    return {X: [_msg(X, 0, a), _msg(X, 1, b)], Y: [_msg(Y, 0, c)]}


def test_hardened_ring_every_interleaving_two_slots():
    """Two senders ([a, b] and [c]), N=2, R=2 units, every footprint mix; at most
    one crash and one take-over from a live owner: never stuck, the busy-slot
    invariant holds in every state, the tail never moves back, no torn payload
    is accepted, Theorem 2 holds, and per-channel delivery is in order without
    duplicates."""
    Lt = Layout(256, 2)
    states = 0
    for a, b, c in itertools.product((1, 2), repeat=3):
        r = explore_faults(Lt, _progs(a, b, c), payload_crc=True)
        states += r.states
        assert not r.stuck and not r.invariant, (a, b, c, r.stuck[:1], r.invariant[:1])
        assert r.rewinds == r.torn == r.unconsumed == r.order == 0, (a, b, c, r)
        assert r.terminals > 0
    assert states > 100_000


@pytest.mark.parametrize("sizes", [(1, 2, 1), (1, 3, 1)])
def test_hardened_ring_three_units(sizes):
    Lt = Layout(384, 2)
    r = explore_faults(Lt, _progs(*sizes), payload_crc=True)
    assert not r.stuck and not r.invariant
    assert r.rewinds == r.torn == r.unconsumed == r.order == 0


def test_header_only_checksum_accepts_a_torn_payload():
    """Q10: the paper's header checksum misses a payload torn by a delayed
    writer; the payload checksum catches it on the same configuration."""
    Lt = Layout(256, 2)
    r = explore_faults(Lt, _progs(1, 2, 1), payload_crc=False, stop_at="torn")
    assert r.torn
    r = explore_faults(Lt, _progs(1, 2, 1), payload_crc=True)
    assert r.torn == 0


def test_plain_store_uh_moves_the_tail_backwards():
    """Q22: with the paper-literal plain UH a taken-over sender's late UH rewinds
    the tail (reachable on the smallest ring); the CAS UH never does."""
    Lt = Layout(256, 2)
    r = explore_faults(Lt, _progs(1, 1, 1), payload_crc=True, uh="store", stop_at="rewinds")
    assert r.rewinds
    r = explore_faults(Lt, _progs(1, 1, 1), payload_crc=True, uh="cas")
    assert r.rewinds == 0 and not r.stuck


def test_untagged_slots_deliver_a_duplicate():
    """R21: without a sequence tag in the size slot, a delayed WL CAS lands on a
    slot the receiver already recycled; a later GH repair publishes it and Z
    reads the old bytes again (a duplicate).  Tagged slots are cleared instead."""
    Lt = Layout(256, 2)
    r = explore_faults(Lt, _progs(1, 2, 1), payload_crc=True, slot_tag=False, stop_at="order")
    assert r.order
    r = explore_faults(Lt, _progs(1, 2, 1), payload_crc=True, slot_tag=True)
    assert r.order == 0 and not r.stuck
