"""Pins for the reserve-then-commit oracle (CPU only):
every interleaving on 2-3 slot rings of 2-4 units with two producers is free of
deadlock, never claims over a live entry, and delivers every channel exactly
once, in order, byte-exact; with one sender lost anywhere the ring stays live
(lock take-over, hole -> PAD).  Each rule is shown necessary: a tail that may
pass an uncommitted (reserved) slot lets the receiver read an entry before it
is written, and without hole filling a lost reservation stalls the ring."""
import itertools

import pytest

import oracle.reserve as rv
from oracle.reserve import explore_rc
from oracle.ring import BUSY, Layout, Msg, unpack, used_slots


def _progs(sizes):
    out = {}
    for pid, sz in enumerate(sizes):
        msgs = []
        for k, u in enumerate(sz):
            n = u * 128 - 64 - 4 * pid
            msgs.append(Msg(n, bytes([(16 * pid + k + i) & 255 for i in range(n)])))
        out[pid] = msgs
    return out


def _configs(N_values, R_units, shapes):
    for N in N_values:
        for Ru in R_units:
            for shape in shapes:
                for combo in itertools.product(range(1, Ru + 1), repeat=sum(shape)):
                    it = iter(combo)
                    yield Layout(Ru * 128, N), [[next(it) for _ in range(m)] for m in shape]


def test_reserve_commit_every_interleaving():
    n = states = 0
    for L, sizes in _configs((2, 3), (2, 3), ((2, 1), (1, 1))):
        for depth in (1, 2):
            r = explore_rc(L, _progs(sizes), depth=depth)
            n += 1
            states += r.states
            assert not r.deadlocks and not r.violations, (L, sizes, depth, r.deadlocks[:1], r.violations[:1])
            assert r.terminals > 0
    assert n >= 100 and states > 100_000


def test_tail_must_not_pass_a_reserved_slot(monkeypatch):
    def loose(self):
        _, t_q = unpack(self.tail)
        _, h_q = unpack(self.head)
        _, r_q = unpack(self.resv)
        w = self.slots[t_q % self.L.N]
        return t_q != r_q and used_slots(t_q, h_q) < self.L.N and bool(w & (BUSY | rv.RESV))
    monkeypatch.setattr(rv.RCSim, "_can_advance", loose)
    found = False
    for L, sizes in _configs((2,), (2, 3), ((1, 1),)):
        r = explore_rc(L, _progs(sizes), depth=1)
        if r.violations:
            found = True
            break
    assert found


def test_lost_sender_anywhere_keeps_the_ring_live():
    """One sender lost at any point (its lock taken over after TL, its
    uncommitted reservation turned into a PAD by the next sender that waits on
    it or claims): never stuck, the other channel complete and in order, the
    lost channel an in-order prefix."""
    n = 0
    for L, sizes in _configs((2,), (2, 3), ((2, 1), (1, 1))):
        r = explore_rc(L, _progs(sizes), depth=1, crash=True)
        n += 1
        assert not r.deadlocks and not r.violations, (L, sizes, r.deadlocks[:1], r.violations[:1])
    assert n >= 30


def test_lost_reservation_without_hole_filling_stalls(monkeypatch):
    monkeypatch.setattr(rv.RCSim, "_hole", lambda self: None)
    stuck = False
    for L, sizes in _configs((2,), (2, 3), ((1, 1),)):
        r = explore_rc(L, _progs(sizes), depth=1, crash=True)
        if r.deadlocks:
            stuck = True
            break
    assert stuck
