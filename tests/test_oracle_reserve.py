"""Pins for the reserve-then-commit oracle (CPU only):
every interleaving on 2-3 slot rings of 2-4 units with two producers is free of
deadlock, never claims over a live entry, and delivers every channel exactly
once, in order, byte-exact -- and each of the variant's two rules is shown to
be necessary: a tail that may pass an uncommitted (reserved) slot lets the
receiver read an entry before it is written, and a sender that waits for
credit without first publishing the PAD it just claimed deadlocks."""
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


def test_waiting_sender_must_publish_its_pad_first(monkeypatch):
    orig = rv.RCSim._producer

    def no_publish(self, p):
        if p.pc == "UnlockFull":
            assert self.lock == p.pid + 1
            self.lock = 0
            p.pc = "RH"
            return f"Unlock({p.pid})"
        return orig(self, p)
    monkeypatch.setattr(rv.RCSim, "_producer", no_publish)
    r = explore_rc(Layout(256, 2), _progs([[1, 1], [2]]), depth=1)
    assert r.deadlocks
