"""Brute-force pins for the oracle (CPU only): every interleaving on 2-4 slot
rings (BASELINE.json configs[0]; north star "deadlock-freedom brute-forced over
all producer/consumer interleavings on rings of 2 to 4 slots").

Also checks the checker itself: plausible wrong rules (SPEC.md:192-193's
"[H_b, P_b)" occupied-range rule with pre-wrap; a non-strict '<=' pointer
formula; the naive 'used + pad <= R' space rule) must each be caught."""
import itertools

import pytest

import oracle.ring as ring
from oracle.bruteforce import explore, byte_programs, sweep
from oracle.ring import Layout


def _all_ok(N_values, R_values, shapes, depths, size_cap=None):
    n = states = 0
    for cfg, r in sweep(N_values, R_values, shapes, depths, size_cap=size_cap):
        n += 1
        states += r.states
        assert r.ok, (cfg, r.deadlocks[:1], r.violations[:1])
        assert r.terminals > 0, cfg
    return n, states


def test_bruteforce_two_slot_ring():
    n, states = _all_ok((2,), (2, 3, 4, 5, 6), ((2,), (3,), (1, 1), (2, 1)), (1, 2))
    assert n > 1000 and states > 50_000


def test_bruteforce_three_and_four_slots():
    n, states = _all_ok((3, 4), (2, 3, 4, 5), ((3,), (2, 1), (1, 1, 1)), (1, 2), size_cap=4)
    assert n > 500


def test_bruteforce_two_producers_two_messages_each():
    _all_ok((2,), (2, 3, 4), ((2, 2),), (1,))


def _find_failure(N_values=(2, 3), R_values=(2, 3, 4), shapes=((3,), (2, 1)), depths=(1, 2)):
    for cfg, r in sweep(N_values, R_values, shapes, depths):
        if not r.ok:
            return cfg, r
    return None


def test_checker_catches_spec_occupied_range_rule(monkeypatch):
    """SPEC.md:192-193 'pre-wrap, then abort if the new range enters [H_b, P_b)':
    admits an overwrite of an unreleased entry."""
    def spec_rule(L, p_b, p_q, h_b, h_q, f):
        if p_q == h_q:
            return True
        lo, hi = h_b, p_b                      # occupied [H_b, P_b) taken literally
        if lo <= hi:
            return not (p_b < hi and p_b + f > lo) and not (lo <= p_b < hi)
        return True
    monkeypatch.setattr(ring, "interval_free", spec_rule)
    assert _find_failure() is not None


def test_checker_catches_non_strict_pointer_formula(monkeypatch):
    monkeypatch.setattr(ring, "adv", lambda L, s, f: s + f if s + f <= L.R else 0)
    assert _find_failure() is not None


def test_checker_catches_head_ignored(monkeypatch):
    """A space check that ignores the head (only counts slots) overwrites."""
    monkeypatch.setattr(ring, "interval_free", lambda L, p_b, p_q, h_b, h_q, f: True)
    assert _find_failure() is not None


def test_checker_catches_pad_released_late(monkeypatch):
    """If a PAD seen with nothing held were NOT released at once, a producer
    waiting for that space could deadlock (reading R3)."""
    orig = ring.Sim._get

    def lazy_get(self):
        c = self.cons
        w = self.mem.slots[c.g_q % self.L.N]
        if w & ring.PADBIT:
            f = w & ring.FMASK
            self.pad_events.append((c.g_q, c.g_b, f))
            c.held.append((c.g_q, f, True))
            c.g_b, c.g_q = ring.adv(self.L, c.g_b, f), ring.seq_next(c.g_q)
            return "RL(Z)"
        return orig(self)
    monkeypatch.setattr(ring.Sim, "_get", lazy_get)
    assert _find_failure() is not None
