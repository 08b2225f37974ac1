"""Reserve-then-commit MPSC variant (TEST INFRASTRUCTURE ONLY).

The paper's sender holds the lock through the whole append, copy included
(PAPER.md:697-706), so producers of one ring copy one at a time.  In this
variant the lock only guards the *claim*: under the lock a sender reads the
reservation frontier and the head, applies the same space rule (
readings R3-R5: PAD entry at the wrap, interval rule, sequence counters),
marks the size slot "reserved" with its footprint and advances the frontier,
then unlocks; it writes the entry (WB) outside the lock and commits it with
WL (reserved -> busy).  The tail -- what the receiver reads (reading R7) --
only ever moves over *committed* slots: any sender, after its commit, moves it
forward over the leading run of busy slots (a CAS per step), so entries are
published in claim order whoever finishes first.  The receiver is unchanged
(PAPER.md:709-718).

Slot words: busy << 63 | pad << 62 | resv << 61 | f.

A sender waits (helping) until the tail has passed its own entry.  With
`crash=True` one sender may be lost at any point; a sender spinning on a lock
held by the lost one takes it over (TL), and a sender whose
entry waits behind the lost one's reservation turns that hole into a PAD
(reserved -> busy|pad, a CAS; on the GPU after the same timeout TL): the
receiver skips it and liveness is kept.  Shares no code with the
product path.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .ring import (BUSY, FMASK, PADBIT, Layout, Msg, adv, decode_header, encode_header, footprint,
                   interval_free, pack, seq_next, unpack, used_slots)

RESV = 1 << 61
F40 = (1 << 40) - 1


class RCProducer:
    __slots__ = ("pid", "msgs", "k", "pc", "p_b", "p_q", "f", "seen_head", "dead")

    def __init__(self, pid, msgs):
        self.pid, self.msgs, self.k = pid, msgs, 0
        self.pc = "Lock" if msgs else "DONE"
        self.p_b = self.p_q = self.f = 0
        self.seen_head = None
        self.dead = False

    def clone(self):
        c = RCProducer.__new__(RCProducer)
        for s in RCProducer.__slots__:
            setattr(c, s, getattr(self, s))
        return c

    def key(self):
        return (self.k, self.pc, self.p_b, self.p_q, self.f, self.seen_head, self.dead)


class RCSim:
    def __init__(self, L: Layout, programs: dict[int, list[Msg]], depth: int = 1, crash: bool = False):
        self.L = L
        self.crashes_left = 1 if crash else 0
        self.resv_owner: dict[int, int] = {}       # slot seq -> claiming sender (bookkeeping)
        self.programs = programs
        self.lock = 0
        self.tail = 0
        self.head = 0
        self.resv = 0
        self.slots = [0] * L.N
        self.data = bytearray(L.R)
        self.owner = [None] * (L.R // L.align)      # unreleased / claimed units (no-overwrite check)
        self.prods = {p: RCProducer(p, list(m)) for p, m in programs.items()}
        self.g_b = self.g_q = 0
        self.held: list[tuple[int, int, int]] = []   # (seq, f, start) gotten, not released
        self.depth = depth
        self.got: list[tuple[int, int, bytes]] = []   # (producer, k, payload) in delivery order
        self.log: list[str] = []

    def clone(self):
        c = RCSim.__new__(RCSim)
        c.L, c.programs, c.depth = self.L, self.programs, self.depth
        c.crashes_left, c.resv_owner = self.crashes_left, dict(self.resv_owner)
        c.lock, c.tail, c.head, c.resv = self.lock, self.tail, self.head, self.resv
        c.slots = list(self.slots)
        c.data = bytearray(self.data)
        c.owner = list(self.owner)
        c.prods = {k: p.clone() for k, p in self.prods.items()}
        c.g_b, c.g_q = self.g_b, self.g_q
        c.held = list(self.held)
        c.got = list(self.got)
        c.log = list(self.log)
        return c

    def key(self):
        return (self.lock, self.tail, self.head, self.resv, tuple(self.slots), bytes(self.data), tuple(self.owner),
                tuple(p.key() for p in self.prods.values()), self.g_b, self.g_q, tuple(self.held),
                tuple(self.got), self.crashes_left)

    # -- enabled actions ---------------------------------------------------------
    def _can_advance(self) -> bool:
        """The slot at the tail is a committed entry of the claimed range
        [tail, resv) (with fewer than N live slots it cannot be an unreleased
        entry of the previous lap)."""
        _, t_q = unpack(self.tail)
        _, h_q = unpack(self.head)
        _, r_q = unpack(self.resv)
        return t_q != r_q and used_slots(t_q, h_q) < self.L.N and bool(self.slots[t_q % self.L.N] & BUSY)

    def _published(self, q: int) -> bool:
        _, t_q = unpack(self.tail)
        return 1 <= used_slots(t_q, q) < (1 << 23)        # the tail is past q (24-bit sequence distance)

    def _hole(self):
        """The tail's slot is reserved by a lost sender."""
        _, t_q = unpack(self.tail)
        _, r_q = unpack(self.resv)
        w = self.slots[t_q % self.L.N]
        if t_q == r_q or not (w & RESV):
            return None
        o = self.resv_owner.get(t_q)
        return t_q if o is not None and self.prods[o].dead else None

    def enabled(self) -> list:
        acts = []
        for pid, p in self.prods.items():
            if p.pc == "DONE" or p.dead:
                continue
            if self.crashes_left:
                acts.append(("crash", pid))
            if p.pc == "Lock" and self.lock != 0:
                if self.prods[self.lock - 1].dead:
                    acts.append(("TL", pid))              # take over a lost sender's lock
                continue
            if p.pc == "RH" and self.head == p.seen_head and not self._can_advance() and self._hole() is None:
                continue                                  # (a committed entry or a hole at the tail: it helps)
            if p.pc in ("Adv", "AdvW") and not self._can_advance():
                if self._hole() is not None:
                    acts.append(("fill", pid))            # reservation of a lost sender -> PAD
                elif p.pc == "AdvW" or self._published(p.p_q):
                    acts.append(("fin", pid))             # own entry published: next message / wait
                continue
            acts.append(("step", pid))
        _, t_q = unpack(self.tail)
        if t_q != self.g_q and len(self.held) < self.depth:
            acts.append(("get", None))
        if self.held:
            acts.append(("rel", None))
        return acts

    def done(self) -> bool:
        _, t_q = unpack(self.tail)
        return all(p.pc == "DONE" or p.dead for p in self.prods.values()) and t_q == self.g_q and not self.held

    def step(self, act) -> str:
        kind, pid = act
        if kind == "get":
            lab = self._get()
        elif kind == "rel":
            lab = self._release()
        elif kind == "crash":
            self.prods[pid].dead = True
            self.crashes_left -= 1
            lab = f"crash({pid})"
        elif kind == "TL":
            self.lock = pid + 1
            self.prods[pid].pc = "Claim"
            lab = f"TL->Lock({pid})"
        elif kind == "fill":
            q = self._hole()
            w = self.slots[q % self.L.N]
            self.slots[q % self.L.N] = BUSY | PADBIT | (w & F40)
            lab = f"Fill({pid})"
        elif kind == "fin":
            p = self.prods[pid]
            if p.pc == "AdvW":                            # published what it could: wait for credit
                p.pc = "RH"
            else:
                p.k += 1
                p.pc = "Lock" if p.k < len(p.msgs) else "DONE"
            lab = f"Done({pid})"
        else:
            lab = self._producer(self.prods[pid])
        self.log.append(lab)
        return lab

    def _claim_units(self, start, f, tag):
        a = self.L.align
        for u in range(start // a, (start + f) // a):
            if self.owner[u] is not None:
                raise AssertionError(f"claim of {tag} over live entry {self.owner[u]} at unit {u}")
            self.owner[u] = tag

    def _producer(self, p: RCProducer) -> str:
        L, me = self.L, p.pid
        if p.pc == "Lock":
            assert self.lock == 0
            self.lock = me + 1
            p.pc = "Claim"
            return f"Lock({me})"
        if p.pc == "Claim":
            # steps 2-4 on the reservation frontier (space rule R4, PAD R3)
            p.p_b, p.p_q = unpack(self.resv)
            h_b, h_q = unpack(self.head)
            p.seen_head = self.head
            p.f = footprint(L, p.msgs[p.k].length)
            if used_slots(p.p_q, h_q) >= L.N:
                p.pc = "UnlockFull"
                return f"Claim({me})"
            if p.p_b + p.f > L.R:
                if not interval_free(L, p.p_b, p.p_q, h_b, h_q, L.R - p.p_b):
                    p.pc = "UnlockFull"
                    return f"Claim({me})"
                # PAD entry: claimed and committed at once (nothing to write)
                self._claim_units(p.p_b, L.R - p.p_b, ("PAD", p.p_q))
                self.slots[p.p_q % L.N] = BUSY | PADBIT | (L.R - p.p_b)
                self.resv = pack(0, seq_next(p.p_q))
                return f"ClaimPad({me})"                   # stays at Claim
            if not interval_free(L, p.p_b, p.p_q, h_b, h_q, p.f):
                p.pc = "UnlockFull"
                return f"Claim({me})"
            assert self.slots[p.p_q % L.N] == 0, "claimed slot not free"
            self._claim_units(p.p_b, p.f, (me, p.k))
            self.slots[p.p_q % L.N] = RESV | p.f
            self.resv_owner[p.p_q] = me
            self.resv = pack(adv(L, p.p_b, p.f), seq_next(p.p_q))
            p.pc = "Unlock"
            return f"Claim({me})"
        if p.pc in ("Unlock", "UnlockFull"):
            assert self.lock == me + 1
            self.lock = 0
            # full: first publish what is committed (e.g. a PAD it just claimed,
            # which the receiver must free before this entry fits, R3), then wait
            p.pc = "WB" if p.pc == "Unlock" else "AdvW"
            return f"Unlock({me})"
        if p.pc == "RH":
            # waiting for credit without the lock: help publish committed
            # entries (e.g. of a sender lost right after its commit, as GH
            # repairs Case 7) and turn a lost reservation into a PAD; claim
            # again once the head has moved
            q = self._hole()
            if q is not None:
                w = self.slots[q % L.N]
                self.slots[q % L.N] = BUSY | PADBIT | (w & F40)
                return f"Fill({me})"
            if self._can_advance():
                t_b, t_q = unpack(self.tail)
                w = self.slots[t_q % L.N]
                self.tail = pack(adv(L, t_b, w & F40), seq_next(t_q))
                return f"UH({me})"
            p.pc = "Lock"
            return f"RH({me})"
        if p.pc == "WB":                                  # outside the lock
            m = p.msgs[p.k]
            h = encode_header(m.uid, m.accepted_at, m.app_id, m.stage, m.length, me, p.k)[: L.hdr]
            self.data[p.p_b: p.p_b + L.hdr] = h
            self.data[p.p_b + L.hdr: p.p_b + L.hdr + m.length] = m.payload
            p.pc = "WL"
            return f"WB({me})"
        if p.pc == "WL":                                  # commit: CAS reserved -> busy
            s = p.p_q % L.N
            assert self.slots[s] == RESV | p.f, "a live sender's reservation was taken"
            self.slots[s] = BUSY | p.f
            p.pc = "Adv"
            return f"WL({me})"
        if p.pc in ("Adv", "AdvW"):                       # move the tail over one committed slot
            t_b, t_q = unpack(self.tail)
            w = self.slots[t_q % L.N]
            self.tail = pack(adv(L, t_b, w & F40), seq_next(t_q))
            return f"UH({me})"
        raise RuntimeError(p.pc)

    def _get(self) -> str:
        L = self.L
        w = self.slots[self.g_q % L.N]
        assert w & BUSY, "published slot not busy"
        f = w & F40
        start = self.g_b
        if not (w & PADBIT):
            d = decode_header(bytes(self.data[start: start + L.hdr]))
            assert d["crc_ok"]
            pay = bytes(self.data[start + L.hdr: start + L.hdr + d["payload_len"]])
            self.got.append((d["producer_id"], d["seq"], pay))
        self.held.append((self.g_q, f, start))
        self.g_b, self.g_q = adv(L, self.g_b, f), seq_next(self.g_q)
        return "RB(Z)"

    def _release(self) -> str:
        L = self.L
        q, f, start = self.held.pop(0)
        h_b, h_q = unpack(self.head)
        assert h_q == q
        self.slots[q % L.N] = 0
        a = L.align
        for u in range(start // a, (start + f) // a):
            self.owner[u] = None
        self.head = pack(adv(L, h_b, f), seq_next(h_q))
        return "REL(Z)"


@dataclass
class RCResult:
    states: int = 0
    terminals: int = 0
    deadlocks: list = field(default_factory=list)
    violations: list = field(default_factory=list)


def explore_rc(L: Layout, programs: dict, depth: int = 1, max_states: int = 2_000_000,
               crash: bool = False) -> RCResult:
    """Every interleaving: no claim over a live entry, the tail only moves over
    committed slots (each receive finds a busy slot and a valid header), every
    channel delivered exactly once in order, no deadlock.  With `crash`, one
    sender may be lost anywhere: the others still finish and the lost one's
    channel is an in-order prefix of its messages (the one it was appending
    when lost is delivered only if it had committed it)."""
    res = RCResult()
    seen = set()
    stack = [RCSim(L, programs, depth, crash)]
    while stack:
        s = stack.pop()
        k = s.key()
        if k in seen:
            continue
        seen.add(k)
        res.states += 1
        if res.states > max_states:
            raise RuntimeError("state budget exceeded")
        if s.done():
            res.terminals += 1
            for pid, msgs in programs.items():
                mine = [(k2, pay) for p2, k2, pay in s.got if p2 == pid]
                ks = [k2 for k2, _ in mine]
                pr = s.prods[pid]
                want = [list(range(len(msgs)))] if not pr.dead else [list(range(pr.k)), list(range(pr.k + 1))]
                if ks not in want or any(pay != bytes(msgs[k2].payload) for k2, pay in mine):
                    res.violations.append(("delivery", pid, s.log))
            continue
        acts = s.enabled()
        if not acts:
            res.deadlocks.append(list(s.log))
            continue
        for a in acts:
            c = s.clone()
            try:
                c.step(a)
            except AssertionError as e:
                res.violations.append((str(e), list(c.log)))
                continue
            stack.append(c)
    return res
