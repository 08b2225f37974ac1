"""Fault-mode oracle of the double ring (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md §6.1 "Deadlock and Liveness": senders may
be lost (crash) or delayed; "if a timer expires, the system assumes the sender
has failed and releases the lock" (TL); "delayed messages
... are allowed to overwrite current buffer entries" and "a checksum is
applied to the data header ... if a mismatch is detected, the data is
discarded".  The eight liveness cases
are schedules of the labelled atomic actions Lock, Unlock, WB, WL, RB, RL, GH,
UH, TL; Theorem 2: "if a sender X
successfully writes data to a position P ... the receiver Z will eventually
access P, but the data at P is not guaranteed to be valid".

This is a separate, plain stepper (`FaultSim`) so that the fault-free oracle
(`oracle.ring.Sim`) stays exactly the 8-step / 5-step protocol.  It adds:
  * `crash(X)`  — X stops forever, at any point of its program;
  * `TL(Y)`     — Y, spinning on the lock (step 1), finds it held by X past the
                  timeout and takes it ("one of the
                  senders releases and reacquires the lock"); modelled as an
                  atomic take-over CAS(X+1 -> Y+1).  X, if alive, continues
                  with its stale view (Cases 2-6, 8);
  * readings from SURVEY.md §8 c-3 that make the recovery sound:
      WL  = CAS(slot, 0 -> busy|f)            (Q23: "WL(X) fails due to the
            busy bit"; a failed WL drops the message: no UH,
            Unlock, next message — no retransmission);
      UH  = CAS(tail, value read at GH -> new) (Q22; `uh="store"` keeps the
            paper-literal plain write, which can move the tail backwards);
      Unlock = CAS(me -> 0)                    (Q22; `unlock="store"` literal);
      payload checksum (Q10; `payload_crc=True`): crc32(payload) in header
            bytes [40, 44), inside the header checksum;
      sequence-tagged size slots (reading R21, `slot_tag=True`): the slot word
            also carries its sequence number mod 2^22 (bits 40-61).  Without it
            a delayed sender's WL CAS can succeed on a slot the receiver has
            already cleared and that now belongs to a later sequence number; a
            GH repair then publishes it and the receiver re-reads stale bytes
            (a duplicate delivery -- found by `explore_faults`, see
            tests/test_oracle_fault.py).  With tags, GH clears a busy slot whose
            tag is not P_seq's (a stale write) instead of publishing it.

Nothing here is fast: one labelled action per `step`, full memory image per
state.  Shares no code with the product path.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .crc32 import crc32
from .ring import (BUSY, FMASK, PADBIT, Layout, Msg, adv, decode_header, encode_header, footprint,
                   interval_free, pack, seq_next, slot_word, unpack, used_slots, MASK24)


TAG_SHIFT = 40
TAG_MASK = (1 << 22) - 1


def tagged(word: int, q: int) -> int:
    return word | ((q & TAG_MASK) << TAG_SHIFT)


def slot_tag(word: int) -> int:
    return (word >> TAG_SHIFT) & TAG_MASK


def slot_f(word: int) -> int:
    return word & ((1 << TAG_SHIFT) - 1)


class FaultProducer:
    __slots__ = ("pid", "msgs", "k", "pc", "p_b", "p_q", "h_b", "h_q", "f", "tail_seen",
                 "fix_tail", "seen_head", "outcomes", "dead")

    def __init__(self, pid: int, msgs: list[Msg]):
        self.pid = pid
        self.msgs = msgs
        self.k = 0
        self.pc = "Lock" if msgs else "DONE"
        self.p_b = self.p_q = self.h_b = self.h_q = self.f = 0
        self.tail_seen = 0          # tail word read at GH: the CAS expectation of UH
        self.fix_tail = None
        self.seen_head = None
        self.outcomes: list[str] = []
        self.dead = False

    def clone(self) -> "FaultProducer":
        c = FaultProducer.__new__(FaultProducer)
        for s in FaultProducer.__slots__:
            setattr(c, s, getattr(self, s))
        c.outcomes = list(self.outcomes)
        return c

    def key(self):
        return (self.k, self.pc, self.p_b, self.p_q, self.h_b, self.h_q, self.f, self.tail_seen,
                self.fix_tail, self.seen_head, tuple(self.outcomes), self.dead)


@dataclass
class Got:
    """One entry as the receiver read it (RL + RB)."""
    seq: int
    start: int
    f: int
    status: str             # "OK" or "CORRUPT"
    ident: tuple | None     # (producer_id, k) from the header when OK
    payload: bytes


class FaultSim:
    def __init__(self, L: Layout, programs: dict[int, list[Msg]], uh: str = "cas", unlock: str = "cas",
                 payload_crc: bool = False, slot_tag: bool = True, max_crashes: int = 1,
                 max_live_steals: int = 1):
        assert L.R < (1 << TAG_SHIFT)
        self.L = L
        self.programs = programs
        self.uh, self.unlock_mode, self.payload_crc = uh, unlock, payload_crc
        self.slot_tag = slot_tag
        self.lock = 0
        self.tail = 0
        self.head = 0
        self.slots = [0] * L.N
        self.data = bytearray(L.R)
        self.g_b = self.g_q = 0                   # receiver cursor (= head: get + release at once)
        self.prods = {pid: FaultProducer(pid, list(m)) for pid, m in programs.items()}
        self.crashes_left = max_crashes
        self.live_steals_left = max_live_steals
        self.got: list[Got] = []
        self.log: list[str] = []
        self.committed: list[int] = []            # seqs whose WL succeeded (Theorem 2)
        self.rewound = False                      # the tail seq ever moved backwards

    # -- search support --------------------------------------------------------
    def clone(self) -> "FaultSim":
        c = FaultSim.__new__(FaultSim)
        c.L, c.programs = self.L, self.programs
        c.uh, c.unlock_mode, c.payload_crc = self.uh, self.unlock_mode, self.payload_crc
        c.slot_tag = self.slot_tag
        c.lock, c.tail, c.head = self.lock, self.tail, self.head
        c.slots = list(self.slots)
        c.data = bytearray(self.data)
        c.g_b, c.g_q = self.g_b, self.g_q
        c.prods = {k: p.clone() for k, p in self.prods.items()}
        c.crashes_left, c.live_steals_left = self.crashes_left, self.live_steals_left
        c.got = list(self.got)
        c.log = list(self.log)
        c.committed = list(self.committed)
        c.rewound = self.rewound
        return c

    def key(self):
        return (self.lock, self.tail, self.head, tuple(self.slots), bytes(self.data), self.g_b, self.g_q,
                tuple(p.key() for p in self.prods.values()), self.crashes_left, self.live_steals_left,
                tuple((g.seq, g.status, g.ident, g.payload) for g in self.got), tuple(self.committed),
                self.rewound)

    # -- enabled actions ---------------------------------------------------------
    def _owner(self):
        return self.lock - 1 if self.lock else None

    def enabled(self) -> list:
        acts = []
        for pid, p in self.prods.items():
            if p.dead or p.pc == "DONE":
                continue
            if p.pc == "Lock":
                if self.lock == 0:
                    acts.append(("step", pid))
                else:
                    o = self.prods[self._owner()]
                    if o.pid != pid and (o.dead or self.live_steals_left > 0):
                        acts.append(("TL", pid))
            elif p.pc == "RH":
                if self.head != p.seen_head:
                    acts.append(("step", pid))
            else:
                acts.append(("step", pid))
            if self.crashes_left > 0:
                acts.append(("crash", pid))
        _, t_q = unpack(self.tail)
        if t_q != self.g_q:
            acts.append(("Z", None))
        return acts

    def done(self) -> bool:
        _, t_q = unpack(self.tail)
        return all(p.dead or p.pc == "DONE" for p in self.prods.values()) and t_q == self.g_q

    # -- one action --------------------------------------------------------------
    def step(self, act) -> str:
        kind, pid = act
        if kind == "Z":
            lab = self._receive()
        elif kind == "crash":
            self.prods[pid].dead = True
            self.crashes_left -= 1
            lab = f"crash({pid})"
        elif kind == "TL":
            o = self.prods[self._owner()]
            if not o.dead:
                self.live_steals_left -= 1
            self.lock = pid + 1
            self.prods[pid].pc = "GH"
            lab = f"TL->Lock({pid})"
        else:
            lab = self._producer_step(self.prods[pid])
        self.log.append(lab)
        self._check()
        return lab

    def _set_tail(self, new: int) -> None:
        _, old_q = unpack(self.tail)
        _, new_q = unpack(new)
        if ((new_q - old_q) & MASK24) > (MASK24 >> 1):
            self.rewound = True
        self.tail = new

    def _next_msg(self, p: FaultProducer) -> None:
        p.k += 1
        p.pc = "Lock" if p.k < len(p.msgs) else "DONE"

    def _decide(self, p: FaultProducer) -> None:
        """Sender step 3 on the view read at GH (readings R3, R4)."""
        L = self.L
        p.f = footprint(L, p.msgs[p.k].length)
        if used_slots(p.p_q, p.h_q) >= L.N:
            p.pc = "UnlockFull"
        elif p.p_b + p.f > L.R:
            p.pc = "WLpad" if interval_free(L, p.p_b, p.p_q, p.h_b, p.h_q, L.R - p.p_b) else "UnlockFull"
        elif interval_free(L, p.p_b, p.p_q, p.h_b, p.h_q, p.f):
            p.pc = "WB"
        else:
            p.pc = "UnlockFull"

    def _header(self, p: FaultProducer) -> bytes:
        m = p.msgs[p.k]
        pc = crc32(bytes(m.payload)) if self.payload_crc else None
        return encode_header(m.uid, m.accepted_at, m.app_id, m.stage, m.length, p.pid, p.k, m.epoch,
                             payload_crc=pc)

    def _unlock(self, p: FaultProducer) -> bool:
        if self.unlock_mode == "cas":
            if self.lock != p.pid + 1:
                return False
        self.lock = 0
        return True

    def _producer_step(self, p: FaultProducer) -> str:
        L, me, pc = self.L, p.pid, p.pc
        if pc == "Lock":                                  # step 1
            assert self.lock == 0
            self.lock = me + 1
            p.pc = "GH"
            return f"Lock({me})"
        if pc == "GH":                                    # steps 2 + 4
            p.tail_seen = self.tail
            p.p_b, p.p_q = unpack(self.tail)
            p.h_b, p.h_q = unpack(self.head)
            p.seen_head = self.head
            nxt = self.slots[p.p_q % L.N]
            if used_slots(p.p_q, p.h_q) < L.N and (nxt & BUSY):
                if self.slot_tag and slot_tag(nxt) != (p.p_q & TAG_MASK):
                    p.fix_tail = nxt                      # a stale write (R21): clear it
                    p.pc = "GHclean"
                else:
                    p.fix_tail = pack(adv(L, p.p_b, slot_f(nxt & FMASK)), seq_next(p.p_q))   # Case 7 repair
                    p.pc = "UHfix"
            else:
                self._decide(p)
            return f"GH({me})"
        if pc == "GHclean":
            s = p.p_q % L.N
            if self.slots[s] == p.fix_tail:               # CAS(stale word -> 0)
                self.slots[s] = 0
            p.fix_tail = None
            p.pc = "GH"
            return f"GHclean({me})"
        if pc == "UHfix":
            if self.uh == "cas" and self.tail != p.tail_seen:
                p.pc = "GH"                               # someone moved it: look again
                return f"UH({me})!"
            self._set_tail(p.fix_tail)
            p.fix_tail = None
            p.pc = "GH"
            return f"UH({me})"
        if pc == "WLpad":                                 # PAD entry (reading R3)
            s = p.p_q % L.N
            if self.slots[s] != 0:
                p.pc = "GH"                               # the slot was taken meanwhile
                return f"WL({me})!"
            w = slot_word(L.R - p.p_b, pad=True)
            self.slots[s] = tagged(w, p.p_q) if self.slot_tag else w
            p.pc = "UHpad"
            return f"WLpad({me})"
        if pc == "UHpad":
            new = pack(0, seq_next(p.p_q))
            if self.uh == "cas" and self.tail != p.tail_seen:
                p.pc = "GH"
                return f"UH({me})!"
            self._set_tail(new)
            p.tail_seen = new
            p.p_b, p.p_q = 0, seq_next(p.p_q)
            self._decide(p)
            return f"UHpad({me})"
        if pc == "WB":                                    # step 5
            m = p.msgs[p.k]
            self.data[p.p_b: p.p_b + L.hdr] = self._header(p)[: L.hdr]
            self.data[p.p_b + L.hdr: p.p_b + L.hdr + m.length] = m.payload
            p.pc = "WL"
            return f"WB({me})"
        if pc == "WL":                                    # step 6, a CAS (Q23)
            s = p.p_q % L.N
            if self.slots[s] != 0:
                p.outcomes.append("DROPPED")              # "WL(X) fails due to the busy bit"
                p.pc = "UnlockDrop"
                return f"WL({me})!"
            self.slots[s] = tagged(slot_word(p.f), p.p_q) if self.slot_tag else slot_word(p.f)
            self.committed.append(p.p_q)
            p.pc = "UH"
            return f"WL({me})"
        if pc == "UH":                                    # step 7
            new = pack(adv(L, p.p_b, p.f), seq_next(p.p_q))
            if self.uh == "cas" and self.tail != p.tail_seen:
                p.outcomes.append("COMMITTED")            # published later by a GH repair
                p.pc = "Unlock"
                return f"UH({me})!"
            self._set_tail(new)
            p.outcomes.append("OK")
            p.pc = "Unlock"
            return f"UH({me})"
        if pc in ("Unlock", "UnlockDrop"):                # step 8
            ok = self._unlock(p)
            self._next_msg(p)
            return f"Unlock({me})" + ("" if ok else "!")
        if pc == "UnlockFull":
            ok = self._unlock(p)
            p.pc = "RH"
            return f"Unlock({me})" + ("" if ok else "!")
        if pc == "RH":
            p.pc = "Lock"
            return f"RH({me})"
        raise RuntimeError(pc)

    def _receive(self) -> str:
        """Receiver steps 1-5 + checksum:
        RL, RB, verify, reset the busy bit, move the head."""
        L = self.L
        s = self.g_q % L.N
        w = self.slots[s]
        assert w & BUSY, "published slot not busy"
        if self.slot_tag:
            assert slot_tag(w) == (self.g_q & TAG_MASK), "published slot carries another sequence number"
        f = slot_f(w & FMASK)
        start = self.g_b
        if w & PADBIT:
            status, ident, payload = "PAD", None, b""
        else:
            h = bytes(self.data[start: start + L.hdr])
            d = decode_header(h)
            ok = d["crc_ok"] and L.hdr + d["payload_len"] <= f
            payload = bytes(self.data[start + L.hdr: start + L.hdr + (d["payload_len"] if ok else 0)])
            if ok and d["payload_crc"] is not None:
                ok = crc32(payload) == d["payload_crc"]
            status = "OK" if ok else "CORRUPT"
            ident = (d["producer_id"], d["seq"]) if ok else None
            if not ok:
                payload = b""
        self.got.append(Got(self.g_q, start, f, status, ident, payload))
        self.slots[s] = 0
        self.g_b, self.g_q = adv(L, self.g_b, f), seq_next(self.g_q)
        self.head = pack(self.g_b, self.g_q)
        return "RL+RB(Z)"

    # -- invariants ------------------------------------------------------------
    def _check(self) -> None:
        """The invariant behind Theorem 2: every slot in
        [H_seq, P_seq) is busy (a busy bit is only ever cleared by Z)."""
        _, t_q = unpack(self.tail)
        _, h_q = unpack(self.head)
        n = used_slots(t_q, h_q)
        if n <= self.L.N:
            for i in range(n):
                if not (self.slots[(h_q + i) % self.L.N] & BUSY):
                    raise AssertionError(f"live slot {(h_q + i) % self.L.N} not busy")


# ----------------------------------------------------------------------------
# Checks over one run / the whole state space
# ----------------------------------------------------------------------------
def torn(sim: FaultSim, g: Got) -> bool:
    """An OK delivery whose bytes are not exactly the message its header names."""
    pid, k = g.ident
    msgs = sim.programs.get(pid)
    return msgs is None or not (0 <= k < len(msgs)) or bytes(msgs[k].payload) != g.payload


@dataclass
class FaultResult:
    states: int = 0
    terminals: int = 0
    stuck: list = field(default_factory=list)        # non-terminal states with nothing enabled
    invariant: list = field(default_factory=list)    # I1 violations
    rewinds: int = 0                                 # terminal states reached through a tail rewind
    torn: int = 0                                    # terminal states with an accepted torn payload
    unconsumed: int = 0                              # Theorem 2: a committed entry skipped or lost
    order: int = 0                                   # per-channel order / duplicate violations


def check_terminal(sim: FaultSim, res: FaultResult) -> None:
    """Theorem 2 at a terminal state: every committed entry
    (successful WL) was accessed by Z, except one whose sender was lost before
    its UH and that no later sender has come to repair yet: it must then sit
    at the tail with its busy slot intact, where the next sender's GH finds it
    ("Z will eventually access P")."""
    _, t_q = unpack(sim.tail)
    seen = {g.seq for g in sim.got}
    for q in sim.committed:
        if q in seen:
            continue
        # an unread committed seq: either it is the pending one at the tail ...
        w = sim.slots[q % sim.L.N]
        pending = q == t_q and (w & BUSY) and (not sim.slot_tag or slot_tag(w) == (q & TAG_MASK))
        # ... or it was a stale WL on a recycled slot (seq below the receiver's
        # cursor when written), which R21 clears and the receiver never reads.
        stale = ((sim.g_q - q) & MASK24) < (MASK24 >> 1) and q != t_q and sim.slot_tag
        if not (pending or stale):
            res.unconsumed += 1
            return
    if any(g.status == "OK" and torn(sim, g) for g in sim.got):
        res.torn += 1
    last = {}
    for g in sim.got:
        if g.status == "OK":
            pid, k = g.ident
            if k <= last.get(pid, -1):
                res.order += 1
                break
            last[pid] = k
    if sim.rewound:
        res.rewinds += 1


def explore_faults(L: Layout, programs: dict, max_states: int = 3_000_000, stop_at: str | None = None,
                   **kw) -> FaultResult:
    """Every interleaving of the labelled actions, crashes and TL take-overs
    (DFS with a visited-state set).  `stop_at` = a FaultResult counter name:
    return as soon as it becomes non-zero (hazard-finding mode)."""
    res = FaultResult()
    root = FaultSim(L, programs, **kw)
    seen = set()
    stack = [root]
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
            check_terminal(s, res)
        else:
            acts = s.enabled()
            if not acts:
                res.stuck.append(list(s.log))
            for a in acts:
                c = s.clone()
                try:
                    c.step(a)
                except AssertionError as e:
                    res.invariant.append((str(e), list(c.log)))
                    continue
                stack.append(c)
        if stop_at is not None and getattr(res, stop_at):
            return res
    return res


# ----------------------------------------------------------------------------
# The paper's eight cases as explicit schedules
# ----------------------------------------------------------------------------
# Actors: X = producer 0, Y = producer 1.  "X lost" = crash(X) at that point.
# Labels name the paper's actions; the receiver drains at the end (RL/RB).
CASES = {
    1: ["Lock(X)", "crash(X)", "TL->Lock(Y)", "GH(Y)", "WB(Y)", "WL(Y)", "UH(Y)", "Unlock(Y)"],
    2: ["Lock(X)", "GH(X)", "TL->Lock(Y)", "GH(Y)", "WB(Y)", "WL(Y)", "UH(Y)", "Unlock(Y)", "WB(X)", "WL(X)"],
    3: ["Lock(X)", "GH(X)", "TL->Lock(Y)", "GH(Y)", "WB(Y)", "WB(X)", "WL(Y)", "UH(Y)", "Unlock(Y)", "WL(X)"],
    4: ["Lock(X)", "GH(X)", "TL->Lock(Y)", "GH(Y)", "WB(Y)", "WB(X)", "WL(X)", "WL(Y)", "UH(X)", "Unlock(X)"],
    5: ["Lock(X)", "GH(X)", "TL->Lock(Y)", "GH(Y)", "WB(X)", "WB(Y)", "WL(Y)", "WL(X)", "UH(Y)", "Unlock(Y)"],
    6: ["Lock(X)", "GH(X)", "TL->Lock(Y)", "GH(Y)", "WB(X)", "WB(Y)", "WL(X)", "WL(Y)", "UH(X)", "Unlock(X)"],
    # Case 7: PAPER.md:817 lists Y's actions as GH UH WB WL Unlock; Y's own final
    # UH is missing (reading Q15: a typo) and is added before Unlock(Y).
    7: ["Lock(X)", "GH(X)", "WB(X)", "WL(X)", "crash(X)", "TL->Lock(Y)", "GH(Y)", "UH(Y)", "GH(Y)", "WB(Y)",
        "WL(Y)", "UH(Y)", "Unlock(Y)"],
    # Case 8: PAPER.md:821 ends "UH(X) -> Unlock(X)" after WL(Y); reading Q15:
    # X, still holding what it thinks is its lock, performs its late Unlock
    # (a CAS that fails against Y's ownership), and Y completes UH + Unlock.
    8: ["Lock(X)", "GH(X)", "WB(X)", "WL(X)", "UH(X)", "TL->Lock(Y)", "GH(Y)", "WB(Y)", "WL(Y)", "UH(Y)",
        "Unlock(X)", "Unlock(Y)"],
}

_NAME = {"X": 0, "Y": 1}


def _act_for(sim: FaultSim, label: str):
    """Translate a paper label into one enabled action (asserting it is enabled
    and that the actor's next step is that action)."""
    name, who = label.rstrip(")").split("(")
    pid = _NAME[who]
    if name == "crash":
        return ("crash", pid)
    if name == "TL->Lock":
        return ("TL", pid)
    p = sim.prods[pid]
    expect = {"Lock": ("Lock",), "GH": ("GH",), "UH": ("UH", "UHfix", "UHpad"), "WB": ("WB",),
              "WL": ("WL", "WLpad"), "Unlock": ("Unlock", "UnlockDrop", "UnlockFull")}[name]
    assert p.pc in expect, f"{label}: {who} is at {p.pc}"
    return ("step", pid)


def replay_case(n: int, L: Layout, x_len: int, y_len: int, progs: dict | None = None, **kw) -> FaultSim:
    """Run case n with one message per sender (lengths x_len, y_len, or the
    given one-message programs), then let the receiver drain.  Returns the
    simulator (inspect `.got`, `.log`)."""
    if progs is None:
        progs = {0: [Msg(x_len, bytes([0xA0 + i % 16 for i in range(x_len)]))],
                 1: [Msg(y_len, bytes([0xB0 + i % 16 for i in range(y_len)]))]}
    sim = FaultSim(L, progs, max_crashes=1, max_live_steals=1, **kw)
    for lab in CASES[n]:
        a = _act_for(sim, lab)
        assert a in sim.enabled(), (lab, sim.enabled())
        sim.step(a)
    while ("Z", None) in sim.enabled():
        sim.step(("Z", None))
    return sim
