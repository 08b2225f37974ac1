"""Plain, slow CPU oracle of the paper's double-ring buffer (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md §6.1 "Ring Buffer" step by step, in the
paper's order and notation, over an in-memory image of the four regions the
paper lists: a lock region, a fixed header holding the head
and tail pointers, a variable-size buffer region and a size region whose slots
carry a busy bit that only the consumer clears.  Where the paper is silent or
ambiguous the reading taken is the one listed in DESIGN.md §"Readings"
(R1..R14); each use below names its reading.

Nothing here is fast or clever: one Python object per region word, one
labelled atomic action per call of `Sim.step`, no batching, no reordering.
The product path (`paper_2601_20655_b200/`) shares no code with this file.

Word formats (DESIGN.md §"Formats"; fixed by this build, not by the paper):
  tail / head word : (byte_offset << 24) | (seq mod 2^24)          (R8, R5)
  size-slot word   : busy << 63 | pad << 62 | footprint            (R9, R3)
  lock word        : 0 = free, producer_id + 1 = held               (R14)
  entry            : 64-byte header, payload, padding to `align`    (R11)
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

from .crc32 import crc32

MASK24 = (1 << 24) - 1
BUSY = 1 << 63
PADBIT = 1 << 62
FMASK = (1 << 62) - 1

# ----------------------------------------------------------------------------
# Layout and pointer formulas
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class Layout:
    """Ring geometry.  PAPER.md:735 and 744 use one symbol `RegionSize` for both
    regions; reading R2 splits it into R (buffer-region bytes) and N (size-region
    slots).  `align`/`hdr` are the entry framing (R11): 128/64 for the GPU
    format, 1/0 for the byte-level examples of the paper's formula."""
    R: int
    N: int
    align: int = 128
    hdr: int = 64

    def __post_init__(self):
        if self.R <= 0 or self.N <= 0:
            raise ValueError("R and N must be positive")
        if self.R % self.align:
            raise ValueError("R must be a multiple of align")
        if self.N > (1 << 23):
            raise ValueError("N must fit the 24-bit sequence space with room (R5)")
        if self.R >= (1 << 40):
            raise ValueError("R must fit 40 bits (R8)")


def align_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


def footprint(L: Layout, length: int) -> int:
    """Bytes an entry occupies in the buffer region: header + payload rounded up
    to `align` (R9: the size slot records this footprint, so the pointer formula
    advances exactly by it)."""
    return align_up(L.hdr + length, L.align)


def adv(L: Layout, p_b: int, size: int) -> int:
    """Buffer-region pointer update, PAPER.md:731-739 (§6.1 "Buffer Region and
    Size Region"):  P_b = P_b + size(P_size) if P_b + size(P_size) < RegionSize,
    else 0.  Strict '<': an entry that ends exactly at R wraps the pointer to 0."""
    return p_b + size if p_b + size < L.R else 0


def seq_next(q: int) -> int:
    """Size-region pointer update:  P_size = (P_size+1) mod
    RegionSize.  Reading R5: the counter is kept modulo 2^24 and the slot index
    is seq mod N, so "size ring full" (P_seq - H_seq = N) is distinguishable
    from "next slot already busy" (sender step 4)."""
    return (q + 1) & MASK24


def pack(b: int, q: int) -> int:
    """One header word per pointer pair; "both the pointers will be
    updated in the header in atomic operations" (R8)."""
    return (b << 24) | (q & MASK24)


def unpack(w: int) -> tuple[int, int]:
    return w >> 24, w & MASK24


def used_slots(p_q: int, h_q: int) -> int:
    return (p_q - h_q) & MASK24


def interval_free(L: Layout, p_b: int, p_q: int, h_b: int, h_q: int, f: int) -> bool:
    """Sender step 3, "If insufficient space remains", reading R4:
    the bytes [p_b, p_b+f) (with p_b+f <= R) are free iff they do not intersect
    the live cyclic range [h_b, p_b) of unreleased entries."""
    assert p_b + f <= L.R
    if p_q == h_q:          # empty ring
        return True
    if p_b > h_b:           # live range [h_b, p_b): everything from p_b to R is free
        return True
    if p_b < h_b:           # live range wraps: free bytes are [p_b, h_b)
        return p_b + f <= h_b
    return False            # p_b == h_b and non-empty: full


def slot_word(f: int, pad: bool = False) -> int:
    """Size-region slot: "the size of each data entry ... includes a busy bit"
    (PAPER.md:685-688); pad flag = reading R3."""
    return BUSY | (PADBIT if pad else 0) | f


# ----------------------------------------------------------------------------
# Entry header (PAPER.md:410-427 fields + build extensions, R11)
# ----------------------------------------------------------------------------
HDR_BYTES = 64
CRC_END = 56          # CRC covers header bytes [4, 56); [56, 64) is t_put (R10)


HDR_FLAG_PAYLOAD_CRC = 1   # flags bit 0: bytes [40, 44) hold crc32(payload) (fault path, Q10)


def encode_header(uid: bytes, accepted_at: int, app_id: int, stage: int, payload_len: int,
                  producer_id: int, seq: int, epoch: int = 0, flags: int = 0, t_put: int = 0,
                  payload_crc: int | None = None) -> bytes:
    """64-byte entry header.  Fields 4..44 follow the paper's message header
    (UUID, proxy timestamp, application ID, stage) in SPEC.md's
    order (uid16 accepted_at8 app_id4 stage2 payload_len4
    reserved6); bytes 44..56 are build extensions (producer id, channel seq,
    route epoch, flags) that make "message context / origin" visible
    (PAPER.md:630-631); bytes 56..64 hold a timing stamp outside the checksum.
    Checksum: "a checksum is applied to the data header".  With
    `payload_crc` (the fault path's hardening: a header-only
    checksum accepts torn payloads) bytes [40, 44) carry crc32(payload) and
    flags bit 0 is set; both lie inside the header checksum."""
    assert len(uid) == 16
    reserved = bytes(6)
    if payload_crc is not None:
        reserved = bytes(2) + struct.pack("<I", payload_crc)
        flags |= HDR_FLAG_PAYLOAD_CRC
    body = (bytes(uid)
            + struct.pack("<QIHI", accepted_at, app_id, stage, payload_len)
            + reserved
            + struct.pack("<IIHH", producer_id, seq, epoch, flags))
    assert len(body) == CRC_END - 4
    return struct.pack("<I", crc32(body)) + body + struct.pack("<Q", t_put)


def decode_header(h: bytes) -> dict:
    crc, = struct.unpack_from("<I", h, 0)
    uid = bytes(h[4:20])
    accepted_at, app_id, stage, payload_len = struct.unpack_from("<QIHI", h, 20)
    producer_id, seq, epoch, flags = struct.unpack_from("<IIHH", h, 44)
    t_put, = struct.unpack_from("<Q", h, 56)
    payload_crc, = struct.unpack_from("<I", h, 40)
    return dict(crc=crc, uid=uid, accepted_at=accepted_at, app_id=app_id, stage=stage,
                payload_len=payload_len, producer_id=producer_id, seq=seq, epoch=epoch,
                flags=flags, t_put=t_put, crc_ok=(crc32(bytes(h[4:CRC_END])) == crc),
                payload_crc=payload_crc if flags & HDR_FLAG_PAYLOAD_CRC else None)


# ----------------------------------------------------------------------------
# Memory image (lock region, header, buffer region, size region)
# ----------------------------------------------------------------------------
class RingImage:
    __slots__ = ("L", "lock", "tail", "head", "slots", "data", "owner")

    def __init__(self, L: Layout):
        self.L = L
        self.lock = 0
        self.tail = 0
        self.head = 0
        self.slots = [0] * L.N
        self.data = bytearray(L.R)
        # owner[u] = id of the unreleased entry covering align-unit u, or None.
        # Bookkeeping for the "no overwrite of an unreleased entry" check only.
        self.owner = [None] * (L.R // L.align)

    def clone(self) -> "RingImage":
        c = RingImage.__new__(RingImage)
        c.L = self.L
        c.lock, c.tail, c.head = self.lock, self.tail, self.head
        c.slots = list(self.slots)
        c.data = bytearray(self.data)
        c.owner = list(self.owner)
        return c

    def key(self):
        return (self.lock, self.tail, self.head, tuple(self.slots), bytes(self.data), tuple(self.owner))


# ----------------------------------------------------------------------------
# Producer (sender), as an explicit-state machine
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Msg:
    length: int
    payload: bytes
    uid: bytes = bytes(16)
    accepted_at: int = 0
    app_id: int = 0
    stage: int = 0
    epoch: int = 0


class Producer:
    """One sender.  `pc` names the next labelled atomic action:
    Lock, GH, UH(repair), WLpad/UHpad (reading R3), WB, WL, UH, Unlock, and RH
    (re-read the head while waiting for credit, reading R12 BLOCK)."""
    __slots__ = ("pid", "msgs", "k", "pc", "p_b", "p_q", "h_b", "h_q", "f", "seen_head",
                 "outcomes", "fix_tail", "mpsc", "block")

    def __init__(self, pid: int, msgs: list[Msg], mpsc: bool, block: bool):
        self.pid = pid
        self.msgs = msgs
        self.k = 0
        self.mpsc = mpsc
        self.block = block
        self.pc = self._first_pc() if msgs else "DONE"
        self.p_b = self.p_q = self.h_b = self.h_q = self.f = 0
        self.seen_head = None
        self.fix_tail = None
        self.outcomes: list[str] = []

    def _first_pc(self):
        # Sender step 1 "Acquire the lock"; with a single producer
        # the lock is elided (reading R14: no competitor exists).
        return "Lock" if self.mpsc else "GH"

    def clone(self) -> "Producer":
        c = Producer.__new__(Producer)
        for s in Producer.__slots__:
            setattr(c, s, getattr(self, s))
        c.outcomes = list(self.outcomes)
        return c

    def key(self):
        return (self.k, self.pc, self.p_b, self.p_q, self.h_b, self.h_q, self.f,
                self.seen_head, self.fix_tail, tuple(self.outcomes))


# ----------------------------------------------------------------------------
# Consumer (receiver)
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Delivered:
    start: int          # byte offset of the entry in the buffer region
    f: int              # footprint from the size slot
    seq_slot: int       # size-region sequence number of the entry
    status: str         # "OK" or "CORRUPT"
    header: bytes       # the entry header bytes [0, hdr) as read
    payload: bytes      # the payload bytes as read


class Consumer:
    """Single consumer, co-located with the ring (never fails).
    G = private read cursor, H = published head (reading R13: get and release
    are split; release is in order)."""
    __slots__ = ("g_b", "g_q", "held", "delivered", "depth")

    def __init__(self, depth: int = 1):
        self.g_b = 0
        self.g_q = 0
        self.held: list[tuple[int, int, bool]] = []    # (seq, f, is_pad) gotten, not released
        self.delivered: list[Delivered] = []
        self.depth = depth

    def clone(self) -> "Consumer":
        c = Consumer.__new__(Consumer)
        c.g_b, c.g_q, c.depth = self.g_b, self.g_q, self.depth
        c.held = list(self.held)
        c.delivered = list(self.delivered)
        return c

    def key(self):
        return (self.g_b, self.g_q, tuple(self.held), len(self.delivered))

    def n_held_msgs(self):
        return sum(1 for _, _, pad in self.held if not pad)


class ProtocolViolation(AssertionError):
    pass


# ----------------------------------------------------------------------------
# The stepper
# ----------------------------------------------------------------------------
class Sim:
    """Deterministic stepper over labelled atomic actions.

    `enabled()` lists the actors that can take a step; `step(actor)` performs
    exactly one action and returns its label, e.g. "WB(1)" or "REL(Z)".
    Actor ids: producer pid (int) or "Z" (the consumer).
    """

    def __init__(self, L: Layout, programs: dict[int, list[Msg]], mpsc: bool | None = None,
                 block: bool = True, depth: int = 1, check: bool = True):
        self.L = L
        self.mem = RingImage(L)
        if mpsc is None:
            mpsc = len(programs) > 1
        self.mpsc = mpsc
        self.producers = {pid: Producer(pid, list(msgs), mpsc, block) for pid, msgs in programs.items()}
        self.cons = Consumer(depth)
        self.check = check
        self.programs = programs
        self.last_k = {pid: -1 for pid in programs}      # last delivered stream index per channel
        self.log: list[str] = []
        self.pad_events: list[tuple[int, int, int]] = []   # (seq, start, f) of PAD entries consumed

    # -- cloning for search ---------------------------------------------------
    def clone(self) -> "Sim":
        c = Sim.__new__(Sim)
        c.L, c.mpsc, c.check, c.programs = self.L, self.mpsc, self.check, self.programs
        c.last_k = dict(self.last_k)
        c.mem = self.mem.clone()
        c.producers = {k: p.clone() for k, p in self.producers.items()}
        c.cons = self.cons.clone()
        c.log = list(self.log)
        c.pad_events = list(self.pad_events)
        return c

    def key(self):
        return (self.mem.key(), tuple(p.key() for p in self.producers.values()), self.cons.key(),
                tuple(self.last_k.values()))

    # -- enabled actions --------------------------------------------------------
    def producer_enabled(self, p: Producer) -> bool:
        if p.pc == "DONE":
            return False
        if p.pc == "Lock":
            return self.mem.lock == 0          # CAS-based spinlock: spins while held
        if p.pc == "RH":
            return self.mem.head != p.seen_head  # waits until the consumer frees space
        return True

    def consumer_get_enabled(self) -> bool:
        # Receiver steps 1-2, reading R7: new data exists
        # iff the published tail sequence differs from the read cursor.
        _, t_q = unpack(self.mem.tail)
        return t_q != self.cons.g_q and self.cons.n_held_msgs() < self.cons.depth

    def enabled(self) -> list:
        acts = [pid for pid, p in self.producers.items() if self.producer_enabled(p)]
        if self.consumer_get_enabled():
            acts.append("Z")
        if self.cons.n_held_msgs() > 0:
            acts.append("Zrel")
        return acts

    def done(self) -> bool:
        _, t_q = unpack(self.mem.tail)
        return (all(p.pc == "DONE" for p in self.producers.values())
                and t_q == self.cons.g_q and not self.cons.held)

    # -- one action ---------------------------------------------------------------
    def step(self, actor) -> str:
        if actor == "Z":
            lab = self._get()
        elif actor == "Zrel":
            lab = self._release()
        else:
            lab = self._producer_step(self.producers[actor])
        self.log.append(lab)
        if self.check:
            self._check_invariants()
        return lab

    # -- sender ---------------------------------------------------------------------
    def _decide(self, p: Producer) -> None:
        """Sender step 3 after step 4's header check (reading R6):
        choose WB, a PAD entry (reading R3) or 'insufficient space'."""
        L = self.L
        msg = p.msgs[p.k]
        p.f = footprint(L, msg.length)
        used = used_slots(p.p_q, p.h_q)
        if used >= L.N:
            return self._full(p)
        if p.p_b + p.f > L.R:
            # The entry would straddle the end of the buffer region; the pointer
            # formula only ever places entries at P_b, so the
            # tail [P_b, R) is covered by a PAD entry first (reading R3).
            if interval_free(L, p.p_b, p.p_q, p.h_b, p.h_q, L.R - p.p_b):
                p.pc = "WLpad"
                return
            return self._full(p)
        if interval_free(L, p.p_b, p.p_q, p.h_b, p.h_q, p.f):
            p.pc = "WB"
            return
        return self._full(p)

    def _full(self, p: Producer) -> None:
        # "If insufficient space remains ... release the lock and abort"
        # (PAPER.md:699).  Reading R12: TRY = abort; BLOCK = release the lock and
        # wait for the consumer to move the head, then start over at step 1.
        if p.mpsc:
            p.pc = "UnlockFull"
        else:
            self._after_full(p)

    def _after_full(self, p: Producer) -> None:
        if p.block:
            p.pc = "RH"
        else:
            p.outcomes.append("FULL")
            self._next_msg(p)

    def _next_msg(self, p: Producer) -> None:
        p.k += 1
        p.pc = p._first_pc() if p.k < len(p.msgs) else "DONE"

    def _producer_step(self, p: Producer) -> str:
        L, mem, me = self.L, self.mem, p.pid
        pc = p.pc
        if pc == "Lock":
            # Step 1: "Acquire the lock using a CAS-based spinlock".
            assert mem.lock == 0
            mem.lock = me + 1
            p.pc = "GH"
            return f"Lock({me})"
        if pc == "GH":
            # Step 2: "Read the current tail position from the shared header"
            # -- tail word holds (P_b, P_size); the head is read
            # for the space check of step 3.  Step 4: "Check
            # whether the next slot in the size region has been updated".
            p.p_b, p.p_q = unpack(mem.tail)
            p.h_b, p.h_q = unpack(mem.head)
            p.seen_head = mem.head
            nxt = mem.slots[p.p_q % L.N]
            if used_slots(p.p_q, p.h_q) < L.N and (nxt & BUSY):
                # A previous sender committed WB+WL but was lost before UH
                # (Case 7): "update the header before writing new data".
                p.fix_tail = pack(adv(L, p.p_b, nxt & FMASK), seq_next(p.p_q))
                p.pc = "UHfix"
            else:
                self._decide(p)
            return f"GH({me})"
        if pc == "UHfix":
            mem.tail = p.fix_tail
            p.fix_tail = None
            p.pc = "GH"
            return f"UH({me})"
        if pc == "WLpad":
            # PAD entry (reading R3): the size slot records the skipped bytes with
            # the pad flag; the busy bit is set as in step 6.
            self._claim_units(p.p_b, L.R - p.p_b, ("PAD", p.p_q))
            s = p.p_q % L.N
            if mem.slots[s] != 0:
                raise ProtocolViolation(f"WLpad on busy slot {s}")
            mem.slots[s] = slot_word(L.R - p.p_b, pad=True)
            p.pc = "UHpad"
            return f"WLpad({me})"
        if pc == "UHpad":
            # Step 7 for the PAD entry: P_b + (R - P_b) = R is not < R, so the
            # formula of PAPER.md:731-739 wraps P_b to 0.
            new_b = adv(L, p.p_b, L.R - p.p_b)
            assert new_b == 0
            p.p_b, p.p_q = new_b, seq_next(p.p_q)
            mem.tail = pack(p.p_b, p.p_q)
            self._decide(p)
            return f"UHpad({me})"
        if pc == "WB":
            # Step 5: "Write the data into the buffer region starting at the
            # buffer tail position".
            msg = p.msgs[p.k]
            self._claim_units(p.p_b, p.f, (me, p.k))
            if L.hdr:
                h = encode_header(msg.uid, msg.accepted_at, msg.app_id, msg.stage, msg.length,
                                  me, p.k, msg.epoch, 0, 0)[: L.hdr]
                mem.data[p.p_b: p.p_b + L.hdr] = h
            mem.data[p.p_b + L.hdr: p.p_b + L.hdr + msg.length] = msg.payload
            p.pc = "WL"
            return f"WB({me})"
        if pc == "WL":
            # Step 6: "Write the data size into the size region at the size tail
            # position and set the busy bit".
            s = p.p_q % L.N
            if mem.slots[s] != 0:
                raise ProtocolViolation(f"WL on busy slot {s}")
            mem.slots[s] = slot_word(p.f)
            p.pc = "UH"
            return f"WL({me})"
        if pc == "UH":
            # Step 7: "Update the tail position in the header",
            # with both pointer formulas.
            p.p_b, p.p_q = adv(L, p.p_b, p.f), seq_next(p.p_q)
            mem.tail = pack(p.p_b, p.p_q)
            p.outcomes.append("OK")
            if p.mpsc:
                p.pc = "Unlock"
            else:
                self._next_msg(p)
            return f"UH({me})"
        if pc == "Unlock":
            # Step 8: "Release the lock".
            assert mem.lock == me + 1
            mem.lock = 0
            self._next_msg(p)
            return f"Unlock({me})"
        if pc == "UnlockFull":
            assert mem.lock == me + 1
            mem.lock = 0
            self._after_full(p)
            return f"Unlock({me})"
        if pc == "RH":
            # Waiting for credit saw the head move: start the append over.
            p.pc = p._first_pc()
            return f"RH({me})"
        raise RuntimeError(f"producer {me} stuck in {pc}")

    def _claim_units(self, start: int, f: int, tag) -> None:
        a = self.L.align
        for u in range(start // a, (start + f) // a):
            if self.mem.owner[u] is not None:
                raise ProtocolViolation(
                    f"write of {tag} over unreleased entry {self.mem.owner[u]} at unit {u}")
            self.mem.owner[u] = tag

    def _free_units(self, start: int, f: int) -> None:
        a = self.L.align
        for u in range(start // a, (start + f) // a):
            self.mem.owner[u] = None

    # -- receiver ---------------------------------------------------------------------
    def _get(self) -> str:
        """Receiver steps 1-3 plus the checksum check
        (PAPER.md:768-769).  A PAD entry is stepped over using its size slot,
        as the paper's consumer "skips invalid entries and proceeds using size
        metadata"; if nothing is held it is released at once so
        that the producer waiting on it can proceed (reading R3)."""
        L, mem, c = self.L, self.mem, self.cons
        w = mem.slots[c.g_q % L.N]
        if not (w & BUSY):
            raise ProtocolViolation(f"published slot {c.g_q % L.N} not busy")
        f = w & FMASK
        if w & PADBIT:
            if c.g_b + f != L.R:
                raise ProtocolViolation("PAD does not end at R")
            self.pad_events.append((c.g_q, c.g_b, f))
            c.held.append((c.g_q, f, True))
            c.g_b, c.g_q = adv(L, c.g_b, f), seq_next(c.g_q)
            if c.n_held_msgs() == 0:
                self._release_front()
            return "RL(Z)"
        start = c.g_b
        if L.hdr:
            h = bytes(mem.data[start: start + L.hdr])
            d = decode_header(h)
            ok = d["crc_ok"] and L.hdr + d["payload_len"] <= f
            length = d["payload_len"] if ok else 0
        else:
            h = b""
            ok, length = True, f
        payload = bytes(mem.data[start + L.hdr: start + L.hdr + length])
        d = Delivered(start, f, c.g_q, "OK" if ok else "CORRUPT", h, payload)
        c.delivered.append(d)
        if self.check and ok:
            self._check_order(d)
        c.held.append((c.g_q, f, False))
        c.g_b, c.g_q = adv(L, c.g_b, f), seq_next(c.g_q)
        return "RB(Z)"

    def _ident(self, d: Delivered) -> tuple[int, int]:
        if self.L.hdr:
            hd = decode_header(d.header)
            return hd["producer_id"], hd["seq"]
        return tag_ident(d.payload)

    def _check_order(self, d: Delivered) -> None:
        """Exactly-once, in-order, byte-exact delivery per channel (the plain
        definition, DESIGN.md c-1), checked at every receive."""
        pid, k = self._ident(d)
        if pid not in self.programs or not (0 <= k < len(self.programs[pid])):
            raise ProtocolViolation(f"delivered unknown message {pid}/{k}")
        last = self.last_k[pid]
        outs = self.producers[pid].outcomes
        if k <= last or any(j >= len(outs) or outs[j] != "FULL" for j in range(last + 1, k)):
            raise ProtocolViolation(f"channel {pid}: got {k} after {last}")
        if d.payload != bytes(self.programs[pid][k].payload):
            raise ProtocolViolation(f"channel {pid}: payload of {k} differs")
        self.last_k[pid] = k

    def _release_front(self) -> None:
        """Receiver steps 4-5 for the oldest held entry:
        "Reset the busy bit in the size region", then "Update the head
        position" with the pointer formulas."""
        L, mem, c = self.L, self.mem, self.cons
        q, f, _ = c.held.pop(0)
        h_b, h_q = unpack(mem.head)
        assert h_q == q, (h_q, q)
        s = q % L.N
        assert mem.slots[s] & BUSY
        mem.slots[s] = 0
        self._free_units(h_b, f)
        mem.head = pack(adv(L, h_b, f), seq_next(h_q))

    def _release(self) -> str:
        # Release the oldest held message and any PAD entries the read cursor
        # has already passed behind it (reading R13: in-order release).
        c = self.cons
        while c.held and c.held[0][2]:
            self._release_front()
        self._release_front()
        while c.held and c.held[0][2]:
            self._release_front()
        return "REL(Z)"

    # -- invariants (checked after every action when check=True) -----------------------
    def _check_invariants(self) -> None:
        L, mem = self.L, self.mem
        t_b, t_q = unpack(mem.tail)
        h_b, h_q = unpack(mem.head)
        n_live = used_slots(t_q, h_q)
        if n_live > L.N:
            raise ProtocolViolation("more live slots than N")
        # Every slot in [H_seq, P_seq) is busy; every other slot is clear, except
        # a slot written (WL) but not yet published (UH) by a sender.
        live_bytes = 0
        for i in range(n_live):
            w = mem.slots[(h_q + i) % L.N]
            if not (w & BUSY):
                raise ProtocolViolation(f"live slot {(h_q + i) % L.N} not busy")
            live_bytes += w & FMASK
        # The live entries tile the cyclic range [H_b, P_b) exactly (pointer
        # formulas + PAD entries leave no unaccounted bytes).
        if n_live == 0:
            expect = 0
            if (t_b, t_q) != (h_b, h_q):
                raise ProtocolViolation("empty ring but head != tail")
        elif t_b == h_b:
            expect = L.R
        else:
            expect = (t_b - h_b) % L.R
        if live_bytes != expect:
            raise ProtocolViolation(f"live bytes {live_bytes} != cyclic distance {expect}")


def tag_msg(pid: int, k: int, length: int) -> Msg:
    """Header-less test message (byte-level layouts, hdr=0): every payload byte
    is the tag 1 + 16*pid + k, so any overwrite or misplacement is visible."""
    assert pid < 15 and k < 16
    return Msg(length, bytes([1 + 16 * pid + k]) * length)


def tag_ident(payload: bytes) -> tuple[int, int]:
    t = payload[0] - 1
    return t // 16, t % 16


# ----------------------------------------------------------------------------
# Drivers
# ----------------------------------------------------------------------------

def run(sim: Sim, policy: str = "rr", seed: int = 0, max_steps: int = 10_000_000) -> Sim:
    """Drive `sim` to quiescence.  policy 'rr' = round-robin over enabled
    actors, 'random' = seeded uniform choice, 'drain' = consumer whenever
    possible.  Raises on deadlock (a non-terminal state with nothing enabled)."""
    import random
    rng = random.Random(seed)
    i = 0
    for _ in range(max_steps):
        if sim.done():
            return sim
        acts = sim.enabled()
        if not acts:
            raise ProtocolViolation("deadlock: nothing enabled; log tail " + " ".join(sim.log[-12:]))
        if policy == "rr":
            a = acts[i % len(acts)]
            i += 1
        elif policy == "random":
            a = rng.choice(acts)
        elif policy == "drain":
            a = "Z" if "Z" in acts else ("Zrel" if "Zrel" in acts else acts[0])
        else:
            raise ValueError(policy)
        sim.step(a)
    raise ProtocolViolation("step budget exhausted")


def fifo_definition(programs: dict[int, list[Msg]]) -> dict[int, list[bytes]]:
    """The plain definition the ring must reach: for every
    channel, the delivered payloads equal the put payloads, exactly once, in
    put order (fault-free runs; "if a producer writes data
    starting at address R, the consumer will eventually read that same data")."""
    return {pid: [bytes(m.payload) for m in msgs] for pid, msgs in programs.items()}


def delivered_by_channel(sim: Sim) -> dict[int, list[tuple[int, bytes]]]:
    """Group the consumer's delivered entries by header producer id."""
    out: dict[int, list[tuple[int, bytes]]] = {}
    for d in sim.cons.delivered:
        hd = decode_header(d.header)
        out.setdefault(hd["producer_id"], []).append((hd["seq"], d.payload))
    return out


def spsc_image(L: Layout, lengths: list[int], consumed: int | None = None) -> dict:
    """Oracle prediction for a single-producer BLOCK stream: run the stepper with
    a draining consumer and report, per size-region sequence number, the entry
    (start, footprint, pad) the consumer saw.  Placement is a pure function of
    the length sequence (the head only decides *when* a sender proceeds, never
    *where*: PAPER.md:731-745 move P_b by sizes alone)."""
    msgs = [Msg(n, bytes(n)) for n in lengths]
    sim = Sim(L, {0: msgs}, mpsc=False, block=True, depth=1, check=False)
    run(sim, policy="drain")
    ents = []
    pads = {q: (s, f) for q, s, f in sim.pad_events}
    di = iter(sim.cons.delivered)
    total = len(lengths) + len(pads)
    q = 0
    for _ in range(total):
        if q in pads:
            s, f = pads[q]
            ents.append((q, s, f, True))
        else:
            d = next(di)
            assert d.seq_slot == q
            ents.append((q, d.start, d.f, False))
        q = seq_next(q)
    return dict(entries=ents, tail=sim.mem.tail, head=sim.mem.head)
