"""Exhaustive interleaving search on tiny rings (TEST INFRASTRUCTURE ONLY).

BASELINE.json configs[0]: "brute-force interleavings on a 2-slot ring"; the
north star asks for deadlock-freedom "brute-forced over all producer/consumer
interleavings on rings of 2 to 4 slots".  This module enumerates every
interleaving of the labelled atomic actions of `oracle.ring.Sim`
 by depth-first search with a visited-state set and checks,
in every reachable state:
  * no write (WB, or a PAD entry) lands on bytes of an unreleased entry
    (data written at R is read from R);
  * every slot in [H_seq, P_seq) is busy and the live entries tile [H_b, P_b)
    exactly (pointer formulas; busy bit);
  * each delivery is the next message of its channel, byte-exact;
and at the leaves:
  * deadlock freedom: every non-terminal state has an enabled action
    (the consumer is never blocked, producers wait only on
    conflict);
  * terminal states have delivered every message exactly once (BLOCK mode).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

from .ring import Layout, Sim, ProtocolViolation, tag_msg


@dataclass
class Result:
    states: int = 0
    terminals: int = 0
    deadlocks: list = field(default_factory=list)
    violations: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.deadlocks and not self.violations


def explore(L: Layout, programs: dict, mpsc: bool | None = None, block: bool = True,
            depth: int = 1, max_states: int = 2_000_000) -> Result:
    res = Result()
    root = Sim(L, programs, mpsc=mpsc, block=block, depth=depth, check=True)
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
            if block:
                for pid, msgs in programs.items():
                    if s.last_k[pid] != len(msgs) - 1:
                        res.violations.append(("incomplete", pid, s.last_k[pid], s.log))
            continue
        acts = s.enabled()
        if not acts:
            res.deadlocks.append(list(s.log))
            continue
        for a in acts:
            c = s.clone()
            try:
                c.step(a)
            except AssertionError as e:   # ProtocolViolation and internal asserts
                res.violations.append((str(e), list(c.log)))
                continue
            stack.append(c)
    return res


def byte_programs(sizes_per_producer: list[list[int]]) -> dict:
    """Header-less tagged messages for byte-level rings (align=1, hdr=0)."""
    return {pid: [tag_msg(pid, k, n) for k, n in enumerate(sizes)]
            for pid, sizes in enumerate(sizes_per_producer)}


def sweep(N_values=(2, 3, 4), R_values=(2, 3, 4, 5, 6), shapes=((3,), (2, 1), (2, 2)),
          depths=(1, 2), block=True, size_cap=None):
    """Run `explore` over every ring geometry, producer/message shape and
    footprint combination (footprints 1..R units cover exact fit, f = R and the
    PAD path).  Yields (config, Result)."""
    for N in N_values:
        for R in R_values:
            L = Layout(R, N, align=1, hdr=0)
            top = R if size_cap is None else min(R, size_cap)
            for shape in shapes:
                total = sum(shape)
                for combo in itertools.product(range(1, top + 1), repeat=total):
                    it = iter(combo)
                    sizes = [[next(it) for _ in range(m)] for m in shape]
                    for d in depths:
                        cfg = dict(N=N, R=R, sizes=sizes, depth=d, block=block)
                        yield cfg, explore(L, byte_programs(sizes), block=block, depth=d)
