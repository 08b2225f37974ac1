"""Multi-GPU wiring of double rings, one process per GPU (host plumbing only).

Every hop between two stages is one ring owned by the consuming GPU
(the queue and its consumer are co-located).  This module
decides which rings each rank creates, which rings it attaches to as a
producer (and with which producer id), and whose head mirrors it binds, for
the BASELINE.json topologies, and performs the handle exchange over a
torch.distributed group (an all_gather of 256-byte handles -- the RDMA
queue-pair / registered-address setup of PAPER.md:637-641; never on the data
path).  The ring calls are injected, so the wiring itself is testable on CPU
with a gloo group.

Topologies
  pairs     rank r -> ring on rank (r+1) % N (every GPU one egress + one ingress
            stream; C3-shaped traffic, weak scaling)
  pipeline  stage s on rank s -> ring on rank s+1; the last stage -> a sink ring
            on rank 0 (C4: text-encoder -> VAE-encode -> DiT -> VAE-decode -> sink)
  fanin     ranks 1..N-1 -> one shared MPSC ring on rank 0 (C5); with
            `spare_consumer`, rank N-1 also owns a second ring that producers
            1..N-2 attach to, for the mid-stream reassignment (C5b)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable


@dataclass(frozen=True)
class RingSpec:
    name: str
    owner: int
    data_bytes: int
    n_slots: int
    max_producers: int = 1
    flags: int = 0         # ring_create flags (e.g. reserve-then-commit)


@dataclass(frozen=True)
class Attach:
    producer: int       # rank
    ring: str           # RingSpec.name
    producer_id: int    # unique per ring, < max_producers


@dataclass
class Wiring:
    rings: list[RingSpec] = field(default_factory=list)
    attach: list[Attach] = field(default_factory=list)

    def validate(self, world: int) -> None:
        names = {r.name: r for r in self.rings}
        assert len(names) == len(self.rings), "ring names must be unique"
        for r in self.rings:
            assert 0 <= r.owner < world and r.max_producers >= 1
        seen = set()
        for a in self.attach:
            assert a.ring in names, a
            assert 0 <= a.producer < world, a
            assert 0 <= a.producer_id < names[a.ring].max_producers, a
            assert (a.ring, a.producer_id) not in seen, a
            seen.add((a.ring, a.producer_id))


def plan_pairs(world: int, data_bytes: int = 64 << 20, n_slots: int = 64) -> Wiring:
    w = Wiring()
    for r in range(world):
        w.rings.append(RingSpec(f"in{r}", r, data_bytes, n_slots, 1))
    for r in range(world):
        w.attach.append(Attach(r, f"in{(r + 1) % world}", 0))
    return w


def plan_pipeline(world: int, hop_bytes: list[int], hop_slots: list[int]) -> Wiring:
    """Stage s (rank s) feeds rank s+1; the last stage feeds the sink on rank 0.
    `hop_bytes[s]` / `hop_slots[s]` size the ring of hop s (owned by its consumer)."""
    assert world >= 2 and len(hop_bytes) == world and len(hop_slots) == world
    w = Wiring()
    for s in range(world):
        w.rings.append(RingSpec(f"hop{s}", (s + 1) % world, hop_bytes[s], hop_slots[s], 1))
        w.attach.append(Attach(s, f"hop{s}", 0))
    return w


def plan_fanin(world: int, data_bytes: int = 1 << 30, n_slots: int = 256, spare_consumer: bool = False,
               flags: int = 0) -> Wiring:
    assert world >= 2
    w = Wiring()
    w.rings.append(RingSpec("fan0", 0, data_bytes, n_slots, world - 1, flags))
    for p in range(1, world):
        w.attach.append(Attach(p, "fan0", p - 1))
    if spare_consumer and world >= 3:
        spare = world - 1
        w.rings.append(RingSpec("fan1", spare, data_bytes, n_slots, world - 2))
        for p in range(1, spare):
            w.attach.append(Attach(p, "fan1", p - 1))
    return w


def plan_fanin_set(world: int, data_bytes: int = 512 << 20, n_slots: int = 256) -> Wiring:
    """Lock-free fan-in: one single-producer ring per
    producer rank 1..world-1, all owned by rank 0 (served by ring_set_consume)."""
    assert world >= 2
    w = Wiring()
    for p in range(1, world):
        w.rings.append(RingSpec(f"sub{p}", 0, data_bytes, n_slots, 1))
        w.attach.append(Attach(p, f"sub{p}", 0))
    return w


@dataclass
class Wired:
    rings: dict            # name -> ring handle (rings this rank owns)
    peers: dict            # name -> peer handle (rings this rank produces into)
    producer_ids: dict     # name -> producer id used by this rank


def wire(w: Wiring, rank: int, world: int, group, *, device: int,
         create: Callable, export: Callable, attach: Callable, bind: Callable,
         all_gather_object: Callable | None = None) -> Wired:
    """Create / export / attach / bind for this rank.

    create(spec, device) -> ring; export(ring) -> bytes;
    attach(handle_bytes, device, producer_id) -> (peer, mirror_bytes);
    bind(ring, producer_id, mirror_bytes) -> None.
    """
    w.validate(world)
    if all_gather_object is None:
        import torch.distributed as dist

        def all_gather_object(out, obj):
            dist.all_gather_object(out, obj, group=group)
    own = {r.name: create(r, device) for r in w.rings if r.owner == rank}
    mine = {name: export(ring) for name, ring in own.items()}
    handles_by_rank = [None] * world
    all_gather_object(handles_by_rank, mine)
    handles = {k: v for d in handles_by_rank for k, v in d.items()}
    peers, pids, mirrors = {}, {}, {}
    for a in w.attach:
        if a.producer == rank:
            peer, mh = attach(handles[a.ring], device, a.producer_id)
            peers[a.ring] = peer
            pids[a.ring] = a.producer_id
            mirrors[(a.ring, a.producer_id)] = mh
    mirrors_by_rank = [None] * world
    all_gather_object(mirrors_by_rank, mirrors)
    for d in mirrors_by_rank:
        for (ring_name, pid), mh in d.items():
            if ring_name in own:
                bind(own[ring_name], pid, mh)
    return Wired(own, peers, pids)
