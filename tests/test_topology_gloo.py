"""CPU tests of the multi-GPU wiring (paper_2601_20655_b200/topology.py): the
plans for the BASELINE topologies, and the handle exchange run for real over a
world_size-2 (and 4) gloo process group on 127.0.0.1 with recording fakes in
place of the CUDA calls."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_20655_b200 import topology as T


def test_plans_validate():
    for world in (2, 3, 4, 8):
        T.plan_pairs(world).validate(world)
        T.plan_fanin(world).validate(world)
        T.plan_fanin(world, spare_consumer=True).validate(world)
        T.plan_pipeline(world, [1 << 20] * world, [8] * world).validate(world)


def test_pairs_every_rank_one_egress_one_ingress():
    w = T.plan_pairs(4)
    assert sorted(a.producer for a in w.attach) == [0, 1, 2, 3]
    owners = {r.name: r.owner for r in w.rings}
    assert sorted(owners[a.ring] for a in w.attach) == [0, 1, 2, 3]
    assert all(owners[a.ring] == (a.producer + 1) % 4 for a in w.attach)


def test_fanin_shared_mpsc_ring_and_spare():
    w = T.plan_fanin(8, spare_consumer=True)
    fan0 = [a for a in w.attach if a.ring == "fan0"]
    assert sorted(a.producer for a in fan0) == list(range(1, 8))
    assert sorted(a.producer_id for a in fan0) == list(range(7))
    spec = {r.name: r for r in w.rings}
    assert spec["fan0"].max_producers == 7 and spec["fan0"].owner == 0
    assert spec["fan1"].owner == 7 and sorted(a.producer for a in w.attach if a.ring == "fan1") == list(range(1, 7))


def test_pipeline_chain_and_sink():
    w = T.plan_pipeline(4, [1, 2, 3, 4], [8, 8, 8, 8])
    owners = {r.name: r.owner for r in w.rings}
    assert [(a.producer, owners[a.ring]) for a in w.attach] == [(0, 1), (1, 2), (2, 3), (3, 0)]


def test_validate_rejects_duplicate_producer_ids():
    w = T.Wiring([T.RingSpec("x", 0, 1024, 8, 2)], [T.Attach(0, "x", 0), T.Attach(1, "x", 0)])
    with pytest.raises(AssertionError):
        w.validate(2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    plan = {"pairs": lambda: T.plan_pairs(world),
            "fanin": lambda: T.plan_fanin(world, 1 << 20, 16, spare_consumer=True)}[kind]()

    def create(spec, device):
        calls.append(("create", spec.name, device))
        return ("ring", spec.name)

    def export(ring):
        return f"H:{ring[1]}@{rank}".encode()

    def attach(handle, device, pid):
        calls.append(("attach", handle.decode(), pid))
        return ("peer", handle.decode(), pid), f"M:{handle.decode()}:{pid}@{rank}".encode()

    def bind(ring, pid, mh):
        calls.append(("bind", ring[1], pid, mh.decode()))

    wired = T.wire(plan, rank, world, None, device=rank, create=create, export=export, attach=attach, bind=bind)
    q.put((rank, calls, sorted(wired.rings), sorted(wired.peers)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("pairs", 2), ("fanin", 4)])
def test_wire_over_gloo(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, calls, rings, peers = q.get(timeout=120)
        res[rank] = (calls, rings, peers)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plan = T.plan_pairs(world) if kind == "pairs" else T.plan_fanin(world, 1 << 20, 16, spare_consumer=True)
    owners = {r.name: r.owner for r in plan.rings}
    for a in plan.attach:
        calls = res[a.producer][0]
        # the producer attached with the owner's exported handle and its producer id
        assert ("attach", f"H:{a.ring}@{owners[a.ring]}", a.producer_id) in calls
        # the owner bound exactly that producer's mirror
        mh = f"M:H:{a.ring}@{owners[a.ring]}:{a.producer_id}@{a.producer}"
        assert ("bind", a.ring, a.producer_id, mh) in res[owners[a.ring]][0]
    for rank in range(world):
        assert res[rank][1] == sorted(r.name for r in plan.rings if r.owner == rank)
