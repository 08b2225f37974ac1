"""Theorem-1 sizing and fast reject driving the stage router (
PAPER.md:556-614).  CPU part: the library's ring_required_instances (host
arithmetic) equals the oracle's Theorem-1 formula.  GPU part: a route sized by
router_size_route for the paper's second pipeline figure (T_X = 4, T_Y = 12,
K = 2 -> M = 6 instances of Y) admits requests by their proxy timestamps
exactly as the oracle's burst-1 token bucket does, never sends a rejected one,
and spreads the admitted ones round robin over the six rings in order."""
import random

import numpy as np
import pytest

import synth
from oracle.pipeline import fast_reject, required_instances
from oracle.ring import decode_header


def test_required_instances_matches_theorem1():
    from paper_2601_20655_b200 import ring as R
    rng = random.Random(11)
    cases = [(4, 12, 1), (4, 12, 2), (5, 5, 1), (4, 10, 3), (1, 1 << 40, 7)]
    cases += [(rng.randint(1, 10**9), rng.randint(1, 10**10), rng.randint(1, 64)) for _ in range(500)]
    for t_x, t_y, k in cases:
        assert R.ring_required_instances(t_x, t_y, k) == required_instances(t_x, t_y, k)
    assert R.ring_required_instances(0, 5, 1) == 0 and R.ring_required_instances(5, 5, 0) == 0


@pytest.mark.gpu
def test_sized_route_admission_and_round_robin():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring as R
    from gpu_util import upload, msg_tensor, views_host
    T_X, T_Y, K = 4000, 12000, 2                  # the paper's figure, in microseconds -> ns-like units
    M = required_instances(T_X, T_Y, K)
    assert M == 6
    rings, peers = [], []
    for _ in range(7):                            # a pool of 7 instances; Theorem 1 uses 6
        r = R.ring_create(0, 1 << 20, 64, 1, R.RING_CREATE_LOCAL)
        pe, mh = R.ring_attach_peer(R.ring_export(r), 0, 0)
        R.ring_bind_mirror(r, 0, mh)
        rings.append(r)
        peers.append(pe)
    router = R.router_create(0, 8)
    assert R.router_size_route(router, 9, 3, T_X, T_Y, K, peers) == M
    n = 60
    stream = synth.random_stream(synth.SEED_BASE + 50, 0, n, 1, 3000, app_id=9, stage=3)
    rng = np.random.Generator(np.random.PCG64(synth.SEED_BASE + 50))
    arrivals = np.cumsum(rng.integers(0, 3500, n)).tolist()        # bursts and gaps around T_X/K = 2000
    for m, t in zip(stream, arrivals):
        m.accepted_at = int(t)
    buf, srcs = upload(stream, "cuda:0")
    msgs = msg_tensor(stream, srcs, "cuda:0")
    st = torch.full((n,), 10, dtype=torch.int32, device="cuda:0")
    dest = torch.full((n,), 99, dtype=torch.int32, device="cuda:0")
    R.ring_put_routed(router, msgs, n, 0, st, dest)
    torch.cuda.synchronize()
    admit = fast_reject(arrivals, T_X, K)
    assert 5 < sum(admit) < n                     # the stream exercises both outcomes
    stv = [int(x) for x in st.cpu().tolist()]
    assert stv == [0 if a else R.RING_EREJECTED for a in admit]
    dv = [int(x) for x in dest.cpu().tolist()]
    accepted = [i for i in range(n) if admit[i]]
    assert [dv[i] for i in accepted] == [j % M for j in range(len(accepted))]
    for j in range(M + 1):
        want = accepted[j::M] if j < M else []
        vt = torch.zeros(max(len(want), 1) * 128, dtype=torch.uint8, device="cuda:0")
        R.ring_consume(rings[j], max(len(want), 1), vt, None, 0, R.RING_TRY)
        torch.cuda.synchronize()
        v = views_host(vt)
        if not want:
            assert v[0]["status"] == R.RING_EMPTY          # the 7th instance is not used
            continue
        hs = [decode_header(bytes(x["header"])) for x in v]
        assert all(x["status"] == 0 for x in v)
        assert [h["uid"] for h in hs] == [stream[i].uid for i in want]
        assert [h["accepted_at"] for h in hs] == [arrivals[i] for i in want]
        assert [h["seq"] for h in hs] == list(range(len(want)))     # rejected requests take no channel seq
        for x, i in zip(v, want):
            assert R.ring_read_data(rings[j], int(x["offset"]), int(x["len"])) == stream[i].payload.tobytes()
    R.router_destroy(router)
    for pe in peers:
        R.ring_detach(pe)
    for r in rings:
        R.ring_destroy(r)
