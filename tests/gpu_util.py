"""Helpers for the GPU parity tests: drive the CUDA path through the C ABI and
predict the same run with the oracle.  (Test code: imports both sides; the
product path and the oracle never import each other.)"""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle.ring import Layout, Sim, Msg, run, encode_header, decode_header
from paper_2601_20655_b200 import ring as R


def to_oracle_msgs(stream) -> list[Msg]:
    return [Msg(m.length, m.payload.tobytes(), m.uid, m.accepted_at, m.app_id, m.stage) for m in stream]


def oracle_spsc(L: Layout, msgs: list[Msg], producer_id: int = 0, depth: int = 1) -> Sim:
    """The oracle's run of one producer's stream, BLOCK mode, draining consumer."""
    sim = Sim(L, {producer_id: msgs}, mpsc=False, block=True, depth=depth)
    run(sim, policy="drain")
    return sim


def upload(stream, device) -> tuple[torch.Tensor, list[int]]:
    """Concatenate payloads into one device buffer (256-B aligned offsets)."""
    offs, total = [], 0
    for m in stream:
        offs.append(total)
        total += (m.length + 255) // 256 * 256
    host = np.zeros(max(total, 256), dtype=np.uint8)
    for m, o in zip(stream, offs):
        host[o:o + m.length] = m.payload
    buf = torch.from_numpy(host).to(device)
    base = buf.data_ptr()
    return buf, [base + o for o in offs]


def msg_tensor(stream, srcs, device) -> torch.Tensor:
    a = R.make_msgs(srcs, [m.length for m in stream], [m.uid for m in stream], [m.accepted_at for m in stream],
                    [m.app_id for m in stream], [m.stage for m in stream])
    return torch.from_numpy(a.view(np.uint8).copy()).to(device)


def batches(stream, L: Layout, max_batch: int = 10**9):
    """Split a stream into batches that a ring with everything consumed can
    absorb without waiting for credit: count + 1 (a PAD) <= N and
    sum(f) + max(f) <= R (at most one wrap).  Lets one GPU run put then get in
    stream order without two kernels spinning on each other."""
    out, cur, fsum, fmax = [], [], 0, 0
    for i, m in enumerate(stream):
        f = R.ring_footprint(m.length)
        if cur and (len(cur) + 2 > L.N or fsum + f + max(fmax, f) > L.R or len(cur) >= max_batch):
            out.append(cur)
            cur, fsum, fmax = [], 0, 0
        cur.append(i)
        fsum += f
        fmax = max(fmax, f)
    if cur:
        out.append(cur)
    return out


def views_host(t: torch.Tensor) -> np.ndarray:
    return R.parse_views(t.cpu().numpy())


def expected_header(m, producer_id: int, seq: int, epoch: int = 0) -> bytes:
    return encode_header(m.uid, m.accepted_at, m.app_id, m.stage, m.length, producer_id, seq, epoch, 0, 0)[:56]


def check_views_against_oracle(views: np.ndarray, sim: Sim, first: int, stream, producer_id: int = 0):
    """Views [first, first+len(views)) against the oracle's delivered entries."""
    for j, v in enumerate(views):
        d = sim.cons.delivered[first + j]
        m = stream[first + j]
        assert R.STATUS_NAMES[int(v["status"])] == "OK", (first + j, int(v["status"]))
        assert (int(v["start"]), int(v["footprint"]), int(v["slot_seq"])) == (d.start, d.f, d.seq_slot), \
            (first + j, int(v["start"]), d.start)
        hdr = bytes(v["header"])
        assert hdr[:56] == expected_header(m, producer_id, first + j), first + j
        assert hdr[:56] == d.header[:56]
        assert int(v["len"]) == m.length
        assert int(v["offset"]) == d.start + 64
