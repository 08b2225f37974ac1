"""Helpers for the GPU parity tests: drive the CUDA path through the C ABI and
predict the same run with the oracle.  (Test code: imports both sides; the
product path and the oracle never import each other.)"""
from __future__ import annotations

import numpy as np
import torch

import synth
from synth import device as SD
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


def devices(k: int, cross: bool) -> list[int]:
    """k device ids: distinct GPUs when `cross` (skips the test if there are
    fewer), else all on GPU 0 -- rings created without RING_CREATE_LOCAL then
    take the system-scope (NVLink) kernels with producer and consumer kernels
    spinning concurrently on one GPU."""
    import pytest
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if cross:
        if torch.cuda.device_count() < k:
            pytest.skip(f"needs {k} GPUs")
        return list(range(k))
    return [0] * k


def device_sources(specs, seed: int, device="cuda"):
    """Payload sources generated on the device: specs = [(channel, seq, length)];
    one buffer with 256-B aligned offsets, filled with synth.payload_bytes of
    each (seed, channel, seq).  Returns (buffer, [device addresses])."""
    offs, total = [], 0
    for _, _, n in specs:
        offs.append(total)
        total += (n + 255) // 256 * 256
    buf = torch.empty(max(total, 256), dtype=torch.uint8, device=device)
    ptrs = [buf.data_ptr() + o for o in offs]
    with torch.cuda.device(buf.device):
        keep = SD.fill(ptrs, [n for _, _, n in specs], [c for c, _, _ in specs], [q for _, q, _ in specs], seed)
        torch.cuda.synchronize()
    del keep
    return buf, ptrs


def dev_u64(vals, device="cuda") -> torch.Tensor:
    return torch.tensor([v - 2**64 if v >= 2**63 else v for v in vals], dtype=torch.int64, device=device)


def verify_views(ring, vt: torch.Tensor, n: int, seed: int, chans=None, seqs=None, stream=None, lut=None,
                 lut_stride=0):
    """On-device, exact compare of the payloads that n view records point at
    (inside the ring: view mode, before release) with the seeded generator.
    Keys default to the header's (producer_id, seq) [R11 bytes 44-52]; pass
    device tensors to key otherwise, or a device table `lut` that maps the
    header's (producer_id, seq) to the generator's seq: lut[pid * lut_stride +
    seq].  Only device work on `stream` (no host synchronisation).  Returns the
    device tensor of first-bad offsets (-1 = ok)."""
    base = R.ring_get_info(ring).data
    s = stream if stream is not None else torch.cuda.current_stream(vt.device)
    return SD.verify_views(vt, n, base, seed, chans, seqs, lut, lut_stride, s)


def replay_mpsc(L, progs, order, check=True):
    """Oracle run that follows an observed lock order (R16): only the producer
    whose message is next may step until that message is published; the
    consumer drains whenever it can."""
    sim = Sim(L, progs, mpsc=True, block=True, depth=1, check=check)
    for pid in order:
        p = sim.producers[pid]
        target = len(p.outcomes) + 1
        # until the message is published AND the lock released (Unlock follows UH)
        while len(p.outcomes) < target or p.pc not in ("Lock", "DONE"):
            if sim.producer_enabled(p):
                sim.step(pid)
            elif "Z" in sim.enabled():
                sim.step("Z")
            elif "Zrel" in sim.enabled():
                sim.step("Zrel")
            else:
                raise AssertionError("replay stuck")
    run(sim, policy="drain")
    return sim
