"""Fused device-side put: a stage kernel computes
out = bf16(in * scale) and its threads write the result straight into the peer
ring, publishing it themselves (csrc/ring_stage.cuh).  Checked against plain
PyTorch CPU for the payload (the same fp32 product rounded to nearest even) and
the oracle for placement (start, footprint, PAD entries at the wraps), header
fields and per-channel sequence — mixed with ordinary ring_put_batch launches
on the same attachment, on one GPU and across NVLink."""
import numpy as np
import pytest

import synth
from oracle.ring import Layout, decode_header, spsc_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_20655_b200 import ring
    ring.ring_set_timeout_ns(2_000_000_000)
    return ring


def _bf16_input(k, n, dev):
    g = torch.Generator().manual_seed(synth.SEED_BASE + 60 + k)
    return torch.randn(n + 1, generator=g).to(torch.bfloat16).to(dev)


@pytest.mark.parametrize("ring_dev", [0, 1])
def test_fused_stage_put_matches_cpu_and_oracle(R, ring_dev):
    if ring_dev >= torch.cuda.device_count():
        pytest.skip("needs 2 GPUs")
    L = Layout(1 << 20, 16)
    flags = R.RING_CREATE_LOCAL if ring_dev == 0 else R.RING_CREATE_DEFAULT
    ring = R.ring_create(ring_dev, L.R, L.N, 1, flags)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    view = R.ring_peer_device_view(peer)
    assert view["sys"] == (1 if ring_dev else 0) and view["N"] == L.N
    # alternate fused stage puts (even k) and ordinary batch puts (odd k);
    # element counts exercise ragged tails, an unaligned input and the wraps
    counts = [100_000, 3, 131_000, 77_777, 250_000, 1, 40_000, 262_000, 9, 150_000]
    lengths = [2 * n for n in counts]
    scales = [0.5, 1.75, -3.0, 1.0, 0.125, 2.0, -0.75, 1.5, 4.0, 0.3]
    st = torch.full((len(counts),), 10, dtype=torch.int32, device="cuda:0")
    expect_payload, keep = [], []
    s = torch.cuda.Stream(0)
    views = torch.zeros(8 * 128, dtype=torch.uint8, device=f"cuda:{ring_dev}")
    got = []
    for k, (n, sc) in enumerate(zip(counts, scales)):
        x = _bf16_input(k, n, "cuda:0")
        xin = x[1:] if k == 4 else x[:n]                         # k = 4: a 2-byte-aligned input
        ref = (xin.cpu().float() * sc).to(torch.bfloat16)
        expect_payload.append(ref.view(torch.uint8).numpy().tobytes())
        uid = bytes([k] * 16)
        if k % 2 == 0:
            R.ring_stage_scale_bf16_put(peer, xin, n, sc, uid, 1000 + k, 5, 2, 0, st[k:k + 1], s)
        else:
            y = (xin.float() * sc).to(torch.bfloat16)            # the unfused path: compute, then put
            keep.append(y)
            a = R.make_msgs([y.data_ptr()], [2 * n], [uid], [1000 + k], [5], [2])
            d = torch.from_numpy(a.view(np.uint8).copy()).cuda(0)
            keep.append(d)
            R.ring_put_batch(peer, d, 1, 0, st[k:k + 1], s)
        keep.append(x)
        s.synchronize()
        R.ring_consume(ring, 1, views, None, 0, R.RING_TRY)     # the ring holds few of these at once
        torch.cuda.synchronize(ring_dev)
        got.append(R.parse_views(views[:128].cpu().numpy())[0].copy())
        ent = got[-1]
        assert ent["status"] == 0, (k, ent["status"])
        assert R.ring_read_data(ring, int(ent["offset"]), int(ent["len"])) == expect_payload[k], k
    assert st.cpu().tolist() == [0] * len(counts)
    img = spsc_image(L, lengths)
    ents = [e for e in img["entries"] if not e[3]] if isinstance(img, dict) and "entries" in img else None
    for k, ent in enumerate(got):
        h = decode_header(bytes(ent["header"]))
        assert (h["seq"], h["payload_len"], h["uid"], h["accepted_at"], h["app_id"], h["stage"]) == \
            (k, lengths[k], bytes([k] * 16), 1000 + k, 5, 2)
        assert h["crc_ok"]
        assert int(ent["footprint"]) == ((64 + lengths[k] + 127) // 128) * 128
        if ents is not None:
            assert (int(ent["slot_seq"]), int(ent["start"]), int(ent["footprint"])) == tuple(ents[k][:3])
    R.ring_detach(peer)
    R.ring_destroy(ring)
