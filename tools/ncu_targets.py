"""Kernels to capture with ncu (not a test; ncu serialises kernels, so every
launch here runs to completion without waiting on another kernel):

  nvlink   GPU0 -> a 1 GiB / 256-slot ring on GPU1: 6 put launches of 32 x
           4,194,304 B (put_kernel<2>, the NVLink instance; the ring holds all
           of them, so no credit wait), then one copy-out consume of the last
           launch's 32 entries on GPU1 (get_kernel<true>).
  split    BASELINE.json configs[2] one way with the split placement: a 256 MiB /
           64-slot ring whose buffer region is on GPU0 and control words on
           GPU1; 63 Wan2.1 tensors (4,194,304 / 4,193,280 B alternating) put
           locally on GPU0, then one copy-out consume on GPU1 pulls them over
           NVLink (get_kernel<true>, line-aligned remote loads).
  copyout  C2 ring (64 MiB, 64 slots) on one GPU: put 64 x 1,048,512 B, then
           a copy-out consume of them (get_kernel<false>, the default grid);
           3 rounds.

  ncu --set full -k regex:put_kernel -s 3 -c 1 -o ... python tools/ncu_targets.py nvlink
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_20655_b200 import ring as R  # noqa: E402


def msgs(src, size, m, device):
    a = R.make_msgs([src.data_ptr() + (q * size) % (src.numel() - size) // 256 * 256 for q in range(m)], [size] * m,
                    [bytes(16)] * m, [0] * m, [7] * m, [2] * m)
    return torch.from_numpy(a.view(np.uint8).copy()).to(device)


def nvlink():
    ring = R.ring_create(1, 1 << 30, 256, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    if os.environ.get("PUT_CFG"):       # ctas:threads:copy_mode, e.g. 17:0:1 = the TMA engine on 17 SMs
        R.ring_peer_config(peer, *(int(x) for x in os.environ["PUT_CFG"].split(":")))
    m, size = 32, 4194304
    src = torch.randint(0, 255, (256 << 20,), dtype=torch.uint8, device="cuda:0")
    d = msgs(src, size, m, "cuda:0")
    st = torch.zeros(m, dtype=torch.int32, device="cuda:0")
    for _ in range(6):
        R.ring_put_batch(peer, d, m, 0, st)
        torch.cuda.synchronize(0)
        assert (st == 0).all().item()
    vt = torch.zeros(6 * m * 128, dtype=torch.uint8, device="cuda:1")
    dst = torch.empty(6 * m * size, dtype=torch.uint8, device="cuda:1")
    with torch.cuda.device(1):
        R.ring_consume(ring, 6 * m, vt, dst, size, 0)
        torch.cuda.synchronize(1)
    assert (R.parse_views(vt.cpu().numpy())["status"] == 0).all()
    R.ring_detach(peer)
    R.ring_destroy(ring)


def split():
    ring = R.ring_create_split(1, 0, 256 << 20, 64, 1, 0)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    m = 63
    lens = [4194304 if q % 2 == 0 else 4193280 for q in range(m)]
    src = torch.randint(0, 255, (m * 4194304,), dtype=torch.uint8, device="cuda:0")
    a = R.make_msgs([src.data_ptr() + q * 4194304 for q in range(m)], lens, [bytes(16)] * m, [0] * m, [7] * m,
                    [2] * m)
    d = torch.from_numpy(a.view(np.uint8).copy()).to("cuda:0")
    st = torch.zeros(m, dtype=torch.int32, device="cuda:0")
    vt = torch.zeros(m * 128, dtype=torch.uint8, device="cuda:1")
    dst = torch.empty(m * 4194304, dtype=torch.uint8, device="cuda:1")
    for _ in range(3):
        R.ring_put_batch(peer, d, m, 0, st)
        torch.cuda.synchronize(0)
        assert (st == 0).all().item()
        with torch.cuda.device(1):
            R.ring_consume(ring, m, vt, dst, 4194304, 0)
            torch.cuda.synchronize(1)
        assert (R.parse_views(vt.cpu().numpy())["status"] == 0).all()
    assert torch.equal(dst.view(-1)[: lens[0]].cpu(), src[: lens[0]].cpu())
    R.ring_detach(peer)
    R.ring_destroy(ring)


def copyout():
    ring = R.ring_create(0, 64 << 20, 64, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
    R.ring_bind_mirror(ring, 0, mh)
    m, size = 64, 1048512
    src = torch.randint(0, 255, (256 << 20,), dtype=torch.uint8, device="cuda:0")
    d = msgs(src, size, m, "cuda:0")
    st = torch.zeros(m, dtype=torch.int32, device="cuda:0")
    vt = torch.zeros(m * 128, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(m * size, dtype=torch.uint8, device="cuda:0")
    for _ in range(3):
        R.ring_put_batch(peer, d, m, 0, st)
        R.ring_consume(ring, m, vt, dst, size, 0)
        torch.cuda.synchronize()
        assert (st == 0).all().item()
        assert (R.parse_views(vt.cpu().numpy())["status"] == 0).all()
    R.ring_detach(peer)
    R.ring_destroy(ring)


if __name__ == "__main__":
    R.ring_set_timeout_ns(20_000_000_000)
    {"nvlink": nvlink, "split": split, "copyout": copyout}[sys.argv[1]]()
    print("ncu_targets", sys.argv[1], "ok", flush=True)
