"""Diagnostic: reserve-then-commit fan-in on one GPU (K producers on streams)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_20655_b200 import ring as R
R.ring_set_timeout_ns(500_000_000)
K = int(os.environ.get("K", "3")); M = int(os.environ.get("M", "1000")); size = int(os.environ.get("SIZE", "4096"))
N = int(os.environ.get("N", "256")); RB = int(os.environ.get("RB", str(1 << 30)))
flags = R.RING_CREATE_RESERVE_COMMIT if os.environ.get("RC", "1") == "1" else 0
PDEV = int(os.environ.get("PDEV", "0"))
ring = R.ring_create(0, RB, N, K, flags | (R.RING_CREATE_LOCAL if PDEV == 0 else 0))
h = R.ring_export(ring)
peers = []
for p in range(K):
    pe, mh = R.ring_attach_peer(h, PDEV, p); R.ring_bind_mirror(ring, p, mh); peers.append(pe)
torch.cuda.set_device(PDEV)
src = torch.randint(0, 255, (size + 256,), dtype=torch.uint8, device="cuda")
a = R.make_msgs([src.data_ptr()] * M, [size] * M, [bytes(16)] * M, [0] * M, [0] * M, [0] * M)
d = torch.from_numpy(a.view(np.uint8).copy()).cuda()
sts = [torch.full((M,), 10, dtype=torch.int32, device="cuda") for _ in range(K)]
vt = torch.zeros(K * M * 128, dtype=torch.uint8, device="cuda:0")
sc = torch.cuda.Stream(0); ss = [torch.cuda.Stream() for _ in range(K)]
t0 = time.time()
R.ring_consume(ring, K * M, vt, None, 0, 0, sc)
for p in range(K):
    R.ring_put_batch(peers[p], d, M, 0, sts[p], ss[p])
for dd in {0, PDEV}: torch.cuda.synchronize(dd)
print("time", round(time.time() - t0, 3))
for p in range(K):
    s = sts[p].cpu().numpy(); print("producer", p, {int(k): int(v) for k, v in zip(*np.unique(s, return_counts=True))})
v = R.parse_views(vt.cpu().numpy())
print("views", {int(k): int(c) for k, c in zip(*np.unique(v["status"], return_counts=True))})
print("image", {k: (hex(x) if isinstance(x, int) else None) for k, x in R.ring_read_image(ring).items() if k != "slots"})
sl = R.ring_read_image(ring)["slots"]
print("slots nonzero", [(i, hex(w)) for i, w in enumerate(sl) if w][:12])

if os.environ.get("B200RING_TRACE"):
    for p in range(K):
        t = R.ring_peer_trace(peers[p])
        for half in (t[:2048], t[2048:]):
            print("peer", p, "takeovers", int(half[1890]), "holes", int(half[1891]), "commit fails", int(half[1892]),
                  "slot", hex(int(half[1893])), "want", hex(int(half[1894])))
