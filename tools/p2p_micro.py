"""Micro-benchmark (not a test): one-direction P2P streaming GPU0 -> ring on
GPU1 in one process, for grid sizes / copy engines / message sizes.  Each case:
`steps` launch pairs (consume on GPU1 first, put on GPU0) of `m` messages."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_20655_b200 import ring as R

R.ring_set_timeout_ns(3_000_000_000)
ring = R.ring_create(1, int(os.environ.get("RB", str(64 << 20))), int(os.environ.get("N", "64")), 1, 0)
peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
R.ring_bind_mirror(ring, 0, mh)
src = torch.randint(0, 255, (160 << 20,), dtype=torch.uint8, device="cuda:0")
sp, sc = torch.cuda.Stream(0), torch.cuda.Stream(1)
vw = torch.zeros(64 * 128, dtype=torch.uint8, device="cuda:1")
st = torch.zeros(64, dtype=torch.int32, device="cuda:0")
sizes = [int(x) for x in os.environ.get("SIZES", str(4194304)).split(",")]
cfgs = [tuple(int(v) for v in c.split(":")) for c in os.environ.get("CFGS", "33:0,65:0,129:0,17:1,33:1,65:1").split(",")]
steps = int(os.environ.get("STEPS", "20"))
for size in sizes:
    m = max(1, min(32, (128 << 20) // size))
    a = R.make_msgs([src.data_ptr() + (q * size) % (96 << 20) // 256 * 256 for q in range(m)], [size] * m,
                    [bytes(16)] * m, [0] * m, [7] * m, [2] * m)
    d = torch.from_numpy(a.view(np.uint8).copy()).cuda(0)
    for ctas, mode in cfgs:
        R.ring_peer_config(peer, ctas, 512, mode)
        for rep in range(2):
            torch.cuda.synchronize(0); torch.cuda.synchronize(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(1):
                e0.record(sc)
            if os.environ.get("ONE_CONSUME"):          # one consumer launch for every step's messages
                vall = torch.zeros(m * steps * 128, dtype=torch.uint8, device="cuda:1")
                R.ring_consume(ring, m * steps, vall, None, 0, 0, sc)
            for s in range(steps):
                if not os.environ.get("ONE_CONSUME"):
                    R.ring_consume(ring, m, vw, None, 0, 0, sc)
                R.ring_put_batch(peer, d, m, 0, st, sp)
            with torch.cuda.device(1):
                e1.record(sc)
            torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        ok = bool((st[:m] == 0).all().item())
        if os.environ.get("B200RING_TRACE"):
            t = R.ring_peer_trace(peer).astype(np.int64)
            for nm, h in (("prev", t[2048:]), ("last", t[:2048])):
                z = t[2048 + 252]
                rel = lambda v: round((v - z) / 1e3, 1) if v else None
                rounds = [(rel(h[4 * r]), rel(h[4 * r + 1]), int(h[4 * r + 3])) for r in range(64) if h[4 * r]]
                fl = [(rel(h[256 + 2 * j]), int(h[257 + 2 * j])) for j in range(512) if h[256 + 2 * j]]
                print(f"  {nm}: entry {rel(h[252])} end {rel(h[253])} rounds(start,placed,g) {rounds[:12]}")
                print(f"  {nm}: flushes {fl[:40]}")
        ms = e0.elapsed_time(e1)
        print(f"size={size:>10} m={m:3d} ctas={ctas:4d} mode={mode} {m * steps * size / ms / 1e6:8.1f} GB/s ok={ok}",
              flush=True)
