"""Micro-benchmark (not a test): put-kernel time on a same-GPU ring for
different message mixes and grid sizes, to separate control overhead
(leader / publisher) from copy throughput.  Prints one line per case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_20655_b200 import ring as R

torch.cuda.set_device(0)
Rb, N = 64 << 20, 64
ring = R.ring_create(0, Rb, N, 1, R.RING_CREATE_LOCAL)
peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
R.ring_bind_mirror(ring, 0, mh)
src = torch.randint(0, 255, (256 << 20,), dtype=torch.uint8, device="cuda")
views = torch.zeros(64 * 128, dtype=torch.uint8, device="cuda")
status = torch.zeros(64, dtype=torch.int32, device="cuda")
cases = [("64 x 0 B", 64, 0), ("64 x 4 KiB", 64, 4096), ("63 x 1 MiB-64", 63, 1048512),
         ("15 x 4 MiB-64", 15, 4194240)]
TRACE = bool(os.environ.get("B200RING_TRACE"))


def show_trace():
    t = R.ring_peer_trace(peer).astype(np.int64)
    t0 = t[0]
    rounds = [(r, (t[4*r] - t0) / 1e3, (t[4*r+1] - t0) / 1e3, (t[4*r+2] - t0) / 1e3, int(t[4*r+3]))
              for r in range(64) if t[4*r]]
    print("   leader rounds (start, placed, released us; g):", [(r, round(a, 2), round(b, 2), round(c, 2), g) for r, a, b, c, g in rounds])
    per = [round((t[128 + l] - t0) / 1e3, 2) for l in range(32) if t[128 + l]]
    print("   round-0 per-message placement starts (us):", per[:4]); print("   msg1 phases (us):", [round((t[i] - t0) / 1e3, 3) for i in (129, 160, 161, 162, 130)])
    pub = [((t[256+2*j] - t0) / 1e3, int(t[257+2*j]) >> 16, int(t[257+2*j]) & 0xffff) for j in range(512) if t[256+2*j]]
    print(f"   publisher start {(t[255]-t0)/1e3:.2f} us; runs (t us, first item, run):", [(round(a, 2), b, c) for a, b, c in pub[:40]], "... n =", len(pub))
grids = [int(x) for x in (sys.argv[1:] or ["148", "296"])]
MODES = [int(x) for x in os.environ.get("COPY_MODES", "0,1").split(",")]
for ctas in grids:
  for mode in MODES:
    for threads in (512,):
        R.ring_peer_config(peer, ctas, threads, mode)
        print(f"copy_mode={mode}")
        for name, m, plen in cases:
            a = R.make_msgs([src.data_ptr() + q * (plen + 256) % (192 << 20) for q in range(m)], [plen] * m,
                            [bytes(16)] * m, [0] * m, [7] * m, [1] * m)
            d = torch.from_numpy(a.view(np.uint8).copy()).cuda()
            ts = []
            for it in range(12):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                R.ring_put_batch(peer, d, m, 0, status)
                e1.record()
                R.ring_consume(ring, m, views)
                torch.cuda.synchronize()
                assert (status[:m] == 0).all().item()
                if it >= 2:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            us = float(np.median(ts))
            gbs = m * plen / us / 1e3
            print(f"ctas={ctas:4d} thr={threads:5d} {name:16s} put {us:8.2f} us  payload {gbs:8.1f} GB/s  "
                  f"r+w {2 * gbs:8.1f} GB/s", flush=True)
            if TRACE:
                show_trace()
