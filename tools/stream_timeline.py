"""Diagnostic (not a test): event timeline of the C2 streaming loop.  Records
CUDA events around every put (stream sp) and consume (stream sc) and prints,
per step, when each kernel started / ended relative to the first put, to show
where the gaps between consecutive put launches come from.
Env: THREADS (put CTA size), STEPS, PRIO=1 (high-priority consumer stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_20655_b200 import ring as R

torch.cuda.set_device(0)
Rb, N, plen, m = 64 << 20, 64, 1048512, 64
ring = R.ring_create(0, Rb, N, 1, R.RING_CREATE_LOCAL)
peer, mh = R.ring_attach_peer(R.ring_export(ring), 0, 0)
R.ring_bind_mirror(ring, 0, mh)
R.ring_peer_config(peer, 148, int(os.environ.get("THREADS", "256")), 0)
if os.environ.get("GET_CFG"):
    gc, gt = (int(x) for x in os.environ["GET_CFG"].split(":"))
    R.ring_config(ring, gc, gt)
stride = 1 << 20
src = torch.randint(0, 255, (4 * m * stride,), dtype=torch.uint8, device="cuda")
d_msgs = []
for s in range(4):
    a = R.make_msgs([src.data_ptr() + (s * m + q) * stride for q in range(m)], [plen] * m,
                    [bytes(16)] * m, [0] * m, [7] * m, [1] * m)
    d_msgs.append(torch.from_numpy(a.view(np.uint8).copy()).cuda())
status = torch.zeros(m, dtype=torch.int32, device="cuda")
views = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
dst = torch.empty(m * plen, dtype=torch.uint8, device="cuda") if os.environ.get("COPYOUT") else None
sp = torch.cuda.Stream()
sc = torch.cuda.Stream(priority=-1) if os.environ.get("PRIO") else torch.cuda.Stream()
steps = int(os.environ.get("STEPS", "12"))
for i in range(6):
    R.ring_put_batch(peer, d_msgs[i % 4], m, 0, status, sp)
    R.ring_consume(ring, m, views, dst, plen if dst is not None else 0, 0, sc)
torch.cuda.synchronize()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
with torch.cuda.stream(sp):
    torch.cuda._sleep(2_000_000)
for i in range(steps):
    ev[i][0].record(sp)
    R.ring_put_batch(peer, d_msgs[i % 4], m, 0, status, sp)
    ev[i][1].record(sp)
    ev[i][2].record(sc)
    R.ring_consume(ring, m, views, dst, plen if dst is not None else 0, 0, sc)
    ev[i][3].record(sc)
torch.cuda.synchronize()
z = ev[0][0]
print("step  put_start put_end  cons_start cons_end   (us from put 0 start)")
for i in range(steps):
    t = [z.elapsed_time(e) * 1e3 for e in ev[i]]
    print(f"{i:4d}  {t[0]:9.1f} {t[1]:8.1f}  {t[2]:9.1f} {t[3]:8.1f}   put {t[1] - t[0]:6.1f}  "
          f"gap to next put {(z.elapsed_time(ev[i + 1][0]) * 1e3 - t[1]) if i + 1 < steps else 0:5.1f}")
per = (z.elapsed_time(ev[-1][1]) * 1e3) / steps
print(f"per step {per:.2f} us  payload {m * plen / per / 1e3:.1f} GB/s")
