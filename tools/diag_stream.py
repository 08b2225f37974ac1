"""Diagnostic (not a test): multi-launch P2P streaming in ONE process, 2 GPUs.
Prints per-step put statuses / view statuses to locate failures."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2601_20655_b200 import ring as R

R.ring_set_timeout_ns(1_000_000_000)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
world = 2
rings, peers = [], []
for r in range(world):
    torch.cuda.set_device(r)
    rings.append(R.ring_create(r, 64 << 20, 64, 1, 0))
for r in range(world):
    pe, mh = R.ring_attach_peer(R.ring_export(rings[(r + 1) % world]), r, 0)
    peers.append(pe)
    R.ring_bind_mirror(rings[(r + 1) % world], 0, mh)
srcs, msgs, st, vw, sp, sc = [], [], [], [], [], []
for r in range(world):
    torch.cuda.set_device(r)
    src = torch.randint(0, 255, (m * 4194304,), dtype=torch.uint8, device=f"cuda:{r}")
    srcs.append(src)
    lens = [4194304 if q % 2 == 0 else 4193280 for q in range(m)]
    a = R.make_msgs([src.data_ptr() + q * 4194304 for q in range(m)], lens, [bytes(16)] * m, [0] * m, [7] * m, [2] * m)
    msgs.append(torch.from_numpy(a.view(np.uint8).copy()).to(f"cuda:{r}"))
    st.append(torch.zeros(m, dtype=torch.int32, device=f"cuda:{r}"))
    vw.append(torch.zeros(m * 128, dtype=torch.uint8, device=f"cuda:{r}"))
    sp.append(torch.cuda.Stream(r)); sc.append(torch.cuda.Stream(r))
for s in range(steps):
    t0 = time.time()
    for r in range(world):
        R.ring_consume(rings[r], m, vw[r], None, 0, 0, sc[r])
    for r in range(world):
        R.ring_put_batch(peers[r], msgs[r], m, 0, st[r], sp[r])
    for r in range(world):
        torch.cuda.synchronize(r)
    dt = time.time() - t0
    ps = [st[r].cpu().numpy() for r in range(world)]
    vs = [R.parse_views(vw[r].cpu().numpy())["status"] for r in range(world)]
    bad = [(r, np.unique(ps[r]).tolist(), np.unique(vs[r]).tolist()) for r in range(world)]
    print(f"step {s}: {dt*1e3:.2f} ms  put/view statuses {bad}", flush=True)
    if any(len(b[1]) > 1 or b[1][0] != 0 or len(b[2]) > 1 or b[2][0] != 0 for b in bad):
        for r in range(world):
            img = R.ring_read_image(rings[r])
            print("ring", r, {k: hex(v) for k, v in img.items() if k != "slots"}, [hex(x) for x in img["slots"][:8]])
        break
