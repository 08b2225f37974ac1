"""Diagnostic (not a test): the bench's ring-of-pairs pattern, one process per
GPU (torchrun), handles exchanged with a gloo process group.  Prints statuses
and ring images on failure."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2601_20655_b200 import ring as R

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
dist.init_process_group(os.environ.get("DIAG_BACKEND", "gloo"))
R.ring_set_timeout_ns(1_000_000_000)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ring = R.ring_create(dev, 64 << 20, 64, 1, 0)
hs = [None] * world
dist.all_gather_object(hs, R.ring_export(ring))
peer, mh = R.ring_attach_peer(hs[(rank + 1) % world], dev, 0)
ms = [None] * world
dist.all_gather_object(ms, mh)
R.ring_bind_mirror(ring, 0, ms[(rank - 1) % world])
dist.barrier()
src = torch.randint(0, 255, (m * 4194304,), dtype=torch.uint8, device="cuda")
lens = [4194304 if q % 2 == 0 else 4193280 for q in range(m)]
a = R.make_msgs([src.data_ptr() + q * 4194304 for q in range(m)], lens, [bytes(16)] * m, [0] * m, [7] * m, [2] * m)
msgs = torch.from_numpy(a.view(np.uint8).copy()).cuda()
st = torch.zeros(m, dtype=torch.int32, device="cuda")
vw = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
sp, sc = torch.cuda.Stream(), torch.cuda.Stream()
for s in range(steps):
    dist.barrier()
    t0 = time.time()
    R.ring_consume(ring, m, vw, None, 0, 0, sc)
    R.ring_put_batch(peer, msgs, m, 0, st, sp)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ps = np.unique(st.cpu().numpy()).tolist()
    vs = np.unique(R.parse_views(vw.cpu().numpy())["status"]).tolist()
    img = R.ring_read_image(ring)
    print(f"rank {rank} step {s}: {dt*1e3:.2f} ms put {ps} views {vs} tail {img['tail']:#x} head {img['head']:#x} cur {img['cursor']:#x}", flush=True)
dist.barrier()
R.ring_detach(peer)
dist.barrier()
R.ring_destroy(ring)
dist.destroy_process_group()
