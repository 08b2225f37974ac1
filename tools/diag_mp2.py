"""Diagnostic (not a test): bench-like pipelined steps (no sync between steps),
one process per GPU; optional nvidia-smi sampling during the loop."""
import sys, os, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2601_20655_b200 import ring as R

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
R.ring_set_timeout_ns(1_000_000_000)
m, steps, smi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ring = R.ring_create(dev, 64 << 20, 64, 1, 0)
hs = [None] * world
dist.all_gather_object(hs, R.ring_export(ring))
peer, mh = R.ring_attach_peer(hs[(rank + 1) % world], dev, 0)
ms = [None] * world
dist.all_gather_object(ms, mh)
R.ring_bind_mirror(ring, 0, ms[(rank - 1) % world])
src = torch.randint(0, 255, (m * 4194304,), dtype=torch.uint8, device="cuda")
lens = [4194304 if q % 2 == 0 else 4193280 for q in range(m)]
a = R.make_msgs([src.data_ptr() + q * 4194304 for q in range(m)], lens, [bytes(16)] * m, [0] * m, [7] * m, [2] * m)
msgs = torch.from_numpy(a.view(np.uint8).copy()).cuda()
sts = [torch.full((m,), 10, dtype=torch.int32, device="cuda") for _ in range(steps)]
vws = [torch.zeros(m * 128, dtype=torch.uint8, device="cuda") for _ in range(steps)]
sp, sc = torch.cuda.Stream(), torch.cuda.Stream()
p = None
if smi and rank == 0:
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=index,clocks.sm", "--format=csv,noheader", "-lms", "100"],
                         stdout=subprocess.DEVNULL)
    time.sleep(0.3)
dist.barrier()
t0 = time.time()
for s in range(steps):
    R.ring_consume(ring, m, vws[s], None, 0, 0, sc)
    R.ring_put_batch(peer, msgs, m, 0, sts[s], sp)
torch.cuda.synchronize()
dt = time.time() - t0
if p: p.terminate()
first_bad = None
for s in range(steps):
    ps = np.unique(sts[s].cpu().numpy()).tolist()
    vs = np.unique(R.parse_views(vws[s].cpu().numpy())["status"]).tolist()
    if ps != [0] or vs != [0]:
        first_bad = (s, ps, vs)
        break
img = R.ring_read_image(ring)
print(f"rank {rank} smi={smi} steps={steps} {dt*1e3:.1f} ms first_bad={first_bad} tail {img['tail']:#x} head {img['head']:#x} cur {img['cursor']:#x}", flush=True)
dist.barrier()
R.ring_detach(peer)
dist.barrier()
R.ring_destroy(ring)
dist.destroy_process_group()
