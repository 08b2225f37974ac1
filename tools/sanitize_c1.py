"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) over the
ring's kernels: the C1 stream (BASELINE.json configs[0]: 32-KiB ring, 8
slots, U[1, 4096]-B payloads) through put, get, release and consume, on one
stream so that no kernel waits for another one that a serialising tool would
hold back (every put batch fits in the free ring: no credit wait).

Variants: LOCAL ring (gpu scope) and system-scope ring; view and copy-out
consume; get + release; a two-producer MPSC ring (paper lock); a
fault-tolerant ring.  Each payload is checked against synth.payload_bytes.

  compute-sanitizer --tool memcheck python tools/sanitize_c1.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_util import upload, msg_tensor, views_host  # noqa: E402
from paper_2601_20655_b200 import ring as R  # noqa: E402


def run(flags, n_prod=1, copy=False, get_release=False, n=48, batch=4, seed_off=0):
    L_R, L_N = 32768, 8
    ring = R.ring_create(0, L_R, L_N, max(n_prod, 1 if not flags & R.RING_CREATE_FAULT_TOLERANT else 2), flags)
    h = R.ring_export(ring)
    peers = []
    for pid in range(n_prod):
        pe, mh = R.ring_attach_peer(h, 0, pid)
        R.ring_bind_mirror(ring, pid, mh)
        R.ring_peer_config(pe, 4, 128, 0)
        peers.append(pe)
    R.ring_config(ring, 4, 128)
    streams = [synth.random_stream(synth.SEED_BASE + 30 + seed_off, pid, n, 1, 4096) for pid in range(n_prod)]
    bufs, msgs = [], []
    for st in streams:
        b, srcs = upload(st, "cuda")
        bufs.append(b)
        msgs.append(msg_tensor(st, srcs, "cuda"))
    status = torch.full((batch,), 10, dtype=torch.int32, device="cuda")
    vt = torch.zeros(batch * 128, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(batch * 4096, dtype=torch.uint8, device="cuda")
    got = []
    for k0 in range(0, n, batch):
        for pid in range(n_prod):
            R.ring_put_batch(peers[pid], msgs[pid][k0 * 48:(k0 + batch) * 48], batch, 0, status)
            if get_release:
                R.ring_get(ring, batch, vt, dst if copy else None, 4096 if copy else 0, 0)
                R.ring_release(ring, batch)
            else:
                R.ring_consume(ring, batch, vt, dst if copy else None, 4096 if copy else 0, 0)
            torch.cuda.synchronize()
            assert (status == 0).all().item(), status.tolist()
            v = views_host(vt)
            assert all(int(x["status"]) == 0 for x in v), [int(x["status"]) for x in v]
            if copy:
                d = dst.cpu().numpy()
                for j in range(batch):
                    assert d[j * 4096: j * 4096 + int(v[j]["len"])].tobytes() == \
                        streams[pid][k0 + j].payload.tobytes()
            got.append(len(v))
    for pe in peers:
        R.ring_detach(pe)
    R.ring_destroy(ring)
    return sum(got)


if __name__ == "__main__":
    R.ring_set_timeout_ns(120_000_000_000)   # the tools slow every kernel down
    done = 0
    done += run(R.RING_CREATE_LOCAL)
    done += run(R.RING_CREATE_LOCAL, copy=True)
    done += run(R.RING_CREATE_LOCAL, get_release=True, copy=True)
    done += run(0)                                        # system scope
    done += run(0, copy=True, get_release=True)
    done += run(0, n_prod=2, n=24, batch=2)               # MPSC, paper lock
    done += run(R.RING_CREATE_FAULT_TOLERANT, n=16, batch=2)
    print(f"sanitize_c1: {done} messages delivered and checked", flush=True)
