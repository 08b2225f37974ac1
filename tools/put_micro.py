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
         ("15 x 4 MiB-64", 15, 4194240), ("1 x 4 KiB", 1, 4096)]
TRACE = bool(os.environ.get("B200RING_TRACE"))
if os.environ.get("CASES"):
    cases = [cases[int(c)] for c in os.environ["CASES"].split(",")]


def show_trace():
    t = R.ring_peer_trace(peer).astype(np.int64)[:2048]
    t0 = t[0]
    rounds = [(r, (t[4*r] - t0) / 1e3, (t[4*r+1] - t0) / 1e3, (t[4*r+2] - t0) / 1e3, int(t[4*r+3]))
              for r in range(64) if t[4*r]]
    print("   leader rounds (start, placed, released us; g):", [(r, round(a, 2), round(b, 2), round(c, 2), g) for r, a, b, c, g in rounds])
    per = [round((t[128 + l] - t0) / 1e3, 2) for l in range(32) if t[128 + l]]
    print("   round-0 per-message placement starts (us):", per[:4]); print("   msg1 phases (us):", [round((t[i] - t0) / 1e3, 3) for i in (129, 160, 161, 162, 130)])
    pub = [((t[256+2*j] - t0) / 1e3, int(t[257+2*j])) for j in range(512) if t[256+2*j]]
    cw = [(b, *[(t[1280 + 4*b + k] - t0) / 1e3 for k in range(4)]) for b in range(148) if t[1280 + 4*b]]
    cw.sort(key=lambda r: r[1])
    print("   copy warps (cta, grab, planned, found, done us):", [tuple(round(x, 2) for x in r) for r in cw[:6]], "...",
          [tuple(round(x, 2) for x in r) for r in cw[-3:]])
    if cw:
        print("   copy start spread: planned %.2f-%.2f found %.2f-%.2f done %.2f-%.2f" % (
            min(r[2] for r in cw), max(r[2] for r in cw), min(r[3] for r in cw), max(r[3] for r in cw),
            min(r[4] for r in cw), max(r[4] for r in cw)))
    print(f"   kernel entry {(t[252]-t0)/1e3:.2f} us publisher end {(t[253]-t0)/1e3:.2f} us")
    print(f"   publisher start {(t[255]-t0)/1e3:.2f} us; flushes (t us, items published):", [(round(a, 2), b) for a, b in pub[:40]], "... n =", len(pub))
if os.environ.get("COPYREF"):
    for nb in (63 * 1048512, 64 << 20):
        a_, b_ = src[:nb], src[128 << 20:(128 << 20) + nb]
        for _ in range(3): b_.copy_(a_)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000); e0.record()
        for _ in range(20): b_.copy_(a_)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        print(f"torch copy_ {nb} B: {us:.2f} us  r+w {2 * nb / us / 1e3:.1f} GB/s (L2-warm source)")
grids = [int(x) for x in (sys.argv[1:] or ["148", "296"])]
MODES = [int(x) for x in os.environ.get("COPY_MODES", "0,1").split(",")]
for ctas in grids:
  for mode in MODES:
    for threads in [int(x) for x in os.environ.get("THREADS", "256").split(",")]:
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
            # back-to-back: puts on one stream, consumes on another (as bench.py)
            sp = torch.cuda.Stream()
            sc = torch.cuda.Stream(priority=-1) if os.environ.get("PRIO") else torch.cuda.Stream()
            ev = [torch.cuda.Event() for _ in range(40)]
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(sp):
                torch.cuda._sleep(2_000_000)
                e0.record(sp)
            import time as _t
            h0 = _t.perf_counter()
            for it in range(40):
                R.ring_put_batch(peer, d, m, 0, status, sp)
                R.ring_consume(ring, m, views, None, 0, 0, sc)
            h1 = _t.perf_counter()
            e1.record(sp)
            torch.cuda.synchronize()
            st_us = e0.elapsed_time(e1) * 1e3 / 40
            print(f"      host enqueue {(h1 - h0) / 40 * 1e6:.2f} us/step")
            print(f"      streamed: {st_us:8.2f} us/step  payload {m * plen / st_us / 1e3:8.1f} GB/s", flush=True)
            if TRACE:
                t = R.ring_peer_trace(peer).astype(np.int64)
                prev, last = t[2048:], t[:2048]
                z = prev[252]
                v = R.parse_views(views.cpu().numpy())
                tv = v["t_visible"][:m].astype(np.int64)
                tp = np.array([int.from_bytes(bytes(v["header"][q][56:64]), "little") for q in range(m)], dtype=np.int64)
                print(f"      last consume: t_put {(tp.min() - z) / 1e3:.2f}-{(tp.max() - z) / 1e3:.2f} t_visible {(tv.min() - z) / 1e3:.2f}-{(tv.max() - z) / 1e3:.2f}")
                for nm, h in (("prev", prev), ("last", last)):
                    rel = lambda v: round((v - z) / 1e3, 2) if v else None
                    rounds = [(rel(h[4*r]), rel(h[4*r+1]), rel(h[4*r+2])) for r in range(4) if h[4*r]]
                    fl = [(rel(h[256+2*j]), int(h[257+2*j])) for j in range(8) if h[256+2*j]]
                    cw = [h[1280 + 4*b + 1] for b in range(148) if h[1280 + 4*b + 1]]
                    cg = [h[1280 + 4*b + 0] for b in range(148) if h[1280 + 4*b + 0]]
                    print(f"      {nm}: copy grab {rel(min(cg)) if cg else None}-{rel(max(cg)) if cg else None}; "
                          f"cta1 grab/planned/found/done {[rel(h[1280 + 4 + k]) for k in range(4)]}")
                    cf = [h[1280 + 4*b + 2] for b in range(148) if h[1280 + 4*b + 2]]
                    cd = [h[1280 + 4*b + 3] for b in range(148) if h[1280 + 4*b + 3]]
                    print(f"      {nm}: copy-warp last exit {rel(h[254])} spec(cta1): units {h[1880]} run {h[1881]} "
                          f"H {h[1882] >> 24}/{h[1882] & 0xffffff} P {h[1883] >> 24}/{h[1883] & 0xffffff} at {rel(h[1884])}")
                    print(f"      {nm}: entry {rel(h[252])} rounds(start,placed,hdr) {rounds} copies planned "
                          f"{rel(min(cw)) if cw else None}-{rel(max(cw)) if cw else None} found {rel(min(cf)) if cf else None}-{rel(max(cf)) if cf else None} "
                          f"done {rel(min(cd)) if cd else None}-{rel(max(cd)) if cd else None} flushes {fl} end {rel(h[253])}")
