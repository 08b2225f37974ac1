"""Multi-GPU topologies of BASELINE.json beyond the default ring of pairs
(invoked through `bench.py --topology pipeline|fanin|reassign` under torchrun):

  pipeline  C4: text-encoder -> VAE-encode -> DiT -> VAE-decode -> sink, one
            stage per GPU, each hop a double ring owned by the next stage's GPU;
            stages forward synthetic outputs of the Wan2.1 shapes (stage compute
            = 0), so the run measures the transport term Network(q) of
            T(q) = T_X + T_Y + Network(q).
  fanin     C5a: GPUs 1..N-1 -> one shared MPSC ring (paper lock) on GPU 0,
            message-size sweep 4 KiB .. 256 MiB (x4 steps).
  reassign  C5b: as fanin with Wan-shaped messages; at 50% of each producer's
            messages the router flips (NodeManager reassignment):
            GPU N-1 stops producing and becomes a second consumer, producers
            1..N-2 round-robin over {GPU 0, GPU N-1} (ResultDeliver).

Every number is device-timed (CUDA events, max over ranks); latencies are
t_visible - t_put on the host clock (ring_clock_offset_ns).  Rank 0 prints one
JSON line per topology.
"""
from __future__ import annotations

import os
import time

import numpy as np
import torch
import torch.distributed as dist

import synth
from paper_2601_20655_b200 import ring as R
from paper_2601_20655_b200 import topology as T

METRIC = "ring transfer GB/s per GPU vs 900 GB/s NVLink; p50/p99 msg latency at 1/2/4/8 GPU"
NVLINK_PEAK_MEASURED = 770.0
# one GPU's NVLink ingress fed by k GPUs' SM pushes at once (profiles/r02b_p2p_fanin.txt)
FANIN_INGRESS = {1: 680.0, 2: 715.6, 3: 718.3}

# Wan2.1 I2V intermediate tensors
EMB = synth.wan_bytes("umt5_emb")                       # 4,194,304
LAT720 = synth.wan_bytes("latent_720p")                 # 9,676,800
FRAMES = synth.wan_bytes("frames_720p")                 # 447,897,600
STAGE_OUT = [EMB, LAT720 + EMB, LAT720, FRAMES]         # text-enc, VAE-enc, DiT, VAE-dec outputs


def _pct(x, q):
    return round(float(np.percentile(np.asarray(x, dtype=np.float64), q)), 2) if len(x) else None


def _views(vt):
    return R.parse_views(vt.cpu().numpy())


def _lat_us(v, off_cons, off_prod_by_id, by_ring=False):
    """t_visible - t_put on the host clock; the producer is the header's
    producer id, or (ring sets, every ring's producer has id 0) the ring index."""
    t_put = np.frombuffer(v["header"][:, 56:64].tobytes(), dtype="<u8").astype(np.int64)
    if by_ring:
        pid = v["reserved"][:, 0].astype(np.int64)
    else:
        pid = np.frombuffer(v["header"][:, 44:48].tobytes(), dtype="<u4").astype(np.int64)
    offp = np.array([off_prod_by_id[int(p)] for p in pid], dtype=np.int64)
    return (((v["t_visible"].astype(np.int64) - off_cons) - (t_put - offp)) / 1e3).tolist()


def _msgs(srcs, lens, app_id=7, stage=1, seed=0, rank=0):
    n = len(lens)
    hdr = [synth.header_fields(synth.SEED_BASE + seed, rank, q) for q in range(n)]
    a = R.make_msgs(srcs, lens, [h[0] for h in hdr], [h[1] for h in hdr], [app_id] * n, [stage] * n)
    return torch.from_numpy(a.view(np.uint8).copy()).cuda()


def _fill(nbytes, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    t = torch.empty((nbytes + 1) // 2, dtype=torch.bfloat16, device="cuda")
    t.normal_(generator=g)
    return t.view(torch.uint8)[:nbytes]


def _seeded_source(nbytes, seed):
    """A source buffer holding synth.payload_bytes(seed, 0, 0, nbytes) (device
    generator): every message put from it can be checked on the device."""
    from synth import device as SD
    t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    SD.fill([t.data_ptr()], [nbytes], [0], [0], seed)
    torch.cuda.synchronize()
    return t


def _verify_pass(ring, total, seed, stream):
    """Consumer side of a verification pass: every entry is taken with ring_get,
    its payload compared in place (before release) with the generator on the
    device (synth/csrc/synth_dev.cu), then released.  Returns (bad payloads,
    per-producer order ok, views)."""
    from synth import device as SD
    vt = torch.zeros(total * 128, dtype=torch.uint8, device="cuda")
    zc = torch.zeros(1, dtype=torch.int32, device="cuda")
    zs = torch.zeros(1, dtype=torch.int64, device="cuda")
    base = R.ring_get_info(ring).data
    bads = []
    for j in range(total):
        v = vt[j * 128:(j + 1) * 128]
        R.ring_get(ring, 1, v, None, 0, 0, stream)
        bads.append(SD.verify_views(v, 1, base, seed, zc, zs, None, 0, stream))
        R.ring_release(ring, 1, stream)
    stream.synchronize()
    nbad = sum(int((b.cpu() != -1).sum()) for b in bads)
    vv = _views(vt)
    pid = np.frombuffer(vv["header"][:, 44:48].tobytes(), dtype="<u4")
    seq = np.frombuffer(vv["header"][:, 48:52].tobytes(), dtype="<u4")
    order_ok = all(bool(np.all(np.diff(seq[pid == p].astype(np.int64)) == 1)) for p in np.unique(pid))
    return nbad, order_ok and bool((vv["status"] == 0).all()), vv


def _wire(plan, rank, world, grp, dev, split=()):
    """Rings named in `split` take the split placement (ring_create_split, R28):
    control words at the consumer, buffer region on the producer's GPU -- the
    consumer pulls every payload over NVLink with its copy-out.  The producer of
    ring "hop{s}" is rank s (device s)."""
    def create(s, d):
        if s.name in split:
            return R.ring_create_split(d, int(s.name[3:]) % torch.cuda.device_count(), s.data_bytes, s.n_slots,
                                       s.max_producers, s.flags)
        return R.ring_create(d, s.data_bytes, s.n_slots, s.max_producers, s.flags)
    return T.wire(plan, rank, world, grp, device=dev, create=create,
                  export=R.ring_export, attach=R.ring_attach_peer, bind=R.ring_bind_mirror)


def _teardown(wired, grp):
    dist.barrier(group=grp)
    for p in wired.peers.values():
        R.ring_detach(p)
    dist.barrier(group=grp)
    for r in wired.rings.values():
        R.ring_destroy(r)


def run_pipeline(args, rank, world, grp, offsets):
    dev = torch.cuda.current_device()
    outs = (STAGE_OUT[:world - 1] + [FRAMES]) if world < 4 else STAGE_OUT + [EMB] * (world - 4)
    hop_bytes = [(1 << 30) if b >= (256 << 20) else (256 << 20) for b in outs]
    hop_slots = [8 if b >= (256 << 20) else 64 for b in outs]
    # frames-sized hops (>= 256 MiB) pulled by their consumer (split placement):
    # one way, pulls carry 1.125 wire bytes per payload byte against 1.21 for
    # peer stores; the smaller hops stay pushed
    split = {f"hop{s}" for s, b in enumerate(outs) if b >= (256 << 20)} if getattr(args, "c4_split", True) else set()
    wired = _wire(T.plan_pipeline(world, hop_bytes, hop_slots), rank, world, grp, dev, split)
    B = args.msgs_per_step or 2
    out_bytes = outs[rank]
    src = _fill(out_bytes, 1000 + rank)
    d_msgs = _msgs([src.data_ptr()] * B, [out_bytes] * B, stage=rank + 1, seed=4, rank=rank)
    peer = wired.peers[f"hop{rank}"]
    in_ring = wired.rings[f"hop{(rank - 1) % world}"]
    st = torch.zeros(B, dtype=torch.int32, device="cuda")
    vt = torch.zeros(B * 128, dtype=torch.uint8, device="cuda")
    s_put, s_get = torch.cuda.Stream(), torch.cuda.Stream()
    in_name = f"hop{(rank - 1) % world}"
    in_bytes = outs[(rank - 1) % world]
    pulled = torch.empty(B * in_bytes, dtype=torch.uint8, device="cuda") if in_name in split else None

    def consume():
        R.ring_consume(in_ring, B, vt, pulled, in_bytes if pulled is not None else 0, 0, s_get)

    def step():
        if rank == 0:      # new requests enter; the sink drains independently
            R.ring_put_batch(peer, d_msgs, B, 0, st, s_put)
            consume()
        else:              # store-and-forward stage: receive the request, emit the next tensor
            consume()
            s_put.wait_stream(s_get)
            R.ring_put_batch(peer, d_msgs, B, 0, st, s_put)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier(group=grp)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s_put)
    e[1].record(s_get)
    for _ in range(args.steps):
        step()
    e[2].record(s_put)
    e[3].record(s_get)
    torch.cuda.synchronize()
    ms = max(e[0].elapsed_time(e[2]), e[1].elapsed_time(e[3]), e[0].elapsed_time(e[3]), e[1].elapsed_time(e[2]))
    v = _views(vt)
    ok = bool((st == 0).all().item()) and bool((v["status"] == 0).all())
    prev = (rank - 1) % world
    lat = _lat_us(v, offsets[rank], {0: offsets[prev]})
    t = torch.tensor([ms, 0.0 if ok else 1.0], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=grp)
    lats = [None] * world
    dist.all_gather_object(lats, lat, group=grp)
    _teardown(wired, grp)
    if rank != 0:
        return None
    ms_max = float(t[0])
    reqs = B * args.steps
    hop_gbs = [round(b * reqs / (ms_max / 1e3) / 1e9, 2) for b in outs]
    total = sum(outs) * reqs / (ms_max / 1e3) / 1e9
    hop_lat = {f"hop{(s - 1) % world}": {"p50": _pct(lats[s], 50), "p99": _pct(lats[s], 99)} for s in range(world)}
    return {"metric": METRIC, "topology": "pipeline", "value": round(total, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
            "requests_per_s": round(reqs / (ms_max / 1e3), 2), "per_gpu_gbs": round(total / world, 2),
            "hop_bytes": outs, "hop_gbs": hop_gbs,
            "hop_frac_of_770": [round(g / NVLINK_PEAK_MEASURED, 4) for g in hop_gbs],
            "hop_latency_us": hop_lat,
            "e2e_transport_latency_p50_us": round(sum(h["p50"] for h in hop_lat.values() if h["p50"] is not None), 2),
            "config": {"workload": "C4 Wan2.1-I2V stage pipeline (store-and-forward per batch of requests)",
                       "requests_per_step": B, "hop_ring_bytes": hop_bytes, "hop_slots": hop_slots,
                       "hop_placement": ["split (consumer pulls)" if f"hop{s}" in split else "push"
                                         for s in range(world)]},
            "higher_is_better": True, "dtype": "u8", "data": "synthetic", "ok": ok == 1 and float(t[1]) == 0.0}


def run_fanin(args, rank, world, grp, offsets):
    dev = torch.cuda.current_device()
    mode = getattr(args, "fanin_mode", "mpsc")
    lockfree = mode == "set"
    plan = T.plan_fanin_set(world, 512 << 20, 256) if lockfree else \
        T.plan_fanin(world, 1 << 30, 256, flags=R.RING_CREATE_RESERVE_COMMIT if mode == "rc" else 0)
    wired = _wire(plan, rank, world, grp, dev)
    my_ring = f"sub{rank}" if lockfree else "fan0"
    rset = R.ring_set_create([wired.rings[f"sub{p}"] for p in range(1, world)]) if lockfree and rank == 0 else None
    sizes = [4096 << (2 * i) for i in range(9)]          # 4 KiB .. 256 MiB
    if args.sizes:
        sizes = [int(x) for x in args.sizes.split(",")]
    verify = getattr(args, "verify", False)
    vseed = synth.SEED_BASE + 5
    if rank > 0:
        src = _seeded_source(max(sizes), vseed) if verify else _fill(max(sizes), 2000 + rank)
    else:
        src = None
    rows = []
    for size in sizes:
        M = int(min(1000, max(4, (2 << 30) // size // max(1, world - 1))))
        if rank > 0:
            d_msgs = _msgs([src.data_ptr()] * M, [size] * M, seed=5, rank=rank)
            st = torch.zeros(M, dtype=torch.int32, device="cuda")
        else:
            total = M * (world - 1)
            vt = torch.zeros(total * 128, dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        res = []
        for it in range(2):                                # warm-up pass, timed pass
            dist.barrier(group=grp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if rank == 0:
                if lockfree:
                    R.ring_set_consume(rset, total, vt, None, 0, s)
                else:
                    R.ring_consume(wired.rings["fan0"], total, vt, None, 0, 0, s)
            else:
                R.ring_put_batch(wired.peers[my_ring], d_msgs, M, 0, st, s)
            e1.record(s)
            torch.cuda.synchronize()
            res = [e0.elapsed_time(e1)]
        ok = True
        lat = []
        if rank == 0:
            v = _views(vt)
            ok = bool((v["status"] == 0).all())
            lat = _lat_us(v, offsets[0], {p - 1: offsets[p] for p in range(1, world)}, by_ring=lockfree)
        else:
            ok = bool((st == 0).all().item())
        t = torch.tensor([res[0], 0.0 if ok else 1.0], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=grp)
        lats = [None] * world
        dist.all_gather_object(lats, lat, group=grp)
        ms = float(t[0])
        allb = size * M * (world - 1)
        lat0 = lats[0]
        row = {"size": size, "msgs_per_producer": M, "ms": round(ms, 4),
               "ingress_gbs": round(allb / (ms / 1e3) / 1e9, 2),
               "msgs_per_s": round(M * (world - 1) / (ms / 1e3), 1),
               "lat_p50_us": _pct(lat0, 50), "lat_p99_us": _pct(lat0, 99), "lat_samples": len(lat0),
               "ok": float(t[1]) == 0.0}
        if verify and not lockfree:
            # verification pass (untimed): the same puts again; every payload
            # compared in place on the device, per-producer order from the headers
            dist.barrier(group=grp)
            vres = [0, 1]
            if rank == 0:
                nbad, order_ok, _ = _verify_pass(wired.rings["fan0"], M * (world - 1), vseed, s)
                vres = [nbad, 1 if order_ok else 0]
            else:
                R.ring_put_batch(wired.peers[my_ring], d_msgs, M, 0, st, s)
                s.synchronize()
                vres = [0, 1 if bool((st == 0).all().item()) else 0]
            vt_ = torch.tensor([vres[0], 1 - vres[1]], dtype=torch.float64)
            dist.all_reduce(vt_, op=dist.ReduceOp.MAX, group=grp)
            row["verified"] = {"payload_mismatches": int(vt_[0]), "order_and_status_ok": float(vt_[1]) == 0.0,
                               "what": "second pass, ring_get -> device compare in place -> ring_release per entry"}
        rows.append(row)
    if rset is not None:
        R.ring_set_destroy(rset)
    _teardown(wired, grp)
    if rank != 0:
        return None
    best = max(r["ingress_gbs"] for r in rows)
    return {"metric": METRIC, "topology": "fanin" + ("-" + mode if mode != "mpsc" else ""), "value": best,
            "unit": "GB/s", "n_gpus": world,
            "fanin_mode": {"set": "lock-free: one SPSC ring per producer, one consumer warp",
                           "rc": "reserve-then-commit MPSC ring: claim under the lock, copy outside it",
                           "mpsc": "paper MPSC ring with the lock"}[mode],
            "producers": world - 1, "sweep": rows,
            "roofline": {"bound": "nvlink (consumer ingress)", "achieved": best,
                         "peak": FANIN_INGRESS.get(world - 1, NVLINK_PEAK_MEASURED),
                         "frac": round(best / FANIN_INGRESS.get(world - 1, NVLINK_PEAK_MEASURED), 4),
                         "peak_source": ("profiles/r02b_p2p_fanin.txt: bare SM pushes from the producers' GPUs into "
                                         "one GPU at once (tools/p2p_fanin.cu)" if world - 1 in FANIN_INGRESS else
                                         "B200_PROFILING.md peer copy 770 GB/s (no measured ingress for this fan-in)")},
            "config": {"workload": ("C5a variant (SURVEY.md sec 8 f3): GPUs 1..N-1 -> one 512 MiB SPSC ring each on GPU 0, "
                                    "one consumer warp" if lockfree else
                                    "C5a variant (SURVEY.md sec 8 f3 ii): GPUs 1..N-1 -> one reserve-then-commit MPSC "
                                    "ring on GPU 0, size sweep" if mode == "rc" else
                                    "C5a: GPUs 1..N-1 -> one MPSC ring (paper lock) on GPU 0, size sweep"),
                       "R_bytes": (512 << 20) if lockfree else 1 << 30, "n_slots": 256},
            "higher_is_better": True, "dtype": "u8", "data": "synthetic"}


def run_reassign(args, rank, world, grp, offsets):
    """C5b: stage reassignment mid-stream through the router's epoch flip."""
    assert world >= 3, "reassign needs >= 3 GPUs"
    dev = torch.cuda.current_device()
    spare = world - 1
    plan = T.plan_fanin(world, 1 << 30, 256, spare_consumer=True)
    wired = _wire(plan, rank, world, grp, dev)
    M = args.msgs_per_step or 200                           # per producer, even
    half = M // 2
    lens = [EMB, synth.wan_bytes("latent_480p")]
    verify = getattr(args, "verify", False)
    vseed = synth.SEED_BASE + 6
    src = (_seeded_source(EMB, vseed) if verify else _fill(EMB, 3000 + rank)) if rank > 0 else None
    vres = {}
    router = None
    if 0 < rank:
        router = R.router_create(dev, 4)
        R.router_set_route(router, 7, 2, [wired.peers["fan0"]])
        d1 = _msgs([src.data_ptr()] * half, [lens[q % 2] for q in range(half)], app_id=7, stage=2, seed=6, rank=rank)
        d2 = _msgs([src.data_ptr()] * half, [lens[(half + q) % 2] for q in range(half)], app_id=7, stage=2, seed=7,
                   rank=rank)
        st = torch.zeros(M, dtype=torch.int32, device="cuda")
        dests = torch.zeros(M, dtype=torch.int32, device="cuda")
    # expected counts: fan0 gets every first half, and half of producers 1..N-2's second halves
    n_rr = (world - 2) * half
    fan0_total = (world - 1) * half + n_rr // 2
    fan1_total = n_rr - n_rr // 2
    s = torch.cuda.Stream()
    dist.barrier(group=grp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    if rank == 0:
        vt = torch.zeros(fan0_total * 128, dtype=torch.uint8, device="cuda")
        if verify:        # every payload compared in place before its release (timed with it)
            nbad, order_ok, _vv = _verify_pass(wired.rings["fan0"], fan0_total, vseed, s)
            vt = torch.from_numpy(np.ascontiguousarray(_vv).view(np.uint8).reshape(-1).copy())
            vres = {"payload_mismatches": nbad, "order_and_status_ok": order_ok}
        else:
            R.ring_consume(wired.rings["fan0"], fan0_total, vt, None, 0, 0, s)
    else:
        R.ring_put_routed(router, d1, half, 0, st[:half], dests[:half], s)
    if rank == spare:
        vt = torch.zeros(fan1_total * 128, dtype=torch.uint8, device="cuda")
        s2 = torch.cuda.Stream()
        s.synchronize()                 # the spare finishes its first half, then becomes a consumer
        if verify:
            nbad, order_ok, _vv = _verify_pass(wired.rings["fan1"], fan1_total, vseed, s2)
            vt = torch.from_numpy(np.ascontiguousarray(_vv).view(np.uint8).reshape(-1).copy())
            vres = {"payload_mismatches": nbad, "order_and_status_ok": order_ok}
        else:
            R.ring_consume(wired.rings["fan1"], fan1_total, vt, None, 0, 0, s2)
        s.wait_stream(s2)
    elif rank > 0:
        # NodeManager reassignment: the new route takes effect for later puts (epoch flip)
        R.router_set_route(router, 7, 2, [wired.peers["fan0"], wired.peers["fan1"]], s)
        R.ring_put_routed(router, d2, half, 0, st[half:], dests[half:], s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ok = True
    info = {}
    if rank == 0 or rank == spare:
        v = _views(vt)
        ok = bool((v["status"] == 0).all())
        hd = [R.parse_views(vt.cpu().numpy())["header"][i] for i in range(len(v))]
        epochs = [int.from_bytes(bytes(h[52:54]), "little") for h in hd]
        info = {"received": len(v), "epochs": sorted(set(epochs))} | ({"verified": vres} if vres else {})
    if rank > 0:
        ok = ok and bool((st == 0).all().item())
    t = torch.tensor([ms, 0.0 if ok else 1.0], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=grp)
    infos = [None] * world
    dist.all_gather_object(infos, info, group=grp)
    if router is not None:
        R.router_destroy(router)
    _teardown(wired, grp)
    if rank != 0:
        return None
    total_bytes = sum(lens[q % 2] for q in range(M)) * (world - 1)
    ms_max = float(t[0])
    return {"metric": METRIC, "topology": "reassign", "value": round(total_bytes / (ms_max / 1e3) / 1e9, 2),
            "unit": "GB/s", "n_gpus": world, "ms": round(ms_max, 3), "consumer0": infos[0],
            "consumer_spare": infos[spare], "expected": {"fan0": fan0_total, "fan1": fan1_total},
            "config": {"workload": "C5b: fan-in with router epoch flip at 50%; GPU N-1 becomes a 2nd consumer",
                       "msgs_per_producer": M},
            "ok": float(t[1]) == 0.0, "higher_is_better": True, "dtype": "u8", "data": "synthetic"}


RUNNERS = {"pipeline": run_pipeline, "fanin": run_fanin, "reassign": run_reassign}


def main(args, rank, world, grp):
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    offsets = [None] * world
    dist.all_gather_object(offsets, R.ring_clock_offset_ns(dev), group=grp)
    return RUNNERS[args.topology](args, rank, world, grp, offsets)
