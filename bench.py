#!/usr/bin/env python
"""Benchmark of the double-ring tensor transport (BASELINE.json metric:
"ring transfer GB/s per GPU vs 900 GB/s NVLink; p50/p99 msg latency").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

N = 1 -> BASELINE.json configs[1] (C2): a same-GPU ring of 64 slots x 1 MiB
(R = 64 MiB), 1,048,512-B payloads (footprint exactly 1 MiB).  One step = one
pass of the whole hot path over one batch: ring_put_batch of 64 messages
(claim, header + CRC, copy, publish) then ring_consume of the 64 entries (poll,
slot + header read, CRC verify, release + credit), in stream order on one GPU
(two kernels spinning on each other must never share a GPU; R20).
N >= 2 -> C3-shaped messages (umT5 embeddings 4,194,304 B / 480p latents
4,193,280 B, alternating) over NVLink: rank r puts into the ring on rank
(r+1) % N while consuming its own ring (fed by rank r-1), both streaming
concurrently with credit flowing back; weak scaling (fixed work per GPU).

Prints ONE JSON line on rank 0.  `value` = payload bytes delivered by all
ranks / max-over-ranks device time of the K timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ring transfer GB/s per GPU vs 900 GB/s NVLink; p50/p99 msg latency at 1/2/4/8 GPU"
UNIT = "GB/s"
NVLINK_PEAK_MEASURED = 770.0   # B200_PROFILING.md: measured peer copy, per direction per GPU
NVLINK_NOMINAL = 900.0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ---------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.25)

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8 or not parts[0].isdigit() or int(parts[0]) != self.idx:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# CPU baseline: the oracle as it stands on the host cores (bounded sample)
# ---------------------------------------------------------------------------------------
def oracle_throughput(payload_lens, R_bytes, N_slots, budget_s: float = 12.0, seed: int = 0):
    """Run the CPU oracle (oracle/ring.py, one producer, draining consumer) over
    repeated batches of the workload's messages for about `budget_s` seconds.
    Returns (GB/s of payload, messages, seconds)."""
    import synth
    from oracle.ring import Layout, Sim, Msg, run
    L = Layout(R_bytes, N_slots)
    payloads = [synth.payload_bytes(synth.SEED_BASE + seed, 0, q, n).tobytes() for q, n in enumerate(payload_lens)]
    msgs = [Msg(n, p, bytes(16), 0, 7, 1) for n, p in zip(payload_lens, payloads)]
    t0 = time.perf_counter()
    done_msgs = done_bytes = 0
    while True:
        sim = Sim(L, {0: msgs}, mpsc=False, block=True, depth=1, check=False)
        run(sim, policy="drain")
        done_msgs += len(msgs)
        done_bytes += sum(payload_lens)
        dt = time.perf_counter() - t0
        if dt >= budget_s:
            break
    return done_bytes / dt / 1e9, done_msgs, dt


# ---------------------------------------------------------------------------------------
# N = 1: C2 same-GPU ring
# ---------------------------------------------------------------------------------------
def bench_c2(args):
    import torch
    import synth
    from paper_2601_20655_b200 import ring as R

    dev = 0
    torch.cuda.set_device(dev)
    Rb, N, plen = 64 << 20, 64, 1048512
    m = args.msgs_per_step or 64
    sets = 4                                   # 4 x 64 MiB rotating inputs > 126 MB L2
    ring = R.ring_create(dev, Rb, N, 1, R.RING_CREATE_LOCAL)
    peer, mh = R.ring_attach_peer(R.ring_export(ring), dev, 0)
    R.ring_bind_mirror(ring, 0, mh)
    if args.copy_ctas or args.threads:
        R.ring_peer_config(peer, args.copy_ctas, args.threads, 0)
    stride = (plen + 255) // 256 * 256
    src = torch.empty(sets * m * stride, dtype=torch.uint8, device="cuda")
    for s in range(sets):
        for q in range(m):
            k = s * m + q
            src[k * stride: k * stride + plen] = torch.from_numpy(synth.payload_bytes(synth.SEED_BASE + 2, 0, k, plen))
    d_msgs = []
    for s in range(sets):
        srcs = [src.data_ptr() + (s * m + q) * stride for q in range(m)]
        hdr = [synth.header_fields(synth.SEED_BASE + 2, 0, s * m + q) for q in range(m)]
        a = R.make_msgs(srcs, [plen] * m, [h[0] for h in hdr], [h[1] for h in hdr], [7] * m, [1] * m)
        d_msgs.append(torch.from_numpy(a.view(np.uint8).copy()).cuda())
    status = torch.zeros(m, dtype=torch.int32, device="cuda")
    views = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(i, timed=None):
        if timed is not None:
            timed[0].record(stream)
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, stream)
        if timed is not None:
            timed[1].record(stream)
        R.ring_consume(ring, m, views, None, 0, 0, stream)
        if timed is not None:
            timed[2].record(stream)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    assert (status == 0).all().item(), "put failed in warm-up"
    v = R.parse_views(views.cpu().numpy())
    assert (v["status"] == 0).all(), "consume failed in warm-up"

    clk = Clocks(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]) if False else dev)
    clk.start()
    l0 = R.ring_launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_start.record(stream)
    for i in range(args.steps):
        step(args.warmup + i, ev[i])
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = R.ring_launch_count() - l0
    clocks = clk.stop()
    ms = t_start.elapsed_time(t_end)
    put_ms = [a.elapsed_time(b) for a, b, c in ev]
    get_ms = [b.elapsed_time(c) for a, b, c in ev]
    assert (status == 0).all().item()
    v = R.parse_views(views.cpu().numpy())
    assert (v["status"] == 0).all()
    # latency of the last step's messages: t_visible - t_put (same GPU clock)
    t_put = np.frombuffer(v["header"][:, 56:64].tobytes(), dtype="<u8")
    lat_us = (v["t_visible"].astype(np.int64) - t_put.astype(np.int64)) / 1e3

    payload = m * plen * args.steps
    value = payload / (ms / 1e3) / 1e9
    f = R.ring_footprint(plen)
    put_bytes = m * (plen + f)                 # read s, write f per message
    put_avg_ms = statistics.mean(put_ms)
    peaks, src_kind = load_peaks()
    achieved = put_bytes / (put_avg_ms / 1e3) / 1e9

    # e2e: host payloads (pinned) -> device every step, put + consume, views -> host
    host_src = torch.empty(m * stride, dtype=torch.uint8).pin_memory()
    host_src.copy_(src[: m * stride].cpu())
    host_views = torch.empty(m * 128, dtype=torch.uint8).pin_memory()
    e_steps = max(3, min(args.steps, 50))
    for i in range(2):
        src[: m * stride].copy_(host_src, non_blocking=True)
        step(0)
        host_views.copy_(views, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e_steps):
        src[: m * stride].copy_(host_src, non_blocking=True)
        step(0)
        host_views.copy_(views, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e = m * plen * e_steps / (e2e_ms / 1e3) / 1e9

    cpu_gbs, cpu_msgs, cpu_s = oracle_throughput([plen] * m, Rb, N, budget_s=args.cpu_budget)

    R.ring_detach(peer)
    R.ring_destroy(ring)
    return {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C2 (BASELINE.json configs[1]): 1xB200 same-GPU double ring, 64 slots x 1 MiB "
                               "(R=64 MiB), 1,048,512-B payloads (footprint 1 MiB), put batch -> consume batch",
                   "R_bytes": Rb, "n_slots": N, "msgs_per_step": m, "payload_bytes": plen,
                   "l2": "inputs larger than L2 (4 x 64 MiB rotating source sets + 64 MiB ring)",
                   "consume_mode": "view (zero copy)", "parallelism": "replicas only (1 ring)"},
        "msgs_per_s": round(m * args.steps / (ms / 1e3), 1),
        "latency_us": {"p50": round(float(np.percentile(lat_us, 50)), 2),
                       "p99": round(float(np.percentile(lat_us, 99)), 2),
                       "what": "t_visible - t_put of the last step's 64 messages (batched put: includes queueing)"},
        "kernels_ms": {"put_avg": round(put_avg_ms, 5), "consume_avg": round(statistics.mean(get_ms), 5)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": None,
                     "kernel": "put_kernel", "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src_kind})",
                     "algorithmic_bytes_per_launch": put_bytes},
        "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": m * stride,
                "d2h_bytes_per_step": m * 128},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "cpu_baseline": {"value": round(cpu_gbs, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{cpu_msgs} x 1,048,512-B messages through the Python oracle ring "
                                   f"(R=64 MiB, N=64) in {cpu_s:.1f} s"},
    }


# ---------------------------------------------------------------------------------------
# N >= 2: ring of pairs over NVLink (C3-shaped messages)
# ---------------------------------------------------------------------------------------
def bench_pairs(args, rank, world):
    import torch
    import torch.distributed as dist
    import synth
    from paper_2601_20655_b200 import ring as R

    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    Rb, N = 64 << 20, 64
    m = args.msgs_per_step or 32
    lens = [synth.wan_bytes("umt5_emb"), synth.wan_bytes("latent_480p")]
    ring = R.ring_create(dev, Rb, N, 1, 0)
    handles = [None] * world
    dist.all_gather_object(handles, R.ring_export(ring))
    nxt = (rank + 1) % world
    peer, mh = R.ring_attach_peer(handles[nxt], dev, 0)
    if args.copy_ctas or args.threads:
        R.ring_peer_config(peer, args.copy_ctas, args.threads, 0)
    mirrors = [None] * world
    dist.all_gather_object(mirrors, mh)
    R.ring_bind_mirror(ring, 0, mirrors[(rank - 1) % world])
    dist.barrier()
    sets = 2
    stride = 4194304
    src = torch.empty(sets * m * stride, dtype=torch.uint8, device="cuda")
    d_msgs = []
    for s in range(sets):
        srcs, ln = [], []
        for q in range(m):
            k = s * m + q
            kind = ("umt5_emb", "latent_480p")[k % 2]
            shape, distn = synth.WAN_SHAPES[kind]
            b = synth.bf16_tensor_bytes(synth.SEED_BASE + 3, rank, k, shape, distn)
            src[k * stride: k * stride + b.size] = torch.from_numpy(b)
            srcs.append(src.data_ptr() + k * stride)
            ln.append(b.size)
        hdr = [synth.header_fields(synth.SEED_BASE + 3, rank, s * m + q) for q in range(m)]
        a = R.make_msgs(srcs, ln, [h[0] for h in hdr], [h[1] for h in hdr], [7] * m, [2] * m)
        d_msgs.append(torch.from_numpy(a.view(np.uint8).copy()).cuda())
    payload_step = sum(lens[q % 2] for q in range(m))
    status = torch.zeros(m, dtype=torch.int32, device="cuda")
    views = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
    sp = torch.cuda.Stream()
    sc = torch.cuda.Stream()

    def step(i):
        R.ring_consume(ring, m, views, None, 0, 0, sc)
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    dist.barrier()
    clk = Clocks(dev) if rank == 0 else None
    if clk:
        clk.start()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = R.ring_launch_count()
    t0c, t0p = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t1c, t1p = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0c.record(sc)
    t0p.record(sp)
    for i in range(args.steps):
        step(args.warmup + i)
    t1c.record(sc)
    t1p.record(sp)
    torch.cuda.synchronize()
    launches = R.ring_launch_count() - l0
    ms = max(t0c.elapsed_time(t1c), t0p.elapsed_time(t1p), t0c.elapsed_time(t1p), t0p.elapsed_time(t1c))
    dist.barrier()
    clocks = clk.stop() if clk else None
    ok = bool((status == 0).all().item()) and bool((R.parse_views(views.cpu().numpy())["status"] == 0).all())
    v = R.parse_views(views.cpu().numpy())
    t_put = np.frombuffer(v["header"][:, 56:64].tobytes(), dtype="<u8")
    lat_us = ((v["t_visible"].astype(np.int64) - t_put.astype(np.int64)) / 1e3).tolist()
    t = torch.tensor([ms, 0.0 if ok else 1.0, float(launches)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    lats = [None] * world
    dist.all_gather_object(lats, lat_us)
    ms_max, bad = float(t[0]), float(t[1])
    dist.barrier()
    R.ring_detach(peer)
    dist.barrier()
    R.ring_destroy(ring)
    if rank != 0:
        return None
    all_lat = np.array([x for l in lats for x in l])
    value = payload_step * args.steps * world / (ms_max / 1e3) / 1e9
    per_gpu = value / world
    return {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C3-shaped ring of pairs: rank r -> ring on rank (r+1)%N over NVLink, Wan2.1 "
                               "umT5 emb 512x4096 bf16 / 480p latent 16x21x60x104 bf16 alternating",
                   "R_bytes": Rb, "n_slots": N, "msgs_per_step_per_rank": m,
                   "l2": "inputs larger than L2 per rank (2 x 128 MiB source sets)",
                   "parallelism": f"{world} concurrent SPSC rings (egress+ingress per GPU)"},
        "per_gpu_gbs": round(per_gpu, 2),
        "nvlink_frac_of_900": round(per_gpu / NVLINK_NOMINAL, 4),
        "latency_us": {"p50": round(float(np.percentile(all_lat, 50)), 2),
                       "p99": round(float(np.percentile(all_lat, 99)), 2),
                       "what": "t_visible - t_put (globaltimer; streaming, loaded)"},
        "roofline": {"bound": "nvlink", "achieved": round(per_gpu, 1), "peak": NVLINK_PEAK_MEASURED, "unit": "GB/s",
                     "frac": round(per_gpu / NVLINK_PEAK_MEASURED, 4), "traffic": None, "kernel": "put_kernel",
                     "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction (900 nominal)"},
        "gpu_launches": int(t[2]) * world,
        "clocks": clocks,
        "ok": bad == 0.0,
    }


def reference_arm(args):
    """--impl reference: the CPU oracle as it stands, on the host cores, on our
    arm's config / metric / unit; each step a bounded sample of the workload."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    if world == 1:
        lens, Rb, N, wl = [1048512] * 16, 64 << 20, 64, "C2 sample: 16 x 1,048,512-B messages per step"
    else:
        lens, Rb, N, wl = [4194304, 4193280] * 4, 64 << 20, 64, "C3 sample: 8 x ~4 MiB messages per step"
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        gbs, nm, dt = oracle_throughput(lens, Rb, N, budget_s=0.0, seed=i)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = sum(lens) * len(times) / tot / 1e9
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / len(times) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl, "R_bytes": Rb, "n_slots": N},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": wl + " through oracle/ring.py (single thread)"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--msgs-per-step", type=int, default=0)
    ap.add_argument("--copy-ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if not args.steps:
            args.steps = 5
        out = reference_arm(args)
        if out:
            print(json.dumps(out), flush=True)
        return
    if world == 1:
        if not args.steps:
            args.steps = 2000
        out = bench_c2(args)
        print(json.dumps(out), flush=True)
        return
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    if not args.steps:
        args.steps = 200
    dist.init_process_group("nccl", device_id=None)
    try:
        out = bench_pairs(args, rank, world)
        if out:
            print(json.dumps(out), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
