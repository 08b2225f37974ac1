#!/usr/bin/env python
"""Benchmark of the double-ring tensor transport (BASELINE.json metric:
"ring transfer GB/s per GPU vs 900 GB/s NVLink; p50/p99 msg latency at 1/2/4/8 GPU").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

N = 1 -> BASELINE.json configs[1] (C2): a same-GPU ring of 64 slots x 1 MiB
(R = 64 MiB), 1,048,512-B payloads (footprint exactly 1 MiB).  One step = one
pass of the whole hot path over one batch: ring_put_batch of 64 messages
(claim, header + CRC, copy, publish) then ring_consume of the 64 entries (poll,
slot + header read, CRC verify, release + credit), in stream order on one GPU
(two kernels spinning on each other must never share a GPU).
N >= 2 -> C3-shaped messages (umT5 embeddings 4,194,304 B / 480p latents
4,193,280 B, alternating) over NVLink: rank r puts into the ring on rank
(r+1) % N while consuming its own ring (fed by rank r-1), both streaming
concurrently with credit flowing back; weak scaling (fixed work per GPU).
Handles are exchanged over a gloo group of torch.distributed (plumbing only:
no collective and no NCCL on the data path).

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
C3_LENS = (4194304, 4193280)   # umT5 embeddings 512x4096 bf16 / 480p latents 16x21x60x104 bf16


def log(*a):
    print(f"[bench r{os.environ.get('RANK', '0')} {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic(name: str, kernel: str = "put_kernel"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from
    the committed summary of one `ncu --set full` capture of the same bench
    command (profiles/<name>, written by tools/ncu_summary.py), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            for d in json.load(f):
                if kernel in d.get("kernel", "") and "dram_traffic_bytes" in d:
                    return int(d["dram_traffic_bytes"])
    except (OSError, ValueError):
        pass
    return None


def pct(x, q):
    return round(float(np.percentile(np.asarray(x, dtype=np.float64), q)), 2) if len(x) else None


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
def oracle_inputs(payload_lens, seed: int = 0):
    import synth
    from oracle.ring import Msg
    return [Msg(n, synth.payload_bytes(synth.SEED_BASE + seed, 0, q, n).tobytes(), bytes(16), 0, 7, 1)
            for q, n in enumerate(payload_lens)]


def oracle_pass(msgs, R_bytes, N_slots):
    """One pass of the CPU oracle (oracle/ring.py: one producer, draining consumer)."""
    from oracle.ring import Layout, Sim, run
    sim = Sim(Layout(R_bytes, N_slots), {0: msgs}, mpsc=False, block=True, depth=1, check=False)
    run(sim, policy="drain")
    return sim


def cpu_baseline(R_bytes, N_slots, producers, per, lo, hi, budget_s: float, what: str):
    """The CPU baseline of BASELINE.md §6: oracle/ring_threaded.cpp (the same
    protocol over host memory, one pinned thread per producer plus the
    consumer, memcpy payloads, std::atomic acquire/release) on a bounded sample
    of the workload; the single-thread Python stepper's rate is kept beside it."""
    from oracle import threaded as T
    r = T.run(R_bytes, N_slots, producers, per, lo, hi, 20260120)
    py = cpu_baseline_python([lo] * 16 if lo == hi else [lo, hi] * 8, R_bytes, N_slots, budget_s)
    return {"value": round(r["gbs"], 4), "unit": UNIT, "cores": r["threads"], "kind": "oracle-threaded",
            "sample": f"{r['messages']} messages ({what}) through oracle/ring_threaded.cpp: {producers} producer "
                      f"thread(s) + 1 consumer thread, pinned, R={R_bytes >> 20} MiB, N={N_slots}, {r['seconds']:.2f} s"
                      f"{'' if r['bad'] == 0 else ', DELIVERY ERRORS'}",
            "msgs_per_s": r["msgs_per_s"], "p50_us": r["p50_us"], "p99_us": r["p99_us"],
            "cpu_model": r["cpu_model"], "host_cpus": os.cpu_count(), "delivery_ok": r["bad"] == 0,
            "python_oracle": py}


def cpu_baseline_python(payload_lens, R_bytes, N_slots, budget_s: float):
    msgs = oracle_inputs(payload_lens)
    t0 = time.perf_counter()
    n = 0
    while True:
        oracle_pass(msgs, R_bytes, N_slots)
        n += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s:
            break
    return {"value": round(sum(payload_lens) * n / dt / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{n} x {len(payload_lens)} messages of {payload_lens[0]:,} B through oracle/ring.py "
                      f"(R={R_bytes >> 20} MiB, N={N_slots}), single thread, {dt:.1f} s"}


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
    if args.ctas or args.threads or args.copy_mode:
        R.ring_peer_config(peer, args.ctas, args.threads, args.copy_mode)
    engine = bool(args.engine) and not args.copy_mode
    put_flags = R.RING_ASYNC if engine else 0
    stride = (plen + 255) // 256 * 256
    src = torch.empty(sets * m * stride, dtype=torch.uint8, device="cuda")
    for k in range(sets * m):
        src[k * stride: k * stride + plen] = torch.from_numpy(synth.payload_bytes(synth.SEED_BASE + 2, 0, k, plen))
    d_msgs = []
    for s in range(sets):
        srcs = [src.data_ptr() + (s * m + q) * stride for q in range(m)]
        hdr = [synth.header_fields(synth.SEED_BASE + 2, 0, s * m + q) for q in range(m)]
        a = R.make_msgs(srcs, [plen] * m, [h[0] for h in hdr], [h[1] for h in hdr], [7] * m, [1] * m)
        d_msgs.append(torch.from_numpy(a.view(np.uint8).copy()).cuda())
    status = torch.zeros(m, dtype=torch.int32, device="cuda")
    views = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
    # Producer and consumer kernels on separate streams (configs[1]), streaming:
    # consume(s) drains batch s while put(s) writes it, and put(s+1) (after
    # put(s) on its stream) takes credit as consume(s) releases entries.  The
    # waits form a chain, never a cycle: put(s+1) -> consume(s) -> put(s), and
    # the consumer kernel is one warp, so it is always resident next to a put.
    # With --no-overlap, put(s+1) waits for consume(s) to finish (event).
    sp, sc = torch.cuda.Stream(), torch.cuda.Stream()
    stream = sp
    def sync(limit_s: float = 60.0):
        # never torch.cuda.synchronize() while the engine runs: it waits for the
        # resident engine kernel, which only exits when stopped.  A stream that
        # does not finish within limit_s ends the bench with a diagnosis
        # (every device spin has its own timeout, so this means a kernel that
        # cannot be scheduled).
        t0 = time.time()
        for s_ in (sp, sc, torch.cuda.current_stream()):
            while not s_.query():
                if time.time() - t0 > limit_s:
                    log(f"C2: stream {s_} stuck; engine {R.ring_peer_engine_state(peer) if engine else None}; "
                        f"sp={sp.query()} sc={sc.query()} main={torch.cuda.current_stream().query()}")
                    os._exit(3)
                time.sleep(0.0002)

    if engine:
        R.ring_peer_engine_start(peer, sp)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(min(args.steps, 64))]
    consumed = [torch.cuda.Event()]           # holder: events recorded in a graph capture stay in it
    consumed[0].record(sc)
    capturing = [False]

    def step(i, timed=None, before_put=None):
        if capturing[0]:
            if args.no_overlap:
                sp.wait_stream(sc)                # graph edge: put(s+1) after consume(s)
        elif args.no_overlap or before_put is not None:
            sp.wait_event(consumed[0])            # the previous batch has been consumed
        if before_put is not None:
            before_put()
        if timed is not None:
            timed[0].record(sp)
        R.ring_put_batch(peer, d_msgs[i % sets], m, put_flags, status, sp)
        if timed is not None:
            timed[1].record(sp)
            timed[2].record(sc)
        R.ring_consume(ring, m, views, None, 0, 0, sc)
        if timed is not None:
            timed[3].record(sc)
        if not capturing[0]:
            consumed[0].record(sc)

    log(f"C2: engine={engine}, warm-up")
    for i in range(args.warmup):
        step(i)
    if engine:
        R.ring_peer_engine_wait(peer, sp)
    sync()
    log("C2: warm-up done")
    assert (status == 0).all().item(), "put failed in warm-up"
    assert (R.parse_views(views.cpu().numpy())["status"] == 0).all(), "consume failed in warm-up"

    # Per-kernel durations: an eager pass with events around every launch.
    n_ev = min(len(ev), 64)
    for i in range(n_ev):
        step(i, ev[i])
    if engine:
        R.ring_peer_engine_wait(peer, sp)
    sync()
    put_ms = [a.elapsed_time(b) for a, b, c, d in ev[:n_ev]]
    get_ms = [c.elapsed_time(d) for a, b, c, d in ev[:n_ev]]

    # Timed region: eager launches (the host issues a step in ~15 us, the GPU
    # takes ~36 us), or with --graph a CUDA graph of G steps replayed; G is even,
    # so each launch context keeps alternating its two counter sets.
    G = 16
    graph = None
    if args.graph:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        capturing[0] = True
        with torch.cuda.graph(graph, stream=cap, capture_error_mode="relaxed"):
            sp.wait_stream(cap)
            sc.wait_stream(cap)
            for i in range(G):
                step(i)
            cap.wait_stream(sp)
            cap.wait_stream(sc)
        capturing[0] = False
        consumed[0] = torch.cuda.Event()
        consumed[0].record(sc)
        for _ in range(2):
            graph.replay()
        sync()
        assert (status == 0).all().item(), "put failed in graph warm-up"
    steps = (args.steps + G - 1) // G * G if graph is not None else args.steps
    log("C2: timed region")
    clk = Clocks(dev)
    clk.start()
    l0 = R.ring_launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the put kernel's average launch duration, live over the timed region: CUDA
    # events on its own stream sp around the whole loop (sp carries only the
    # put launches, back to back; events between launches would break the
    # back-to-back launch and cost ~2-3 us each)
    sp_start, sp_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sync()
    main = torch.cuda.current_stream()
    t_start.record(main)
    if graph is not None:
        for _ in range(steps // G):
            graph.replay()
    else:
        sp.wait_stream(main)
        sc.wait_stream(main)
        sp_start.record(sp)
        for i in range(steps):
            step(args.warmup + i)
        sp_end.record(sp)
        if engine:
            R.ring_peer_engine_wait(peer, sp)
        main.wait_stream(sp)
        main.wait_stream(sc)
    t_end.record(main)
    sync()
    launches = (2 * steps) if graph is not None else R.ring_launch_count() - l0
    clocks = clk.stop()
    ms = t_start.elapsed_time(t_end)
    args.steps = steps
    assert (status.cpu() == 0).all()
    v = R.parse_views(views.cpu().numpy())
    assert (v["status"] == 0).all()
    # repetitions (5 runs, median with min / max): the timed
    # region above plus 4 more passes of the same K steps, eager launches
    rep_gbs = [m * plen * steps / (ms / 1e3) / 1e9]
    for r in range(4):
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sync()
        r0.record(main)
        sp.wait_stream(main)
        sc.wait_stream(main)
        for i in range(steps):
            step(i)
        if engine:
            R.ring_peer_engine_wait(peer, sp)
        main.wait_stream(sp)
        main.wait_stream(sc)
        r1.record(main)
        sync()
        rep_gbs.append(m * plen * steps / (r0.elapsed_time(r1) / 1e3) / 1e9)
    assert (status.cpu() == 0).all()
    # loaded latency, pooled over >= 1,000 messages: a further
    # streaming pass (outside the timed region) with one view buffer per step,
    # first 10 % dropped as warm-up
    lat_steps = 20
    lviews = [torch.zeros(m * 128, dtype=torch.uint8, device="cuda") for _ in range(lat_steps)]
    for i in range(lat_steps):
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)
        R.ring_consume(ring, m, lviews[i], None, 0, 0, sc)
    sync()
    lat_all = []
    for lv in lviews:
        vv = R.parse_views(lv.cpu().numpy())
        tp = np.frombuffer(vv["header"][:, 56:64].tobytes(), dtype="<u8").astype(np.int64)
        lat_all += ((vv["t_visible"].astype(np.int64) - tp) / 1e3).tolist()
    lat_us = lat_all[len(lat_all) // 10:]
    del lviews

    # unloaded latency: one message in flight, put -> consume,
    # t_visible - t_put (t_put: the put's leader takes the message up, before
    # the claim); 4 KiB, the C2 payload and a C3-sized 4 MiB payload
    log("C2: unloaded latency, flag round trip, small messages")
    unl = {}
    one_v = torch.zeros(128, dtype=torch.uint8, device="cuda")
    one_st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for size in (4096, plen, 4194304 - 64):
        one = R.make_msgs([src.data_ptr()], [size], [bytes(16)], [0], [7], [1])
        d_one = torch.from_numpy(one.view(np.uint8).copy()).cuda()
        lat = []
        for i in range(110):
            R.ring_consume(ring, 1, one_v, None, 0, 0, sc)     # the consumer waits for it
            R.ring_put_batch(peer, d_one, 1, 0, one_st, sp)
            sync()
            vv = R.parse_views(one_v.cpu().numpy())
            tp = int(np.frombuffer(vv["header"][0, 56:64].tobytes(), dtype="<u8")[0])
            lat.append((int(vv["t_visible"][0]) - tp) / 1e3)
        unl[size] = lat[10:]
    # flag round trip between two kernels on this GPU: the
    # small-message roofline msgs/s <= 1 / (t_RTT * k), k = 1 for SPSC
    rtt = R.ring_probe_rtt(dev, dev, 2000)
    # small messages streaming: 4 KiB, 1,024 per step (view consume)
    small_m, small_steps = 1024, 20
    smalls = R.make_msgs([src.data_ptr() + 4096 * q for q in range(small_m)], [4096] * small_m,
                         [bytes(16)] * small_m, [0] * small_m, [7] * small_m, [1] * small_m)
    d_small = torch.from_numpy(smalls.view(np.uint8).copy()).cuda()
    small_st = torch.zeros(small_m, dtype=torch.int32, device="cuda")
    small_v = torch.zeros(small_m * 128, dtype=torch.uint8, device="cuda")
    for i in range(3):
        R.ring_put_batch(peer, d_small, small_m, 0, small_st, sp)
        R.ring_consume(ring, small_m, small_v, None, 0, 0, sc)
    sync()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(main)
    sp.wait_stream(main)
    sc.wait_stream(main)
    for i in range(small_steps):
        R.ring_put_batch(peer, d_small, small_m, 0, small_st, sp)
        R.ring_consume(ring, small_m, small_v, None, 0, 0, sc)
    main.wait_stream(sp)
    main.wait_stream(sc)
    s1.record(main)
    sync()
    small_ok = bool((small_st.cpu() == 0).all()) and bool((R.parse_views(small_v.cpu().numpy())["status"] == 0).all())
    small_msgs_s = small_m * small_steps / (s0.elapsed_time(s1) / 1e3)

    payload = m * plen * args.steps
    value = payload / (ms / 1e3) / 1e9
    f = R.ring_footprint(plen)
    put_bytes = m * (plen + f)                 # read s, write f per message
    # engine: one resident put grid; its time per batch in the stream IS the step
    # (the events around a doorbell would only time the doorbell)
    if engine:
        put_avg_ms = ms / args.steps
        put_avg_src = "engine: timed region / steps"
    elif graph is None:
        put_avg_ms = sp_start.elapsed_time(sp_end) / args.steps
        put_avg_src = f"CUDA events on the put stream around the {args.steps} put launches of the timed region"
    else:
        put_avg_ms = statistics.mean(put_ms)
        put_avg_src = "CUDA events around 64 put launches of a separate eager pass (graph mode)"
    peaks, src_kind = load_peaks()
    achieved = put_bytes / (put_avg_ms / 1e3) / 1e9

    # e2e: host payloads (pinned) -> device every step, put + consume, views -> host
    host_src = torch.empty(m * stride, dtype=torch.uint8).pin_memory()
    host_src.copy_(src[: m * stride].cpu())
    host_views = torch.empty(m * 128, dtype=torch.uint8).pin_memory()
    e_steps = max(3, min(args.steps, 50))

    def h2d():
        with torch.cuda.stream(sp):
            src[: m * stride].copy_(host_src, non_blocking=True)

    def e2e_step():
        step(0, before_put=h2d)              # source set 0 = the buffer just copied in
        with torch.cuda.stream(sc):
            host_views.copy_(views, non_blocking=True)

    for i in range(2):
        e2e_step()
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e_steps):
        e2e_step()
    sp.wait_stream(sc)
    e1.record(stream)
    sync()
    e2e = m * plen * e_steps / (e0.elapsed_time(e1) / 1e3) / 1e9

    # secondary line: copy-out consume (the consumer copies every payload out of
    # the ring before releasing it: 4 bytes of HBM traffic per payload byte)
    dst = torch.empty(m * plen, dtype=torch.uint8, device="cuda")
    co_steps = max(4, min(args.steps, 400))
    for i in range(3):
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)
        R.ring_consume(ring, m, views, dst, plen, 0, sc)
    sync()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(main)
    sp.wait_stream(main)
    sc.wait_stream(main)
    for i in range(co_steps):
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)
        R.ring_consume(ring, m, views, dst, plen, 0, sc)
    main.wait_stream(sp)
    main.wait_stream(sc)
    c1.record(main)
    sync()
    co_ms = c0.elapsed_time(c1)
    co_ok = bool((status == 0).all().item()) and bool((R.parse_views(views.cpu().numpy())["status"] == 0).all())
    co_launch = m * plen * co_steps / (co_ms / 1e3) / 1e9
    # the same with the persistent put engine feeding the ring (one resident put
    # grid: the next batch's copies overlap the current batch's copy-out)
    co_engine, co_eng_ms, co_eng_ok = None, None, None
    if not engine and not args.copy_mode:      # (the engine drives LSU copy warps only)
        R.ring_peer_engine_start(peer, sp)
        for i in range(3):
            R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)
            R.ring_consume(ring, m, views, dst, plen, 0, sc)
        R.ring_peer_engine_wait(peer, sp)
        sync()
        c2, c3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c2.record(main)
        sp.wait_stream(main)
        sc.wait_stream(main)
        for i in range(co_steps):
            R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)
            R.ring_consume(ring, m, views, dst, plen, 0, sc)
        R.ring_peer_engine_wait(peer, sp)
        main.wait_stream(sp)
        main.wait_stream(sc)
        c3.record(main)
        sync()
        co_eng_ms = c2.elapsed_time(c3)
        co_eng_ok = bool((status == 0).all().item()) and \
            bool((R.parse_views(views.cpu().numpy())["status"] == 0).all())
        R.ring_peer_engine_stop(peer, sp)
        sync()
        co_engine = m * plen * co_steps / (co_eng_ms / 1e3) / 1e9
    best_engine = co_engine is not None and co_eng_ok and co_engine > co_launch
    copy_out = {"value": round(co_engine if best_engine else co_launch, 2), "unit": UNIT,
                "put": "persistent engine" if best_engine else "one put launch per step",
                "ms_per_step": round((co_eng_ms if best_engine else co_ms) / co_steps, 5), "steps": co_steps,
                "ok": co_ok and (co_eng_ok is not False),
                "launches_gbs": round(co_launch, 2), "engine_gbs": round(co_engine, 2) if co_engine else None,
                "roofline_payload_gbs": round(peaks["hbm_gbs"] / 4, 1),
                "what": "same stream with ring_consume copying each payload out (copy-out mode, SURVEY.md d-3); "
                        "value = the better of the put launched per step and the persistent put engine"}
    del dst

    if engine:
        R.ring_peer_engine_stop(peer, sp)
        sync()
    cpu = cpu_baseline(Rb, N, 1, 2000, plen, plen, args.cpu_budget, "C2 shape: 1,048,512-B payloads")
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
                   "consume_mode": "view (zero copy)",
                   "put": "persistent engine, one async doorbell per batch" if engine else "one put launch per batch", "parallelism": "replicas only (1 ring)",
                   "streams": "put on one stream, consume on another; consume(s) overlaps put(s), "
                              "put(s+1) takes credit as consume(s) releases entries (device-side waits)"},
        "msgs_per_s": round(m * args.steps / (ms / 1e3), 1),
        "latency_us": {"p50": pct(lat_us, 50), "p99": pct(lat_us, 99), "samples": len(lat_us),
                       "what": "loaded: t_visible - t_put over 20 streamed steps (first 10 % dropped; same GPU "
                               "clock; batched put, so it includes the wait behind earlier messages of the batch)"},
        "repetitions": {"n": len(rep_gbs), "median": round(statistics.median(rep_gbs), 2),
                        "min": round(min(rep_gbs), 2), "max": round(max(rep_gbs), 2), "unit": UNIT,
                        "what": "the timed region plus 4 more passes of the same K steps"},
        "latency_unloaded_us": {
            f"{s}B": {"p50": pct(l, 50), "p99": pct(l, 99), "samples": len(l)} for s, l in unl.items()} | {
            "what": "one message in flight (the consumer already waiting), t_visible - t_put, t_put = the "
                    "put leader taking the message up (before the claim); first 10 of 110 dropped"},
        "small_messages": {"size": 4096, "msgs_per_s": round(small_msgs_s, 1), "ok": small_ok,
                           "rtt_min_us": round(rtt["rtt_min_ns"] / 1e3, 3),
                           "rtt_p50_us": round(rtt["rtt_p50_ns"] / 1e3, 3),
                           "unbatched_bound_msgs_per_s": round(1e9 / rtt["rtt_p50_ns"], 1),
                           "ratio_to_unbatched_bound": round(small_msgs_s / (1e9 / rtt["rtt_p50_ns"]), 3),
                           "what": "4 KiB messages, 1,024 per put launch, streamed 20 launches.  SURVEY.md d-3's "
                                   "bound 1 / (t_RTT * k), k = 1 (SPSC), holds for one message per publication; "
                                   "the put publishes a run of complete entries with one fence, so a batch "
                                   "exceeds it by the run length.  t_RTT = median in-run flag round trip between "
                                   "two kernels on this GPU (ring_probe_rtt, system scope)"},
        "kernels_ms": {"put_avg": round(put_avg_ms, 5), "put_avg_source": put_avg_src,
                       "put_avg_events_per_launch": round(statistics.mean(put_ms), 5),
                       "consume_avg": round(statistics.mean(get_ms), 5)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": ncu_traffic("r02b_ncu_put_c2.json"),
                     "traffic_source": "profiles/r02b_ncu_put_c2.json (ncu --set full, put_kernel, same config)",
                     "kernel": "put_kernel<0> (persistent engine: time per batch = step time)" if engine
                     else "put_kernel<0> (average launch duration on its stream over the timed region; "
                          "ncu launch list: put 66 % of kernel time, profiles/r02b_ncu_launches_c2.json)",
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src_kind})",
                     "algorithmic_bytes_per_launch": put_bytes},
        "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": m * stride,
                "d2h_bytes_per_step": m * 128},
        "copy_out": copy_out,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "cpu_baseline": cpu,
    }


# ---------------------------------------------------------------------------------------
# N >= 2: ring of pairs over NVLink (C3-shaped messages)
# ---------------------------------------------------------------------------------------
def bench_pairs(args, rank, world, grp):
    import torch
    import torch.distributed as dist
    import synth
    from paper_2601_20655_b200 import ring as R

    from paper_2601_20655_b200 import topology as T
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    # 256 MiB rings, 128 messages (512 MiB) per put / consume launch: per-launch
    # start and drain amortised over ~0.8 ms (64 MiB / 32 per launch: -9 %,
    # profiles/r02_c3_sweep.txt)
    Rb, N = (args.ring_mb or 256) << 20, 64
    m = args.msgs_per_step or 128
    pull = bool(args.pull)
    own = None
    if args.pull == 2:
        # split placement: the ring's control words + header copies on this rank,
        # its buffer region on the previous rank's GPU (the producer writes
        # locally, this rank pulls each payload over NVLink)
        prev, nxt = (rank - 1) % world, (rank + 1) % world
        ndev = torch.cuda.device_count()
        ring = R.ring_create_split(dev, (dev - 1) % ndev, Rb, N, 1, 0)
        hs = [None] * world
        dist.all_gather_object(hs, R.ring_export(ring), group=grp)
        peer, mh = R.ring_attach_peer(hs[nxt], dev, 0)
        mhs = [None] * world
        dist.all_gather_object(mhs, mh, group=grp)
        R.ring_bind_mirror(ring, 0, mhs[prev])
        if args.cons_ctas or args.cons_threads:
            R.ring_config(ring, args.cons_ctas, args.cons_threads)
        dist.barrier(group=grp)
    elif pull:
        # pull placement: each rank's egress ring lives in its OWN memory; the
        # next rank opens it and pulls every payload over NVLink (ring_open)
        own = R.ring_create(dev, Rb, N, 1, 0)
        h = R.ring_export(own)
        peer, mh = R.ring_attach_peer(h, dev, 0)
        hs = [None] * world
        dist.all_gather_object(hs, (h, mh), group=grp)
        prev = (rank - 1) % world
        ring = R.ring_open(hs[prev][0], dev)
        R.ring_bind_mirror(ring, 0, hs[prev][1])
        if args.cons_ctas or args.cons_threads:
            R.ring_config(ring, args.cons_ctas, args.cons_threads)
        dist.barrier(group=grp)
    else:
        wired = T.wire(T.plan_pairs(world, Rb, N), rank, world, grp, device=dev,
                       create=lambda s, d: R.ring_create(d, s.data_bytes, s.n_slots, s.max_producers, 0),
                       export=R.ring_export, attach=R.ring_attach_peer, bind=R.ring_bind_mirror)
        ring = wired.rings[f"in{rank}"]
        peer = wired.peers[f"in{(rank + 1) % world}"]
    if args.ctas or args.threads or args.copy_mode:
        R.ring_peer_config(peer, args.ctas, args.threads, args.copy_mode)
    offsets = [None] * world
    dist.all_gather_object(offsets, R.ring_clock_offset_ns(dev), group=grp)
    log("rings attached; clock offsets (gpu - host, ns):", offsets)
    sets, stride = 2, 4194304
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
    payload_step = sum(C3_LENS[q % 2] for q in range(m))
    status = torch.zeros(m, dtype=torch.int32, device="cuda")
    views = torch.zeros(m * 128, dtype=torch.uint8, device="cuda")
    pull_dst = torch.empty(m * stride, dtype=torch.uint8, device="cuda") if pull else None
    sp, sc = torch.cuda.Stream(), torch.cuda.Stream()

    def step(i):
        # consumer first: it waits for data.  Pull: its copy-out brings every
        # payload over NVLink into pull_dst (push: the put already wrote it here)
        R.ring_consume(ring, m, views, pull_dst, stride if pull else 0, 0, sc)
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)

    def latencies():
        v = R.parse_views(views.cpu().numpy())
        t_put = np.frombuffer(v["header"][:, 56:64].tobytes(), dtype="<u8").astype(np.int64)
        prev = (rank - 1) % world
        # both stamps on the host clock: t - offset(gpu)
        return (((v["t_visible"].astype(np.int64) - offsets[rank]) - (t_put - offsets[prev])) / 1e3).tolist(), v

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ok_w = bool((status == 0).all().item()) and bool((latencies()[1]["status"] == 0).all())
    log("warm-up done, ok =", ok_w)
    dist.barrier(group=grp)
    clk = Clocks(dev) if rank == 0 else None
    if clk:
        clk.start()
    dist.barrier(group=grp)
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
    dist.barrier(group=grp)
    clocks = clk.stop() if clk else None
    _, v = latencies()
    ok = bool((status == 0).all().item()) and bool((v["status"] == 0).all())
    log(f"timed region {ms:.3f} ms, ok = {ok}")
    # sampled payload check: 4 messages of the last timed step, byte for byte
    # against the producer's seeded tensors (push: in the ring, released but
    # not yet overwritten -- the step's last 32 messages, the ring holds 63;
    # pull / split: in the copy-out buffer)
    last, prev_r = args.warmup + args.steps - 1, (rank - 1) % world
    mism, sampled = 0, 0
    for q in sorted({max(0, m - 32), max(0, m - 16), max(0, m - 2), m - 1}):
        k = (last % sets) * m + q
        shape, distn = synth.WAN_SHAPES[("umt5_emb", "latent_480p")[k % 2]]
        exp = synth.bf16_tensor_bytes(synth.SEED_BASE + 3, prev_r, k, shape, distn).tobytes()
        n = int(v[q]["len"])
        got = (pull_dst[q * stride: q * stride + n].cpu().numpy().tobytes() if pull
               else R.ring_read_data(ring, int(v[q]["offset"]), n))
        sampled += 1
        mism += int(got != exp)
    ok = ok and mism == 0
    # loaded latency pooled over further streamed steps (outside the timed
    # region), one view buffer per step, first 10 % dropped
    lat_steps = 20
    lviews = [torch.zeros(m * 128, dtype=torch.uint8, device="cuda") for _ in range(lat_steps)]
    dist.barrier(group=grp)
    for i in range(lat_steps):
        R.ring_consume(ring, m, lviews[i], pull_dst, stride if pull else 0, 0, sc)
        R.ring_put_batch(peer, d_msgs[i % sets], m, 0, status, sp)
    torch.cuda.synchronize()
    lat_loaded = []
    prev_rank = (rank - 1) % world
    for lv in lviews:
        vv = R.parse_views(lv.cpu().numpy())
        tp = np.frombuffer(vv["header"][:, 56:64].tobytes(), dtype="<u8").astype(np.int64)
        lat_loaded += (((vv["t_visible"].astype(np.int64) - offsets[rank]) - (tp - offsets[prev_rank])) / 1e3).tolist()
    lat_loaded = lat_loaded[len(lat_loaded) // 10:]
    del lviews

    # unloaded latency: one message in flight (consumer waiting first), 4 KiB and one C3 tensor
    unl = {}
    for size in (4096, C3_LENS[0]):
        lat = []
        one = torch.from_numpy(R.make_msgs([src.data_ptr()], [size], [bytes(16)], [0], [7], [2]).view(np.uint8).copy()).cuda()
        for it in range(args.lat_iters):
            dist.barrier(group=grp)
            R.ring_consume(ring, 1, views, pull_dst, stride if pull else 0, 0, sc)
            time.sleep(0.0002)
            R.ring_put_batch(peer, one, 1, 0, status, sp)
            torch.cuda.synchronize()
            lv, vv = latencies()
            if it >= args.lat_iters // 10 and int(vv["status"][0]) == 0:
                lat.append(lv[0])
        unl[size] = lat

    # e2e: host payloads (pinned) -> device each step, then the step, views -> host
    host_src = torch.empty(m * stride, dtype=torch.uint8).pin_memory()
    host_src.copy_(src[: m * stride].cpu())
    host_views = torch.empty(m * 128, dtype=torch.uint8).pin_memory()
    e_steps = max(3, min(args.steps, 20))
    dist.barrier(group=grp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sp)
    for i in range(e_steps):
        with torch.cuda.stream(sp):
            src[: m * stride].copy_(host_src, non_blocking=True)
        R.ring_consume(ring, m, views, pull_dst, stride if pull else 0, 0, sc)
        R.ring_put_batch(peer, d_msgs[0], m, 0, status, sp)
        sp.wait_stream(sc)
        with torch.cuda.stream(sp):
            host_views.copy_(views, non_blocking=True)
    e1.record(sp)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)

    summary = torch.tensor([ms, e2e_ms, 0.0 if ok else 1.0, float(launches)], dtype=torch.float64)
    dist.all_reduce(summary, op=dist.ReduceOp.MAX, group=grp)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lat_loaded, unl[4096], unl[C3_LENS[0]], mism, sampled), group=grp)
    cpu = None
    ce, rtt = None, None
    if rank == 0:
        try:
            ce = measure_ce(dev, (dev + 1) % torch.cuda.device_count())
        except Exception as e:          # reference only: the line keeps the guide's peak
            log("copy-engine reference failed:", repr(e))
            ce = None
        rtt = R.ring_probe_rtt(dev, (dev + 1) % torch.cuda.device_count(), 2000)
        rtt["host_mapped_offset_ns"] = int(offsets[1] - offsets[0])
        cpu = cpu_baseline(Rb, N, 1, 500, C3_LENS[1], C3_LENS[0], args.cpu_budget,
                           "C3 shape: U[4,193,280, 4,194,304]-B payloads")
    dist.barrier(group=grp)
    if args.pull == 2:
        R.ring_detach(peer)
        dist.barrier(group=grp)
        R.ring_destroy(ring)
    elif pull:
        R.ring_destroy(ring)            # the mapping of the previous rank's ring
        dist.barrier(group=grp)
        R.ring_detach(peer)
        R.ring_destroy(own)
    else:
        R.ring_detach(peer)
        dist.barrier(group=grp)
        R.ring_destroy(ring)
    if rank != 0:
        return None
    ms_max, e2e_max, bad = float(summary[0]), float(summary[1]), float(summary[2])
    loaded = [x for g in gathered for x in g[0]]
    u4k = [x for g in gathered for x in g[1]]
    u4m = [x for g in gathered for x in g[2]]
    value = payload_step * args.steps * world / (ms_max / 1e3) / 1e9
    per_gpu = value / world
    e2e = payload_step * e_steps * world / (e2e_max / 1e3) / 1e9
    return {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": ("C3-shaped ring of pairs, SPLIT placement: control words + header copies at the "
                                "consumer, buffer region at the producer, payloads pulled over NVLink (copy-out)"
                                if args.pull == 2 else
                                "C3-shaped ring of pairs, PULL placement: rank r's egress ring lives on rank r, rank "
                                "(r+1)%N opens it and pulls every payload over NVLink (copy-out consume)" if pull else
                                "C3-shaped ring of pairs: rank r -> ring on rank (r+1)%N over NVLink") +
                               ", Wan2.1 umT5 emb 512x4096 bf16 / 480p latent 16x21x60x104 bf16 alternating",
                   "placement": {0: "push (ring at the consumer)", 1: "pull (ring_open)",
                                 2: "split (ring_create_split)"}[args.pull],
                   "R_bytes": Rb, "n_slots": N, "msgs_per_step_per_rank": m,
                   "l2": f"inputs larger than L2 per rank (2 x {m * 4} MiB source sets)",
                   "parallelism": f"{world} concurrent SPSC rings (one egress + one ingress stream per GPU)"},
        "per_gpu_gbs": round(per_gpu, 2),
        "verified": {"sampled_messages": sum(g[4] for g in gathered), "payload_mismatches": sum(g[3] for g in gathered),
                     "what": "per rank, 4 messages of the last timed step compared byte for byte with the "
                             "producer's seeded Wan2.1 tensors (synth.bf16_tensor_bytes)"},
        # forward bytes on the link per message = footprint +
        # size slot + tail word (the ncu counters add the link protocol on top:
        # profiles/r02_ncu_nvlink_counters.csv, 1.21 wire bytes per payload byte)
        "wire_gbs_per_gpu_algorithmic": round(per_gpu * sum(R.ring_footprint(C3_LENS[q % 2]) + 16 for q in range(m))
                                              / payload_step, 2),
        "nvlink_frac_of_900": round(per_gpu / NVLINK_NOMINAL, 4),
        "nvlink_ce": ce,
        "nvlink_frac_of_ce": round(per_gpu / ce["bidir_per_direction_gbs"], 4) if ce else None,
        "flag_rtt": {"rtt_min_us": round(rtt["rtt_min_ns"] / 1e3, 3), "rtt_p50_us": round(rtt["rtt_p50_ns"] / 1e3, 3),
                     "ntp_offset_ns": rtt["offset_b_minus_a_ns"], "host_mapped_offset_ns": rtt["host_mapped_offset_ns"],
                     "offset_disagreement_ns": rtt["offset_b_minus_a_ns"] - rtt["host_mapped_offset_ns"],
                     "what": "flag ping-pong GPU r <-> GPU r+1 (ring_probe_rtt, system scope, 2,000 rounds): RTT, "
                             "and the NTP-style clock offset from the min-RTT round next to the host-mapped offset "
                             "(ring_clock_offset_ns) the latencies use"} if rtt else None,
        "msgs_per_s": round(m * args.steps * world / (ms_max / 1e3), 1),
        "latency_us": {
            "loaded_p50": pct(loaded, 50), "loaded_p99": pct(loaded, 99),
            "unloaded_4KiB_p50": pct(u4k, 50), "unloaded_4KiB_p99": pct(u4k, 99),
            "unloaded_4MiB_p50": pct(u4m, 50), "unloaded_4MiB_p99": pct(u4m, 99),
            "samples": {"loaded": len(loaded), "unloaded_4KiB": len(u4k), "unloaded_4MiB": len(u4m)},
            "what": "t_visible (consumer GPU) - t_put (producer GPU), both %globaltimer mapped to the host "
                    "CLOCK_MONOTONIC with ring_clock_offset_ns; loaded = 20 streamed steps after the timed "
                    "region, unloaded = one message in flight; first 10 % of each dropped"},
        "roofline": {"bound": "nvlink", "achieved": round(per_gpu, 1),
                     "peak": ce["bidir_per_direction_gbs"] if ce else NVLINK_PEAK_MEASURED, "unit": "GB/s",
                     "frac": round(per_gpu / (ce["bidir_per_direction_gbs"] if ce else NVLINK_PEAK_MEASURED), 4),
                     "traffic": None, "kernel": "get_kernel<true> copy-out (pull)" if pull else "put_kernel<2>",
                     "peak_source": ("in-run cudaMemcpyPeerAsync, both directions at once (nvlink_ce); "
                                     if ce else "B200_PROFILING.md measured peer copy 770 GB/s; ") +
                                    "900 GB/s nominal per direction: nvlink_frac_of_900"},
        "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": m * stride * world,
                "d2h_bytes_per_step": m * 128 * world},
        "gpu_launches": int(summary[3]) * world,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "ok": bad == 0.0,
    }


def bench_c3_one_way(args, rank, world, grp, placement: str, put_cfg=None):
    """BASELINE.json configs[2] as the north star states its target: ONE ring,
    GPU 0 -> GPU 1, 4-MB Wan2.1 tensors, GB/s per direction against 900.
    placement "split" (ring_create_split, R28: control words and header copies
    at the consumer, buffer region at the producer; the copy-out consume pulls
    every payload over NVLink) or "push" (the paper's one-sided write into the
    consumer's ring).  256 MiB ring, 64 messages per put / consume launch.
    Payloads come from the seeded device generator; the last timed launch's
    copy-out (split) or ring entries (push) are compared with it on the device.
    Ranks >= 2 only take part in the collectives.  Returns the result on rank 0."""
    import torch
    import torch.distributed as dist
    from paper_2601_20655_b200 import ring as R
    from synth import device as SD
    dev = int(os.environ.get("LOCAL_RANK", rank))
    Rb, N, K, launches, warm = 256 << 20, 64, 64, int(os.environ.get("B200RING_C3_LAUNCHES", 120)), 2
    stride, seed = 4194304, synth_seed_c3()
    lens = [C3_LENS[q % 2] for q in range(K)]
    split = placement == "split"
    ring = peer = None
    hs = [None] * world
    if rank == 1:
        ring = (R.ring_create_split(dev, (dev - 1) % torch.cuda.device_count(), Rb, N, 1, 0) if split
                else R.ring_create(dev, Rb, N, 1, 0))
        hs[1] = R.ring_export(ring)
    dist.all_gather_object(hs, hs[1] if rank == 1 else None, group=grp)
    mh = None
    if rank == 0:
        peer, mh = R.ring_attach_peer(hs[1], dev, 0)
        if put_cfg:                       # (ctas, threads, copy_mode): e.g. the TMA engine on 17 SMs
            R.ring_peer_config(peer, *put_cfg)
    mhs = [None] * world
    dist.all_gather_object(mhs, mh, group=grp)
    if rank == 1:
        R.ring_bind_mirror(ring, 0, mhs[0])
    res = torch.zeros(4, dtype=torch.float64)
    active = rank in (0, 1)          # every rank walks the same collectives; ranks >= 2 do no work
    if active:
        s = torch.cuda.Stream()
        if rank == 0:
            src = torch.empty(K * stride, dtype=torch.uint8, device="cuda")
            keep = SD.fill([src.data_ptr() + q * stride for q in range(K)], lens, [0] * K, list(range(K)), seed)
            a = R.make_msgs([src.data_ptr() + q * stride for q in range(K)], lens, [bytes(16)] * K, [0] * K,
                            list(range(K)), [2] * K)
            d_msgs = torch.from_numpy(a.view(np.uint8).copy()).cuda()
            status = torch.zeros(K, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            del keep
            run = lambda: R.ring_put_batch(peer, d_msgs, K, 0, status, s)
        else:
            views = torch.zeros(K * 128, dtype=torch.uint8, device="cuda")
            dst = torch.empty(K * stride, dtype=torch.uint8, device="cuda") if split else None
            run = lambda: R.ring_consume(ring, K, views, dst, stride if split else 0, 0, s)
        for _ in range(warm):
            run()
        torch.cuda.synchronize()
    dist.barrier(group=grp)
    if active:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(launches):
            run()
        e1.record(s)
        torch.cuda.synchronize()
        res[0] = e0.elapsed_time(e1)
        if rank == 0:
            res[1] = float(bool((status == 0).all().item()))
        else:
            v = R.parse_views(views.cpu().numpy())
            res[1] = float(bool((v["status"] == 0).all()))
            if split:
                bad = SD.verify([dst.data_ptr() + q * stride for q in range(K)], lens, [0] * K, list(range(K)), seed)
            else:
                # push: the last launch's entries are still in the ring (released, not overwritten)
                base = R.ring_get_info(ring).data
                bad = SD.verify([base + int(o) for o in v["offset"]], lens, [0] * K, list(range(K)), seed)
            torch.cuda.synchronize()
            res[2] = float(int((bad.cpu() != -1).sum()))
        res[3] = 1.0
    dist.barrier(group=grp)
    out = [None] * world
    dist.all_gather_object(out, res.tolist(), group=grp)
    if rank == 0:
        R.ring_detach(peer)
    dist.barrier(group=grp)
    if rank == 1:
        R.ring_destroy(ring)
    if rank != 0:
        return None
    ms = max(out[0][0], out[1][0])
    gbs = sum(lens) * launches / (ms / 1e3) / 1e9
    return {"placement": placement, "put": ({"ctas": put_cfg[0], "copy_mode": put_cfg[2]} if put_cfg else "default"),
            "value": round(gbs, 1), "unit": "GB/s (payload, one direction)",
            "nvlink_frac_of_900": round(gbs / NVLINK_NOMINAL, 4), "ms": round(ms, 3),
            "ms_producer": round(out[0][0], 3), "ms_consumer": round(out[1][0], 3),
            "ok": out[0][1] == 1.0 and out[1][1] == 1.0 and out[1][2] == 0.0,
            "verified": {"payload_mismatches": int(out[1][2]), "messages": K,
                         "what": "the last timed launch's payloads compared on the consumer GPU with the seeded "
                                 "generator (synth/csrc/synth_dev.cu)"},
            "config": {"workload": "C3 (BASELINE.json configs[2]) one ring GPU 0 -> GPU 1, Wan2.1 umT5 emb / 480p "
                                   "latent alternating (4,194,304 / 4,193,280 B)",
                       "R_bytes": Rb, "n_slots": N, "msgs_per_launch": K, "launches_timed": launches,
                       "timing": "CUDA events on the producer's and the consumer's stream, max of the two"}}


def synth_seed_c3():
    import synth
    return synth.SEED_BASE + 33


def measure_ce(a: int, b: int, nbytes: int = 256 << 20, reps: int = 10) -> dict:
    """In-run copy-engine NVLink reference: cudaMemcpyPeerAsync (cuda-python),
    GPU a -> GPU b alone, then a -> b and b -> a at the same time, each
    direction issued on a stream of its source GPU and timed by its own CUDA
    events (per direction: the slower of the two)."""
    import torch
    from cuda.bindings import runtime as rt
    for x, y in ((a, b), (b, a)):
        with torch.cuda.device(x):
            rt.cudaDeviceEnablePeerAccess(y, 0)     # "already enabled" is fine
    xa = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a}")
    yb = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{b}")
    xb = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{b}")
    ya = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a}")
    sa, sb = torch.cuda.Stream(a), torch.cuda.Stream(b)

    def copies(dst, dd, src, sd, st):
        for _ in range(reps):
            err, = rt.cudaMemcpyPeerAsync(dst.data_ptr(), dd, src.data_ptr(), sd, nbytes, st.cuda_stream)
            assert err == rt.cudaError_t.cudaSuccess, err

    def timed(jobs):
        for d in (a, b):
            torch.cuda.synchronize(d)
        ev = []
        for dst, dd, src, sd, st in jobs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(sd):
                e0.record(st)
                copies(dst, dd, src, sd, st)
                e1.record(st)
            ev.append((e0, e1))
        for d in (a, b):
            torch.cuda.synchronize(d)
        return [nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9 for e0, e1 in ev]

    timed([(yb, b, xa, a, sa)])                                   # warm
    one = timed([(yb, b, xa, a, sa)])[0]
    bi = timed([(yb, b, xa, a, sa), (ya, a, xb, b, sb)])
    del xa, yb, xb, ya
    return {"one_direction_gbs": round(one, 1), "bidir_per_direction_gbs": round(min(bi), 1),
            "bidir_gbs": [round(x, 1) for x in bi],
            "what": f"cudaMemcpyPeerAsync {nbytes >> 20} MiB x {reps}, GPU {a} -> {b} alone and with {b} -> {a} "
                    "concurrently (each direction on a stream of its source GPU, its own CUDA events)"}


def R_clock_offset(dev):
    from paper_2601_20655_b200 import ring as R
    return R.ring_clock_offset_ns(dev)


def reference_arm(args):
    """--impl reference: the CPU oracle as it stands, on the host cores, on our
    arm's config / metric / unit; each step a bounded sample of the workload."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import threaded as T
    if world == 1:
        lo = hi = 1048512
        per, Rb, N, wl = 64, 64 << 20, 64, "C2 sample: 64 x 1,048,512-B messages per step (one ring's worth)"
    else:
        lo, hi = C3_LENS[1], C3_LENS[0]
        per, Rb, N, wl = 128, 256 << 20, 64, "C3 sample: 128 x ~4 MiB messages per step (one pair launch's worth)"
    times, nbytes, res = [], 0, None
    for i in range(args.warmup + args.steps):
        res = T.run(Rb, N, 1, per, lo, hi, 20260120 + i)
        if i >= args.warmup:
            times.append(res["seconds"])
            nbytes += res["bytes"]
    tot = sum(times)
    value = nbytes / tot / 1e9
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / len(times) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl, "R_bytes": Rb, "n_slots": N},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": res["threads"],
                             "kind": "oracle-threaded", "cpu_model": res["cpu_model"], "host_cpus": os.cpu_count(),
                             "sample": wl + " through oracle/ring_threaded.cpp (1 producer + 1 consumer thread, "
                                            "pinned, memcpy payloads)"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--msgs-per-step", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0, help="put grid size (0 = library default)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--copy-mode", type=int, default=0, help="0: LSU copy warps, 1: TMA engine")
    ap.add_argument("--topology", default="pairs", choices=["pairs", "pipeline", "fanin", "reassign"],
                    help="N>1: pairs (default bench line) or the C4 / C5a / C5b runs of bench_multi.py")
    ap.add_argument("--sizes", default="", help="fanin: comma-separated message sizes")
    ap.add_argument("--fanin-mode", default="mpsc", choices=["mpsc", "set", "rc"],
                    help="fanin: the paper's locked MPSC ring, one SPSC ring per producer + ring_set_consume, "
                         "or a reserve-then-commit MPSC ring")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--lat-iters", type=int, default=560,
                    help="N>1: unloaded-latency round trips per size per rank (>= 1,000 samples pooled at N=2)")
    ap.add_argument("--no-overlap", action="store_true", help="N=1: put(s+1) waits for consume(s)")
    ap.add_argument("--ring-mb", type=int, default=0, help="N>1 pairs: ring data region in MiB (0 = 256)")
    ap.add_argument("--cons-ctas", type=int, default=0, help="N>1 pull: consumer copy-out grid (0 = default)")
    ap.add_argument("--cons-threads", type=int, default=0)
    ap.add_argument("--pull", type=int, default=0,
                    help="N>1 pairs: 1 = pull placement (ring at the producer, consumer pulls over NVLink), "
                         "2 = split placement (control at the consumer, buffer region at the producer)")
    ap.add_argument("--engine", type=int, default=0,
                    help="N=1: 1 = persistent put engine (doorbells), 0 = one put launch per step")
    ap.add_argument("--graph", action="store_true",
                    help="N=1: replay a CUDA graph of 16 steps in the timed region (default: eager launches)")
    ap.add_argument("--watchdog", type=float, default=0.0,
                    help="seconds: dump every Python stack and exit if the run takes longer (debugging)")
    args = ap.parse_args()
    if args.watchdog > 0:
        import faulthandler
        faulthandler.dump_traceback_later(args.watchdog, exit=True)
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
            args.steps = 24000
        print(json.dumps(bench_c2(args)), flush=True)
        return
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    if not args.steps:
        args.steps = 200
    # NCCL is the process group of record; the handle exchange and the
    # max-over-ranks reduction run on a gloo group (CPU objects only).
    dist.init_process_group("nccl")
    local = int(os.environ.get("LOCAL_RANK", rank))
    import torch
    torch.cuda.set_device(local)
    dist.barrier(device_ids=[local])      # once, off the data path: NCCL saw every rank
    grp = dist.new_group(backend="gloo")
    try:
        if args.topology != "pairs":
            import bench_multi
            if not args.steps or args.steps == 200:
                args.steps = 10
            out = bench_multi.main(args, rank, world, grp)
        else:
            out = bench_pairs(args, rank, world, grp)
            # the configs BASELINE.json maps to this GPU count, in the
            # same line: C4 at >= 4 GPUs, C5a (verified sweep) and C5b (verified flip)
            # at >= 3 (the 8-GPU shape is 7 producers -> 1 consumer)
            import copy
            import bench_multi
            extra = {}
            offsets = [None] * world
            dist.all_gather_object(offsets, R_clock_offset(local), group=grp)
            extra["c3_one_way"] = {pl: bench_c3_one_way(args, rank, world, grp, pl) for pl in ("split", "push")}
            # the paper's L3 concern (transfers off the SMs): the push by
            # the TMA engine on 17 SMs (no LSU copy)
            extra["c3_one_way"]["push_tma_17sm"] = bench_c3_one_way(args, rank, world, grp, "push", (17, 0, 1))
            if world >= 4:
                a4 = copy.copy(args)
                a4.steps, a4.warmup, a4.msgs_per_step = 10, 3, 2
                extra["c4"] = bench_multi.run_pipeline(a4, rank, world, grp, offsets)
            if world >= 3:
                a5 = copy.copy(args)
                a5.sizes, a5.verify, a5.fanin_mode = "4096,4194304,268435456", True, "mpsc"
                extra["c5a"] = bench_multi.run_fanin(a5, rank, world, grp, offsets)
                a5b = copy.copy(args)
                a5b.msgs_per_step, a5b.verify = 48, True
                extra["c5b"] = bench_multi.run_reassign(a5b, rank, world, grp, offsets)
            if out is not None:
                for k, v in extra.items():
                    if v is not None:
                        out[k] = v
                if out.get("c3_one_way"):
                    ce1 = (out.get("nvlink_ce") or {}).get("one_direction_gbs")
                    for r in out["c3_one_way"].values():
                        r["nvlink_frac_of_ce_one_way"] = round(r["value"] / ce1, 4) if ce1 else None
                    best = max(out["c3_one_way"].items(), key=lambda kv: kv[1]["value"] if kv[1]["ok"] else 0)
                    out["c3_one_way"]["best"] = best[0]
                    out["c3_one_way"]["what"] = (
                        "north-star target (>= 80 % of 900 GB/s per direction, >= 4 MB messages) on ONE ring; "
                        "split: the consumer's copy-out pulls over NVLink (1.125 wire bytes per payload byte, "
                        "profiles/r02b_ncu_split_counters.csv), push: peer stores (1.21), push_tma_17sm: the "
                        "same push by the TMA engine on 17 SMs (6 engine warps per CTA, no LSU copy)")
        if out:
            print(json.dumps(out), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
