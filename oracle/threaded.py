"""Build and run oracle/ring_threaded.cpp, the threaded host-memory run of the
double ring (TEST / BENCH INFRASTRUCTURE ONLY -- see
oracle/__init__.py for who may call it).  Plain g++, no CUDA, nothing shared
with the product library."""
from __future__ import annotations

import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ring_threaded.cpp")
BIN = os.path.join(HERE, "ring_threaded")


def build(force: bool = False) -> str:
    if force or not os.path.exists(BIN) or os.path.getmtime(SRC) > os.path.getmtime(BIN):
        tmp = BIN + ".tmp"
        subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-Wall", "-o", tmp, SRC], check=True)
        os.replace(tmp, BIN)
    return BIN


def run(R: int, N: int, producers: int, per: int, lo: int, hi: int, seed: int, core0: int = 0,
        timeout: float = 600) -> dict:
    """One run; returns the runner's JSON result (gbs, msgs_per_s, p50_us,
    p99_us, messages, bytes, seconds, threads, bad, cpu_model, host_cpus)."""
    build()
    out = subprocess.run([BIN, str(R), str(N), str(producers), str(per), str(lo), str(hi), str(seed), "run",
                          str(core0)], capture_output=True, text=True, timeout=timeout)
    if out.returncode not in (0, 1):
        raise RuntimeError(f"ring_threaded failed: {out.stderr[-500:]}")
    return json.loads(out.stdout.strip().splitlines()[-1])


def placements(R: int, N: int, per: int, lo: int, hi: int, seed: int) -> list[tuple[int, int, int]]:
    """SPSC run in "place" mode: (start, footprint, slot seq) of every delivered message."""
    build()
    out = subprocess.run([BIN, str(R), str(N), "1", str(per), str(lo), str(hi), str(seed), "place"],
                         capture_output=True, text=True, timeout=600, check=True)
    return [tuple(int(x) for x in line.split()) for line in out.stdout.splitlines() if line.strip()]


def lengths(seed: int, channel: int, per: int, lo: int, hi: int) -> list[int]:
    """The runner's message lengths: U[lo, hi] from splitmix64 (ring_threaded.cpp msg_len)."""
    M = (1 << 64) - 1

    def sm(x):
        z = (x + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    if lo == hi:
        return [lo] * per
    return [lo + sm(sm(seed ^ 0x5151) ^ (channel << 32) ^ k) % (hi - lo + 1) for k in range(per)]
