"""Seeded synthetic inputs: message sizes, header fields, payload bytes.

Recipe:
  * seed base 20260120; per-config seed = base + config id.
  * payload bytes: counter-based splitmix64 keyed by (seed, channel, seq); any
    message's bytes can be regenerated on its own, at any size.
  * Wan2.1-shaped bf16 tensors: standard normal (embeddings, latents) or
    U[-1, 1] (decoded frames), rounded to bf16 (round-to-nearest-even), drawn
    from numpy's PCG64 seeded by (seed, channel, seq).
  * header fields (uid, accepted_at, app_id, stage) drawn from PCG64(seed).
Nothing here knows about rings, footprints or checksums.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

SEED_BASE = 20260120

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _key(seed: int, channel: int, seq: int) -> np.uint64:
    k = splitmix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))
    k = splitmix64(k ^ np.uint64(channel & 0xFFFFFFFF))
    k = splitmix64(k ^ np.uint64(seq & 0xFFFFFFFFFFFF))
    return k[0]


def payload_bytes(seed: int, channel: int, seq: int, length: int) -> np.ndarray:
    """`length` pseudo-random bytes for message (channel, seq): uint8 array."""
    if length == 0:
        return np.zeros(0, dtype=np.uint8)
    nw = (length + 7) // 8
    with np.errstate(over="ignore"):
        ctr = _key(seed, channel, seq) + np.arange(nw, dtype=np.uint64)
    return splitmix64(ctr).view(np.uint8)[:length].copy()


def _f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    with np.errstate(over="ignore"):
        return ((u + rounding) >> np.uint32(16)).astype(np.uint16)


def bf16_tensor_bytes(seed: int, channel: int, seq: int, shape, dist: str = "normal") -> np.ndarray:
    """A bf16 tensor of `shape` as raw little-endian bytes (uint8 array)."""
    n = int(np.prod(shape))
    rng = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, channel, seq]))
    if dist == "normal":
        x = rng.standard_normal(n, dtype=np.float32)
    elif dist == "uniform":
        x = rng.uniform(-1.0, 1.0, n).astype(np.float32)
    else:
        raise ValueError(dist)
    return _f32_to_bf16_bits(x).view(np.uint8)


# Wan2.1 image-to-video intermediate tensors (BASELINE.json configs)
WAN_SHAPES = {
    "umt5_emb": ((512, 4096), "normal"),                 # 4,194,304 B
    "latent_480p": ((16, 21, 60, 104), "normal"),        # 4,193,280 B
    "latent_720p": ((16, 21, 90, 160), "normal"),        # 9,676,800 B
    "frames_720p": ((81, 3, 720, 1280), "uniform"),      # 447,897,600 B
}


def wan_bytes(kind: str) -> int:
    shape, _ = WAN_SHAPES[kind]
    return int(np.prod(shape)) * 2


@dataclass
class Message:
    """One workflow message (PAPER.md:410-427 fields) plus its payload length."""
    channel: int          # producer id
    seq: int              # per-channel sequence number
    length: int           # payload bytes
    uid: bytes            # 16 B
    accepted_at: int      # u64
    app_id: int           # u32
    stage: int            # u16
    payload: np.ndarray | None = field(default=None, repr=False)


def header_fields(seed: int, channel: int, seq: int, app_id: int = 7, stage: int = 1):
    rng = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, channel, seq, 0xABCD]))
    uid = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
    accepted_at = int(rng.integers(0, 2**63, dtype=np.int64))
    return uid, accepted_at, app_id, stage


def random_stream(seed: int, channel: int, count: int, lo: int, hi: int,
                  with_payload: bool = True, app_id: int = 7, stage: int = 1) -> list[Message]:
    """`count` messages with payload length ~ U[lo, hi] (inclusive)."""
    rng = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, channel, 0x5151]))
    lens = rng.integers(lo, hi + 1, count)
    out = []
    for q in range(count):
        uid, acc, app, stg = header_fields(seed, channel, q, app_id, stage)
        m = Message(channel, q, int(lens[q]), uid, acc, app, stg)
        if with_payload:
            m.payload = payload_bytes(seed, channel, q, m.length)
        out.append(m)
    return out


def fixed_stream(seed: int, channel: int, count: int, length: int,
                 with_payload: bool = True, app_id: int = 7, stage: int = 1) -> list[Message]:
    out = []
    for q in range(count):
        uid, acc, app, stg = header_fields(seed, channel, q, app_id, stage)
        m = Message(channel, q, length, uid, acc, app, stg)
        if with_payload:
            m.payload = payload_bytes(seed, channel, q, length)
        out.append(m)
    return out


def wan_stream(seed: int, channel: int, count: int, kinds=("umt5_emb", "latent_480p"),
               with_payload: bool = True, app_id: int = 7, stage: int = 1) -> list[Message]:
    """Alternating Wan2.1-shaped bf16 tensors (C3: umT5 embeddings / 480p latents)."""
    out = []
    for q in range(count):
        kind = kinds[q % len(kinds)]
        shape, dist = WAN_SHAPES[kind]
        uid, acc, app, stg = header_fields(seed, channel, q, app_id, stage)
        m = Message(channel, q, wan_bytes(kind), uid, acc, app, stg)
        if with_payload:
            m.payload = bf16_tensor_bytes(seed, channel, q, shape, dist)
        out.append(m)
    return out
