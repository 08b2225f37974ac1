"""Thin ctypes binding of the C ABI in include/b200ring.h (argument marshalling only).

Every function has the name of its C entry point and raises `RingError` when the
C call returns a non-OK status.  No protocol step runs in Python: puts, gets and
releases are kernels launched by libb200ring.so on the given CUDA stream.  There
is no fallback: if the shared library is missing or does not load, importing
this module raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libb200ring.so")

# ---- status codes / flags (include/b200ring.h) ------------------------------------
RING_OK, RING_EINVAL, RING_ENOMEM, RING_EMSGSIZE, RING_FULL, RING_EMPTY = 0, 1, 2, 3, 4, 5
RING_ETIMEDOUT, RING_ECORRUPT, RING_ECUDA, RING_EPEER, RING_EPENDING, RING_EDROPPED = 6, 7, 8, 9, 10, 11
RING_EREJECTED, RING_ECLOSED = 12, 13
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "EMSGSIZE", 4: "FULL", 5: "EMPTY", 6: "ETIMEDOUT",
                7: "ECORRUPT", 8: "ECUDA", 9: "EPEER", 10: "EPENDING", 11: "EDROPPED", 12: "EREJECTED", 13: "ECLOSED"}
RING_BLOCK, RING_TRY, RING_NO_TIMESTAMP, RING_ASYNC = 0, 1, 2, 4
RING_CREATE_DEFAULT, RING_CREATE_LOCAL, RING_CREATE_FAULT_TOLERANT, RING_CREATE_RESERVE_COMMIT = 0, 1, 2, 4
RING_AT_LOCK, RING_AT_GH, RING_AT_WB, RING_AT_WL, RING_AT_UH = 1, 2, 3, 4, 5
RING_HDR_BYTES, RING_ENTRY_ALIGN = 64, 128


class ring_hdr_t(C.Structure):
    _fields_ = [("uid", C.c_uint8 * 16), ("accepted_at", C.c_uint64), ("app_id", C.c_uint32),
                ("stage", C.c_uint16), ("reserved", C.c_uint16)]


class ring_handle_t(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 256)]


class ring_fault_t(C.Structure):
    _fields_ = [("die_after", C.c_uint32), ("pause_mask", C.c_uint32), ("msg", C.c_uint32),
                ("reserved", C.c_uint32), ("arrived", C.c_void_p), ("go", C.c_void_p)]


class ring_dev_peer_t(C.Structure):
    _fields_ = [("ring", C.c_uint64), ("data", C.c_uint64), ("state", C.c_uint64), ("ctl", C.c_uint64),
                ("crc_table", C.c_uint64), ("R", C.c_uint64), ("N", C.c_uint32), ("producer_id", C.c_uint32),
                ("sys", C.c_uint32), ("reserved", C.c_uint32)]


class ring_info_t(C.Structure):
    _fields_ = [("device", C.c_int), ("n_slots", C.c_uint32), ("max_producers", C.c_uint32),
                ("data_bytes", C.c_uint64), ("base", C.c_uint64), ("data", C.c_uint64),
                ("data_offset", C.c_uint64), ("alloc_bytes", C.c_uint64)]


# numpy mirrors of the device-side records (for building / parsing device arrays)
MSG_DTYPE = np.dtype([("src", "<u8"), ("len", "<u8"), ("uid", "u1", 16), ("accepted_at", "<u8"),
                      ("app_id", "<u4"), ("stage", "<u2"), ("reserved", "<u2")])
VIEW_DTYPE = np.dtype([("offset", "<u8"), ("len", "<u8"), ("footprint", "<u8"), ("start", "<u8"),
                       ("slot_seq", "<u4"), ("status", "<u4"), ("t_visible", "<u8"), ("reserved", "<u8", 2),
                       ("header", "u1", 64)])
assert MSG_DTYPE.itemsize == 48 and VIEW_DTYPE.itemsize == 128


class RingError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str = ""):
        self.status = status
        super().__init__(f"{fn}: {STATUS_NAMES.get(status, status)}" + (f" ({detail})" if detail else ""))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2601_20655_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P, U32, U64, I = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    sig = {
        "ring_create": [I, U64, U32, U32, U32, C.POINTER(P)],
        "ring_create_split": [I, I, U64, U32, U32, U32, C.POINTER(P)],
        "ring_open": [C.POINTER(ring_handle_t), I, C.POINTER(P)],
        "ring_destroy": [P],
        "ring_get_info": [P, C.POINTER(ring_info_t)],
        "ring_export": [P, C.POINTER(ring_handle_t)],
        "ring_attach_peer": [C.POINTER(ring_handle_t), I, U32, C.POINTER(P), C.POINTER(ring_handle_t)],
        "ring_bind_mirror": [P, U32, C.POINTER(ring_handle_t)],
        "ring_detach": [P],
        "ring_put_batch": [P, P, U32, U32, P, P],
        "ring_put": [P, P, U64, C.POINTER(ring_hdr_t), U32, P, P],
        "ring_peer_config": [P, U32, U32, U32],
        "ring_peer_engine_start": [P, P],
        "ring_peer_engine_wait": [P, P],
        "ring_peer_engine_stop": [P, P],
        "ring_peer_engine_state": [P, C.POINTER(C.c_uint64)],
        "ring_get": [P, U32, P, P, U64, U32, P],
        "ring_release": [P, U32, P],
        "ring_consume": [P, U32, P, P, U64, U32, P],
        "ring_config": [P, U32, U32],
        "ring_read_image": [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                            C.POINTER(C.c_uint64), P],
        "ring_read_data": [P, U64, U64, P],
        "ring_write_data": [P, U64, U64, P],
        "router_create": [I, U32, C.POINTER(P)],
        "router_destroy": [P],
        "router_set_route": [P, U32, C.c_uint16, C.POINTER(P), U32, P],
        "ring_put_routed": [P, P, U32, U32, P, P, P],
        "ring_set_timeout_ns": [U64],
        "ring_clock_offset_ns": [I, C.POINTER(C.c_int64)],
        "ring_probe_rtt": [I, I, U32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int64)],
        "ring_peer_trace": [P, P, U32],
        "ring_get_trace": [P, P, U32],
        "ring_peer_set_fault": [P, C.POINTER(ring_fault_t)],
        "ring_set_lock_timeout_ns": [U64],
        "ring_set_hole_timeout_ns": [U64],
        "router_set_admission": [P, U32, C.c_uint16, U64, U32, P],
        "ring_peer_device_view": [P, C.POINTER(ring_dev_peer_t)],
        "ring_set_create": [C.POINTER(P), U32, C.POINTER(P)],
        "ring_set_destroy": [P],
        "ring_set_consume": [P, U32, P, P, U32, P],
        "ring_stage_scale_bf16_put": [P, P, U64, C.c_float, C.POINTER(ring_hdr_t), U32, P, P],
        "router_size_route": [P, U32, C.c_uint16, U64, U64, U32, C.POINTER(P), U32, C.POINTER(U32), P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.ring_strerror.argtypes = [C.c_int]
    lib.ring_strerror.restype = C.c_char_p
    lib.ring_last_cuda_error.argtypes = []
    lib.ring_last_cuda_error.restype = C.c_char_p
    lib.ring_launch_count.argtypes = []
    lib.ring_launch_count.restype = C.c_uint64
    lib.ring_footprint.argtypes = [C.c_uint64]
    lib.ring_footprint.restype = C.c_uint64
    lib.ring_peer_submitted.argtypes = [P]
    lib.ring_peer_submitted.restype = C.c_uint64
    lib.ring_required_instances.argtypes = [U64, U64, U32]
    lib.ring_required_instances.restype = C.c_uint64
    return lib


lib = _load()


def _check(fn: str, st: int):
    if st != RING_OK:
        detail = lib.ring_last_cuda_error().decode() if st == RING_ECUDA else ""
        raise RingError(fn, st, detail)


def _stream(stream) -> int | None:
    """Accept a torch.cuda.Stream, a raw cudaStream_t int, or None (legacy default stream)."""
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream)) or None


def _ptr(x) -> int | None:
    """Device pointer of a torch tensor (or an int), None for None."""
    if x is None:
        return None
    return int(x.data_ptr()) if hasattr(x, "data_ptr") else int(x)


# ---- lifetime ---------------------------------------------------------------------------
def ring_create(device: int, data_bytes: int, n_slots: int, max_producers: int = 1, flags: int = 0) -> int:
    out = C.c_void_p()
    _check("ring_create", lib.ring_create(device, data_bytes, n_slots, max_producers, flags, C.byref(out)))
    return out.value


def ring_create_split(device: int, data_device: int, data_bytes: int, n_slots: int, max_producers: int = 1,
                      flags: int = 0) -> int:
    """Split placement: control words + header copies on `device` (the consumer),
    the buffer region on `data_device` (the producer's GPU)."""
    out = C.c_void_p()
    _check("ring_create_split", lib.ring_create_split(device, data_device, data_bytes, n_slots, max_producers, flags,
                                                      C.byref(out)))
    return out.value


def ring_open(handle: bytes, device: int) -> int:
    """Consumer side of a ring living in another GPU's memory (pull placement)."""
    out = C.c_void_p()
    _check("ring_open", lib.ring_open(C.byref(_handle(handle)), device, C.byref(out)))
    return out.value


def ring_destroy(ring: int) -> None:
    _check("ring_destroy", lib.ring_destroy(ring))


def ring_get_info(ring: int) -> ring_info_t:
    info = ring_info_t()
    _check("ring_get_info", lib.ring_get_info(ring, C.byref(info)))
    return info


def ring_export(ring: int) -> bytes:
    h = ring_handle_t()
    _check("ring_export", lib.ring_export(ring, C.byref(h)))
    return bytes(h.bytes)


def _handle(b: bytes) -> ring_handle_t:
    h = ring_handle_t()
    C.memmove(h.bytes, bytes(b), 256)
    return h


def ring_attach_peer(handle: bytes, producer_device: int, producer_id: int) -> tuple[int, bytes]:
    """Returns (peer, mirror_handle)."""
    out = C.c_void_p()
    mh = ring_handle_t()
    _check("ring_attach_peer", lib.ring_attach_peer(C.byref(_handle(handle)), producer_device, producer_id,
                                                    C.byref(out), C.byref(mh)))
    return out.value, bytes(mh.bytes)


def ring_bind_mirror(ring: int, producer_id: int, mirror_handle: bytes) -> None:
    _check("ring_bind_mirror", lib.ring_bind_mirror(ring, producer_id, C.byref(_handle(mirror_handle))))


def ring_detach(peer: int) -> None:
    _check("ring_detach", lib.ring_detach(peer))


# ---- producer ---------------------------------------------------------------------------
def ring_put_batch(peer: int, d_msgs, n: int, flags: int, d_status, stream=None) -> None:
    _check("ring_put_batch", lib.ring_put_batch(peer, _ptr(d_msgs), n, flags, _ptr(d_status), _stream(stream)))


def ring_put(peer: int, d_payload, length: int, hdr: ring_hdr_t, flags: int, d_status, stream=None) -> None:
    _check("ring_put", lib.ring_put(peer, _ptr(d_payload), length, C.byref(hdr), flags, _ptr(d_status),
                                    _stream(stream)))


def ring_peer_config(peer: int, copy_ctas: int = 0, threads: int = 0, copy_mode: int = 0) -> None:
    _check("ring_peer_config", lib.ring_peer_config(peer, copy_ctas, threads, copy_mode))


def ring_peer_engine_start(peer: int, stream=None) -> None:
    _check("ring_peer_engine_start", lib.ring_peer_engine_start(peer, _stream(stream)))


def ring_peer_engine_wait(peer: int, stream=None) -> None:
    _check("ring_peer_engine_wait", lib.ring_peer_engine_wait(peer, _stream(stream)))


def ring_peer_engine_stop(peer: int, stream=None) -> None:
    _check("ring_peer_engine_stop", lib.ring_peer_engine_stop(peer, _stream(stream)))


def ring_peer_engine_state(peer: int) -> dict:
    out = (C.c_uint64 * 4)()
    _check("ring_peer_engine_state", lib.ring_peer_engine_state(peer, out))
    return dict(posted=out[0], planned=out[1], done=out[2], closed=out[3])


def ring_peer_submitted(peer: int) -> int:
    return int(lib.ring_peer_submitted(peer))


def ring_get_trace(ring: int, n: int = 1024) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    _check("ring_get_trace", lib.ring_get_trace(ring, out.ctypes.data, n))
    return out


def ring_peer_trace(peer: int, n: int = 4096) -> np.ndarray:
    """Debug timelines (needs B200RING_TRACE=1): words [0, 2048) the last put
    launch, [2048, 4096) the launch before it."""
    out = np.zeros(n, dtype=np.uint64)
    _check("ring_peer_trace", lib.ring_peer_trace(peer, out.ctypes.data, n))
    return out


# ---- consumer ---------------------------------------------------------------------------
def ring_get(ring: int, n: int, d_views, d_dst=None, dst_stride: int = 0, flags: int = 0, stream=None) -> None:
    _check("ring_get", lib.ring_get(ring, n, _ptr(d_views), _ptr(d_dst), dst_stride, flags, _stream(stream)))


def ring_release(ring: int, count: int, stream=None) -> None:
    _check("ring_release", lib.ring_release(ring, count, _stream(stream)))


def ring_consume(ring: int, n: int, d_views, d_dst=None, dst_stride: int = 0, flags: int = 0, stream=None) -> None:
    _check("ring_consume", lib.ring_consume(ring, n, _ptr(d_views), _ptr(d_dst), dst_stride, flags,
                                            _stream(stream)))


def ring_config(ring: int, copy_ctas: int = 0, threads: int = 0) -> None:
    _check("ring_config", lib.ring_config(ring, copy_ctas, threads))


def ring_read_image(ring: int) -> dict:
    info = ring_get_info(ring)
    lock, tail, head, cur = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    slots = np.zeros(info.n_slots, dtype=np.uint64)
    _check("ring_read_image", lib.ring_read_image(ring, C.byref(lock), C.byref(tail), C.byref(head), C.byref(cur),
                                                  slots.ctypes.data))
    return dict(lock=lock.value, tail=tail.value, head=head.value, cursor=cur.value,
                slots=[int(x) for x in slots])


def ring_read_data(ring: int, offset: int, length: int) -> bytes:
    buf = (C.c_ubyte * max(length, 1))()
    _check("ring_read_data", lib.ring_read_data(ring, offset, length, C.addressof(buf)))
    return bytes(buf[:length])


def ring_write_data(ring: int, offset: int, data: bytes) -> None:
    buf = (C.c_ubyte * max(len(data), 1)).from_buffer_copy(bytes(data) or b"\0")
    _check("ring_write_data", lib.ring_write_data(ring, offset, len(data), C.addressof(buf)))


# ---- router -------------------------------------------------------------------------------
def router_create(device: int, max_routes: int = 64) -> int:
    out = C.c_void_p()
    _check("router_create", lib.router_create(device, max_routes, C.byref(out)))
    return out.value


def router_destroy(router: int) -> None:
    _check("router_destroy", lib.router_destroy(router))


def router_set_route(router: int, app_id: int, stage: int, dests: list[int], stream=None) -> None:
    arr = (C.c_void_p * max(len(dests), 1))(*dests)
    _check("router_set_route", lib.router_set_route(router, app_id, stage, arr, len(dests), _stream(stream)))


def ring_put_routed(router: int, d_msgs, n: int, flags: int, d_status, d_dest=None, stream=None) -> None:
    _check("ring_put_routed", lib.ring_put_routed(router, _ptr(d_msgs), n, flags, _ptr(d_status), _ptr(d_dest),
                                                  _stream(stream)))


# ---- misc ---------------------------------------------------------------------------------
def ring_set_timeout_ns(ns: int) -> None:
    _check("ring_set_timeout_ns", lib.ring_set_timeout_ns(ns))


def ring_probe_rtt(dev_a: int, dev_b: int, iters: int = 1000) -> dict:
    mn, p50, off = C.c_uint64(), C.c_uint64(), C.c_int64()
    _check("ring_probe_rtt", lib.ring_probe_rtt(dev_a, dev_b, iters, C.byref(mn), C.byref(p50), C.byref(off)))
    return {"rtt_min_ns": mn.value, "rtt_p50_ns": p50.value, "offset_b_minus_a_ns": off.value}


def ring_clock_offset_ns(device: int) -> int:
    """GPU globaltimer minus host CLOCK_MONOTONIC, in ns (measurement support)."""
    out = C.c_int64()
    _check("ring_clock_offset_ns", lib.ring_clock_offset_ns(device, C.byref(out)))
    return int(out.value)


def ring_strerror(status: int) -> str:
    return lib.ring_strerror(status).decode()


def ring_launch_count() -> int:
    return int(lib.ring_launch_count())


def ring_footprint(length: int) -> int:
    return int(lib.ring_footprint(length))


# ---- record helpers (host-side marshalling of the device arrays) --------------------------
def make_msgs(srcs, lens, uids, accepted_at, app_ids, stages) -> np.ndarray:
    """Build a host array of ring_msg_t records (upload it with torch to the producer GPU)."""
    n = len(lens)
    a = np.zeros(n, dtype=MSG_DTYPE)
    a["src"] = np.asarray(srcs, dtype=np.uint64)
    a["len"] = np.asarray(lens, dtype=np.uint64)
    a["uid"] = np.frombuffer(b"".join(bytes(u) for u in uids), dtype=np.uint8).reshape(n, 16) if n else 0
    a["accepted_at"] = np.asarray(accepted_at, dtype=np.uint64)
    a["app_id"] = np.asarray(app_ids, dtype=np.uint32)
    a["stage"] = np.asarray(stages, dtype=np.uint16)
    return a


def parse_views(raw: np.ndarray) -> np.ndarray:
    """Interpret a uint8 host array of n*128 bytes as ring_view_t records."""
    return np.ascontiguousarray(raw, dtype=np.uint8).view(VIEW_DTYPE)


# ---- fault injection (tests of RING_CREATE_FAULT_TOLERANT rings) ---------------------
def ring_peer_set_fault(peer: int, die_after: int = 0, pause_mask: int = 0, msg: int = 0,
                        arrived=None, go=None) -> None:
    """Make message `msg` of later launches stop for good after action `die_after`
    (RING_AT_*) and/or pause after the actions in `pause_mask` until the host
    sets go[l]; `arrived` / `go` are pinned host tensors (>= 8 int32 words).
    All zeros clears."""
    if not (die_after or pause_mask):
        _check("ring_peer_set_fault", lib.ring_peer_set_fault(peer, None))
        return
    f = ring_fault_t(die_after, pause_mask, msg, 0, _ptr(arrived), _ptr(go))
    _check("ring_peer_set_fault", lib.ring_peer_set_fault(peer, C.byref(f)))


def ring_set_lock_timeout_ns(ns: int) -> None:
    _check("ring_set_lock_timeout_ns", lib.ring_set_lock_timeout_ns(int(ns)))


# ---- pipeline sizing / admission --------------------------------
def router_set_admission(router: int, app_id: int, stage: int, t_x: int, k: int, stream=None) -> None:
    _check("router_set_admission", lib.router_set_admission(router, app_id, stage, int(t_x), int(k), _stream(stream)))


def ring_required_instances(t_x: int, t_y: int, k: int) -> int:
    return int(lib.ring_required_instances(int(t_x), int(t_y), int(k)))


def router_size_route(router: int, app_id: int, stage: int, t_x: int, t_y: int, k: int, pool, stream=None) -> int:
    arr = (C.c_void_p * len(pool))(*pool)
    m = C.c_uint32()
    _check("router_size_route", lib.router_size_route(router, app_id, stage, int(t_x), int(t_y), int(k), arr,
                                                      len(pool), C.byref(m), _stream(stream)))
    return m.value


# ---- fused device-side put -----------------------------------------
def ring_peer_device_view(peer: int) -> dict:
    v = ring_dev_peer_t()
    _check("ring_peer_device_view", lib.ring_peer_device_view(peer, C.byref(v)))
    return {name: getattr(v, name) for name, _ in ring_dev_peer_t._fields_}


def ring_stage_scale_bf16_put(peer: int, d_in, n_elems: int, scale: float, uid: bytes = bytes(16),
                              accepted_at: int = 0, app_id: int = 0, stage: int = 0, flags: int = 0,
                              d_status=None, stream=None) -> None:
    """Synthetic stage with a fused put epilogue: out = bf16(in * scale) written
    by the computing kernel straight into the peer ring (one message)."""
    h = ring_hdr_t()
    C.memmove(h.uid, bytes(uid), 16)
    h.accepted_at, h.app_id, h.stage, h.reserved = accepted_at, app_id, stage, 0
    _check("ring_stage_scale_bf16_put", lib.ring_stage_scale_bf16_put(peer, _ptr(d_in), int(n_elems), float(scale),
                                                                      C.byref(h), flags, _ptr(d_status),
                                                                      _stream(stream)))


# ---- lock-free fan-in set -----------------------------------------
def ring_set_create(rings) -> int:
    arr = (C.c_void_p * len(rings))(*rings)
    out = C.c_void_p()
    _check("ring_set_create", lib.ring_set_create(arr, len(rings), C.byref(out)))
    return out.value


def ring_set_destroy(s: int) -> None:
    _check("ring_set_destroy", lib.ring_set_destroy(s))


def ring_set_consume(s: int, n: int, d_views, d_ring_idx=None, flags: int = 0, stream=None) -> None:
    _check("ring_set_consume", lib.ring_set_consume(s, n, _ptr(d_views), _ptr(d_ring_idx), flags, _stream(stream)))


def ring_set_hole_timeout_ns(ns: int) -> None:
    _check("ring_set_hole_timeout_ns", lib.ring_set_hole_timeout_ns(int(ns)))
