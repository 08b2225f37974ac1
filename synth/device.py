"""ctypes binding of libb200synth.so: the seeded payload generator of
synth/streams.py run on the GPU (fill) and an exact compare against it
(verify).  Test / bench infrastructure only: it shares no code with the
product library and holds none of the ring's arithmetic.  Arrays are torch
tensors on the current CUDA device (or Python lists, uploaded here)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libb200synth.so")
SRC = os.path.join(HERE, "csrc", "synth_dev.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NO_ERROR = 2**64 - 1


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(SRC) > os.path.getmtime(LIB_PATH):
        tmp = LIB_PATH + ".tmp"
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                        "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", SRC, "-o", tmp], check=True)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run synth.device.build()")
        L = C.CDLL(LIB_PATH)
        P, U32, U64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.synth_fill.argtypes = [P, P, P, P, U32, U64, P]
        L.synth_fill.restype = C.c_int
        L.synth_verify.argtypes = [P, P, P, P, U32, U64, P, P]
        L.synth_verify.restype = C.c_int
        L.synth_verify_views.argtypes = [P, U32, U64, P, P, P, U64, U64, P, P, P]
        L.synth_verify_views.restype = C.c_int
        L.synth_hold_sms.argtypes = [U64, U64, P]
        L.synth_hold_sms.restype = C.c_int
        L.synth_word.argtypes = [U64, U32, U64, U64]
        L.synth_word.restype = U64
        _lib = L
    return _lib


def _dev(x, dtype):
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    vals = [int(v) for v in x]
    if dtype == torch.int64:
        vals = [v - 2**64 if v >= 2**63 else v for v in vals]       # same bits, signed
    return torch.tensor(vals, dtype=dtype).to("cuda")


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _args(ptrs, lens, chans, seqs):
    import torch
    p, l, c, q = _dev(ptrs, torch.int64), _dev(lens, torch.int64), _dev(chans, torch.int32), _dev(seqs, torch.int64)
    assert p.numel() == l.numel() == c.numel() == q.numel()
    return p, l, c, q


def fill(ptrs, lens, chans, seqs, seed: int, stream=None):
    """Write synth.payload_bytes(seed, chans[i], seqs[i], lens[i]) at device address ptrs[i]."""
    p, l, c, q = _args(ptrs, lens, chans, seqs)
    st = lib().synth_fill(p.data_ptr(), l.data_ptr(), c.data_ptr(), q.data_ptr(), p.numel(), seed & (2**64 - 1),
                          _stream(stream))
    if st:
        raise RuntimeError(f"synth_fill: cudaError {st}")
    return (p, l, c, q)   # keep the argument arrays alive until the stream has run


def verify(ptrs, lens, chans, seqs, seed: int, stream=None):
    """Device tensor (int64, n): offset of the first byte of range i that differs
    from synth.payload_bytes(seed, chans[i], seqs[i], lens[i]), or -1 (all equal)."""
    import torch
    p, l, c, q = _args(ptrs, lens, chans, seqs)
    bad = torch.empty(p.numel(), dtype=torch.int64, device="cuda")
    st = lib().synth_verify(p.data_ptr(), l.data_ptr(), c.data_ptr(), q.data_ptr(), p.numel(), seed & (2**64 - 1),
                            bad.data_ptr(), _stream(stream))
    if st:
        raise RuntimeError(f"synth_verify: cudaError {st}")
    bad._keep = (p, l, c, q)
    return bad


def verify_views(views, n: int, data_base: int, seed: int, chans=None, seqs=None, lut=None, lut_stride: int = 0,
                 stream=None):
    """verify() of the payloads that n view records (ring_view_t, 128 B each, a
    device uint8 tensor) point at inside a ring whose buffer region starts at
    device address data_base.  Keys: the header's (producer_id, seq) unless
    chans (int32) / seqs (int64) device tensors are given; lut (int64 device
    tensor) maps (producer_id, seq) to the generator's seq.  Launches only this
    library's kernels (no torch kernel, no host synchronisation)."""
    import torch
    dev = views.device
    for t in (chans, seqs, lut):
        assert t is None or (t.device == dev and t.is_contiguous())
    assert chans is None or chans.dtype == torch.int32
    assert seqs is None or seqs.dtype == torch.int64
    assert lut is None or lut.dtype == torch.int64
    bad = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    work = torch.empty(max(n, 1) * 4, dtype=torch.int64, device=dev)
    ptr = (lambda t: t.data_ptr() if t is not None else None)
    with torch.cuda.device(dev):
        st = lib().synth_verify_views(views.data_ptr(), n, data_base, ptr(chans), ptr(seqs), ptr(lut), lut_stride,
                                      seed & (2**64 - 1), work.data_ptr(), bad.data_ptr(), _stream(stream))
    if st:
        raise RuntimeError(f"synth_verify_views: cudaError {st}")
    bad._keep = (views, chans, seqs, lut, work)
    return bad[:n]


def word(seed: int, channel: int, seq: int, i: int) -> int:
    return int(lib().synth_word(seed & (2**64 - 1), channel, seq, i))


def hold_sms(base_ns: int, step_ns: int, stream=None):
    """Test scaffolding: occupy every SM of the current device (all shared
    memory) and release them one at a time, SM i after base_ns + i * step_ns."""
    st = lib().synth_hold_sms(base_ns, step_ns, _stream(stream))
    if st:
        raise RuntimeError(f"synth_hold_sms: cudaError {st}")
