"""B200-native double-ring tensor transport (arXiv 2601.20655 §6, re-done on NVLink 5).

`paper_2601_20655_b200.ring` is a thin ctypes binding of the C ABI declared in
include/b200ring.h and implemented by the in-tree libb200ring.so (sm_100a
kernels + host runtime in csrc/).  `paper_2601_20655_b200.dist` exchanges ring
handles across processes with torch.distributed (plumbing only).
"""
__all__ = ["ring"]
