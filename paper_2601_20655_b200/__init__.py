"""B200-native double-ring tensor transport (arXiv 2601.20655 §6, re-done on NVLink 5).

`paper_2601_20655_b200.ring` is a thin ctypes binding of the C ABI declared in
include/b200ring.h and implemented by the in-tree libb200ring.so (sm_100a
kernels + host runtime in csrc/).  `paper_2601_20655_b200.topology` wires rings
across ranks (handles exchanged with torch.distributed over gloo: plumbing
only, no collective on the data path).  `paper_2601_20655_b200.build` compiles
the library for sm_100a.
"""
__all__ = ["ring", "topology", "build"]
