"""CPU oracle of the paper's double-ring buffer (arXiv 2601.20655, §6 "RDMA Network").

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import, call or
execute anything under `oracle/`.  The product path
(`paper_2601_20655_b200/`) never imports it, and the oracle never imports the
product path: the two share no code, headers, tables or constants.  The only
module both sides use is `synth/` (seeded input generators, no ring arithmetic).

Contents (each function cites the PAPER.md passage it follows):
  crc32.py      — CRC-32/IEEE, bit by bit (checksum of PAPER.md:768-769).
  ring.py       — layout constants, pointer formulas, entry
                  header, the sender's 8 steps
                   and the receiver's 5 steps
                   as an explicit-state stepper over labelled
                  atomic actions, and FIFO drivers.
  bruteforce.py — exhaustive interleaving search on tiny rings (2-4 slots):
                  no overwrite of an unreleased entry, pointer invariants,
                  busy-bit protocol, exactly-once in-order delivery, and
                  deadlock freedom.

Floating point: none.  Everything here is integer / byte arithmetic, so parity
with the CUDA path is bit-exact.

Parity pins (see DESIGN.md §"Oracle pins"): CRC check value + zlib, the
hand-derived worked examples in tests/golden/ (from the formulas at
PAPER.md:731-747), closed forms for constant-size streams, and the brute-force
invariants.  Throughput/latency have no published numbers: "parity unpinned"
applies to those (they are not oracle functions).
"""
