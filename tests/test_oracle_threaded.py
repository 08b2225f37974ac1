"""The threaded host-memory runner (oracle/ring_threaded.cpp, the CPU
baseline of BASELINE.md §6) pinned to the Python oracle: for one producer the
placement of every entry is a function of the message lengths alone, so its
(start, footprint, slot) sequence must equal oracle.ring.spsc_image's on the
same lengths -- through wraps, PAD entries and credit waits; and every run
checks exactly-once, in-order delivery of the seeded payload bytes itself
(`bad` = 0), with one and with several producers (MPSC, paper lock)."""
import pytest

from oracle import threaded as T
from oracle.ring import Layout, spsc_image


@pytest.mark.parametrize("R,N,per,lo,hi", [(32768, 8, 1000, 1, 4096), (1 << 20, 16, 400, 1, 70000),
                                           (65536, 4, 300, 30000, 60000)])
def test_threaded_placements_equal_oracle(R, N, per, lo, hi):
    seed = 20260121
    got = T.placements(R, N, per, lo, hi, seed)
    img = spsc_image(Layout(R, N), T.lengths(seed, 0, per, lo, hi))
    want = [(start, f, q) for (q, start, f, pad) in img["entries"] if not pad]
    assert len(got) == per
    assert got == want


@pytest.mark.parametrize("producers", [1, 3])
def test_threaded_delivery_exact(producers):
    r = T.run(1 << 20, 16, producers, 300, 1, 70000, 7)
    assert r["bad"] == 0 and r["messages"] == 300 * producers, r
    assert r["threads"] == producers + 1
