"""Pins for oracle/pipeline.py (CPU only): Theorem 1 sizing and the fast-reject
admission of PAPER.md §5, pinned by the paper's two
pipeline figures (T_X = 4 s, T_Y = 12 s: one worker -> 3 instances, output
every 4 s; two workers -> 6 instances, output every 2 s), the latency formula
T(q) = T_X + T_Y + Network(q), brute-force token-bucket counting, and a
negative control (M - 1 instances queue without bound)."""
import itertools
import random
from fractions import Fraction

from oracle.pipeline import fast_reject, required_instances, simulate, steady_output_interval


def test_figures_of_the_paper():
    # PAPER.md:537-552 captions: T_X=4, T_Y=12; 1 worker -> outputs every 4 s
    # (3 instances of Y), 2 workers -> 6 instances, outputs every 2 s.
    assert required_instances(4, 12, 1) == 3
    assert steady_output_interval(4, 1) == 4
    assert required_instances(4, 12, 2) == 6
    assert steady_output_interval(4, 2) == 2
    assert required_instances(5, 5, 1) == 1
    assert required_instances(4, 10, 3) == 8           # ceil(30/4)
    assert steady_output_interval(3, 2) == Fraction(3, 2)


def test_theorem1_steady_state_and_no_queueing():
    """Arrivals at exactly the admitted rate K/T_X, M = ceil(K T_Y/T_X): Y emits
    one output every T_X/K after the first, and every request's latency is
    T_X + T_Y + Network (no request waits inside the instances)."""
    rng = random.Random(7)
    for _ in range(200):
        t_x = rng.randint(1, 20)
        t_y = rng.randint(t_x + 1, 80)
        k = rng.randint(1, 4)
        net = rng.randint(0, 3)
        m = required_instances(t_x, t_y, k)
        step = Fraction(t_x, k)
        arr = [i * step for i in range(120)]
        run = simulate(arr, t_x, t_y, k, m, net)
        done = [r[3] for r in run]
        assert all(b - a == step for a, b in zip(done, done[1:]))
        assert all(r[3] - a == t_x + t_y + net for r, a in zip(run, arr))


def test_under_provisioned_y_queues_without_bound():
    t_x, t_y, k = 4, 12, 2
    m = required_instances(t_x, t_y, k) - 1
    step = Fraction(t_x, k)
    arr = [i * step for i in range(300)]
    lat = [r[3] - a for r, a in zip(simulate(arr, t_x, t_y, k, m), arr)]
    assert lat[-1] > lat[100] > lat[10] > t_x + t_y


def test_fast_reject_examples():
    assert fast_reject([0, 1, 2, 3, 4], 4, 1) == [True, False, False, False, True]
    assert all(fast_reject([0, 10, 20, 30], 4, 1))
    assert fast_reject([0, 1, 2, 3, 4], 4, 2) == [True, False, True, False, True]


def test_fast_reject_never_exceeds_the_limit():
    """Over any window of W, the accepted count is <= ceil(W K / T_X) + 1
    (burst 1), and a request is rejected only if accepting it would break the
    spacing T_X/K from the previous accepted one."""
    rng = random.Random(3)
    for _ in range(100):
        t_x, k = rng.randint(1, 9), rng.randint(1, 3)
        arr = sorted(rng.randint(0, 200) for _ in range(rng.randint(1, 60)))
        acc = [t for t, ok in zip(arr, fast_reject(arr, t_x, k)) if ok]
        step = Fraction(t_x, k)
        assert all(b - a >= step for a, b in zip(acc, acc[1:]))
        for lo, hi in itertools.combinations(sorted(set(arr)), 2):
            n = sum(1 for t in acc if lo <= t <= hi)
            assert n <= (hi - lo) / step + 1
