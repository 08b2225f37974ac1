"""Pipeline sizing and admission (TEST INFRASTRUCTURE ONLY).

PAPER.md §5 "Pipelining": two stages X and Y with execution
times T_X < T_Y; with K parallel workers in X, Theorem 1 assigns
M = ceil(K * T_Y / T_X) instances to Y so that both stages produce outputs at
the rate K / T_X; the proxy's Request Monitor rejects requests arriving faster
than K / T_X ("fast reject"); a request's latency is
T(q) = T_X + T_Y + Network(q).

Plain integer / Fraction arithmetic (no floats), a burst-1 token bucket for
the admission (the strictest reading of "the incoming request rate exceeds
K/T_X"), and a discrete-event simulation of the two stages used to check
Theorem 1 and the no-queueing claim.  Shares no code with the product path.
"""
from __future__ import annotations

from fractions import Fraction


def required_instances(t_x: int, t_y: int, k: int) -> int:
    """Theorem 1: M = ceil(T_Y / T_X * K)."""
    assert t_x > 0 and t_y > 0 and k >= 1
    return -(-(k * t_y) // t_x)


def steady_output_interval(t_x: int, k: int) -> Fraction:
    """'the proxy can submit requests every T_X/K seconds'."""
    return Fraction(t_x, k)


def fast_reject(arrivals: list[int], t_x: int, k: int) -> list[bool]:
    """Admission at rate K/T_X with burst 1 (PAPER.md:612-613 'whenever the
    incoming request rate exceeds K/T_X, the proxy rejects additional
    requests'): a request arriving at t is accepted iff t >= next, and then
    next = max(next, t) + T_X/K.  Exact rationals."""
    step = Fraction(t_x, k)
    nxt = None
    out = []
    for t in arrivals:
        if nxt is None or t >= nxt:
            out.append(True)
            nxt = (t if nxt is None else max(nxt, Fraction(t))) + step
        else:
            out.append(False)
    return out


def simulate(arrivals: list, t_x, t_y, k: int, m: int, network=0):
    """Discrete-event run of X (K workers) -> Y (M instances), round-robin
    dispatch to Y as the ResultDeliver does.  Each request
    goes to the earliest-free worker of X, then to the next Y instance in
    round-robin order; it starts there when that instance is free.  Returns
    per request (start_x, done_x, start_y, done_y)."""
    free_x = [Fraction(0)] * k
    free_y = [Fraction(0)] * m
    out = []
    for i, a in enumerate(arrivals):
        w = min(range(k), key=lambda j: (free_x[j], j))
        sx = max(Fraction(a), free_x[w])
        dx = sx + t_x
        free_x[w] = dx
        y = i % m
        sy = max(dx + network, free_y[y])
        dy = sy + t_y
        free_y[y] = dy
        out.append((sx, dx, sy, dy))
    return out
