"""TEST INFRASTRUCTURE ONLY -- restated binomial checkpoint schedule.

Follows ``pkg/src/odegrad/checkpointing.py``: the closed-form minimal
recomputation count (``revolve_count``, :32-41), the stage-storing split
recurrence (``_dp``, :44-51; ``_argmin_split``, :61-67) and the action
generator (``revolve_schedule``, :83-170) with its two segment kinds (a plain
segment whose start state is positioned, and a segment whose last record is
already slotted).  Actions are tuples ``(kind, step, start, stop)`` with kind
in {"advance", "store", "restore", "reverse"}.
"""

from __future__ import annotations

import math
from functools import lru_cache


def revolve_count(nt: int, nc: int) -> int:
    """Closed-form minimal extra forward steps (checkpointing.py:32-41)."""
    if nt < 1 or nc < 1:
        raise ValueError("need nt >= 1 and nc >= 1")
    if nt == 1:
        return 0
    t = 1
    while True:
        lo = math.comb(nc + t - 1, t - 1)
        hi = math.comb(nc + t, t)
        if lo < nt <= hi:
            break
        t += 1
    return (t - 1) * nt - math.comb(nc + t, t - 1) + 1


@lru_cache(maxsize=None)
def split_cost(length: int, slots: int) -> int:
    """Recomputation cost of reversing ``length`` steps with ``slots`` records
    (checkpointing.py:44-51)."""
    if length <= 1 or slots >= length - 1:
        return 0
    if slots == 1:
        return (length - 1) * (length - 2) // 2
    return min((m - 1) + split_cost(length - m, slots - 1) + split_cost(m, slots)
               for m in range(1, length))


def dp_optimal_count(nt: int, nc: int) -> int:
    if nt < 1 or nc < 1:
        raise ValueError("need nt >= 1 and nc >= 1")
    return split_cost(nt, nc)


def best_split(length: int, slots: int) -> int:
    """Smallest m attaining the split minimum (checkpointing.py:61-67)."""
    costs = [(m - 1) + split_cost(length - m, slots - 1) + split_cost(m, slots)
             for m in range(1, length)]
    return 1 + costs.index(min(costs))


def revolve_schedule(nt: int, nc: int):
    """Action list reversing steps nt-1..0 with <= nc live records."""
    if nt < 1 or nc < 1:
        raise ValueError("need nt >= 1 and nc >= 1")
    out = []
    A = lambda i, j: out.append(("advance", -1, i, j))   # noqa: E731
    S = lambda k: out.append(("store", k, -1, -1))        # noqa: E731
    L = lambda k: out.append(("restore", k, -1, -1))      # noqa: E731
    R = lambda k: out.append(("reverse", k, -1, -1))      # noqa: E731

    def plain(o, n, c, anchor):
        if n == 0:
            return
        last = o + n - 1
        if n == 1:
            A(o, o + 1)
            R(o)
        elif c >= n - 1:
            for k in range(o, last):
                A(k, k + 1)
                S(k)
            A(last, last + 1)
            R(last)
            for k in range(last - 1, o - 1, -1):
                L(k)
                R(k)
        elif c == 1:
            A(o, o + 1)
            S(o)
            A(o + 1, o + n)
            R(last)
            for k in range(last - 1, o, -1):
                L(o)
                A(o + 1, k + 1)
                R(k)
            L(o)
            R(o)
        else:
            m = best_split(n, c)
            A(o, o + m)
            S(o + m - 1)
            plain(o + m, n - m, c - 1, o + m - 1)
            L(anchor)
            slotted(o, m, c, anchor)

    def slotted(o, n, c, anchor):
        last = o + n - 1
        if n == 1:
            R(o)
        elif c >= n - 1:
            for k in range(o, last - 1):
                A(k, k + 1)
                S(k)
            A(last - 1, last)
            R(last)
            R(last - 1)
            for k in range(last - 2, o - 1, -1):
                L(k)
                R(k)
        elif c == 1:
            R(last)
            for k in range(last - 1, o - 1, -1):
                L(anchor)
                A(o, k + 1)
                R(k)
        else:
            m = best_split(n, c)
            A(o, o + m)
            S(o + m - 1)
            slotted(o + m, n - m, c - 1, o + m - 1)
            L(anchor)
            slotted(o, m, c, anchor)

    plain(0, nt, nc, -1)
    return out


def audit(nt: int, nc: int):
    """Dry run: (extra advanced steps after the first reverse, max live slots)
    (checkpointing.py:343-390)."""
    acts = revolve_schedule(nt, nc)
    live, peak, pos, hand, extra, advanced, started = set(), 0, 0, None, 0, 0, False
    rev = []
    for kind, step, a, b in acts:
        if kind == "advance":
            assert a == pos, (a, pos)
            advanced += b - a
            if started:
                extra += b - a
            pos, hand = b, b - 1
        elif kind == "store":
            assert step == hand
            live.add(step)
            peak = max(peak, len(live))
        elif kind == "restore":
            pos, hand = step + 1, None
        else:
            if hand != step:
                assert step in live, (step, live)
                live.remove(step)
            if not started:
                assert advanced == nt
                started = True
            rev.append(step)
    assert rev == list(range(nt - 1, -1, -1))
    return extra, peak
