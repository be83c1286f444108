"""rebalance_pair driven through the real engine.

A one-pair AcceLLM cluster gets a 1-token request that occupies member 0's
prefill, then k prompts arriving together while it runs: they are prefilled
in one job on member 0, get copies on member 1, join member 0's batch, and
member 0's next boundary runs rebalance_pair over exactly that batch with an
empty partner (SPEC.md:311's shape: A = {k requests}, B = {}). The MOVE
events of that boundary give the greedy's partition, which is checked
against an exhaustive search over all 2^k assignments ("oracle =
exhaustive search over <= 2^4 assignments")."""
from __future__ import annotations

import itertools

from paper_2411_05555_b200.abi import make_point


def case(prompts, decode=50):
    arr = [0.0] + [0.001] * len(prompts)
    pl = [20] + list(prompts)
    dl = [1] + [decode] * len(prompts)
    p = make_point(model="llama2-70b", device="h100", policy="accellm", instances=2, num_requests=len(arr),
                   trace_index=0, eff=(0.5, 0.8, 0.8))
    return p, (arr, pl, dl)


def objectives(a, b):
    """(count objective, token objective) of SPEC.md:308 for partition A|B."""
    c = len(a) - len(b)
    return max(0, abs(c) - 1), abs(sum(a) - sum(b))


def exhaustive_best(sizes):
    best = None
    for mask in itertools.product((0, 1), repeat=len(sizes)):
        a = [s for s, m in zip(sizes, mask) if not m]
        b = [s for s, m in zip(sizes, mask) if m]
        o = objectives(a, b)
        if best is None or o < best:
            best = o
    return best


def first_rebalance(events, prompts):
    """Partition after member 0's first rebalance: the MOVE events (kind 6)
    from instance 0 at the first time any request moves."""
    moves = [e for e in events if e.kind == 6 and e.inst == 0]
    if not moves:
        return list(prompts), []
    t0 = min(e.t for e in moves)
    moved = {e.a for e in moves if e.t == t0}  # request ids (1..k)
    a = [s for i, s in enumerate(prompts, start=1) if i not in moved]
    b = [s for i, s in enumerate(prompts, start=1) if i in moved]
    return a, b
