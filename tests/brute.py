"""Brute-force references used to pin the oracle (tests only; pure Python, tiny inputs).

Each routine is the textbook definition, independent of oracle/saga_oracle.cpp:
  * brute_next_use: O(N^2) scan of the definition next_use[p] = min{q > p : b_q = b_p}.
  * brute_min: exhaustive search over every eviction decision sequence of demand paging
    without bypass (Belady 1966; "exhaustive search over all eviction decision
    sequences"), memoised on (position, cache set).
  * interval_greedy: OPTgen-style interval form of MIN -- a reuse interval (prev, p] can be a
    hit iff the cache has room over all of its interior points; intervals taken by right end.
  * brute_epoch_opt: exhaustive search over every epoch-batched policy (DESIGN.md reading
    "batch admission"): at each epoch any k-subset of the non-requested residents may be evicted.
"""
from __future__ import annotations

import functools
import itertools

INF = 0xFFFFFFFF


def brute_next_use(seq):
    out = []
    for p, b in enumerate(seq):
        nxt = INF
        for q in range(p + 1, len(seq)):
            if seq[q] == b:
                nxt = q
                break
        out.append(nxt)
    return out


def brute_min(seq, C):
    """minimum number of misses over all no-bypass demand-paging executions with capacity C."""
    seq = tuple(seq)

    @functools.lru_cache(maxsize=None)
    def go(i, cache):
        if i == len(seq):
            return 0
        b = seq[i]
        if b in cache:
            return go(i + 1, cache)
        if len(cache) < C:
            return 1 + go(i + 1, cache | frozenset([b]))
        best = None
        for v in cache:
            r = 1 + go(i + 1, (cache - frozenset([v])) | frozenset([b]))
            best = r if best is None else min(best, r)
        return best

    return go(0, frozenset())


def interval_greedy(seq, C):
    """misses of MIN via the interval formulation: hits = max #reuse intervals selectable such
    that at every interior point at most C-1 other selected intervals are open."""
    n = len(seq)
    last = {}
    intervals = []  # (prev, p): block held from prev to p
    for p, b in enumerate(seq):
        if b in last:
            intervals.append((last[b], p))
        last[b] = p
    occ = [0] * n  # number of selected intervals covering the open point set (prev, p)
    hits = 0
    for (a, b) in sorted(intervals, key=lambda x: (x[1], x[0])):
        if all(occ[x] < C - 1 for x in range(a + 1, b)) if b > a + 1 else True:
            # the interval also occupies one slot at each interior point
            if C >= 1:
                for x in range(a + 1, b):
                    occ[x] += 1
                hits += 1
    return n - hits


def brute_epoch_opt(epochs, owner_of, C):
    """epochs: list of (inv_owners:set, records:list of lids).  Minimal misses over all
    epoch-batched eviction choices; None if some epoch needs more than C distinct blocks."""
    epochs = [(frozenset(inv), tuple(rec)) for inv, rec in epochs]
    for _, rec in epochs:
        if len(set(rec)) > C:
            return None

    @functools.lru_cache(maxsize=None)
    def go(j, S):
        if j == len(epochs):
            return 0
        inv, rec = epochs[j]
        S = frozenset(b for b in S if owner_of[b] not in inv)
        if not rec:
            return go(j + 1, S)
        A = frozenset(rec)
        miss = len(A - S)
        k = len(S) + miss - C
        cand = sorted(S - A)
        if k <= 0:
            return miss + go(j + 1, S | A)
        best = None
        for V in itertools.combinations(cand, k):
            r = miss + go(j + 1, (S - frozenset(V)) | A)
            best = r if best is None else min(best, r)
        return best

    return go(0, frozenset())
