"""Pins of the F4 online-statistics oracle (oracle/tool_stats.py): textbook nearest-rank
percentiles, the EMA's closed forms and its recurrence, the window and causality rules, and the
cold start -- nothing here calls the CUDA path.
"""
import math
import random

import numpy as np
import pytest

from gen import default_place_cfg, make, pattern_labels
from oracle.tool_stats import ema_truncated, nearest_rank, samples, t_end, tool_stats


def test_nearest_rank_textbook():
    # the standard worked example of the nearest-rank method: {15, 20, 35, 40, 50}
    v = [15, 20, 35, 40, 50]
    assert [nearest_rank(v, p) for p in (50, 300, 400, 500, 1000)] == [15, 20, 20, 35, 50]
    assert nearest_rank(range(1, 101), 950) == 95          # 1..100: P95 = 95
    assert nearest_rank([7], 950) == 7
    assert nearest_rank(range(256, 0, -1), 950) == 244     # rank ceil(0.95 * 256) = 244


def test_ema_identical_observations_equal_L():
    # after N identical observations of length L the estimate equals L (prior n0 = L)
    for L in (0, 1, 175, 850, 1250, 6000, 100_000):
        for k in (0, 1, 5, 64, 65, 300):
            assert ema_truncated([L] * min(k, 64), k, L, 64) == L


def test_ema_matches_the_recurrence():
    # n <- 0.8 n + 0.2 obs from n0; the truncated sum differs by at most 0.8^64 * max + rounding
    rng = random.Random(3)
    for _ in range(200):
        k = rng.randint(0, 400)
        obs = [rng.randint(0, 5000) for _ in range(k)]
        n0 = rng.randint(0, 5000)
        n = float(n0)
        for o in obs:
            n = 0.8 * n + 0.2 * o
        m = min(k, 64)
        got = ema_truncated(obs[k - m:], k, n0, 64)
        assert abs(got - n) <= 0.5 + 5000 * 0.8 ** 64 + 1e-6, (got, n)
        if k <= 64:
            assert abs(got - n) <= 0.5 + 1e-6


def _stats_trace():
    """one node, tools alternate per step: sessions of 6 calls, tool = step % 2"""
    d = make("C2", n_sessions=60, n_nodes=2)
    lab = (np.asarray(d.call_aeg_node) % 2).astype(np.uint32)
    return d, default_place_cfg(0), lab


def test_history_is_causal_and_windowed():
    d, pc, lab = _stats_trace()
    S = samples(d, pc, lab)
    ttl, obs = tool_stats(d, pc, lab, 2, p_pm=950, window=8, min_samples=3)
    for c in range(0, d.n_calls, 7):
        x = int(lab[c])
        ts, lats, obss = S.get(x, ([], [], []))
        T = t_end(d, pc, c)
        hist = [i for i in range(len(ts)) if ts[i] <= T]           # completed by the tool start
        assert hist == list(range(len(hist)))                       # a prefix in completion order
        n = min(len(hist), 8)
        if n >= 3:
            w = sorted(lats[len(hist) - n:len(hist)])
            assert ttl[c] == min(w[math.ceil(0.95 * n) - 1], 10 ** 9)
        else:
            assert ttl[c] == d.node_ttl_base_us[d.call_aeg_node[c]]  # cold start


def test_window_excludes_old_samples():
    d, pc, lab = _stats_trace()
    # a huge latency only in the oldest samples cannot reach the last-8 window
    ttl8, _ = tool_stats(d, pc, lab, 2, window=8, min_samples=1)
    ttl_all, _ = tool_stats(d, pc, lab, 2, window=1024, min_samples=1)
    S = samples(d, pc, lab)
    some = False
    for c in range(d.n_calls):
        ts, lats, _ = S.get(int(lab[c]), ([], [], []))
        k = sum(1 for t in ts if t <= t_end(d, pc, c))
        if k > 8:
            assert ttl8[c] == nearest_rank(lats[k - 8:k], 950)
            assert ttl_all[c] == nearest_rank(lats[max(0, k - 1024):k], 950)
            some = True
    assert some


def test_labels_checked():
    d, pc, lab = _stats_trace()
    with pytest.raises(ValueError):
        tool_stats(d, pc, lab, 1)
