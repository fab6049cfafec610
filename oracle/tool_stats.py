"""CPU oracle of F4's online tool statistics (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module; it
shares no code with paper_2605_00528_b200/.  Plain Python, written from:

  Alg. 1 line 2: "ttl_base <- Percentile(H_t, p)" over the latency history H_t of tool t;
    P:694 "We maintain per-tool-type latency distributions ... and set TTL to the p-th percentile
    of expected duration, where p is configurable (default 95%)".
  P:685: "n_obs is the expected observation length estimated from tool-type-specific
    distributions maintained via exponential moving averages".
  S:273 (SPEC design decision): "nearest-rank on the sorted sample window (window = last 256
    samples per tool type)"; S:245 / S:159: EMA smoothing 0.2; "after N identical observations of
    length L, the estimate equals L".

Readings (DESIGN.md §3 R-online): a tool sample is a call d with a successor d' in its session
(latency t(d') - t_end(d), clamped to [0, 2^32 - 1]; observation = new tokens of d'), completed
at t(d'); the history of call c is its tool's samples completed at or before c's tool start
t_end(c); below min_samples the node's static TTL base is kept (cold start); the EMA starts at
the node's observation length and is evaluated as its explicit sum over the newest `terms`
samples (dropped weight 0.8^terms), in fp64 in a fixed order, rounded half up.
"""
from __future__ import annotations

import bisect

import numpy as np


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def t_end(d, pc, c: int) -> int:
    """Tool start of call c: t_c + prefill(new) + decode(out) (R-el)."""
    return int(d.call_t_us[c]) + ceil_div(int(d.call_new_tokens[c]) * 1_000_000, pc["prefill_tok_s"]) + \
        ceil_div(int(d.call_output_tokens[c]) * 1_000_000, pc["decode_tok_s"])


def nearest_rank(values, p_pm: int) -> int:
    """Nearest-rank percentile: the ceil(p n / 1000)-th smallest of n >= 1 values."""
    v = sorted(int(x) for x in values)
    r = max(1, (p_pm * len(v) + 999) // 1000)
    return v[r - 1]


def ema_weights(terms: int):
    """0.2 * 0.8^i and 0.8^i (i = 0..terms), by repeated fp64 multiplication."""
    w = [0.2]
    for _ in range(1, max(terms, 1)):
        w.append(w[-1] * 0.8)
    p = [1.0]
    for _ in range(terms):
        p.append(p[-1] * 0.8)
    return w, p


def ema_truncated(newest, k: int, n0: float, terms: int) -> int:
    """round-half-up of [k <= terms] 0.8^k n0 + sum_{i=m-1..0} 0.2 0.8^i obs_{k-1-i}, m = min(k, terms);
    `newest` = obs_{k-m} .. obs_{k-1} (oldest first) of a history of k samples."""
    m = min(k, terms)
    assert len(newest) == m
    w, p = ema_weights(terms)
    acc = p[k] * float(n0) if k <= terms else 0.0
    for i in range(m - 1, -1, -1):
        acc = acc + w[i] * float(newest[m - 1 - i])
    return int(np.floor(acc + 0.5))


def samples(d, pc, label):
    """Per tool: (completion times, latencies, observations) in completion (trace) order."""
    n_s = int(np.asarray(d.session_type).shape[0])
    seqs = [[] for _ in range(n_s)]
    for c, s in enumerate(np.asarray(d.call_session).tolist()):
        seqs[s].append(c)
    per = {}
    for q in seqs:
        for a, b in zip(q[:-1], q[1:]):
            lat = min(max(int(d.call_t_us[b]) - t_end(d, pc, a), 0), 0xFFFFFFFF)
            per.setdefault(int(label[a]), []).append((b, int(d.call_t_us[b]), lat, int(d.call_new_tokens[b])))
    out = {}
    for x, lst in per.items():
        lst.sort()  # completion order = index of d'
        out[x] = ([t for _, t, _, _ in lst], [l for _, _, l, _ in lst], [o for _, _, _, o in lst])
    return out


def tool_stats(d, pc, label, n_labels, p_pm=950, window=256, min_samples=20, terms=64, calls=None):
    """(ttl int64 [len(calls)], obs uint32 [len(calls)]) for the given calls (default: all)."""
    label = np.asarray(label)
    if (label >= n_labels).any():
        raise ValueError("label >= n_labels")
    S = samples(d, pc, label)
    calls = range(d.n_calls) if calls is None else calls
    ttl, obs = [], []
    for c in calls:
        x = int(label[c])
        ts, lats, obss = S.get(x, ([], [], []))
        k = bisect.bisect_right(ts, t_end(d, pc, c))
        v = int(d.call_aeg_node[c])
        n = min(k, window)
        if n >= min_samples and n > 0:
            ttl.append(min(nearest_rank(lats[k - n:k], p_pm), 1_000_000_000))
        else:
            ttl.append(int(d.node_ttl_base_us[v]))
        m = min(k, terms)
        obs.append(min(ema_truncated(obss[k - m:k], k, int(d.node_obs_tokens[v]), terms), 0xFFFFFFFF))
    return np.array(ttl, np.int64), np.array(obs, np.uint32)
