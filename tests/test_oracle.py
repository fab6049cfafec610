"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU needed).

Every test compares the oracle with something other than itself: SPEC worked examples,
values printed in PAPER.md / computed independently in the survey (tests/golden/),
closed forms (Observation 1, Theorem 2 limit case), brute force on tiny inputs, exact
rational arithmetic and invariants.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from gen import (default_place_cfg, make, make_c1, make_chain_limit, make_obs1, make_random_small,
                 make_stream_trace, sweep_caps)
from tests.brute import brute_epoch_opt, brute_min, brute_next_use, interval_greedy

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def misses(ctr, O):
    return int(ctr[O.CI["MISSES"]] + ctr[O.CI["MIG_MISSES"]] + ctr[O.CI["PF_MISSES"]])


def hits(ctr, O):
    return int(ctr[O.CI["HITS"]] + ctr[O.CI["MIG_HITS"]] + ctr[O.CI["PF_HITS"]])


# ------------------------------------------------------------------------------------------
# A5 scalar formulas: SPEC worked examples
# ------------------------------------------------------------------------------------------

def _score_inputs(R, S):
    """(d, tau, size, smax) with d/tau = R and size/smax = S exactly in fp32 (the examples' values)."""
    d, tau = {0.0: (0, 1), 0.5: (1, 2), 1.0: (7, 7)}[R]
    size, smax = {0.0: (0, 1), 0.25: (1, 4), 1.0: (3, 3)}[S]
    return d, tau, size, smax


def test_eviction_score_examples(O):
    # through the oracle's score() (eq:recency / eq:size normalisation included)
    for ex in gold("spec_examples.json")["eviction_score"]:
        d, tau, size, smax = _score_inputs(ex["R"], ex["S"])
        s, q = O.score32(0.3, 0.5, 0.2, d, tau, size, smax, ex["P"])
        assert np.float32(s) == np.float32(ex["fp32"]), ex["cite"]
        assert q == ex["q"], ex["cite"]
        # fp64 evaluation of eq:eviction agrees within 1e-6
        assert abs(0.3 * ex["R"] + 0.5 * (1 - ex["P"]) + 0.2 * ex["S"] - s) < 1e-6


def test_reuse_examples(O):
    for ex in gold("spec_examples.json")["reuse"]:
        P = O.reuse32(ex["p"], ex["q16"], ex["ncur"], ex["nobs"])
        assert np.float32(P) == np.float32(ex["fp32"]), ex["cite"]


def test_overlap_examples(O):
    # eq:overlap linear form n_cur / (n_cur + n_obs) via a single p=1 whole-context edge
    for ex in gold("spec_examples.json")["overlap"]:
        P = O.reuse32([1.0], [65536], ex["ncur"], ex["nobs"])
        assert np.float32(P) == np.float32(ex["value"]), ex["cite"]


def test_fig2_aeg_reuse_and_keys(O):
    g = gold("fig2_aeg.json")
    for v in range(5):
        es = [(p, 65536) for (u, _, p) in g["edges"] if u == v]
        P = O.reuse32([p for p, _ in es], [q for _, q in es], g["ncur"], g["obs"][v])
        assert np.float32(P) == np.float32(g["p_reuse_fp32"][v]), v
        _, q = O.score32(0.3, 0.5, 0.2, 0, 0, 750, 750, P)   # R = 0 (tau = 0), S = 1
        assert q == g["q_at_R0_S1"][v], v


def _ttl_rational(el, ttl_base, ttl_max, occ, cap, low=700, high=900):
    """Alg. alg:ttl + eq:pressure in exact rationals: protected iff el < min(ttl*(1-m/2), TTL_max)."""
    m = (Fraction(occ, cap) - Fraction(low, 1000)) / (Fraction(high - low, 1000))
    m = min(max(m, Fraction(0)), Fraction(1))
    return el < min(Fraction(ttl_base) * (1 - m / 2), Fraction(ttl_max))


def test_ttl_examples(O):
    for ex in gold("spec_examples.json")["ttl"]:
        cap = 1000
        occ = ex["occ_pm"]
        eff = ex["effective_us"]
        assert O.ttl_protect(eff - 1, ex["ttl_base_us"], 300_000_000, occ, cap), ex["cite"]
        assert not O.ttl_protect(eff, ex["ttl_base_us"], 300_000_000, occ, cap), ex["cite"]


def test_ttl_predicate_matches_rational_definition(O):
    rng = np.random.default_rng(7)
    for _ in range(20000):
        cap = int(rng.integers(1, 5000))
        occ = int(rng.integers(0, cap + 1))
        ttl = int(rng.integers(0, 1_000_000_001))
        ttl_max = int(rng.choice([300_000_000, int(rng.integers(1, 10 ** 9))]))
        el = int(rng.integers(-10 ** 6, 10 ** 9))
        assert O.ttl_protect(el, ttl, ttl_max, occ, cap) == _ttl_rational(el, ttl, ttl_max, occ, cap)


def test_splitmix64_reference(O):
    ex = gold("spec_examples.json")["splitmix64"]
    assert O.splitmix64(ex["in"]) == ex["out"]


# ------------------------------------------------------------------------------------------
# A4 next use / local ids / first touches by brute force
# ------------------------------------------------------------------------------------------

def _check_next_use(o, w):
    s = o.stream(w)
    seq = [int(x) for x in s["block"]]
    nu = o.next_use(w)
    assert list(nu["next_use"]) == brute_next_use(seq)
    uniq = sorted(set(seq))
    assert list(nu["local_id"]) == [uniq.index(b) for b in seq]
    assert list(nu["ftn"]) == [int(b not in seq[:p]) for p, b in enumerate(seq)]
    # first in epoch: no earlier record of the same epoch touches the block
    ev_of = np.zeros(len(seq), np.int64)
    pos = 0
    gi = 0
    for j, ev in enumerate(s["events"]):
        for _ in range(ev[1]):
            p0, ln = s["groups"][gi][0], s["groups"][gi][1]
            ev_of[p0:p0 + ln] = j
            gi += 1
    fie = [int(all(not (seq[q] == b and ev_of[q] == ev_of[p]) for q in range(p))) for p, b in enumerate(seq)]
    assert list(nu["fie"]) == fie
    # W_lo / W_hi by direct counting over record epochs
    rec_epochs = sorted(set(ev_of.tolist()))
    wlo = max(len(set(seq[p] for p in range(len(seq)) if ev_of[p] == j)) for j in rec_epochs) if seq else 0
    first = {}
    last = {}
    for p, b in enumerate(seq):
        first.setdefault(b, p)
        last[b] = p
    whi = 0
    for j in rec_epochs:
        ps = [p for p in range(len(seq)) if ev_of[p] == j]
        st, en = min(ps), max(ps)
        whi = max(whi, sum(1 for b in first if first[b] <= en and last[b] >= st))
    assert o.sweep_range(w) == (wlo, whi)


def test_next_use_c1_bruteforce(O):
    o = O.Oracle(make_c1(), default_place_cfg())
    _check_next_use(o, 0)
    g = gold("c1.json")
    assert o.sweep_range(0) == (g["w_lo"], g["w_hi"])
    assert sweep_caps(g["w_lo"], g["w_hi"], 8, 64) == g["caps"]
    assert o.stream(0)["block"].size == g["n_accesses"] and o.n_local(0) == g["n_distinct"]


@pytest.mark.parametrize("seed", range(12))
def test_next_use_random_bruteforce(O, seed):
    d = make_random_small(seed, n_sessions=6, n_nodes=2)
    o = O.Oracle(d, default_place_cfg(seed))
    for w in range(d.n_nodes):
        _check_next_use(o, w)


# ------------------------------------------------------------------------------------------
# MIN: brute force = interval greedy = oracle heap
# ------------------------------------------------------------------------------------------

def test_belady_spec_example(O):
    ex = gold("spec_examples.json")["belady"]
    o = O.Oracle(make_stream_trace(ex["seq"]), default_place_cfg())
    assert o.min_misses(0, ex["cap"]) == ex["misses"] == brute_min(ex["seq"], ex["cap"])


def test_min_bruteforce_random(O):
    rng = np.random.default_rng(11)
    for _ in range(400):
        nb = int(rng.integers(2, 7))
        n = int(rng.integers(1, 13))
        seq = [int(x) for x in rng.integers(0, nb, size=n)]
        o = O.Oracle(make_stream_trace(seq), default_place_cfg())
        for C in range(1, 6):
            m = o.min_misses(0, C)
            assert m == brute_min(seq, C), (seq, C)
            assert m == interval_greedy(seq, C), (seq, C)


# ------------------------------------------------------------------------------------------
# LRU / LRU + Prefix baselines (Table tab:competitive; DESIGN.md R-lru): with one
# access per epoch the epoch-batched replay is per-access paging, which must equal a textbook
# LRU simulation (ordered dictionary) -- victims, in order, and misses.
# ------------------------------------------------------------------------------------------

def _textbook_lru(seq, C, shared=0):
    """Per-access LRU without bypass; with `shared` > 0 blocks < shared are evicted only when no
    other block is resident (prefix caching)."""
    from collections import OrderedDict
    cache, miss, victims = OrderedDict(), 0, []
    for b in seq:
        if b in cache:
            cache.move_to_end(b)
            continue
        miss += 1
        if len(cache) == C:
            priv = [x for x in cache if x >= shared]
            v = priv[0] if priv else next(iter(cache))
            del cache[v]
            victims.append(v)
        cache[b] = True
    return miss, victims


@pytest.mark.parametrize("n_shared", [0, 2])
def test_lru_equals_textbook(O, n_shared):
    rng = np.random.default_rng(21 + n_shared)
    for _ in range(300):
        nb = int(rng.integers(n_shared + 2, n_shared + 8))
        n = int(rng.integers(1, 25))
        seq = [int(x) for x in rng.integers(0, nb, size=n)]
        o = O.Oracle(make_stream_trace(seq, n_shared=n_shared), default_place_cfg())
        lid = o.next_use(0)["local_id"]
        g2l = {int(b): int(l) for b, l in zip(o.stream(0)["block"], lid)}
        for C in range(1, 6):
            for pol, shared in ((O.POL_LRU, 0), (O.POL_LRU_PREFIX, n_shared)):
                m, vic = _textbook_lru(seq, C, shared)
                ctr, log = o.replay(pol, 0, C, log=True)
                assert misses(ctr, O) == m, (seq, C, pol)
                assert [int(x) for x in log] == [g2l[v] for v in vic], (seq, C, pol)


def test_lru_bounded_by_belady_epoch(O):
    for seed in range(6):
        d = make_random_small(seed, n_sessions=6, n_nodes=2, max_calls=5, max_blocks=8)
        o = O.Oracle(d, default_place_cfg(seed))
        for w in range(d.n_nodes):
            lo, hi = o.sweep_range(w)
            for C in range(max(lo, 1), hi + 3):
                b = o.replay(O.POL_BELADY, w, C)
                for pol in (O.POL_LRU, O.POL_LRU_PREFIX):
                    r = o.replay(pol, w, C)
                    assert hits(r, O) <= hits(b, O), (seed, w, C, pol)


# ------------------------------------------------------------------------------------------
# BELADY-epoch = brute-force optimum over epoch-batched policies (incl. invalidations)
# ------------------------------------------------------------------------------------------

def _node_epochs(o, w):
    s = o.stream(w)
    lid = o.next_use(w)["local_id"]
    own = o.lid_owner(w)
    eps = []
    gi = ii = 0
    for ev in s["events"]:
        rec = []
        for _ in range(ev[1]):
            p0, ln = s["groups"][gi][0], s["groups"][gi][1]
            rec += [int(x) for x in lid[p0:p0 + ln]]
            gi += 1
        inv = set(int(x) for x in s["inv"][ii:ii + ev[2]])
        ii += ev[2]
        eps.append((inv, rec))
    return eps, own


def test_belady_epoch_bruteforce_streams(O):
    rng = np.random.default_rng(3)
    for _ in range(150):
        nb = int(rng.integers(2, 7))
        n = int(rng.integers(1, 12))
        seq = [int(x) for x in rng.integers(0, nb, size=n)]
        ep = np.sort(rng.integers(1, max(2, n // 2 + 2), size=n)).tolist()
        o = O.Oracle(make_stream_trace(seq, ep), default_place_cfg())
        eps, own = _node_epochs(o, 0)
        for C in range(1, 6):
            ref = brute_epoch_opt(eps, own, C)
            ctr = o.replay(O.POL_BELADY, 0, C)
            if ref is None:
                assert ctr[O.CI["INFEASIBLE_EPOCH"]] > 0
            else:
                assert ctr[O.CI["INFEASIBLE_EPOCH"]] == 0 and misses(ctr, O) == ref, (seq, ep, C)
                assert misses(ctr, O) >= o.min_misses(0, C)


def test_belady_epoch_bruteforce_with_migrations(O):
    n_inv = 0
    for seed in range(60):
        d = make_random_small(seed, n_sessions=5, n_nodes=2, max_calls=3, max_blocks=4)
        pc = default_place_cfg(seed)
        pc.update(kappa=1, theta_pm=100000)  # force affinity + queues so that stealing happens
        o = O.Oracle(d, pc)
        for w in range(d.n_nodes):
            eps, own = _node_epochs(o, w)
            n_inv += sum(len(i) for i, _ in eps)
            n_lid = o.n_local(w)
            if n_lid > 9:
                continue
            for C in range(1, 6):
                ref = brute_epoch_opt(eps, own, C)
                ctr = o.replay(O.POL_BELADY, w, C)
                if ref is None:
                    assert ctr[O.CI["INFEASIBLE_EPOCH"]] > 0
                else:
                    assert misses(ctr, O) == ref, (seed, w, C)
    assert n_inv > 0  # the fixture did exercise invalidations


# ------------------------------------------------------------------------------------------
# Closed forms: Observation 1 and the Theorem 2 limit case
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("c", [1, 4, 7])
def test_observation1_closed_form(O, c):
    for k in range(1, 21):
        o = O.Oracle(make_obs1(k, c), default_place_cfg())
        big = 2 * c * k
        ev = o.replay(O.POL_EVICT_ALL, 0, big)
        assert misses(ev, O) == 2 * c * k * (k + 1) // 2          # sum_j j*c per session
        ret = o.replay(O.POL_BELADY, 0, big)
        assert misses(ret, O) == 2 * c * k                         # initial prefill only (in blocks)
        assert ev[O.CI["REGEN_TOKENS"]] == 16 * 2 * c * (k * (k + 1) // 2 - k)
        assert ret[O.CI["REGEN_TOKENS"]] == 0


@pytest.mark.parametrize("seed", range(40))
def test_theorem2_limit_case(O, seed):
    d = make_chain_limit(seed)
    o = O.Oracle(d, default_place_cfg(seed))
    wlo, whi = o.sweep_range(0)
    ftn = int(o.next_use(0)["ftn"].sum())
    for C in (whi, whi + 3):
        a = o.replay(O.POL_AEG, 0, C)
        b = o.replay(O.POL_BELADY, 0, C)
        assert misses(a, O) == misses(b, O) == o.min_misses(0, C) == ftn == a[O.CI["COMPULSORY_NODE"]]


# ------------------------------------------------------------------------------------------
# Invariants: capacity, conservation, hits(AEG) <= hits(BELADY-epoch) <= hits(MIN), sweep ends
# ------------------------------------------------------------------------------------------

def _invariants(o, d, O, caps_per_node=True):
    for w in range(d.n_nodes):
        if o.stream(w)["block"].size == 0:
            continue
        wlo, whi = o.sweep_range(w)
        ftn = int(o.next_use(w)["ftn"].sum())
        caps = sorted(set([wlo, (wlo + whi) // 2, whi, whi + 5]))
        for C in caps:
            if C == 0:
                continue
            a = o.replay(O.POL_AEG, w, C)
            b = o.replay(O.POL_BELADY, w, C)
            x = o.replay(O.POL_EVICT_ALL, w, C)
            mn = o.min_misses(w, C)
            n = o.stream(w)["block"].size
            for ctr in (a, b, x):
                assert ctr[O.CI["INFEASIBLE_EPOCH"]] == 0
                assert ctr[O.CI["PEAK_RESIDENT"]] <= C
                assert ctr[O.CI["ACCESSES"]] == n == hits(ctr, O) + misses(ctr, O)
                assert ctr[O.CI["COMPULSORY_NODE"]] == ftn
                assert ctr[O.CI["COMPULSORY_GLOBAL"]] <= ctr[O.CI["MISSES"]]
            assert hits(a, O) <= hits(b, O) <= n - mn
            assert hits(x, O) <= hits(b, O)
            if C >= whi:
                assert mn == ftn
        if wlo > 1:
            inf = o.replay(O.POL_BELADY, w, wlo - 1)
            assert inf[O.CI["INFEASIBLE_EPOCH"]] > 0


def test_invariants_c1(O):
    d = make_c1()
    _invariants(O.Oracle(d, default_place_cfg()), d, O)
    dl = make_c1(limit_case=True)
    o = O.Oracle(dl, default_place_cfg())
    wlo, whi = o.sweep_range(0)
    assert misses(o.replay(O.POL_AEG, 0, whi), O) == misses(o.replay(O.POL_BELADY, 0, whi), O)


@pytest.mark.parametrize("seed", range(10))
def test_invariants_random(O, seed):
    d = make_random_small(seed, n_sessions=8, n_nodes=3, max_calls=5, max_blocks=8)
    pc = default_place_cfg(seed)
    if seed % 2:
        pc.update(kappa=1, theta_pm=100000)
    _invariants(O.Oracle(d, pc), d, O)


def test_invariants_small_c2(O):
    d = make("C2", n_sessions=12, n_nodes=2)
    _invariants(O.Oracle(d, default_place_cfg(2)), d, O)


# ------------------------------------------------------------------------------------------
# A2 placement: SPEC routing / stealing examples and P6 invariants
# ------------------------------------------------------------------------------------------

def _two_call_trace(gap_us, n_nodes=2, ttl=2_000_000, extra_sessions=()):
    """session 0 calls at t=1 and t=gap; optional other sessions (t, calls...)."""
    from gen.tracegen import TraceDesc, _AEGBuilder
    b = _AEGBuilder()
    b.add_node(ttl, 0, False)
    b.add_node(ttl, 0, False)
    b.add_edge(0, 1, 1.0)
    aeg = b.finish()
    calls = [(1, 0, 0), (gap_us, 0, 1)] + list(extra_sessions)
    calls.sort(key=lambda x: (x[0], x[1]))
    ns = max(c[1] for c in calls) + 1
    n = len(calls)
    return TraceDesc(
        name="route", n_nodes=n_nodes, n_blocks=ns, seed=0,
        call_t_us=np.array([c[0] for c in calls], np.int64), call_session=np.array([c[1] for c in calls], np.uint32),
        call_aeg_node=np.array([c[2] for c in calls], np.uint32), call_prompt_tokens=np.full(n, 16, np.uint32),
        call_output_tokens=np.full(n, 3, np.uint32), call_new_tokens=np.full(n, 16, np.uint32),
        call_is_last=np.zeros(n, np.uint8), call_range_off=np.arange(n + 1, dtype=np.uint32),
        range_block_lo=np.array([c[1] for c in calls], np.uint32), range_len=np.ones(n, np.uint32),
        session_type=np.zeros(ns, np.uint16), session_block_lo=np.arange(ns, dtype=np.uint32),
        session_block_len=np.ones(ns, np.uint32), type_shared_lo=np.array([0], np.uint32),
        type_shared_len=np.array([0], np.uint32), **aeg)


def test_route_new_session_argmin(O):
    # a new session goes to the argmin-load worker (ties -> lowest worker id)
    d = _two_call_trace(10 ** 7, extra_sessions=[(2, 1, 0)])
    node, _, _, _ = O.Oracle(d, default_place_cfg()).placement()
    assert node[0] == 0 and node[1] == 1


def test_route_overloaded_affinity_reroutes(O):
    # cached at w but load(w) >= theta -> argmin.  kappa=1 and a long call by session 1
    # at node 0 make load(0) = 1 > 0.8 when session 0 returns.
    from gen.tracegen import TraceDesc
    d = _two_call_trace(300_000, extra_sessions=[(2, 1, 0), (200_001, 1, 1)])
    d.call_output_tokens[:] = 3000  # 100 s decode: calls stay in service
    pc = default_place_cfg()
    pc["kappa"] = 1
    o = O.Oracle(d, pc)
    node, _, _, rr = o.placement()
    assert rr >= 1


def test_steal_fires_and_antithrash(O):
    # a thief idle >= T_idle and a victim holding a pending call -> steal.
    # kappa = 1, affinity forced (theta huge).  e=1: s0 -> node 0, s1 -> node 1 (argmin),
    # s2 -> node 0 (tie on load and active count -> lowest id), queued behind s0 (pending).
    # s1's call is short, so node 1 is idle for a whole epoch at e=3 and steals s2.
    d = _two_call_trace(10 ** 8, n_nodes=2, extra_sessions=[(2, 1, 0), (3, 2, 0)])
    out = np.full(d.n_calls, 300, np.uint32)
    out[d.call_session == 1] = 4  # 137 ms: ties node 0 on load (min(rem, E) = E), done at e=3
    d.call_output_tokens = out
    pc = default_place_cfg()
    pc.update(kappa=1, theta_pm=100000)
    node, mig, steals, _ = O.Oracle(d, pc).placement()
    assert node[0] == 0 and node[1] == 1 and node[2] == 0
    assert steals >= 1
    e, s, v, t = (int(x) for x in mig[0])
    assert (s, v, t) == (2, 0, 1) and e == 4
    # S:321 anti-thrash: s2 is not stolen again (its only call completes at node 1 first)
    assert sum(1 for m in mig if int(m[1]) == 2) == 1
    # loads (0.6, 0.4) style: no idle thief -> no steal
    d2 = _two_call_trace(10 ** 8, n_nodes=2, extra_sessions=[(2, 1, 0), (3, 2, 0)])
    d2.call_output_tokens = np.full(d2.n_calls, 300, np.uint32)
    _, _, steals2, _ = O.Oracle(d2, pc).placement()
    assert steals2 == 0


def test_placement_conservation_and_determinism(O):
    d = make("C2", n_sessions=40, n_nodes=4)
    pc = default_place_cfg(9)
    pc.update(kappa=2)
    a = O.Oracle(d, pc).placement()
    b = O.Oracle(d, pc).placement()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2:] == b[2:]
    assert a[0].size == d.n_calls and a[0].max() < d.n_nodes


def test_invalid_traces_rejected(O):
    d = make_c1()
    d.call_t_us = d.call_t_us.copy()
    d.call_t_us[5], d.call_t_us[6] = d.call_t_us[6], d.call_t_us[5]
    with pytest.raises(ValueError):
        O.Oracle(d, default_place_cfg())
    d = make_c1()
    d.edge_p = d.edge_p.copy()
    d.edge_p[0] = 1.5
    with pytest.raises(ValueError):
        O.Oracle(d, default_place_cfg())
    d = make_c1()
    d.range_block_lo = d.range_block_lo.copy()
    d.range_block_lo[1] = 40  # session 0 touching session 3's blocks
    with pytest.raises(ValueError):
        O.Oracle(d, default_place_cfg())


def test_victim_log_with_epochs(O):
    """replay_log = replay(log=True) plus the epoch of each victim: same victims in the same order,
    epochs non-decreasing, one entry per eviction."""
    for seed in range(4):
        d = make_random_small(seed, n_sessions=6, n_nodes=2, max_calls=5, max_blocks=8)
        o = O.Oracle(d, default_place_cfg(seed))
        for w in range(d.n_nodes):
            lo, hi = o.sweep_range(w)
            for C in range(max(lo, 1), hi + 2):
                for pol in (O.POL_AEG, O.POL_BELADY, O.POL_LRU):
                    c1, lids = o.replay(pol, w, C, log=True)
                    c2, log = o.replay_log(pol, w, C)
                    assert np.array_equal(c1, c2)
                    assert [int(x) & 0xFFFFFFFF for x in log] == [int(x) for x in lids]
                    ep = [int(x) >> 32 for x in log]
                    assert ep == sorted(ep)
                    assert len(log) == c1[O.CI["EVICTIONS"]]
