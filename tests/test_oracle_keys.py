"""Pins of the oracle's WA-LRU key path through the functions replay() really calls.

The scalar pins in test_oracle.py check score() / reuse() / prot() on SPEC's worked examples.
These pins check what those scalars are fed inside a replay: which candidates the normalisers
range over (R-norm), which call is the session's current one (c*), which
context length n_cur and AEG node the reuse term reads, and the TTL's elapsed-time origin
(R-el).  Every expected victim below is derived by hand in the test's comment from eq:eviction
 with alpha, beta, gamma = 0.3, 0.5, 0.2, and each trace is built so that one
plausible mistake flips the victim (scripts/mutate_oracle.py runs those mutations).
"""
import json
import os

import numpy as np
import pytest

from gen import default_place_cfg, make_hand_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")
E = 100_000  # epoch (us)


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def _call(t, s, v, blocks, prompt=15, out=1, **kw):
    return dict(t=t, s=s, v=v, prompt=prompt, out=out, blocks=blocks, **kw)


def victims(o, O, pol, cap):
    _, log = o.replay_log(pol, 0, cap)
    return [(int(x) >> 32, int(x) & 0xFFFFFFFF) for x in log]


# ------------------------------------------------------------------------------------------
# "entry A (older, P_reuse=1) vs B (newer, P_reuse=0) -> Lru evicts A, WaLru evicts B"
# ------------------------------------------------------------------------------------------
def spec_s213_trace():
    # node 0: P_reuse = 1 (one edge p = 1, whole context shared, no observation: overlap 1);
    # node 1: no successor (P_reuse = 0, not terminal); node 2: the newcomer.  TTL base 0: nothing
    # is protected (el > 0 for every candidate at T_3).
    nodes = [dict(ttl=0, edges=[(2, 1.0)]), dict(ttl=0), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 1)]),            # A at e = 1, block 0 (lid 0)
             _call(E + 1, 1, 1, [(1, 1)]),        # B at e = 2, block 1 (lid 1)
             _call(2 * E + 1, 2, 2, [(2, 1)])]    # C at e = 3 needs one slot at capacity 2
    return make_hand_trace(calls, nodes)


def test_spec_s213_lru_evicts_older_walru_evicts_unreused(O):
    # At T_3 = 300 ms: cand = {A, B}, d_A = 299,999 = tau_max, d_B = 199,999; sizes 1 block each.
    # WA-LRU: A = 0.3*1 + 0.5*(1-1) + 0.2*1 = 0.5;  B = 0.3*0.667 + 0.5*(1-0) + 0.2 = 0.9 -> B.
    # LRU: A's latest access is older -> A.
    o = O.Oracle(spec_s213_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 2) == [(3, 1)]
    assert victims(o, O, O.POL_LRU, 2) == [(3, 0)]
    key, s32, _ = o.keys(O.POL_AEG, 0, 3, 2, 2, 0, [0, 1], [1, E + 1], [O.INF, O.INF])
    assert abs(float(s32[0]) - 0.5) < 1e-6 and abs(float(s32[1]) - (0.3 * 199_999 / 299_999 + 0.7)) < 1e-6
    assert key[0] >> 63 == 1 and key[1] >> 63 == 1   # neither is TTL-protected


# ------------------------------------------------------------------------------------------
# Fig. 2 through oracle_keys: the per-owner state comes from the session's newest
# call c* (two calls per session; the second one, e(c*) = 2, has n_cur = 12,000)
# ------------------------------------------------------------------------------------------
def fig2_trace():
    g = json.load(open(os.path.join(GOLD, "fig2_aeg.json")))
    edges = {v: [] for v in range(5)}
    for u, w, p in g["edges"]:
        edges[u].append((w, p))
    nodes = [dict(ttl=0, obs=g["obs"][v], term=int(v == 4), edges=edges[v]) for v in range(5)]
    calls = []
    for v in range(5):
        calls.append(_call(1 + v, v, v, [(2 * v, 1)], prompt=3000, out=500))             # e = 1, n_cur 3,500
        calls.append(_call(E + 1 + v, v, v, [(2 * v + 1, 1)], prompt=11000, out=1000))   # e = 2, n_cur 12,000
    return make_hand_trace(calls, nodes), g


def test_fig2_q_through_oracle_keys(O):
    # t_last = T_e for every candidate -> tau_max = 0 -> R = 0; all sizes 750 blocks -> S = 1.
    # q = floor((0.5 * (1 - P_reuse(v)) + 0.2) * 2^20) = the golden Fig. 2 values
    d, g = fig2_trace()
    o = O.Oracle(d, default_place_cfg())
    Te = 2 * E
    lids = np.arange(1, 10, 2, dtype=np.uint32)   # block 2v+1 of session v (local id = block id)
    key, _, _ = o.keys(O.POL_AEG, 0, 2, 10, 10, 0, lids, np.full(5, Te), np.full(5, O.INF))
    q = [(int(k) >> 32) & 0x7FFFFFFF for k in key]
    assert q == g["q_at_R0_S1"]
    # Alg. 1: every c* is still decoding at T_2 (1,000 tokens at 30 tok/s), so el < 0 and the
    # unfinished sessions v0..v3 are protected; v4 is terminal (fin): never protected
    assert [int(k) >> 63 for k in key] == [0, 0, 0, 0, 1]


# ------------------------------------------------------------------------------------------
# R-norm: tau_max and size_max range over cand = S \ A, never over in-flight blocks
# ------------------------------------------------------------------------------------------
def tau_window_trace():
    # A: P_reuse 0.8; B: 0.5; C: no successor.  Node 3 = sink.
    nodes = [dict(ttl=0, edges=[(3, 0.8)]), dict(ttl=0, edges=[(3, 0.5)]), dict(ttl=0), dict(ttl=0)]
    calls = [_call(1, 2, 2, [(2, 1)]),                      # C1, e = 1: block 2 (old)
             _call(90 * E + 1, 0, 0, [(0, 1)]),             # A1, e = 91: block 0
             _call(99 * E + 1, 1, 1, [(1, 1)]),             # B1, e = 100: block 1
             _call(100 * E + 1, 2, 2, [(2, 1), (3, 1)])]    # C2, e = 101: block 2 in flight + new 3
    return make_hand_trace(calls, nodes)


def test_tau_max_over_candidates_only(O):
    # T_101 = 10.1 s, capacity 3: S = {0, 1, 2}, A = {2, 3}, k = 1, cand = {0, 1}.
    # d_A = 1,099,999 = tau_max (cand), d_B = 199,999; sizes 1.
    #   A = 0.3 + 0.5*0.2 + 0.2 = 0.6;  B = 0.3*0.182 + 0.25 + 0.2 = 0.505  -> evict A (lid 0).
    # tau_max over S would take the in-flight C (d = 10,099,999): A = 0.333 < B = 0.456 -> B.
    o = O.Oracle(tau_window_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 3) == [(101, 0)]


def size_window_trace():
    nodes = [dict(ttl=0, edges=[(3, 0.6)]), dict(ttl=0, edges=[(3, 0.5)]), dict(ttl=0), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 1)], prompt=15, out=1),                # A, e = 1: n_cur 16 -> 1 block
             _call(5 * E + 50_000, 1, 1, [(1, 1)], prompt=63, out=1),   # B, e = 6: n_cur 64 -> 4 blocks
             _call(9 * E + 50_001, 2, 2, [(2, 1)], prompt=6399, out=1),  # C1, e = 10: n_cur 6,400 -> 400
             _call(10 * E + 1, 2, 2, [(2, 1), (3, 1)], prompt=6399, out=1)]  # C2, e = 11: 2 in flight
    return make_hand_trace(calls, nodes)


def test_size_max_over_candidates_only(O):
    # T_11 = 1.1 s, capacity 3, cand = {A, B}: d_A = 1,099,999 = tau_max, d_B = 550,000 (R 0.5).
    # size_max over cand = 4:  A = 0.3 + 0.5*0.4 + 0.2*0.25 = 0.55;  B = 0.15 + 0.25 + 0.2 = 0.6 -> B.
    # size_max over S (in-flight C, 400 blocks): A = 0.5005 > B = 0.402 -> A.  (C's d = 149,999 < d_A.)
    o = O.Oracle(size_window_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 3) == [(11, 1)]


# ------------------------------------------------------------------------------------------
# c* = newest call with e(c*) <= e: a call admitted exactly at this boundary is the current one
# ------------------------------------------------------------------------------------------
def cstar_trace():
    # node 0: P = 1; node 1: B's node, P = 0.6; node 2: A's final step (is_last -> fin -> P = 0)
    nodes = [dict(ttl=0, edges=[(3, 1.0)]), dict(ttl=0, edges=[(3, 0.6)]), dict(ttl=0), dict(ttl=0)]
    calls = [_call(1, 1, 1, [(2, 1)]),                     # B1, e = 1: block 2 (lid 2), oldest
             _call(2, 0, 0, [(0, 1)]),                     # A1, e = 1: block 0 (lid 0)
             _call(5 * E + 1, 0, 2, [(1, 1)], last=1)]     # A2, e = 6: new block 1, A finishes
    return make_hand_trace(calls, nodes)


def test_cstar_includes_call_admitted_at_e(O):
    # T_6, capacity 2: S = {0, 2}, A2 brings block 1 -> k = 1, cand = {0, 2}; sizes 1.
    # c*(A) = A2 (e = 6 <= 6): fin -> P = 0: A = 0.3*0.99999 + 0.5 + 0.2 = 0.99999; B = 0.3 + 0.2 + 0.2 = 0.7
    #   -> evict A's block 0.   With c*(A) = A1 (e(c) < e): P = 1, A = 0.5 < 0.7 -> block 2.
    o = O.Oracle(cstar_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 2) == [(6, 0)]


# ------------------------------------------------------------------------------------------
# R-el: the TTL's elapsed time runs from the tool start t_end(c*) (Alg. 1: TTL set when the tool
# call begins), not from the call's arrival t_c
# ------------------------------------------------------------------------------------------
def ttl_origin_trace():
    nodes = [dict(ttl=2_000_000), dict(ttl=0, edges=[(3, 0.5)]), dict(ttl=0), dict(ttl=0)]
    calls = [_call(50_001, 0, 0, [(0, 1)], prompt=15, out=300),   # A, e = 1: decodes 10 s, tool starts at 10.053 s
             _call(85 * E + 1, 1, 1, [(1, 1)]),                  # B, e = 86
             _call(90 * E + 1, 2, 2, [(2, 1)])]                  # C, e = 91 needs a slot at capacity 2
    return make_hand_trace(calls, nodes)


def test_ttl_elapsed_from_tool_start(O):
    # T_91 = 9.1 s: el_A = 9.1 s - 10.053 s < 0 -> A protected (key bit 63 = 0); B (TTL 0) is not.
    # Unprotected first -> evict B (lid 1), EVICT_PROTECTED = 0.  From t_c, el_A = 9.05 s > 2 s:
    # A unprotected, and A = 0.3 + 0.5 + 0.2 = 1.0 > B = 0.3*0.066 + 0.25 + 0.2 -> A.
    o = O.Oracle(ttl_origin_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 2) == [(91, 1)]
    ctr = o.replay(O.POL_AEG, 0, 2)
    assert ctr[O.CI["EVICT_PROTECTED"]] == 0


def test_hard_pressure_evicts_protected_last(O):
    # same trace at a capacity where both A and B must go: the unprotected B first, then A under
    # hard pressure ("skipped unless no alternative"); one protected victim counted.
    # C touches two new blocks (2, 3): k = 2 at capacity 2
    d2 = make_hand_trace([_call(50_001, 0, 0, [(0, 1)], prompt=15, out=300), _call(85 * E + 1, 1, 1, [(1, 1)]),
                          _call(90 * E + 1, 2, 2, [(2, 2)])],
                         [dict(ttl=2_000_000), dict(ttl=0, edges=[(3, 0.5)]), dict(ttl=0), dict(ttl=0)])
    o = O.Oracle(d2, default_place_cfg())
    assert victims(o, O, O.POL_AEG, 2) == [(91, 1), (91, 0)]   # descending key order
    assert o.replay(O.POL_AEG, 0, 2)[O.CI["EVICT_PROTECTED"]] == 1


HAND_TRACES = {"s213": spec_s213_trace, "tau": tau_window_trace, "size": size_window_trace,
               "cstar": cstar_trace, "ttl": ttl_origin_trace}


# ------------------------------------------------------------------------------------------
# eq:pressure's occupancy is |S| after R1 (before this epoch's admissions), SURVEY §8.C.6
# ------------------------------------------------------------------------------------------
def pressure_trace():
    # A (TTL base 1 s, no successor), B (7 blocks, P 0.5, TTL 0), C brings 3 new blocks at e = 7
    nodes = [dict(ttl=1_000_000), dict(ttl=0, edges=[(3, 0.5)]), dict(ttl=0), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 1)]),                              # A, e = 1: t_end = 36,335
             _call(5 * E + 1, 1, 1, [(1, 7)], prompt=111, out=1),   # B, e = 6: 7 blocks, n_cur 112
             _call(6 * E + 1, 2, 2, [(8, 3)])]                     # C, e = 7: 3 new blocks
    return make_hand_trace(calls, nodes)


def test_pressure_uses_occupancy_before_admission(O):
    # T_7 = 0.7 s, capacity 10: |S| = 8, new = 3 -> k = 1, cand = {A's block 0, B's blocks 1..7}.
    # m = (8/10 - 0.7) / 0.2 = 0.5 -> A's TTL = 1 s * (1 - 0.25) = 0.75 s > el_A = 0.663665 s:
    # A protected; B unprotected -> the victim is B's largest local id, 7.
    # (With |S| + new = 11: m = 1, TTL 0.5 s < el_A: A unprotected and A = 0.3 + 0.5 + 0.2/7 >
    #  B = 0.086 + 0.25 + 0.2 -> A's block 0.)
    o = O.Oracle(pressure_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 10) == [(7, 7)]


# ------------------------------------------------------------------------------------------
# Shared-prefix pseudo-session (DESIGN.md R-shared): P_reuse = act(w, a), act = an unfinished
# session of type a has affinity w
# ------------------------------------------------------------------------------------------
def shared_trace():
    # type 0: shared prefix block 0; A (type 0) finishes at its second call; B is type 1
    nodes = [dict(ttl=0, edges=[(2, 1.0)]), dict(ttl=0, edges=[(2, 0.5)]), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 1), (1, 1)]),                           # A1, e = 1: prefix + block 1
             _call(150_000, 0, 0, [(1, 2)], prompt=31, out=1, last=1),   # A2, e = 2: blocks 1, 2; A done
             _call(2 * E + 1, 1, 1, [(3, 1)])]                          # B1, e = 3: new block 3
    return make_hand_trace(calls, nodes, shared=[(0, 1), (4, 0)], session_types=[0, 1])


def test_shared_prefix_inactive_is_not_reused(O):
    # T_3 = 0.3 s, capacity 3: S = {0, 1, 2}, k = 1.  act(0, type 0) = 0 (A finished).
    # prefix (size 1 of size_max 2): R = 1, P = act = 0 -> 0.3 + 0.5 + 0.1 = 0.9;
    # A's blocks (fin: P = 0, size 2): R = 150,000 / 299,999 -> 0.15 + 0.5 + 0.2 = 0.85  -> block 0.
    # (With P = 1 for the prefix: 0.4 -> A's block 2, the larger local id of the two ties.)
    o = O.Oracle(shared_trace(), default_place_cfg())
    assert victims(o, O, O.POL_AEG, 3) == [(3, 0)]
