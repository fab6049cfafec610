"""Hand-derived pins of placement A2 (eq:routing P:735-743, work stealing P:748-766; SURVEY
§8.C.2 rules P1-P3 and DESIGN.md readings R-load, R-cached, R-argmin, R-steal).

Every expected node / migration is worked out by hand in the test comment, boundary by boundary:
E = 100 ms epochs, a call admitted at e(c) = floor(t/E) + 1, work
omega = ceil(pf*1e6/5000) + ceil(out*1e6/30) us (pf = new tokens when routed to its cached
affinity, else the prompt), load(w) = sum over the queue of min(rem, E), kappa servers per node.
"""
import pytest

from gen import default_place_cfg, make_hand_trace

E = 100_000


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def _call(t, s, v, blocks, prompt=15, out=1, **kw):
    return dict(t=t, s=s, v=v, prompt=prompt, out=out, blocks=blocks, **kw)


def test_argmin_tie_lowest_id_despite_active_sessions(O):
    # S:306 "ties -> lowest worker_id".  e=1: s0 -> node 0 (loads 0, 0), omega = 3,000 + 33,334 <
    # E, so it completes at boundary 2; s0 stays an unfinished session with affinity 0.
    # e=3: s1 (new) sees loads (0, 0) -> node 0, although node 0 has one active session and
    # node 1 none (the round-1 tie-break on active sessions would have picked node 1).
    d = make_hand_trace([_call(1, 0, 0, [(0, 1)]), _call(2 * E + 1, 1, 0, [(1, 1)])],
                        [dict(ttl=10 ** 8)], n_nodes=2)
    node, mig, steals, rr = O.Oracle(d, default_place_cfg()).placement()
    assert list(node) == [0, 0] and steals == 0 and rr == 0


def _ttl_trace(ttl):
    # s0 (node v0, TTL base `ttl`): c1 at t=1, omega 36,334, tool start t_end = 1 + 3,000 + 33,334
    # = 36,335.  s3 at t=2 -> node 1 (load(0) = 36,334 > 0), omega 3,000 + 233,334 = 236,334.
    # e=2: node 0 is empty, node 1 holds s3 (rem 136,334 -> load E): s1 (100 s decode) -> node 0.
    # s3 completes at boundary 4.  e=11 (T = 1.1 s): s0's c2 finds load(0) = E < 0.8*32*E and
    # load(1) = 0; el = 1,100,000 - 36,335 = 1,063,665.
    nodes = [dict(ttl=ttl), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 1)]), _call(2, 3, 1, [(3, 1)], out=7),
             _call(E + 1, 1, 1, [(1, 1)], out=3000), _call(10 * E + 5, 0, 0, [(0, 1)])]
    return make_hand_trace(calls, nodes, n_nodes=2)


@pytest.mark.parametrize("ttl,node,rr", [(1_063_665, 0, 0), (1_063_664, 1, 1), (10 ** 9, 0, 0), (0, 1, 1)])
def test_cached_ttl_boundary(O, ttl, node, rr):
    # cached(w*, s) = T_e - t_end(last) <= ttl_base(last) (Alg. 1 with m = 0, DESIGN.md R-cached):
    # at el == ttl the session is still cached -> its affinity node 0 (load under theta); one
    # microsecond less of TTL -> not cached -> argmin load -> node 1, counted as a reroute.
    o = O.Oracle(_ttl_trace(ttl), default_place_cfg())
    n, _, _, r = o.placement()
    assert list(n[:3]) == [0, 1, 0]
    assert int(n[3]) == node and r == rr


def test_terminal_last_node_is_not_cached(O):
    # same timeline with ttl = 1e9 but s0's first call at a terminal AEG node: not cached -> argmin
    d = _ttl_trace(10 ** 9)
    d.node_terminal = d.node_terminal.copy()
    d.node_terminal[0] = 1
    n, _, _, r = O.Oracle(d, default_place_cfg()).placement()
    assert int(n[3]) == 1 and r == 1


def _steal_trace():
    # kappa = 1, theta = 100,000 permille (a cached session always goes to its affinity).
    # e=1: P1 (s2) -> node 0 (tie).  e=2: P1 done; Q1 (s3) -> node 0 (tie).  e=3: Q1 done;
    # L (s0, 100 s) -> node 0 (tie); I (s1, omega 236,334) -> node 1 (load(0) = E).
    # e=4: P2 (s2) and Q2 (s3) are cached at node 0 -> queue 0 = [L (serving), P2, Q2].
    # Node 1 serves I at boundaries 4 (E), 5 (E) and 6 (the last 36,334 us).  e=7: node 1 served
    # nothing -> idle for T_idle; node 0's load > 2 * min load = 0 -> steal the OLDEST pending
    # session there: s2 (P2) -> migration (7, s2, 0 -> 1).  e=8: node 1 serves P2 (done, s2 no
    # longer `moved`).  e=9: node 1 idle again -> steals s3 (Q2): (9, s3, 0 -> 1).  Later node 0
    # holds only L (in service): no steal.
    nodes = [dict(ttl=10 ** 7)]
    calls = [_call(1, 2, 0, [(2, 1)]), _call(E + 1, 3, 0, [(3, 1)]),
             _call(2 * E + 1, 0, 0, [(0, 1)], out=3000), _call(2 * E + 2, 1, 0, [(1, 1)], out=7),
             _call(3 * E + 1, 2, 0, [(2, 1)]), _call(3 * E + 2, 3, 0, [(3, 1)])]
    return make_hand_trace(calls, nodes, n_nodes=2)


def test_steal_oldest_pending_session_then_next(O):
    pc = default_place_cfg()
    pc.update(kappa=1, theta_pm=100_000)
    o = O.Oracle(_steal_trace(), pc)
    node, mig, steals, rr = o.placement()
    assert list(node) == [0, 0, 0, 1, 0, 0]
    assert [tuple(int(x) for x in m) for m in mig] == [(7, 2, 0, 1), (9, 3, 0, 1)]
    assert steals == 2 and rr == 0


def test_steal_needs_idle_thief_and_load_guard(O):
    # P:361 / P:766(a): the thief must have been idle for T_idle.  With T_idle = 10 epochs node 1
    # (idle from boundary 7 on) first qualifies at boundary 16 and steals s2; it serves P2 at 17,
    # is idle again from 18 and steals s3 at 27.
    pc = default_place_cfg()
    pc.update(kappa=1, theta_pm=100_000, t_idle_us=10 * E)
    node, mig, steals, rr = O.Oracle(_steal_trace(), pc).placement()
    assert [tuple(int(x) for x in m) for m in mig] == [(16, 2, 0, 1), (27, 3, 0, 1)]


def test_moved_session_not_stolen_back(O):
    # P:766(b) / S:335 anti-thrash: a session migrated to node 1 cannot be stolen again until one
    # of its calls completes at its new node.  Two idle-prone nodes, every steal recorded once.
    pc = default_place_cfg()
    pc.update(kappa=1, theta_pm=100_000)
    _, mig, _, _ = O.Oracle(_steal_trace(), pc).placement()
    sess = [int(m[1]) for m in mig]
    assert len(sess) == len(set(sess))


def test_reroute_reprefill_is_regeneration(O):
    # P:881 "tokens prefilled" / Observation 1: in _ttl_trace(0) s0's second call is rerouted to
    # node 1 (not cached) and re-prefills block 0 there.  Node 1's records: s3's block 3 (first
    # touch in the whole trace: compulsory) and s0's block 0 (touched before at node 0: a
    # regenerated block, 16 tokens = 3,200 us at 5,000 tok/s), at any capacity >= 1.
    o = O.Oracle(_ttl_trace(0), default_place_cfg())
    for pol in (O.POL_AEG, O.POL_BELADY):
        c = o.replay(pol, 1, 4)
        assert (c[O.CI["MISSES"]], c[O.CI["COMPULSORY_GLOBAL"]], c[O.CI["COMPULSORY_NODE"]]) == (2, 1, 2)
        assert (c[O.CI["REGEN_TOKENS"]], c[O.CI["REGEN_US"]]) == (16, 3200)
        c0 = o.replay(pol, 0, 4)   # node 0: s0's c1 and s1's call, both first touches
        assert (c0[O.CI["MISSES"]], c0[O.CI["COMPULSORY_GLOBAL"]], c0[O.CI["REGEN_TOKENS"]]) == (2, 2, 0)
