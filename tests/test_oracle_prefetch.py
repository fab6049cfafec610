"""Pins of F4's speculative prefetch records (§4.3; SPEC prefetch_target S:235-243;
DESIGN.md R-prefetch): the plan (which successor, which prefix, which epoch) and the replay of
PREFETCH records, each derived by hand; plus the invariants of §8.C.8 on streams with PREFETCH
records (they are ordinary accesses for paging: MIN and BELADY-epoch still bound every policy)."""
import numpy as np
import pytest

from gen import default_place_cfg, make, make_hand_trace, make_random_small
from tests.brute import brute_epoch_opt
from tests.test_oracle import _invariants, _node_epochs, hits, misses

E = 100_000


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def _call(t, s, v, blocks, prompt=15, out=1, **kw):
    return dict(t=t, s=s, v=v, prompt=prompt, out=out, blocks=blocks, **kw)


def _plan_trace(edges0, term0=0, last=0):
    # A1 at node 0 (n_cur = 63 + 30 = 93 tokens, 10 blocks, tool starts at 1 + 12,600 + 1,000,000
    # -> boundary 11); A2 back at t = 2 s (boundary 21).  Nodes 1, 2, 3 are successors.
    nodes = [dict(ttl=0, term=term0, edges=edges0), dict(ttl=0), dict(ttl=0), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 10)], prompt=63, out=30, last=last), _call(2 * 10 ** 6 + 1, 0, 1, [(0, 11)])]
    return make_hand_trace(calls, nodes)


@pytest.mark.parametrize("edges,want_len", [
    ([(2, 0.6, 65536), (3, 0.4, 32768)], 5),   # S:241 argmax p = 0.6 -> node 2: n_sh = 93 -> 5 blocks
    ([(2, 0.4, 65536), (3, 0.6, 32768)], 2),   # argmax -> node 3, half the context: n_sh = 46 -> 2 blocks
    ([(3, 0.5, 32768), (2, 0.5, 65536)], 5),   # S:243 tie 0.5 / 0.5 -> the lower node id (2)
])
def test_prefetch_target_and_prefix(O, edges, want_len):
    o = O.Oracle(_plan_trace(edges), default_place_cfg(), prefetch=True)
    e, n = o.prefetch_plan()
    assert (int(e[0]), int(n[0])) == (11, want_len)
    assert (int(e[1]), int(n[1])) == (0, 0)      # the last call of the session: nothing follows


def test_no_prefetch_at_terminal_or_last(O):
    for kw in (dict(term0=1), dict(last=1)):     # S:242 terminal -> None; a finished session
        o = O.Oracle(_plan_trace([(2, 1.0)], **kw), default_place_cfg(), prefetch=True)
        assert int(o.prefetch_plan()[0][0]) == 0


def test_no_prefetch_when_next_step_arrives_first(O):
    # A2 admitted at boundary 11, the prefetch boundary: the step itself brings its blocks
    d = _plan_trace([(2, 1.0)])
    d.call_t_us = d.call_t_us.copy()
    d.call_t_us[1] = 10 * E + 5
    o = O.Oracle(d, default_place_cfg(), prefetch=True)
    assert int(o.prefetch_plan()[0][0]) == 0


def _replay_trace():
    # A1 (e=1) blocks 0..3, n_cur 93 -> prefix 5 blocks, capped at A1's 4; tool start -> e_pf = 11.
    # B1 (e=5) blocks 10..13, B's only call.  A2 (e=21) blocks 0..4.
    nodes = [dict(ttl=0, edges=[(1, 1.0)]), dict(ttl=0)]
    calls = [_call(1, 0, 0, [(0, 4)], prompt=63, out=30), _call(4 * E + 1, 1, 1, [(10, 4)], last=1),
             _call(20 * E + 1, 0, 1, [(0, 5)], last=1)]
    return make_hand_trace(calls, nodes)


def test_prefetch_replay_evict_all_hand_counts(O):
    # EVICT_ALL at capacity 100 evicts every non-requested block each epoch:
    #   e=1  A1: 4 CALL misses (first touches).   e=5  B1: A's 4 evicted, 4 misses.
    #   e=11 PREFETCH 0..3: B's 4 evicted, 4 prefetch misses (loaded during A's tool call).
    #   e=21 A2: S = {0..3} inside A -> nothing evicted; 4 hits + block 4 missed (first touch).
    C = O.CI
    o = O.Oracle(_replay_trace(), default_place_cfg(), prefetch=True)
    c = o.replay(O.POL_EVICT_ALL, 0, 100)
    got = {k: int(c[C[k]]) for k in ("ACCESSES", "HITS", "MISSES", "PF_HITS", "PF_MISSES", "COMPULSORY_GLOBAL",
                                      "REGEN_TOKENS", "EVICTIONS")}
    assert got == dict(ACCESSES=17, HITS=4, MISSES=9, PF_HITS=0, PF_MISSES=4, COMPULSORY_GLOBAL=9, REGEN_TOKENS=0,
                       EVICTIONS=8)
    # without the PREFETCH records A2 re-prefills its 4 blocks: 64 regenerated tokens
    c0 = O.Oracle(_replay_trace(), default_place_cfg()).replay(O.POL_EVICT_ALL, 0, 100)
    assert (int(c0[C["MISSES"]]), int(c0[C["REGEN_TOKENS"]]), int(c0[C["PF_MISSES"]])) == (13, 64, 0)


def test_prefetch_stream_order(O):
    # node 0's stream: A1 (0..3) | B1 (10..13) | PREFETCH (0..3) at e=11 | A2 (0..4)
    o = O.Oracle(_replay_trace(), default_place_cfg(), prefetch=True)
    s = o.stream(0)
    assert list(s["block"]) == [0, 1, 2, 3, 10, 11, 12, 13, 0, 1, 2, 3, 0, 1, 2, 3, 4]
    assert [(int(e), int(k)) for e, k in zip(s["events"][:, 0], s["groups"][:, 2])] == [(1, 0), (5, 0), (11, 2), (21, 0)]


@pytest.mark.parametrize("seed", range(8))
def test_prefetch_invariants_random(O, seed):
    d = make_random_small(seed, n_sessions=8, n_nodes=2, max_calls=5, max_blocks=8)
    pc = default_place_cfg(seed)
    o = O.Oracle(d, pc, prefetch=True)
    _invariants(o, d, O)


def test_prefetch_belady_epoch_bruteforce(O):
    n_pf = 0
    for seed in range(30):
        d = make_random_small(seed, n_sessions=4, n_nodes=1, max_calls=3, max_blocks=4)
        o = O.Oracle(d, default_place_cfg(seed), prefetch=True)
        n_pf += int((o.prefetch_plan()[0] > 0).sum())
        if o.n_local(0) > 9:
            continue
        eps, own = _node_epochs(o, 0)
        for C in range(1, 6):
            ref = brute_epoch_opt(eps, own, C)
            ctr = o.replay(O.POL_BELADY, 0, C)
            if ref is None:
                assert ctr[O.CI["INFEASIBLE_EPOCH"]] > 0
            else:
                assert misses(ctr, O) == ref, (seed, C)
    assert n_pf > 0


def test_prefetch_c2_small_counts(O):
    d = make("C2", n_sessions=20, n_nodes=2)
    o = O.Oracle(d, default_place_cfg(2), prefetch=True)
    e, n = o.prefetch_plan()
    assert (e > 0).sum() > 0
    _invariants(o, d, O)
