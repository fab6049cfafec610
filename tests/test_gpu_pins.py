"""The hand-derived pins of tests/test_oracle_keys.py and tests/test_oracle_place.py, asserted on
the GPU path through the C ABI (so both arms are held to the same hand-worked expectations, not
only to each other), plus oracle == GPU on the full counter set of those traces."""
import numpy as np
import pytest

from gen import default_place_cfg
from tests import test_oracle_keys as K
from tests import test_oracle_place as PL
from tests import test_oracle_prefetch as PF

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_00528_b200 import saga  # noqa: E402
from oracle import oracle as O  # noqa: E402

O.build()

# (trace builder, policy, capacity, expected victims [(epoch, local id)] in descending key order)
KEY_PINS = [
    ("s213_aeg", K.spec_s213_trace, saga.POLICY_AEG, 2, [(3, 1)]),
    ("s213_lru", K.spec_s213_trace, saga.POLICY_LRU, 2, [(3, 0)]),
    ("tau_window", K.tau_window_trace, saga.POLICY_AEG, 3, [(101, 0)]),
    ("size_window", K.size_window_trace, saga.POLICY_AEG, 3, [(11, 1)]),
    ("cstar", K.cstar_trace, saga.POLICY_AEG, 2, [(6, 0)]),
    ("ttl_origin", K.ttl_origin_trace, saga.POLICY_AEG, 2, [(91, 1)]),
    ("pressure", K.pressure_trace, saga.POLICY_AEG, 10, [(7, 7)]),
    ("shared", K.shared_trace, saga.POLICY_AEG, 3, [(3, 0)]),
]


@pytest.mark.parametrize("name,build,pol,cap,want", KEY_PINS, ids=[p[0] for p in KEY_PINS])
def test_key_pins_on_gpu(name, build, pol, cap, want):
    d = build()
    t = saga.Trace(d, default_place_cfg())
    t.next_use(0)
    ctr, log = t.replay_victims(dict(policy_mask=pol), cap, 0)
    got = sorted((int(x) >> 32, int(x) & 0xFFFFFFFF) for x in log)
    assert got == sorted(want), name
    o = O.Oracle(d, default_place_cfg())
    rc, _ = o.replay_log(pol, 0, cap)
    assert np.array_equal(ctr, rc), name


def test_fig2_keys_on_gpu():
    d, g = K.fig2_trace()
    t = saga.Trace(d, default_place_cfg())
    t.next_use(0)
    dev = "cuda"
    Te = 2 * K.E
    i32 = lambda a: torch.from_numpy(np.asarray(a, np.uint32).view(np.int32).copy()).to(dev)
    batch = dict(seg_node=i32([0]), seg_epoch=i32([2]), seg_occ=i32([10]), seg_cap=i32([10]), seg_act=i32([0]),
                 seg_off=torch.tensor([0, 5], dtype=torch.int64, device=dev),
                 cand_lid=i32(np.arange(1, 10, 2)), cand_t_last=torch.full((5,), Te, dtype=torch.int64, device=dev),
                 cand_nu=i32(np.full(5, 0xFFFFFFFF)))
    key = torch.empty(5, dtype=torch.int64, device=dev)
    t.aeg_score(batch, {}, key, None, policy=saga.POLICY_AEG)
    torch.cuda.synchronize()
    k = key.cpu().numpy().view(np.uint64)
    assert [(int(x) >> 32) & 0x7FFFFFFF for x in k] == g["q_at_R0_S1"]
    assert [int(x) >> 63 for x in k] == [0, 0, 0, 0, 1]


def test_hard_pressure_on_gpu():
    d = K.make_hand_trace([K._call(50_001, 0, 0, [(0, 1)], prompt=15, out=300), K._call(85 * K.E + 1, 1, 1, [(1, 1)]),
                           K._call(90 * K.E + 1, 2, 2, [(2, 2)])],
                          [dict(ttl=2_000_000), dict(ttl=0, edges=[(3, 0.5)]), dict(ttl=0), dict(ttl=0)])
    t = saga.Trace(d, default_place_cfg())
    t.next_use(0)
    ctr, log = t.replay_victims(dict(policy_mask=saga.POLICY_AEG), 2, 0)
    assert sorted(int(x) for x in log) == [(91 << 32) | 0, (91 << 32) | 1]
    assert ctr[saga.CI["EVICT_PROTECTED"]] == 1


def test_argmin_tie_on_gpu():
    d = PL.make_hand_trace([PL._call(1, 0, 0, [(0, 1)]), PL._call(2 * PL.E + 1, 1, 0, [(1, 1)])],
                           [dict(ttl=10 ** 8)], n_nodes=2)
    node, mig, steals, rr = saga.Trace(d, default_place_cfg()).placement()
    assert list(node) == [0, 0] and steals == 0 and rr == 0


@pytest.mark.parametrize("ttl,node,rr", [(1_063_665, 0, 0), (1_063_664, 1, 1)])
def test_cached_ttl_boundary_on_gpu(ttl, node, rr):
    n, _, _, r = saga.Trace(PL._ttl_trace(ttl), default_place_cfg()).placement()
    assert list(n[:3]) == [0, 1, 0] and int(n[3]) == node and r == rr


@pytest.mark.parametrize("t_idle,want", [(PL.E, [(7, 2, 0, 1), (9, 3, 0, 1)]),
                                         (10 * PL.E, [(16, 2, 0, 1), (27, 3, 0, 1)])])
def test_steal_oldest_pending_on_gpu(t_idle, want):
    pc = default_place_cfg()
    pc.update(kappa=1, theta_pm=100_000, t_idle_us=t_idle)
    node, mig, steals, rr = saga.Trace(PL._steal_trace(), pc).placement()
    assert [tuple(int(x) for x in m) for m in mig] == want
    assert list(node) == [0, 0, 0, 1, 0, 0] and steals == 2 and rr == 0


def test_reroute_reprefill_is_regeneration_on_gpu():
    t = saga.Trace(PL._ttl_trace(0), default_place_cfg())
    for w in range(2):
        t.next_use(w)
    got = torch.zeros((2, 1, 2, saga.NCOUNT), dtype=torch.int64, device="cuda")
    t.replay(dict(policy_mask=3), [4], [0, 1], got)
    torch.cuda.synchronize()
    g = got.cpu().numpy()
    CI = saga.CI
    for pi in range(2):
        n1, n0 = g[pi, 0, 1], g[pi, 0, 0]
        assert (n1[CI["MISSES"]], n1[CI["COMPULSORY_GLOBAL"]], n1[CI["COMPULSORY_NODE"]]) == (2, 1, 2)
        assert (n1[CI["REGEN_TOKENS"]], n1[CI["REGEN_US"]]) == (16, 3200)
        assert (n0[CI["MISSES"]], n0[CI["COMPULSORY_GLOBAL"]], n0[CI["REGEN_TOKENS"]]) == (2, 2, 0)


def test_prefetch_hand_counts_on_gpu():
    """tests/test_oracle_prefetch.py::test_prefetch_replay_evict_all_hand_counts on the GPU path."""
    CI = saga.CI
    for pf, want in ((True, dict(ACCESSES=17, HITS=4, MISSES=9, PF_HITS=0, PF_MISSES=4, COMPULSORY_GLOBAL=9,
                                 REGEN_TOKENS=0, EVICTIONS=8)),
                     (False, dict(MISSES=13, REGEN_TOKENS=64, PF_MISSES=0))):
        t = saga.Trace(PF._replay_trace(), default_place_cfg(), prefetch=pf)
        t.next_use(0)
        got = torch.zeros((1, 1, 1, saga.NCOUNT), dtype=torch.int64, device="cuda")
        t.replay(dict(policy_mask=saga.POLICY_EVICT_ALL), [100], [0], got)
        torch.cuda.synchronize()
        g = got.cpu().numpy()[0, 0, 0]
        assert {k: int(g[CI[k]]) for k in want} == want, pf
    s = saga.Trace(PF._replay_trace(), default_place_cfg(), prefetch=True).node_stream(0)
    assert list(s["block"]) == [0, 1, 2, 3, 10, 11, 12, 13, 0, 1, 2, 3, 0, 1, 2, 3, 4]
    assert [int(k) for k in s["groups"][:, 1]] == [0, 0, 2, 0]
