"""GPU (sm_100a) path == CPU oracle, element by element, through the C ABI.

Bit-exact: placement, node streams, next_use / local_id, W_lo / W_hi, every replay counter
(incl. the victim-set hash), AEG / BELADY keys, selected victims.  Tolerance: the fp32 AEG
score against the oracle's fp64 evaluation of eq:eviction, |g - r| <= 1e-5 |r| + 1e-6
(north_star); the fp32 score itself is compared bit-exactly with the oracle's fp32 evaluation in
the same pinned order.
"""
import numpy as np
import pytest

from gen import (default_place_cfg, make, make_c1, make_chain_limit, make_obs1, make_random_small, place_cfg_for,
                 sweep_caps, N_SWEEP, PHYSICAL_CAP)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_00528_b200 import saga  # noqa: E402  (fails loudly if libsaga.so is missing)
from oracle import oracle as O  # noqa: E402

O.build()


def small_cases():
    cases = [("C1", make_c1(), default_place_cfg(0)), ("C1_limit", make_c1(limit_case=True), default_place_cfg(0))]
    for seed in range(6):
        d = make_random_small(seed, n_sessions=8, n_nodes=3, max_calls=5, max_blocks=8)
        pc = default_place_cfg(seed)
        if seed % 2:
            pc.update(kappa=1, theta_pm=100000)  # queues + stealing
        cases.append((f"rand{seed}", d, pc))
    for name, ns, nn in (("C2", 40, 4), ("C3", 80, 4), ("C4", 120, 4)):
        d = make(name, n_sessions=ns, n_nodes=nn)
        cases.append((d.name, d, place_cfg_for(d)))
    d = make("C4", n_sessions=150, n_nodes=4)
    pc = place_cfg_for(d)
    pc.update(kappa=2)
    cases.append(("C4_hot", d, pc))
    cases.append(("obs1", make_obs1(6, 3), default_place_cfg(0)))
    cases.append(("limit3", make_chain_limit(3), default_place_cfg(3)))
    # C5's shape: 32 nodes (every lane of the placement warp owns a node, owned mask 0xFFFFFFFF),
    # 10 tenants with their own shared prefixes; and a hot variant with queues, steals, reroutes
    d = make("C5", n_sessions=300, n_nodes=32)
    cases.append(("C5_32n", d, place_cfg_for(d)))
    d = make("C5", n_sessions=160, n_nodes=32)
    pc = place_cfg_for(d)
    pc.update(kappa=2)
    cases.append(("C5_32n_hot", d, pc))
    # F4 speculative prefetch records (SAGA_LOAD_PREFETCH) on top of queues, steals and reroutes
    for name, seed in (("rand1", 1), ("rand4", 4)):
        d = make_random_small(seed, n_sessions=8, n_nodes=3, max_calls=5, max_blocks=8)
        pc = default_place_cfg(seed)
        if seed % 2:
            pc.update(kappa=1, theta_pm=100000)
        cases.append((name + "_pf", d, pc, True))
    d = make("C2", n_sessions=40, n_nodes=4)
    cases.append(("C2_pf", d, place_cfg_for(d), True))
    d = make("C5", n_sessions=160, n_nodes=32)
    pc = place_cfg_for(d)
    pc.update(kappa=2)
    cases.append(("C5_32n_hot_pf", d, pc, True))
    return cases


CASES = small_cases()
IDS = [c[0] for c in CASES]


@pytest.fixture(scope="module", params=range(len(CASES)), ids=IDS)
def pair(request):
    name, d, pc = CASES[request.param][:3]
    pf = len(CASES[request.param]) > 3 and CASES[request.param][3]
    o = O.Oracle(d, pc, prefetch=pf)
    t = saga.Trace(d, pc, prefetch=pf)
    t.next_use_nodes(list(range(d.n_nodes)))
    return name, d, pc, o, t


def test_placement_equal(pair):
    name, d, pc, o, t = pair
    on, om, osteal, oreroute = o.placement()
    gn, gm, gsteal, greroute = t.placement()
    assert np.array_equal(on, gn), name
    assert np.array_equal(om, gm), name
    assert (osteal, oreroute) == (gsteal, greroute), name


def test_streams_equal(pair):
    name, d, pc, o, t = pair
    for w in range(d.n_nodes):
        so = o.stream(w)
        sg = t.node_stream(w)
        assert np.array_equal(so["block"], sg["block"]), (name, w)
        rec = so["events"][so["events"][:, 1] > 0]
        assert np.array_equal(rec[:, 0], sg["events"][:-1, 0]), (name, w)
        assert np.array_equal(rec[:, 1], sg["events"][:-1, 2]), (name, w)
        assert sg["events"][-1, 0] == 0xFFFFFFFF and sg["events"][-1, 2] == 0
        assert np.array_equal(so["groups"][:, 0], sg["groups"][:, 0]), (name, w)
        assert np.array_equal(so["groups"][:, 2], sg["groups"][:, 1]), (name, w)
        assert np.array_equal(so["groups"][:, 3], sg["group_t"]), (name, w)
        assert sorted(so["inv"].tolist()) == sorted(sg["inv"].tolist()), (name, w)


def test_next_use_equal(pair):
    name, d, pc, o, t = pair
    for w in range(d.n_nodes):
        n, _ = t.info(w)
        nu = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        lid = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        t.next_use(w, nu, lid)
        torch.cuda.synchronize()
        ref = o.next_use(w)
        assert np.array_equal(nu.cpu().numpy().view(np.uint32)[:n], ref["next_use"]), (name, w)
        assert np.array_equal(lid.cpu().numpy().view(np.uint32)[:n], ref["local_id"]), (name, w)
        assert t.info(w)[1] == o.n_local(w)
        assert t.sweep_range(w) == o.sweep_range(w), (name, w)


def _max_group(o, d):
    # the largest block set one call (or migration / prefetch group) brings to a node: below it a
    # capacity is SAGA_ERR_CAPACITY, from it up to W_lo - 1 it is infeasible-epoch data
    return max([int(o.stream(w)["groups"][:, 1].max()) for w in range(d.n_nodes) if o.stream(w)["groups"].size] or [1])


def _caps_for(o, d, name):
    wlo = max(o.sweep_range(w)[0] for w in range(d.n_nodes))
    whi = max(o.sweep_range(w)[1] for w in range(d.n_nodes))
    caps = sweep_caps(wlo, whi, 5)
    caps += [max(_max_group(o, d), wlo - 1, 1), whi + 7]
    return sorted(set(c for c in caps if c > 0))


@pytest.mark.parametrize("variant", ["narrow", "wide"])
def test_replay_counters_equal(pair, variant, monkeypatch):
    """Both compiled shapes of the replay kernel (512 threads x 1 CTA/SM, 256 x 2; run_replay
    picks by item count, SAGA_REPLAY_WIDE forces one) against the oracle."""
    monkeypatch.setenv("SAGA_REPLAY_WIDE", "1" if variant == "wide" else "0")
    name, d, pc, o, t = pair
    caps = _caps_for(o, d, name)
    # AEG, BELADY, EVICT_ALL and the tab:competitive baselines LRU, LRU + Prefix
    ref = o.replay_many(31, caps)
    got = torch.zeros((5, len(caps), d.n_nodes, saga.NCOUNT), dtype=torch.int64, device="cuda")
    t.replay(dict(policy_mask=31), caps, list(range(d.n_nodes)), got)
    torch.cuda.synchronize()
    g = got.cpu().numpy()
    for pi in range(5):
        for ci in range(len(caps)):
            for w in range(d.n_nodes):
                assert np.array_equal(g[pi, ci, w], ref[pi, ci, w]), (name, pi, caps[ci], w, g[pi, ci, w], ref[pi, ci, w])


def test_replay_deterministic(pair):
    name, d, pc, o, t = pair
    caps = _caps_for(o, d, name)[:2]
    a = torch.zeros((2, len(caps), d.n_nodes, saga.NCOUNT), dtype=torch.int64, device="cuda")
    b = torch.zeros_like(a)
    t.replay(dict(policy_mask=3), caps, list(range(d.n_nodes)), a)
    t.replay(dict(policy_mask=3), caps, list(range(d.n_nodes)), b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def _score_batch(d, o, w, rng, n_seg=3, n=700):
    """Candidates at node w: local ids whose owner has a call admitted by epoch e (valid c*)."""
    E = 100_000
    own = o.lid_owner(w)
    ecall = d.call_t_us // E + 1
    first_e = np.full(d.n_sessions, np.iinfo(np.int64).max)
    np.minimum.at(first_e, d.call_session.astype(np.int64), ecall)
    ev = o.stream(w)["events"]
    segs = []
    for _ in range(n_seg):
        e = int(ev[rng.integers(0, len(ev)), 0])
        ok = np.array([(x >= d.n_sessions) or (first_e[x] <= e) for x in own])
        pool = np.nonzero(ok)[0]
        if pool.size == 0:
            continue
        lid = rng.choice(pool, size=min(n, pool.size), replace=False).astype(np.uint32)
        Te = e * E
        tl = Te - rng.integers(0, 60_000_000, size=lid.size)
        nu = rng.integers(0, 2 ** 32, size=lid.size, dtype=np.uint64).astype(np.uint32)
        cap = int(rng.integers(max(1, lid.size), lid.size * 2 + 2))
        occ = int(rng.integers(lid.size, cap + 1))
        act = int(rng.integers(0, 1 << d.n_types))
        segs.append((w, e, occ, cap, act, lid, tl.astype(np.int64), nu))
    return segs


@pytest.mark.parametrize("policy", [saga.POLICY_AEG, saga.POLICY_BELADY])
def test_score_keys_equal(pair, policy):
    name, d, pc, o, t = pair
    rng = np.random.default_rng(5)
    segs = []
    for w in range(d.n_nodes):
        if o.n_local(w):
            segs += _score_batch(d, o, w, rng)
    if not segs:
        pytest.skip("no candidates")
    dev = "cuda"
    off = np.concatenate([[0], np.cumsum([s[5].size for s in segs])]).astype(np.int64)
    i32 = lambda a: torch.from_numpy(np.asarray(a, np.uint32).view(np.int32).copy()).to(dev)
    batch = dict(seg_node=i32([s[0] for s in segs]), seg_epoch=i32([s[1] for s in segs]),
                 seg_occ=i32([s[2] for s in segs]), seg_cap=i32([s[3] for s in segs]),
                 seg_act=i32([s[4] for s in segs]), seg_off=torch.from_numpy(off).to(dev),
                 cand_lid=i32(np.concatenate([s[5] for s in segs])),
                 cand_t_last=torch.from_numpy(np.concatenate([s[6] for s in segs])).to(dev),
                 cand_nu=i32(np.concatenate([s[7] for s in segs])))
    key = torch.empty(int(off[-1]), dtype=torch.int64, device=dev)
    score = torch.empty(int(off[-1]), dtype=torch.float32, device=dev)
    t.aeg_score(batch, {}, key, score, policy=policy)
    torch.cuda.synchronize()
    gk = key.cpu().numpy().view(np.uint64)
    gs = score.cpu().numpy()
    for i, s in enumerate(segs):
        k, s32, s64 = o.keys(policy, s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7])
        assert np.array_equal(gk[off[i]:off[i + 1]], k), (name, i)
        if policy == saga.POLICY_AEG:
            g = gs[off[i]:off[i + 1]]
            assert np.array_equal(g.view(np.uint32), s32.view(np.uint32)), (name, i)
            assert np.all(np.abs(g.astype(np.float64) - s64) <= 1e-5 * np.abs(s64) + 1e-6), (name, i)


def test_select_equal():
    rng = np.random.default_rng(1)
    sizes = [1, 2, 31, 1000, 4097, 32768, 5]
    keys, ks, offs = [], [], [0]
    for n in sizes:
        x = np.unique(rng.integers(0, 2 ** 63, size=n * 2, dtype=np.uint64))[:n]
        if n > 20:  # clustered keys: many equal high bits (like equal q of one session)
            x = (np.uint64(0x8000002A00000000) | rng.choice(2 ** 20, size=n, replace=False).astype(np.uint64))
        rng.shuffle(x)
        keys.append(x)
        ks.append(int(rng.integers(1, n + 1)) if n > 1 else 1)
        offs.append(offs[-1] + n)
    allk = np.concatenate(keys)
    out_off = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)
    dev = "cuda"
    vk = torch.from_numpy(allk.view(np.int64).copy()).to(dev)
    so = torch.from_numpy(np.array(offs, np.int64)).to(dev)
    kk = torch.from_numpy(np.array(ks, np.int32)).to(dev)
    oo = torch.from_numpy(out_off).to(dev)
    vic = torch.full((int(out_off[-1]),), -1, dtype=torch.int32, device=dev)
    saga.evict_select(vk, so, kk, oo, vic)
    torch.cuda.synchronize()
    g = vic.cpu().numpy()
    for i, x in enumerate(keys):
        ref = O.select_topk(x, ks[i])
        assert np.array_equal(g[out_off[i]:out_off[i + 1]], ref), i


@pytest.mark.parametrize("clustered", [False, True])
def test_select_equal_shared_memory_path(clustered):
    """k <= 4096 with a pivot digit of <= 4096 keys runs the shared-memory path; k > 4096 or a
    crowded pivot digit runs the general path.  Both must equal the full descending sort."""
    rng = np.random.default_rng(11 + clustered)
    cases = [(32768, 1), (32768, 5), (32768, 327), (32768, 4096), (32768, 4097), (9000, 8999), (9000, 9000),
             (4096, 2048), (70000, 700), (3, 2)]
    keys, ks, offs = [], [], [0]
    for n, k in cases:
        if clustered:  # equal high bits: one protection bit and q, lids differ
            x = np.uint64(0x8000002A00000000) | rng.choice(2 ** 22, size=n, replace=False).astype(np.uint64)
        else:
            x = np.unique(rng.integers(0, 2 ** 64 - 1, size=n * 2, dtype=np.uint64))[:n]
        rng.shuffle(x)
        keys.append(x)
        ks.append(k)
        offs.append(offs[-1] + n)
    allk = np.concatenate(keys)
    out_off = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)
    dev = "cuda"
    vk = torch.from_numpy(allk.view(np.int64).copy()).to(dev)
    so = torch.from_numpy(np.array(offs, np.int64)).to(dev)
    kk = torch.from_numpy(np.array(ks, np.int32)).to(dev)
    oo = torch.from_numpy(out_off).to(dev)
    vic = torch.full((int(out_off[-1]),), -1, dtype=torch.int32, device=dev)
    saga.evict_select(vk, so, kk, oo, vic)
    torch.cuda.synchronize()
    g = vic.cpu().numpy()
    for i, x in enumerate(keys):
        ref = O.select_topk(x, ks[i])
        assert np.array_equal(g[out_off[i]:out_off[i + 1]], ref), (i, cases[i])


def test_invalid_trace_rejected():
    d = make_c1()
    d.call_t_us = d.call_t_us.copy()
    d.call_t_us[5], d.call_t_us[6] = d.call_t_us[6], d.call_t_us[5]
    with pytest.raises(saga.SagaError) as ex:
        saga.Trace(d, default_place_cfg())
    assert ex.value.status == 2
    d = make_c1()
    d.range_block_lo = d.range_block_lo.copy()
    d.range_block_lo[1] = 40
    with pytest.raises(saga.SagaError) as ex:
        saga.Trace(d, default_place_cfg())
    assert ex.value.status == 2


def test_state_errors():
    d = make_c1()
    t = saga.Trace(d, default_place_cfg())
    with pytest.raises(saga.SagaError) as ex:
        t.sweep_range(0)
    assert ex.value.status == 4
    c = torch.zeros((1, 1, 1, saga.NCOUNT), dtype=torch.int64, device="cuda")
    with pytest.raises(saga.SagaError):
        t.replay(dict(policy_mask=1), [10], [0], c)
    t.next_use(0)
    with pytest.raises(saga.SagaError) as ex:
        t.replay(dict(policy_mask=1), [0], [0], c)
    assert ex.value.status == 3
    # C1's largest call touches 12 blocks (S:209 CapacityError below it); 12 .. W_lo - 1 = 21 is
    # data: the replay stops at the first epoch whose requests exceed the capacity
    with pytest.raises(saga.SagaError) as ex:
        t.replay(dict(policy_mask=1), [11], [0], c)
    assert ex.value.status == 3
    t.replay(dict(policy_mask=1), [21], [0], c)
    assert int(c[0, 0, 0, saga.CI["INFEASIBLE_EPOCH"]]) > 0


def test_launches_counted():
    before = saga.kernel_launches()
    t = saga.Trace(make_c1(), default_place_cfg())
    t.next_use(0)
    assert saga.kernel_launches() > before


def test_victim_log_equal(pair):
    """saga_replay_victims: every victim of every eviction epoch, (epoch, local id) sets equal to
    the oracle's log for each policy, node and a few capacities; epochs ascending on both sides
    (single-item launches take the 512-thread shape; the counters test covers both shapes)."""
    name, d, pc, o, t = pair
    caps = _caps_for(o, d, name)
    caps = sorted(set([caps[0], caps[len(caps) // 2], caps[-1]]))
    for pol in (O.POL_AEG, O.POL_BELADY, O.POL_EVICT_ALL, O.POL_LRU, O.POL_LRU_PREFIX):
        for w in range(d.n_nodes):
            for cap in caps:
                gc, glog = t.replay_victims(dict(policy_mask=pol), cap, w)
                rc, rlog = o.replay_log(pol, w, cap)
                assert np.array_equal(gc, rc), (name, pol, w, cap)
                assert np.array_equal(np.sort(glog), np.sort(rlog)), (name, pol, w, cap)
                ge = (glog >> np.uint64(32)).astype(np.int64)
                assert np.all(np.diff(ge) >= 0)
