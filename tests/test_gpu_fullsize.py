"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

pipeline.run_step (the call bench.py times) on the full C2 / C3 / C4 traces, compared with the
CPU oracle on sampled outputs it can compute (whole nodes at a few capacities), plus properties
that hold at any size: the access identity, |S| <= C, compulsory misses equal to
first touches and independent of policy and capacity, hits(AEG) <= hits(BELADY) per epoch-batched
optimality, and BELADY misses = compulsory misses at C >= W_hi where no block was invalidated.
"""
import numpy as np
import pytest

from gen import make, place_cfg_for, sweep_caps, N_SWEEP, PHYSICAL_CAP

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_00528_b200 import pipeline, saga  # noqa: E402
from oracle import oracle as O  # noqa: E402

CI = saga.CI


def _run(name):
    d = make(name)
    pc = place_cfg_for(d)
    caps_fn = lambda lo, hi: sweep_caps(lo, hi, N_SWEEP.get(name, 8), PHYSICAL_CAP.get(name))
    t, caps, ctr = pipeline.run_step(d, pc, dict(policy_mask=3), caps_fn)
    torch.cuda.synchronize()
    return d, pc, t, caps, ctr.cpu().numpy()


def _properties(d, t, caps, ctr):
    n_pol, n_caps, n_nodes, _ = ctr.shape
    for w in range(n_nodes):
        n_acc, _ = t.info(w)
        wlo, whi = t.sweep_range(w)
        comp = set()
        for p in range(n_pol):
            for c in range(n_caps):
                r = ctr[p, c, w]
                if r[CI["INFEASIBLE_EPOCH"]]:
                    continue
                assert r[CI["ACCESSES"]] == n_acc
                assert r[CI["ACCESSES"]] == r[CI["HITS"]] + r[CI["MISSES"]] + r[CI["MIG_HITS"]] + r[CI["MIG_MISSES"]]
                assert r[CI["PEAK_RESIDENT"]] <= caps[c]
                comp.add(int(r[CI["COMPULSORY_NODE"]]))
        assert len(comp) <= 1, (w, comp)  # first touches: policy- and capacity-independent
        for c in range(n_caps):
            a, b = ctr[0, c, w], ctr[1, c, w]  # AEG, BELADY
            if a[CI["INFEASIBLE_EPOCH"]] or b[CI["INFEASIBLE_EPOCH"]]:
                continue
            assert a[CI["HITS"]] + a[CI["MIG_HITS"]] <= b[CI["HITS"]] + b[CI["MIG_HITS"]], (w, caps[c])
            if caps[c] >= whi and b[CI["INVALIDATED"]] == 0:
                assert b[CI["MISSES"]] + b[CI["MIG_MISSES"]] == b[CI["COMPULSORY_NODE"]], (w, caps[c])


def _next_use_all_nodes(d, t, o):
    """next_use and local_id of every node, element by element, plus W_lo / W_hi and n_local."""
    for w in range(d.n_nodes):
        n, nl = t.info(w)
        nu = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        lid = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        t.next_use(w, nu, lid)
        torch.cuda.synchronize()
        ref = o.next_use(w)
        assert np.array_equal(nu.cpu().numpy().view(np.uint32)[:n], ref["next_use"]), w
        assert np.array_equal(lid.cpu().numpy().view(np.uint32)[:n], ref["local_id"]), w
        assert t.info(w)[1] == o.n_local(w) and t.sweep_range(w) == o.sweep_range(w), w
        del nu, lid


def test_c2_full_size_equals_oracle():
    d, pc, t, caps, ctr = _run("C2")
    o = O.Oracle(d, pc)
    on, om, osteal, orr = o.placement()
    gn, gm, gsteal, grr = t.placement()
    assert np.array_equal(on, gn)
    assert np.array_equal(om, gm) and (osteal, orr) == (gsteal, grr)
    _next_use_all_nodes(d, t, o)
    lo = max(o.sweep_range(w)[0] for w in range(d.n_nodes))
    hi = max(o.sweep_range(w)[1] for w in range(d.n_nodes))
    assert caps == sweep_caps(lo, hi, N_SWEEP["C2"], PHYSICAL_CAP.get("C2"))
    idx = [0, 2, 4, 6, len(caps) - 1]  # five of the nine sweep points, every node, both policies
    ref = o.replay_many(3, [caps[i] for i in idx])
    assert np.array_equal(ctr[:, idx], ref)
    _properties(d, t, caps, ctr)
    t.free()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_all_nodes(name):
    """C3 (288 items) and C4 (1,024 items) launch more items than SMs: the 256 x 2 replay shape.
    Every node at the tightest sweep point (and, for C3, the physical capacity) against the oracle."""
    d, pc, t, caps, ctr = _run(name)
    _properties(d, t, caps, ctr)
    o = O.Oracle(d, pc)
    on, om, _, _ = o.placement()
    gn, gm, _, _ = t.placement()
    assert np.array_equal(on, gn) and np.array_equal(om, gm)
    idx = [0, len(caps) - 1] if name == "C3" else [0]
    ref = o.replay_many(3, [caps[i] for i in idx])
    assert np.array_equal(ctr[:, idx], ref)
    if name == "C3":
        _next_use_all_nodes(d, t, o)
    t.free()


def test_c5_full_size_sampled_nodes():
    """C5 (100k sessions, 32 nodes, 2.9e9 accesses): placement of all 6.4 M calls, then nodes 0 and
    1 (the only streams either side expands) at two capacities of the sweep, both policies."""
    d = make("C5")
    pc = place_cfg_for(d)
    nodes = [0, 1]
    t = saga.Trace(d, pc, owned_mask=0b11)
    o = O.Oracle(d, pc, node_mask=0b11)
    on, om, osteal, orr = o.placement()
    gn, gm, gsteal, grr = t.placement()
    assert np.array_equal(on, gn) and np.array_equal(om, gm) and (osteal, orr) == (gsteal, grr)
    for w in nodes:
        t.next_use(w)
        assert t.sweep_range(w) == o.sweep_range(w), w
    lo = max(o.sweep_range(w)[0] for w in nodes)
    hi = max(o.sweep_range(w)[1] for w in nodes)
    caps = sweep_caps(lo, hi, N_SWEEP["C5"], PHYSICAL_CAP.get("C5"))
    sel = [caps[0], caps[4]]
    got = torch.zeros((2, len(sel), d.n_nodes, saga.NCOUNT), dtype=torch.int64, device="cuda")
    t.replay(dict(policy_mask=3), sel, nodes, got)
    torch.cuda.synchronize()
    ref = o.replay_many(3, sel, nodes=nodes)
    assert np.array_equal(got.cpu().numpy()[:, :, nodes], ref[:, :, nodes])
    t.free()
