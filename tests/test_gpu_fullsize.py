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


def test_c2_full_size_equals_oracle():
    d, pc, t, caps, ctr = _run("C2")
    o = O.Oracle(d, pc)
    on, om, _, _ = o.placement()
    gn, gm, _, _ = t.placement()
    assert np.array_equal(on, gn)
    assert np.array_equal(om, gm)
    nu = torch.empty(t.info(0)[0], dtype=torch.int32, device="cuda")
    t.next_use(0, nu, None)
    torch.cuda.synchronize()
    assert np.array_equal(nu.cpu().numpy().view(np.uint32), o.next_use(0)["next_use"])
    lo = max(o.sweep_range(w)[0] for w in range(d.n_nodes))
    hi = max(o.sweep_range(w)[1] for w in range(d.n_nodes))
    assert caps == sweep_caps(lo, hi, N_SWEEP["C2"], PHYSICAL_CAP.get("C2"))
    idx = [0, len(caps) - 1]  # the tightest point and the physical capacity, every node
    ref = o.replay_many(3, [caps[i] for i in idx])
    assert np.array_equal(ctr[:, idx], ref)
    _properties(d, t, caps, ctr)
    t.free()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_properties_and_sampled_node(name):
    """C3 (288 items) and C4 (1,024 items) launch more items than SMs: the 256 x 2 replay shape."""
    d, pc, t, caps, ctr = _run(name)
    _properties(d, t, caps, ctr)
    o = O.Oracle(d, pc)
    ref = o.replay_many(3, [caps[0]], nodes=[0])  # one node at the tightest capacity
    assert np.array_equal(ctr[:, :1, 0], ref[:, :, 0])
    t.free()
