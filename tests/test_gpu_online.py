"""F4 online statistics and per-call overrides: GPU == CPU oracle, bit-exact.

* saga_tool_stats (k_stats.cu) vs oracle/tool_stats.py: per-call TTL base (nearest-rank
  percentile of the tool's last `window` latencies completed by the call's tool start) and the
  truncated fp64 EMA of observation lengths -- every call on small traces and random labels /
  windows / cold starts, sampled calls at the full C2 and C4 sizes.
* saga_trace_desc.call_ttl_base_us / call_obs_tokens: random per-call overrides, and the online
  statistics fed back, replayed end to end (placement, streams, replay counters incl. the victim
  hash) against the oracle given the same overrides computed by the oracle itself.
"""
import dataclasses

import numpy as np
import pytest

from gen import (default_place_cfg, make, make_random_small, pattern_labels, place_cfg_for, sweep_caps)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_00528_b200 import pipeline, saga  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle.tool_stats import tool_stats as oracle_tool_stats  # noqa: E402

O.build()


def _gpu_stats(d, pc, label, L, **kw):
    t = saga.Trace(d, pc, defer_expand=True)
    lab = torch.from_numpy(np.ascontiguousarray(label, np.uint32).view(np.int32)).cuda()
    ttl, obs = t.tool_stats(lab, L, **kw)
    torch.cuda.synchronize()
    out = ttl.cpu().numpy(), obs.cpu().numpy().view(np.uint32)
    t.free()
    return out


@pytest.mark.parametrize("seed", range(8))
def test_small_every_call(seed):
    rng = np.random.default_rng(seed)
    if seed % 2:
        d = make("C2", n_sessions=int(rng.integers(20, 120)), n_nodes=2)
        pc = place_cfg_for(d)
    else:
        d = make_random_small(seed, n_sessions=int(rng.integers(2, 40)), n_nodes=2, max_calls=8)
        pc = default_place_cfg(seed)
    L = int(rng.choice([1, 2, 5, 64]))
    label = rng.integers(0, L, size=d.n_calls).astype(np.uint32)
    kw = dict(p_pm=int(rng.choice([1, 500, 950, 1000])), window=int(rng.choice([1, 7, 32, 256, 1024])),
              min_samples=int(rng.integers(0, 4)), ema_terms=int(rng.choice([0, 1, 16, 64, 256])))
    g_ttl, g_obs = _gpu_stats(d, pc, label, L, **kw)
    r_ttl, r_obs = oracle_tool_stats(d, pc, label, L, kw["p_pm"], kw["window"], kw["min_samples"], kw["ema_terms"])
    assert np.array_equal(g_ttl, r_ttl)
    assert np.array_equal(g_obs, r_obs)


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_full_size_sampled(name):
    d = make(name)
    pc = place_cfg_for(d)
    label = pattern_labels(d)
    g_ttl, g_obs = _gpu_stats(d, pc, label, 5)
    calls = np.random.default_rng(1).choice(d.n_calls, size=3000, replace=False)
    r_ttl, r_obs = oracle_tool_stats(d, pc, label, 5, calls=calls)
    assert np.array_equal(g_ttl[calls], r_ttl)
    assert np.array_equal(g_obs[calls], r_obs)
    assert (g_ttl != d.node_ttl_base_us[d.call_aeg_node]).any()  # the online values do differ


def _replay_equal(d, pc, n_caps=4):
    t, caps, ctr = pipeline.run_step(d, pc, dict(policy_mask=31), lambda lo, hi: sweep_caps(lo, hi, n_caps))
    torch.cuda.synchronize()
    got = ctr.cpu().numpy()
    gn, gm, gs, _ = t.placement()
    t.free()
    o = O.Oracle(d, pc)
    on, om, os_, _ = o.placement()
    assert np.array_equal(gn, on) and np.array_equal(gm, om)
    ref = o.replay_many(31, caps)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("seed", range(4))
def test_random_overrides_replay(seed):
    rng = np.random.default_rng(50 + seed)
    d = make("C2", n_sessions=60, n_nodes=3)
    pc = place_cfg_for(d)
    pc.update(kappa=2)  # queues and steals: placement reads the TTL through cached(w, s)
    d = dataclasses.replace(d, call_ttl_base_us=rng.integers(0, 3_000_000, size=d.n_calls).astype(np.int64),
                            call_obs_tokens=rng.integers(0, 3000, size=d.n_calls).astype(np.uint32))
    _replay_equal(d, pc)


def test_online_stats_fed_back_replay():
    d = make("C2", n_sessions=80, n_nodes=4)
    pc = place_cfg_for(d)
    label = pattern_labels(d)
    g_ttl, g_obs = _gpu_stats(d, pc, label, 5, min_samples=5)
    r_ttl, r_obs = oracle_tool_stats(d, pc, label, 5, min_samples=5)
    assert np.array_equal(g_ttl, r_ttl) and np.array_equal(g_obs, r_obs)
    # each side replays with its own statistics (identical by the line above)
    _replay_equal(dataclasses.replace(d, call_ttl_base_us=r_ttl, call_obs_tokens=r_obs), pc)


def test_bad_override_rejected():
    d = make_random_small(2)
    d = dataclasses.replace(d, call_ttl_base_us=np.full(d.n_calls, 2_000_000_000, np.int64))
    with pytest.raises(saga.SagaError):
        saga.Trace(d, default_place_cfg(0))
