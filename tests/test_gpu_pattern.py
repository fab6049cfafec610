"""F3 pattern inference: GPU (saga_pattern_infer, k_pattern.cu) == CPU oracle (oracle/pattern.py).

Bit-exact: transition counts, completed-task counts, predicted successors, held-out
(transitions, predicted, correct), and the fp32 probability of every retained edge (one
round-to-nearest division of two integers on both sides).  Cases: full-size C2 / C3 / C5 with
the generator's tool labels; a known label chain with two agent types; random small traces with
random labels (up to 64), random roles (incl. ignored sessions), theta from 1 to 1000 (ties at
theta <= 500) and small cold starts; the global-histogram path (bins > 12288); bad labels.
"""
import numpy as np
import pytest

from gen import (default_place_cfg, make, make_label_markov, make_random_small, pattern_labels, pattern_roles,
                 place_cfg_for)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_00528_b200 import saga  # noqa: E402
from oracle.pattern import NONE, pattern_infer_desc  # noqa: E402


def _run(d, pc, label, L, role, theta=700, min_tasks=30):
    t = saga.Trace(d, pc, defer_expand=True)  # F3 reads only the A1 tables
    lab = torch.from_numpy(np.ascontiguousarray(label, np.uint32).view(np.int32)).cuda()
    ro = torch.from_numpy(np.ascontiguousarray(role, np.uint8)).cuda()
    out = t.pattern_infer(lab, L, ro, theta, min_tasks)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    t.free()
    ref = pattern_infer_desc(d, label, L, role, theta, min_tasks)
    assert np.array_equal(got["counts"], ref["counts"])
    assert np.array_equal(got["tasks"].astype(np.int64), ref["tasks"])
    assert np.array_equal(got["pred"].view(np.uint32), ref["pred"])
    assert np.array_equal(got["prob"].view(np.uint32), ref["prob"].view(np.uint32))
    assert np.array_equal(got["eval"], ref["eval"])
    return got


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_full_size_tool_labels(name):
    d = make(name)
    got = _run(d, place_cfg_for(d), pattern_labels(d), 5, pattern_roles(d))
    assert got["eval"][:, 0].sum() > 0


def test_known_chain_two_types():
    trans = np.array([[0.0, 0.9, 0.0, 0.0, 0.1], [0.0, 0.0, 0.8, 0.0, 0.2],
                      [0.0, 0.0, 0.0, 0.75, 0.25], [0.85, 0.0, 0.0, 0.0, 0.15]])
    d = make_label_markov(5, 400, trans, n_types=2)
    got = _run(d, default_place_cfg(0), pattern_labels(d), 4, pattern_roles(d))
    assert got["pred"].tolist() == [[1, 2, 3, 0]] * 2


@pytest.mark.parametrize("seed", range(12))
def test_random_small(seed):
    rng = np.random.default_rng(100 + seed)
    d = make_random_small(seed, n_sessions=int(rng.integers(1, 40)), n_nodes=2, max_calls=6, n_types=int(rng.integers(1, 5)))
    L = int(rng.choice([1, 2, 3, 7, 64]))
    label = rng.integers(0, L, size=d.n_calls).astype(np.uint32)
    role = rng.integers(0, 3, size=d.n_sessions).astype(np.uint8)
    theta = int(rng.choice([1, 300, 500, 700, 1000]))
    _run(d, default_place_cfg(seed), label, L, role, theta, int(rng.integers(0, 4)))


def test_global_histogram_path():
    # 4 types x 64 labels x 65 successors = 16,640 bins > 12,288: global atomics
    d = make_random_small(11, n_sessions=120, n_nodes=2, max_calls=8, n_types=4)
    assert d.n_types == 4
    rng = np.random.default_rng(7)
    label = rng.integers(0, 64, size=d.n_calls).astype(np.uint32)
    _run(d, default_place_cfg(0), label, 64, pattern_roles(d), 300, 5)


def test_bad_label_and_args():
    d = make_random_small(1)
    t = saga.Trace(d, default_place_cfg(0))
    lab = torch.zeros(d.n_calls, dtype=torch.int32, device="cuda")
    ro = torch.ones(d.n_sessions, dtype=torch.uint8, device="cuda")
    lab[d.n_calls // 2] = 3
    with pytest.raises(saga.SagaError):
        t.pattern_infer(lab, 3, ro)
    with pytest.raises(saga.SagaError):
        t.pattern_infer(lab, 65, ro)
    with pytest.raises(saga.SagaError):
        t.pattern_infer(lab, 4, ro, theta_pm=0)
    out = t.pattern_infer(lab, 4, torch.zeros_like(ro))  # nothing to count
    assert int(out["counts"].sum()) == 0 and bool((out["pred"] == -1).all())
    t.free()


def test_replay_with_inferred_aeg_equals_oracle():
    """'Score with the inferred AEG': the re-annotated trace loads and replays bit-exactly."""
    from gen import TOOL_LABELS, sweep_caps
    from oracle import oracle as O
    from paper_2605_00528_b200 import pipeline
    d = make("C2", n_sessions=80, n_nodes=4)
    pc = place_cfg_for(d)
    L = len(TOOL_LABELS)
    label, role = pattern_labels(d), pattern_roles(d)
    got = _run(d, pc, label, L, role, 700, 10)
    di = pipeline.inferred_aeg_desc(d, label, L, got["prob"], np.full(L, 2_000_000), np.full(L, 300))
    t, caps, ctr = pipeline.run_step(di, pc, dict(policy_mask=3), lambda lo, hi: sweep_caps(lo, hi, 4))
    torch.cuda.synchronize()
    O.build()
    ref = O.Oracle(di, pc).replay_many(3, caps)
    assert np.array_equal(ctr.cpu().numpy(), ref)
    t.free()
