"""Pins of the F3 pattern-inference oracle (oracle/pattern.py) against the paper, SPEC's worked
examples and closed forms -- nothing here calls the CUDA path.

  * S:131-133 worked examples: 29 completed tasks -> not ready; A->B->B->end x 30 -> A->B only
    (B->B and B->end are 1/2 each); A->B 9/10, A->C 1/10 -> A->B only.
  * S:158 / S:585 recovery: label sequences drawn from a known first-order chain whose edges all
    have probability >= 0.7 recover exactly that edge set; the held-out accuracy matches the
    chain's closed form sum_x n_x p(x -> pred x) / sum_x n_x within 5 binomial sigmas.
  * theta boundary (R-pattern ">="): 7/10 retained at theta 0.7, 69/100 dropped; ties at theta
    0.5 predict the smaller label; the fp32 probability of a retained edge is c / t rounded once.
  * invariants: sum of counts = calls of completed training sessions; tasks = completed training
    sessions; role-0 sessions contribute nothing.
"""
import numpy as np
import pytest

from gen import make, make_label_markov, pattern_labels, pattern_roles
from oracle.pattern import NONE, pattern_infer, pattern_infer_desc

A, B, C_, END3 = 0, 1, 2, 3  # labels of a 3-label alphabet, END = L


def _sessions(seqs, types=None, roles=None, ended=None):
    """flat call arrays of explicit label sequences (sessions interleaved call by call)."""
    n = len(seqs)
    types = types or [0] * n
    roles = roles or [1] * n
    ended = ended or [True] * n
    calls = []  # (time, session, label, last)
    for s, q in enumerate(seqs):
        for k, x in enumerate(q):
            calls.append((k * 1000 + s, s, x, int(ended[s] and k == len(q) - 1)))
    calls.sort()
    cs = np.array([c[1] for c in calls]); lab = np.array([c[2] for c in calls], np.uint32)
    last = np.array([c[3] for c in calls], np.uint8)
    return cs, last, np.array(types, np.uint16), lab, np.array(roles, np.uint8)


def _infer(seqs, L=3, theta=700, min_tasks=30, **kw):
    cs, last, ty, lab, ro = _sessions(seqs, **kw)
    return pattern_infer(cs, last, ty, int(ty.max()) + 1, lab, L, ro, theta, min_tasks)


def test_cold_start_29_vs_30():
    o = _infer([[A, B]] * 29)
    assert o["tasks"][0] == 29 and (o["pred"] == NONE).all()
    o = _infer([[A, B]] * 30)
    assert o["tasks"][0] == 30 and o["pred"][0, A] == B and o["pred"][0, B] == END3


def test_spec_example_abb():
    o = _infer([[A, B, B]] * 30)
    assert o["counts"][0, A].tolist() == [0, 30, 0, 0]
    assert o["counts"][0, B].tolist() == [0, 30, 0, 30]      # B->B 1/2, B->end 1/2
    assert o["pred"][0, A] == B and o["pred"][0, B] == NONE  # 0.5 < 0.7: dropped
    assert o["prob"][0, A, B] == np.float32(1.0) and o["prob"][0, B].tolist() == [0, 0, 0, 0]


def test_spec_example_nine_in_ten():
    o = _infer([[A, B]] * 27 + [[A, C_]] * 3)
    assert o["pred"][0, A] == B
    assert o["prob"][0, A, B] == np.float32(27) / np.float32(30) and o["prob"][0, A, C_] == 0


def test_theta_boundary_and_ties():
    o = _infer([[A, B]] * 21 + [[A, C_]] * 9)                # 7/10 exactly: retained (>=)
    assert o["pred"][0, A] == B
    o = _infer([[A, B]] * 69 + [[A, C_]] * 31)               # 0.69 < 0.7
    assert o["pred"][0, A] == NONE
    o = _infer([[A, C_]] * 15 + [[A, B]] * 15, theta=500)    # tie: both retained, smaller label
    assert o["pred"][0, A] == B
    assert o["prob"][0, A, B] == np.float32(0.5) and o["prob"][0, A, C_] == np.float32(0.5)


def test_unfinished_sessions_and_roles():
    seqs = [[A, B, C_]] * 30 + [[A, B]] * 5 + [[C_, C_]] * 4
    o = _infer(seqs, ended=[True] * 30 + [False] * 5 + [True] * 4, roles=[1] * 35 + [0] * 4)
    assert o["tasks"][0] == 30
    assert o["counts"][0].sum() == 30 * 3 + 5 * 1           # unfinished: no end transition
    assert o["counts"][0, C_, C_] == 0                      # role 0 ignored
    assert o["counts"][0, C_, END3] == 30


def test_types_are_separate():
    seqs = [[A, B]] * 30 + [[A, C_]] * 30
    o = _infer(seqs, types=[0] * 30 + [1] * 30)
    assert o["pred"][0, A] == B and o["pred"][1, A] == C_


def test_held_out_accuracy_deterministic_chain():
    seqs = [[A, B, C_]] * 80
    o = _infer(seqs, roles=[1, 2] * 40)
    ev = o["eval"][0]
    assert ev[0] == 40 * 3 and ev[1] == ev[0] and ev[2] == ev[0]  # every step predicted, all correct


# a chain whose every edge has p >= 0.7 (the rest of each row is the end of the task)
TRANS = np.array([[0.0, 0.9, 0.0, 0.0, 0.1],
                  [0.0, 0.0, 0.8, 0.0, 0.2],
                  [0.0, 0.0, 0.0, 0.75, 0.25],
                  [0.85, 0.0, 0.0, 0.0, 0.15]])


def test_recovers_known_chain_and_accuracy_closed_form():
    d = make_label_markov(3, 600, TRANS, n_types=2)
    lab = pattern_labels(d)
    role = pattern_roles(d)
    o = pattern_infer_desc(d, lab, 4, role)
    for a in range(2):
        assert o["tasks"][a] >= 30
        assert o["pred"][a].tolist() == [1, 2, 3, 0]          # exactly the true edge set
        # held-out: transitions out of x go to pred(x) with probability TRANS[x, pred(x)]
        ev = o["eval"][a]
        assert ev[1] == ev[0]
        n_x = np.zeros(4)
        cs = np.asarray(d.call_session)
        for s in np.nonzero((role == 2) & (np.asarray(d.session_type) == a))[0]:
            for c in np.nonzero(cs == s)[0]:
                n_x[lab[c]] += 1
        p = np.array([TRANS[x, [1, 2, 3, 0][x]] for x in range(4)])
        mean = float((n_x * p).sum())
        sd = float(np.sqrt((n_x * p * (1 - p)).sum()))
        assert n_x.sum() == ev[0]
        assert abs(ev[2] - mean) <= 5 * sd, (ev, mean, sd)


def test_counts_sum_to_training_calls_on_c2():
    d = make("C2")
    lab = pattern_labels(d)
    role = pattern_roles(d)
    o = pattern_infer_desc(d, lab, 5, role)
    cs = np.asarray(d.call_session)
    train_calls = int((role[cs] == 1).sum())
    assert int(o["counts"].sum()) == train_calls           # every session of C2 completes
    assert int(o["tasks"][0]) == int((role == 1).sum())
    # SWE chain read_file -> edit_code -> run_test -> read_file: every edge >= 0.7
    assert o["pred"][0, 0] == 1 and o["pred"][0, 1] == 4 and o["pred"][0, 4] == 0


def test_bad_label_rejected():
    cs, last, ty, lab, ro = _sessions([[A, B]] * 2)
    lab[0] = 7
    with pytest.raises(ValueError):
        pattern_infer(cs, last, ty, 1, lab, 3, ro)
