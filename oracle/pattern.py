"""CPU oracle of F3, pattern-based AEG inference (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module; it
shares no code with paper_2605_00528_b200/.  Plain Python loops over sessions, written from:

  P:645 (§3.3, tier (b)): "when only request streams are observable, we infer AEGs by extracting
    tool-type patterns, computing transition probabilities, and retaining edges exceeding
    theta_conf = 0.7" ... "(c) Cold-start: a new agent type with no history is served as a
    request-level workload until 30 tasks complete, after which pattern inference activates".
  P:1072 (tab:pattern caption): "Accuracy measures the fraction of correctly predicted next-step
    node transitions in held-out traces".
  S:126-134 (SPEC infer_pattern): graph of "exactly the transitions whose empirical probability
    >= theta_conf, probabilities = empirical frequencies"; NotReady below 30 tasks; worked
    examples (29 traces -> NotReady; A->B->B->end x30 -> A->B only; A->B 9/10 -> A->B only).

Readings (DESIGN.md §3 R-pattern): first-order transitions between consecutive calls of one
session; "task ended" is successor y = L, counted at a session's final call when it
carries call_is_last; "exceeding" read as >=; the decision is the integer comparison
1000 * count >= theta_pm * total; the predicted next step is the retained successor with the
largest count (smallest label on ties) -- unique whenever theta_pm > 500.
"""
from __future__ import annotations

import numpy as np

NONE = 0xFFFFFFFF


def session_calls(call_session, n_sessions):
    """Calls of each session in trace order (the trace is sorted by arrival time)."""
    seqs = [[] for _ in range(n_sessions)]
    for c, s in enumerate(np.asarray(call_session).tolist()):
        seqs[s].append(c)
    return seqs


def transitions(seq, label, call_is_last, n_labels):
    """(x, y) pairs of one session: consecutive calls' labels, then (x_last, L) if it ended."""
    out = []
    for k, c in enumerate(seq):
        x = int(label[c])
        if k + 1 < len(seq):
            out.append((x, int(label[seq[k + 1]])))
        elif call_is_last[c]:
            out.append((x, n_labels))
    return out


def pattern_infer(call_session, call_is_last, session_type, n_types, label, n_labels, role,
                  theta_pm=700, min_tasks=30):
    """Returns dict(counts [T][L][L+1] int64, tasks [T] int64, pred [T][L] uint32 (NONE = none),
    prob [T][L][L+1] float32, eval [T][4] int64 = transitions, predicted, correct, 0)."""
    L = int(n_labels)
    session_type = np.asarray(session_type)
    role = np.asarray(role)
    label = np.asarray(label)
    call_is_last = np.asarray(call_is_last)
    n_sessions = session_type.shape[0]
    seqs = session_calls(call_session, n_sessions)
    for s in range(n_sessions):
        if role[s] != 0:
            for c in seqs[s]:
                if int(label[c]) >= L:
                    raise ValueError(f"call_label[{c}] >= n_labels")
    # 1. transition counts and completed tasks over the training sessions
    counts = np.zeros((n_types, L, L + 1), np.int64)
    tasks = np.zeros(n_types, np.int64)
    for s in range(n_sessions):
        if role[s] != 1:
            continue
        a = int(session_type[s])
        for x, y in transitions(seqs[s], label, call_is_last, L):
            counts[a, x, y] += 1
            if y == L:
                tasks[a] += 1
    # 2. retained edges (empirical probability >= theta_conf) once the type is past cold start
    pred = np.full((n_types, L), NONE, np.uint32)
    prob = np.zeros((n_types, L, L + 1), np.float32)
    for a in range(n_types):
        if tasks[a] < min_tasks:
            continue
        for x in range(L):
            total = int(counts[a, x].sum())
            best, best_c = NONE, 0
            for y in range(L + 1):
                c = int(counts[a, x, y])
                if c > 0 and 1000 * c >= theta_pm * total:
                    prob[a, x, y] = np.float32(c) / np.float32(total)
                    if best == NONE or c > best_c:
                        best, best_c = y, c
            pred[a, x] = best
    # 3. next-step accuracy on the held-out sessions
    ev = np.zeros((n_types, 4), np.int64)
    for s in range(n_sessions):
        if role[s] != 2:
            continue
        a = int(session_type[s])
        for x, y in transitions(seqs[s], label, call_is_last, L):
            ev[a, 0] += 1
            if pred[a, x] != NONE:
                ev[a, 1] += 1
                if int(pred[a, x]) == y:
                    ev[a, 2] += 1
    return dict(counts=counts, tasks=tasks, pred=pred, prob=prob, eval=ev)


def pattern_infer_desc(d, label, n_labels, role, theta_pm=700, min_tasks=30):
    """pattern_infer on the fields of a gen.TraceDesc."""
    return pattern_infer(d.call_session, d.call_is_last, d.session_type, d.n_types, label, n_labels, role,
                         theta_pm, min_tasks)
