#!/usr/bin/env python
"""Diagnostic (not a target): what each policy evicts, on a scaled C2 trace with the CPU oracle.

For every victim (epoch e, local id b) of a replay, "dead" = block b is never requested again at
this node after epoch e; "live" = it is, so evicting it costs a re-load later.  Bélády-epoch evicts
dead blocks first (farthest next use); the question is how often WA-LRU and LRU pick live blocks
and whose.  Writes a markdown table to stdout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from gen import make, place_cfg_for, sweep_caps  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main(n_sessions=100, node=0):
    O.build()
    d = make("C2", n_sessions=n_sessions, n_nodes=2)
    o = O.Oracle(d, place_cfg_for(d))
    s = o.stream(node)
    lid = o.next_use(node)["local_id"].astype(np.int64)
    # epoch index of each position
    ev = s["events"]
    pos_e = np.zeros(lid.size, np.int64)
    gi = 0
    for j, row in enumerate(ev):
        for _ in range(row[1]):
            p0, ln = int(s["groups"][gi][0]), int(s["groups"][gi][1])
            pos_e[p0:p0 + ln] = row[0]
            gi += 1
    last_e = np.full(o.n_local(node), -1, np.int64)
    np.maximum.at(last_e, lid, pos_e)          # the block's last requesting epoch at this node
    own = o.lid_owner(node)
    lo, hi = o.sweep_range(node)
    caps = sweep_caps(lo, hi, 8)
    print(f"C2 scaled to {n_sessions} sessions, node {node}; victims that are re-requested later (live) / all victims")
    print("| capacity | " + " | ".join(f"{p} live / victims (regen)" for p in ("WA-LRU", "LRU", "BELADY")) + " |")
    print("|---|---|---|---|")
    for C in caps[::2]:
        cells = []
        for pol in (O.POL_AEG, O.POL_LRU, O.POL_BELADY):
            ctr, log = o.replay_log(pol, node, C)
            e = (log >> np.uint64(32)).astype(np.int64)
            b = (log & np.uint64(0xFFFFFFFF)).astype(np.int64)
            live = int((last_e[b] > e).sum())
            regen = int(ctr[O.CI["MISSES"]] - ctr[O.CI["COMPULSORY_GLOBAL"]] + ctr[O.CI["MIG_MISSES"]])
            cells.append(f"{live} / {len(log)} ({regen})")
        print(f"| {C} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
