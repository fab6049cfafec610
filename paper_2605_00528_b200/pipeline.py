"""One pass of the whole hot path (A1-A8) through the C ABI, as bench.py and the tests run it.

load (A1-A3) -> next use per owned node (A4) -> W_lo/W_hi all-reduce max (A8 #1) -> capacity
sweep -> replay (A5-A7) -> counter all-reduce sum (A8 #2).  Nodes are sharded w mod R = rank
(DESIGN.md §6); C1-style single-node traces shard capacity points instead.
"""
from __future__ import annotations

import numpy as np

from . import saga


def owned_nodes(n_nodes: int, rank: int, world: int):
    return [w for w in range(n_nodes) if w % world == rank]


def run_step(desc, place_cfg: dict, replay_cfg: dict, caps_fn, rank: int = 0, world: int = 1, comm=None,
             device: int = 0, stream=None, host=None, counters=None, shard_caps: bool = False,
             before_expand=None, after_replay=None, mark=None):
    """Returns (trace handle, caps list, counters tensor [n_pol, n_caps, n_nodes, 16]).

    before_expand(stream), when given, defers A3 (SAGA_LOAD_DEFER_EXPAND) and is called between
    placement and the first expansion; after_replay(stream) is called after the replay launch.
    bench.py uses them to keep one step's expansion/next-use/replay behind the previous step's
    replay while its single-SM placement runs beside it."""
    import torch
    if shard_caps:
        nodes = list(range(desc.n_nodes))
        mask = 0
    else:
        nodes = owned_nodes(desc.n_nodes, rank, world)
        mask = sum(1 << w for w in nodes) if nodes else 0
    t = saga.Trace(desc, place_cfg, owned_mask=mask if nodes else (1 << (rank % desc.n_nodes)), device=device,
                   stream=stream, host=host, defer_expand=before_expand is not None)
    if before_expand is not None:
        before_expand(t.stream)
    for w in nodes:
        t.next_use(w)
    if mark is not None:
        mark(t.stream, "nextuse")
    wlo, whi = 0, 0
    for w in nodes:
        a, b = t.sweep_range(w)
        wlo, whi = max(wlo, a), max(whi, b)
    if comm is not None and world > 1:
        rng = torch.tensor([wlo, whi], dtype=torch.int64, device=f"cuda:{device}")
        comm.allreduce(rng, op=1, stream=t.stream)
        t.stream.synchronize()
        wlo, whi = (int(x) for x in rng.cpu())
    caps = caps_fn(wlo, whi)
    if mark is not None:
        mark(t.stream, "swept")
    npol = bin(replay_cfg.get("policy_mask", 3) & 31).count("1")
    if counters is None:
        counters = torch.zeros((npol, len(caps), desc.n_nodes, saga.NCOUNT), dtype=torch.int64,
                               device=f"cuda:{device}")
    else:
        counters.zero_()
    if shard_caps:
        mine = [i for i in range(len(caps)) if i % world == rank]
        for i in mine:
            sub = torch.zeros((npol, 1, desc.n_nodes, saga.NCOUNT), dtype=torch.int64, device=counters.device)
            t.replay(replay_cfg, [caps[i]], nodes, sub)
            counters[:, i:i + 1].copy_(sub)
    elif nodes:
        t.replay(replay_cfg, caps, nodes, counters)
    if mark is not None:
        mark(t.stream, "replay_q")
    if after_replay is not None:
        after_replay(t.stream)
    if comm is not None and world > 1:
        comm.allreduce(counters, op=0, stream=t.stream)
    return t, caps, counters
