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
             before_expand=None, after_replay=None, mark=None, range_comm=None, replay_wait: bool = True,
             range_host_reduce=None):
    """Returns (trace handle, caps list, counters tensor [n_pol, n_caps, n_nodes, 16]).

    range_host_reduce(wlo, whi) -> (wlo, whi), when given, replaces the NCCL max all-reduce of
    (W_lo, W_hi): the values are already on the host (saga_sweep_range synchronises), and an NCCL
    kernel would have to wait for an SM that the replays in flight hold for 100+ ms.
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
    t.next_use_nodes(nodes)   # every owned node in one launch set per kernel (A4)
    if mark is not None:
        mark(t.stream, "nextuse")
    wlo, whi = 0, 0
    for w in nodes:
        a, b = t.sweep_range(w)
        wlo, whi = max(wlo, a), max(whi, b)
    rcomm = comm if (comm is not None and world > 1) else range_comm
    if range_host_reduce is not None:  # A8 #1 as a host exchange of the two host-side values
        wlo, whi = range_host_reduce(wlo, whi)
    elif rcomm is not None:  # A8 #1 (range_comm: independent trials that still share one sweep)
        rng = torch.tensor([wlo, whi], dtype=torch.int64, device=f"cuda:{device}")
        rcomm.allreduce(rng, op=1, stream=t.stream)
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
            t.replay(replay_cfg, [caps[i]], nodes, sub, wait=replay_wait)
            counters[:, i:i + 1].copy_(sub)
    elif nodes:
        t.replay(replay_cfg, caps, nodes, counters, wait=replay_wait)
    if mark is not None:
        mark(t.stream, "replay_q")
    if after_replay is not None:
        after_replay(t.stream)
    if comm is not None and world > 1:
        comm.allreduce(counters, op=0, stream=t.stream)
    return t, caps, counters


def inferred_aeg_desc(desc, label, n_labels: int, prob, ttl_us, obs_tokens):
    """The trace re-annotated with the AEG inferred by saga_pattern_infer (F3: "score with the
    inferred AEG", tier (b) of P:645).  Node (a, x) = a * n_labels + x stands for "agent type a,
    tool x"; call c moves to node (type of its session, label[c]); edges are the retained
    (a, x) -> (a, y), y < n_labels, with P = prob[a, x, y] (the kernel's fp32 frequency) and the
    linear-chain overlap (whole context shared, eq:overlap P:685); no node is terminal (the
    residual mass is the end of the task).  ttl_us / obs_tokens [n_labels] are the per-tool TTL
    base and expected observation length the scheduler keeps per tool (Alg. 1 line 2).
    Host re-indexing only: every number comes from the kernel or the caller."""
    import dataclasses
    prob = np.asarray(prob, np.float32)
    T, L = prob.shape[0], int(n_labels)
    off, dst, p = [0], [], []
    for a in range(T):
        for x in range(L):
            for y in range(L):
                if prob[a, x, y] > 0:
                    dst.append(a * L + y)
                    p.append(prob[a, x, y])
            off.append(len(dst))
    styp = np.asarray(desc.session_type, np.int64)
    node = styp[np.asarray(desc.call_session, np.int64)] * L + np.asarray(label, np.int64)
    return dataclasses.replace(
        desc, name=desc.name + "+inferred", call_aeg_node=node.astype(np.uint32),
        aeg_edge_off=np.array(off, np.uint32), edge_dst=np.array(dst, np.uint32), edge_p=np.array(p, np.float32),
        edge_shared_q16=np.full(len(dst), 65536, np.uint32),
        node_ttl_base_us=np.tile(np.asarray(ttl_us, np.int64), T), node_obs_tokens=np.tile(np.asarray(obs_tokens, np.uint32), T),
        node_terminal=np.zeros(T * L, np.uint8), node_tool=np.tile(np.arange(L, dtype=np.uint32), T))
