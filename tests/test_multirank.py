"""N>1 host logic on CPU: world_size-2 `gloo` process groups.

The multi-GPU path shards one trace by cache node (rank r owns nodes w mod R; a one-node trace
shards capacity points instead) and combines with two all-reduces: max of (W_lo, W_hi) before the
sweep is fixed and sum of the int64 counter tensor after the replay.  Every counter cell is
written by exactly one rank, so the sum is an exact gather.  These tests run that partition and
those reductions over gloo with the CPU oracle standing in for each rank's replay, and check the
combined result against a single-process oracle run: the partition must cover every
(policy, capacity, node) cell exactly once, including the victim-set hash.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import default_place_cfg, make, make_c1, place_cfg_for, sweep_caps
from oracle import oracle as O
from paper_2605_00528_b200.pipeline import owned_nodes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _trace(kind):
    if kind == "C1":
        return make_c1(), default_place_cfg(0)
    d = make("C2", n_sessions=40, n_nodes=4)
    return d, place_cfg_for(d)


def _worker(rank, world, port, kind, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, pc = _trace(kind)
        o = O.Oracle(d, pc)
        shard_caps = d.n_nodes == 1
        nodes = list(range(d.n_nodes)) if shard_caps else owned_nodes(d.n_nodes, rank, world)
        lo = max([o.sweep_range(w)[0] for w in nodes] or [0])
        hi = max([o.sweep_range(w)[1] for w in nodes] or [0])
        rng = torch.tensor([lo, hi], dtype=torch.int64)
        dist.all_reduce(rng, op=dist.ReduceOp.MAX)          # A8 #1
        caps = sweep_caps(int(rng[0]), int(rng[1]), 5)
        ctr = np.zeros((3, len(caps), d.n_nodes, O.NCOUNT), dtype=np.int64)
        if shard_caps:
            mine = [i for i in range(len(caps)) if i % world == rank]
            for i in mine:
                ctr[:, i:i + 1] = o.replay_many(7, [caps[i]], nodes=nodes)[:, :, :, :]
        elif nodes:
            part = o.replay_many(7, caps, nodes=nodes)
            ctr[:, :, nodes] = part[:, :, nodes]
        t = torch.from_numpy(ctr)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)            # A8 #2 (int64, exact)
        if rank == 0:
            np.save(out_path, np.concatenate([rng.numpy(), np.array(caps, dtype=np.int64), t.numpy().ravel()]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["C2", "C1"])
def test_two_rank_partition_and_reduction(tmp_path, kind):
    O.build()
    out = str(tmp_path / "r0.npy")
    mp.spawn(_worker, args=(2, _free_port(), kind, out), nprocs=2, join=True)
    got = np.load(out)
    d, pc = _trace(kind)
    o = O.Oracle(d, pc)
    lo = max(o.sweep_range(w)[0] for w in range(d.n_nodes))
    hi = max(o.sweep_range(w)[1] for w in range(d.n_nodes))
    assert list(got[:2]) == [lo, hi]
    caps = sweep_caps(lo, hi, 5)
    assert list(got[2:2 + len(caps)]) == caps
    ref = o.replay_many(7, caps)
    assert np.array_equal(got[2 + len(caps):].reshape(ref.shape), ref)


@pytest.mark.parametrize("n_nodes,world", [(8, 2), (16, 4), (16, 8), (32, 8), (3, 2), (1, 2)])
def test_node_ownership_is_a_partition(n_nodes, world):
    seen = []
    for r in range(world):
        seen += owned_nodes(n_nodes, r, world)
    assert sorted(seen) == list(range(n_nodes))
