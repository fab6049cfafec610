"""N>1 on real GPUs: one process per GPU over NCCL through the library's own
communicator (saga_comm_init / saga_allreduce_counters, A8).  Each rank owns the cache nodes
w mod R of ONE trace, places it (replicated), sorts / scans / replays only its nodes; the
(W_lo, W_hi) maxima and the counter tensor are all-reduced (max, then sum).  Rank 0 checks the
combined counters against a single-process run of the same step and against the CPU oracle, bit
for bit.  Needs >= 2 GPUs (skipped otherwise; run with `gpurun --gpus 2`)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from gen import make, place_cfg_for, sweep_caps  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {"C2": dict(n_sessions=60, n_nodes=4), "C5": dict(n_sessions=200, n_nodes=32)}


def _worker(rank, world, port, name, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2605_00528_b200 import pipeline, saga
        d = make(name, **CASES[name])
        pc = place_cfg_for(d)
        comm = saga.Comm(rank, world, rank)
        caps_fn = lambda lo, hi: sweep_caps(lo, hi, 5)
        t, caps, ctr = pipeline.run_step(d, pc, dict(policy_mask=31), caps_fn, rank=rank, world=world, comm=comm,
                                         device=rank)
        t.stream.synchronize()
        # the max all-reduce on its own: every rank contributes its rank id
        m = torch.tensor([rank, 10 * rank], dtype=torch.int64, device=f"cuda:{rank}")
        comm.allreduce(m, op=1, stream=t.stream)
        t.stream.synchronize()
        if rank == 0:
            np.save(out_path, np.concatenate([np.array(caps, np.int64), m.cpu().numpy(), ctr.cpu().numpy().ravel()]))
        t.free()
        comm.destroy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", list(CASES))
def test_node_sharded_counters_equal_single_gpu_and_oracle(tmp_path, name):
    world = 2
    out = str(tmp_path / "r0.npy")
    mp.spawn(_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
    got = np.load(out)
    from oracle import oracle as O
    from paper_2605_00528_b200 import pipeline
    d = make(name, **CASES[name])
    pc = place_cfg_for(d)
    caps_fn = lambda lo, hi: sweep_caps(lo, hi, 5)
    t, caps, ctr = pipeline.run_step(d, pc, dict(policy_mask=31), caps_fn)
    torch.cuda.synchronize()
    one = ctr.cpu().numpy()
    nc = len(caps)
    assert list(got[:nc]) == caps
    assert list(got[nc:nc + 2]) == [world - 1, 10 * (world - 1)]
    multi = got[nc + 2:].reshape(one.shape)
    assert np.array_equal(multi, one)           # N = 2 == N = 1, every cell incl. the victim hash
    o = O.Oracle(d, pc)
    ref = o.replay_many(31, caps)
    assert np.array_equal(one, ref)
    t.free()
