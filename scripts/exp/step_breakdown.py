"""Wall-clock breakdown of one pipeline step (each API call bracketed by synchronize)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from gen import make, place_cfg_for, sweep_caps, N_SWEEP, PHYSICAL_CAP
from paper_2605_00528_b200 import saga
torch.cuda.set_device(0)
d = make(sys.argv[1] if len(sys.argv) > 1 else "C2")
pc = place_cfg_for(d)
host = saga.HostDesc(d, pinned=True)
stream = torch.cuda.Stream()
for it in range(3):
    T = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    t = saga.Trace(d, pc, stream=stream, host=host)
    torch.cuda.synchronize(); T['load'] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for w in range(d.n_nodes):
        t.next_use(w)
    torch.cuda.synchronize(); T['next_use'] = time.perf_counter() - t0
    t0 = time.perf_counter()
    lo = max(t.sweep_range(w)[0] for w in range(d.n_nodes)); hi = max(t.sweep_range(w)[1] for w in range(d.n_nodes))
    caps = sweep_caps(lo, hi, N_SWEEP.get("C2", 8), PHYSICAL_CAP.get("C2"))
    ctr = torch.zeros((2, len(caps), d.n_nodes, saga.NCOUNT), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize(); T['sweep+alloc'] = time.perf_counter() - t0
    t0 = time.perf_counter()
    t.replay(dict(policy_mask=3), caps, list(range(d.n_nodes)), ctr)
    torch.cuda.synchronize(); T['replay'] = time.perf_counter() - t0
    t0 = time.perf_counter()
    t.free()
    torch.cuda.synchronize(); T['free'] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in T.items()}, 'total', round(sum(T.values()) * 1e3, 1))
