"""Diagnostic: does one step's next-use work (stream B) run beside a long kernel on stream A?

(a) stream A: torch.cuda._sleep (a single-CTA spin kernel); (b) stream A: a trace load (placement).
Prints stream B's next-use time and the library's per-family times for each case.
"""
import ctypes as C
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen import make, place_cfg_for  # noqa: E402
from paper_2605_00528_b200 import saga  # noqa: E402

PROF = ["load", "place", "expand", "sort", "segscan", "epoch_stats", "replay", "score", "select", "pattern"]


def prof():
    pm = (C.c_double * len(PROF))()
    pn = (C.c_uint64 * len(PROF))()
    saga.lib.saga_profile_read(pm, pn)
    return {PROF[i]: round(pm[i], 2) for i in range(len(PROF)) if pn[i]}


def main():
    torch.cuda.set_device(0)
    d = make("C2")
    pc = place_cfg_for(d)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

    def fresh():
        t = saga.Trace(d, pc, owned_mask=0, stream=sb, defer_expand=True)
        torch.cuda.synchronize()
        return t

    def nextuse_on_b(t):
        saga.lib.saga_profile_enable(1)
        prof()
        t0 = time.perf_counter()
        for w in range(d.n_nodes):
            t.next_use(w)
        sb.synchronize()
        ms = 1e3 * (time.perf_counter() - t0)
        p = prof()
        saga.lib.saga_profile_enable(0)
        t.free()
        return ms, p

    for _ in range(2):
        print("alone            ", nextuse_on_b(fresh()), flush=True)
    t = fresh()
    with torch.cuda.stream(sa):
        torch.cuda._sleep(300_000_000)  # ~150 ms at 1.9 GHz
    print("beside _sleep    ", nextuse_on_b(t), flush=True)
    torch.cuda.synchronize()

    out = {}

    def load_a():
        out["t"] = saga.Trace(d, pc, owned_mask=0, stream=sa, defer_expand=True)

    t = fresh()
    th = threading.Thread(target=load_a)
    th.start()
    time.sleep(0.01)
    print("beside placement ", nextuse_on_b(t), flush=True)
    th.join()
    out["t"].free()

    # replay on B alone and beside a placement on A (SAGA_REPLAY_TRACE=1 adds per-item cycles)
    from gen import sweep_caps, N_SWEEP, PHYSICAL_CAP
    for mode in ("alone", "beside placement", "alone", "beside placement"):
        t = fresh()
        for w in range(d.n_nodes):
            t.next_use(w)
        lo = max(t.sweep_range(w)[0] for w in range(d.n_nodes))
        hi = max(t.sweep_range(w)[1] for w in range(d.n_nodes))
        caps = sweep_caps(lo, hi, N_SWEEP["C2"], PHYSICAL_CAP.get("C2"))
        ctr = torch.zeros((2, len(caps), d.n_nodes, saga.NCOUNT), dtype=torch.int64, device="cuda")
        sb.synchronize()
        if mode != "alone":
            th = threading.Thread(target=load_a)
            th.start()
            time.sleep(0.005)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sb)
        print(f"[diag] replay {mode} begin", file=sys.stderr, flush=True)
        t.replay(dict(policy_mask=3), caps, list(range(d.n_nodes)), ctr)
        e1.record(sb)
        sb.synchronize()
        print(f"replay {mode:17s} {e0.elapsed_time(e1):.1f} ms", flush=True)
        if mode != "alone":
            th.join()
            out["t"].free()
        t.free()


if __name__ == "__main__":
    main()
