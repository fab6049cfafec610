#!/usr/bin/env python
"""Benchmark of the SAGA hot path on B200 (BASELINE.json metric: trace accesses/sec of the whole
AEG score + evict + replay and Belady pipeline; achieved HBM GB/s of the dominant kernel).

One step = one pass of every §8(a) row over one synthetic trace: saga_load_trace (A1 validate,
A2 placement, A3 streams) -> saga_belady_next_use per owned node (A4) -> W_lo/W_hi all-reduce
(A8) -> capacity sweep -> saga_replay AEG + BELADY x caps x nodes (A5-A7) -> counter all-reduce
(A8).  value = access-replays (sum over policies x caps x nodes of the node's stream length)
per second, max over ranks, inputs resident in HBM; e2e = the same through the public API from
pinned host buffers with the H2D copy of the trace and the D2H read of the counters timed.

At N > 1 GPUs the default is `--shard trials`: rank r replays its own seeded trial of the workload
(seed = the config's seed + 1000 r; rank 0 is the canonical trace) -- independent problems, so the
per-GPU work is fixed (weak scaling) -- and the per-trial counter tensors are summed over ranks by
the NCCL all-reduce of A8 every step (the paper averages over seeds).  `--shard nodes` instead
splits ONE trace by cache node (w mod R) with the W_lo/W_hi max-all-reduce and the counter
sum-all-reduce (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--shard trials|nodes] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# steps in flight use one stream each; with the default 8 hardware work queues two of torch's pool
# streams can share a queue, which serialises one step's kernels behind the other's placement
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "trace accesses/sec (AEG score+evict+replay, Bélády); HBM GB/s vs B200 peak"
UNIT = "access-replays/s"
PROF_NAMES = ["load", "place", "expand", "sort", "segscan", "epoch_stats", "replay", "score", "select", "pattern"]
WORKLOADS = {
    "C1": "tiny trace: 8 sessions x 10 calls, 1 node, 64 KV blocks",
    "C2": "SWE-bench-shaped: 2000 sessions, 10-100 calls/task, 16-token blocks, 8 nodes, 8+1 caps",
    "C3": "WebArena-shaped: 5000 sessions, branching AEG, 16 nodes, 8+1 caps",
    "C4": "64-GPU cluster: 20k sessions, affinity + work stealing, 16 nodes, 32 caps",
    "C5": "multi-tenant: 100k sessions, 32 nodes, 32 caps",
}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms; the reported samples are those
    taken during the timed region (begin() .. end()).  The sampler is started before the warm-up,
    so nvidia-smi's own start-up (NVML init, ~1 s of driver work) stays out of the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def begin(self):
        self.t0 = time.perf_counter()

    def end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.t0 is not None:
            t1 = self.t1 if self.t1 is not None else float("inf")
            inside = [x for x in lines if self.t0 <= x[0] <= t1 + 0.2]
            lines = inside or [x for x in lines if x[0] >= self.t0][:1]
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def sweep_for(name):
    from gen import N_SWEEP, PHYSICAL_CAP, sweep_caps
    base = name.split("_")[0]
    return lambda lo, hi: sweep_caps(lo, hi, N_SWEEP.get(base, 8), PHYSICAL_CAP.get(base))


def replay_bytes_per_access(policy_mask):
    """Algorithmic bytes per access-replay of the replay kernel (12 fused / 20
    unfused): the per-position words it streams for each record -- local id|flags, unit|kind and
    next use (12 B, BELADY); AEG / EVICT_ALL / LRU also read the previous occurrence and its unit
    (20 B).  Averaged over the policies of the mask (each policy replays every access once)."""
    pols = [b for b in (1, 2, 4, 8, 16) if policy_mask & b]
    return sum(12 if b == 2 else 20 for b in pols) / max(1, len(pols))


def algorithmic_bytes(cat, n_access, n_replay_access, n_calls, key_bits, policy_mask=3):
    """Algorithmic HBM bytes per step of each kernel family (DESIGN.md §6 "Kernels, rooflines")."""
    passes = max(1, (key_bits + 7) // 8)
    return {
        "sort": n_access * (4 + 12 + 16 * (passes - 1)),     # histogram read + pass 1 + later passes
        "segscan": n_access * 20,                            # sorted (key, pos) read + next/prev/lid scattered
        "epoch_stats": n_access * 16,                         # next, prev, lid read + lid|flags written
        "replay": n_replay_access * replay_bytes_per_access(policy_mask),
        "expand": n_access * 4,                               # stream write
        "place": n_calls * 40,
        "load": n_calls * 40,
    }.get(cat, 0)


def input_bytes_per_launch(cat, n_access):
    """Bytes a launch of the kernel family reads as its main input (compared with the L2 size)."""
    return {"sort": n_access * 8, "segscan": n_access * 8, "epoch_stats": n_access * 12, "expand": n_access * 4,
            "replay": n_access * 20}.get(cat)


def bulk_score_select(t, desc, stream, dev, reps=5, n_seg=1024, seg_len=32768, k_frac=0.01):
    """A5 / A6 in bulk on a C5-shaped snapshot -- n_seg segments of seg_len
    candidates (runs of consecutive local ids, i.e. runs of one session's blocks), inputs >> L2,
    k = 1 % per segment.  Returns per-kernel ms and algorithmic GB/s:
    AEG score 24 B/candidate (lid 4 + t_last 8 + owner 4 -> key 8), BELADY key 16 B (lid 4 + nu 4
    -> key 8), select 8 B/candidate (+ 4 B per victim written)."""
    import torch
    from paper_2605_00528_b200 import saga
    nl = t.info(0)[1]
    if nl < seg_len + 1:
        return None
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    n = n_seg * seg_len
    starts = torch.randint(0, nl - seg_len, (n_seg, 1), generator=g, device=dev, dtype=torch.int64)
    lid = (starts + torch.arange(seg_len, device=dev, dtype=torch.int64)).reshape(-1).to(torch.int32)
    e_last = int(desc.call_t_us.max()) // 100_000 + 1
    Te = e_last * 100_000
    t_last = Te - torch.randint(0, 60_000_000, (n,), generator=g, device=dev, dtype=torch.int64)
    nu = torch.randint(0, 2 ** 31, (n,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    i32 = lambda x: torch.full((n_seg,), x, dtype=torch.int32, device=dev)
    off = torch.arange(0, n + 1, seg_len, dtype=torch.int64, device=dev)
    batch = dict(seg_node=i32(0), seg_epoch=i32(e_last), seg_occ=i32(seg_len), seg_cap=i32(seg_len), seg_act=i32(1),
                 seg_off=off, cand_lid=lid, cand_t_last=t_last, cand_nu=nu)
    key = torch.empty(n, dtype=torch.int64, device=dev)
    kk = max(1, int(seg_len * k_frac))
    kreq = torch.full((n_seg,), kk, dtype=torch.int32, device=dev)
    oo = torch.arange(0, n_seg * kk + 1, kk, dtype=torch.int64, device=dev)
    vic = torch.empty(n_seg * kk, dtype=torch.int32, device=dev)
    out = {}

    def timed(fn):
        with torch.cuda.stream(stream):
            fn()
            stream.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ms = timed(lambda: t.aeg_score(batch, {}, key, None, policy=saga.POLICY_AEG))
    out["score_aeg"] = {"ms": ms, "bytes_per_candidate": 24, "algorithmic_gb_s": n * 24 / (ms / 1e3) / 1e9}
    ms = timed(lambda: t.aeg_score(batch, {}, key, None, policy=saga.POLICY_BELADY))
    out["score_belady"] = {"ms": ms, "bytes_per_candidate": 16, "algorithmic_gb_s": n * 16 / (ms / 1e3) / 1e9}
    t.aeg_score(batch, {}, key, None, policy=saga.POLICY_AEG)
    ms = timed(lambda: saga.evict_select(key, off, kreq, oo, vic, stream=stream))
    out["select"] = {"ms": ms, "bytes_per_candidate": 8,
                     "algorithmic_gb_s": (n * 8 + n_seg * kk * 4) / (ms / 1e3) / 1e9}
    out["snapshot"] = f"{n_seg} segments x {seg_len} candidates (runs of consecutive local ids), k = {kk}"
    return out


def f3_pattern(stream, dev, reps=5, config="C5"):
    """SURVEY §8(f) F3 on the largest config (6.4 M calls): saga_pattern_infer with the generator's
    tool labels, half the sessions held out.  Algorithmic bytes (DESIGN.md §6 F3): every call is
    read by exactly one of the two passes, sc_call 4 + label 4 = 8 B per call; per session role
    1 x 2 passes + type 2 + sc_off 4 + call_is_last 1 = 9 B."""
    import numpy as np
    import torch
    from gen import TOOL_LABELS, pattern_labels, pattern_roles, place_cfg_for
    from paper_2605_00528_b200 import saga
    d = _big_trace(config)
    t = saga.Trace(d, place_cfg_for(d), stream=stream, defer_expand=True)
    lab = torch.from_numpy(pattern_labels(d).view(np.int32)).to(dev)
    role = torch.from_numpy(pattern_roles(d)).to(dev)
    L = len(TOOL_LABELS)
    import ctypes as C
    with torch.cuda.stream(stream):
        out = t.pattern_infer(lab, L, role)
        stream.synchronize()
        saga.lib.saga_profile_enable(1)
        saga.lib.saga_profile_read(None, None)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            out = t.pattern_infer(lab, L, role)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pm = (C.c_double * len(PROF_NAMES))()
    pn = (C.c_uint64 * len(PROF_NAMES))()
    saga.lib.saga_profile_read(pm, pn)
    saga.lib.saga_profile_enable(0)
    k_ms = pm[PROF_NAMES.index("pattern")] / reps  # device time of the three kernels
    ev = out["eval"].cpu().numpy()
    t.free()
    n = d.n_calls
    nbytes = 8 * n + 9 * d.n_sessions
    return {"config": config, "calls": n, "ms_call": ms, "ms": k_ms, "calls_per_s": n / (ms / 1e3), "bytes": nbytes,
            "algorithmic_gb_s": nbytes / (k_ms / 1e3) / 1e9,
            "held_out_accuracy": float(ev[:, 2].sum()) / max(1, int(ev[:, 0].sum())),
            "note": "ms / GB/s: device time of the three kernels (CUDA events around them); ms_call: the whole "
                    "API call incl. memsets and its one sync (label check readback)"}


_BIG = {}


def _big_trace(config):
    """the generated trace of a large config, generated once per process (F3 / F4 legs)"""
    from gen import make
    if config not in _BIG:
        _BIG[config] = make(config)
    return _BIG[config]


def f4_tool_stats(stream, dev, reps=3, config="C5"):
    """SURVEY §8(f) F4 online statistics on the largest config (6.4 M calls): saga_tool_stats with
    the generator's tool labels (window 256, p95, 64-term EMA).  Reports calls/s; the kernels'
    work is dominated by the per-call window select (up to 256 latencies per call, re-read from
    L1/L2 by consecutive calls of a tool), so no HBM fraction is claimed."""
    import numpy as np
    import torch
    import ctypes as C
    from gen import TOOL_LABELS, pattern_labels, place_cfg_for
    from paper_2605_00528_b200 import saga
    d = _big_trace(config)
    t = saga.Trace(d, place_cfg_for(d), stream=stream, defer_expand=True)
    lab = torch.from_numpy(pattern_labels(d).view(np.int32)).to(dev)
    L = len(TOOL_LABELS)
    with torch.cuda.stream(stream):
        t.tool_stats(lab, L)
        stream.synchronize()
        saga.lib.saga_profile_enable(1)
        saga.lib.saga_profile_read(None, None)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ttl, obs = t.tool_stats(lab, L)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pm = (C.c_double * len(PROF_NAMES))()
    pn = (C.c_uint64 * len(PROF_NAMES))()
    saga.lib.saga_profile_read(pm, pn)
    saga.lib.saga_profile_enable(0)
    k_ms = (pm[PROF_NAMES.index("pattern")] + pm[PROF_NAMES.index("sort")]) / reps
    changed = float((ttl.cpu().numpy() != np.asarray(d.node_ttl_base_us)[np.asarray(d.call_aeg_node)]).mean())
    t.free()
    return {"config": config, "calls": d.n_calls, "ms_call": ms, "ms": k_ms, "calls_per_s": d.n_calls / (k_ms / 1e3),
            "frac_calls_ttl_changed": changed,
            "note": "ms: device time of the sample, sort, gather and per-call select kernels; ms_call: the API call"}


def run_reference(args):
    """--impl reference: the CPU oracle (oracle/), as it stands, on a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from gen import make, place_cfg_for
    from oracle import oracle as O
    O.build()
    desc = make(args.config, n_sessions=args.n_sessions)
    pc = place_cfg_for(desc)
    nthreads = os.cpu_count() or 1
    times, reps = [], 0
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        o = O.Oracle(desc, pc)
        lo, hi = 0, 0
        for w in range(desc.n_nodes):
            a, b = o.sweep_range(w) if w == 0 else (0, 0)
            lo, hi = max(lo, a), max(hi, b)
        caps = sweep_for(args.config)(lo, hi)
        cap = [caps[len(caps) // 2]]
        ctr = o.replay_many(3, cap, nodes=[0], nthreads=nthreads)
        dt = time.perf_counter() - t0
        reps = int(ctr[:, :, 0, 0].sum())
        if i >= args.warmup:
            times.append(dt)
        del o
    sec = statistics.median(times)
    v = reps / sec
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64/fp32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOADS.get(args.config, '')}",
                       "sample": f"node 0, AEG+BELADY at capacity {cap[0]}, incl. oracle placement/expansion and node-0 next use"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": f"{args.config} node 0, 2 policies x 1 capacity ({reps} access-replays/step)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(desc, pc, caps, nthreads):
    """Oracle timed on a bounded sample: full oracle build (placement, streams) + next use of every
    node + one replay per (node, policy) at the middle capacity, on every host thread; then node 0's
    two replays again on ONE thread (the per-core rate)."""
    from oracle import oracle as O
    O.build()
    t0 = time.perf_counter()
    o = O.Oracle(desc, pc)
    cap = [caps[len(caps) // 2]]
    ctr = o.replay_many(3, cap, nthreads=nthreads)
    dt = time.perf_counter() - t0
    reps = int(ctr[:, :, :, 0].sum())
    t1 = time.perf_counter()
    c1 = o.replay_many(3, cap, nodes=[0], nthreads=1)
    dt1 = time.perf_counter() - t1
    reps1 = int(c1[:, :, 0, 0].sum())
    return {"value": reps / dt, "unit": UNIT, "cores": nthreads, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{desc.name}: oracle build + all {desc.n_nodes} nodes x AEG+BELADY at capacity {cap[0]} "
                      f"({reps} access-replays in {dt:.1f} s)",
            "single_thread": {"value": reps1 / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"node 0 x AEG+BELADY at capacity {cap[0]} ({reps1} access-replays in {dt1:.1f} s)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n-sessions", type=int, default=None)
    ap.add_argument("--impl", default="saga", choices=["saga", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bulk", action="store_true")
    ap.add_argument("--shard", default=None, choices=["trials", "nodes"])
    ap.add_argument("--inflight", type=int, default=None,
                    help="independent steps in flight on separate streams (default 3 at N=1; 2 + 2R node-sharded, <= 12)")
    ap.add_argument("--overlap", action="store_true",
                    help="overlap steps even above the default size threshold (keeps inflight expanded traces resident)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="chain each step's expansion to the previous step's finished replay")
    ap.add_argument("--range-nccl", action="store_true",
                    help="N > 1: all-reduce (W_lo, W_hi) with the library's NCCL communicator instead of a host (gloo) exchange")
    ap.add_argument("--gate", default="queued", choices=["queued", "none"],
                    help="with overlap: a step's expansion starts after the previous step's replay is queued "
                         "(queued) or right after its own placement (none)")
    ap.add_argument("--stream-priority", type=int, default=-1,
                    help="priority of the step streams (load, placement, expansion, sort); the library runs "
                         "each replay kernel on its own lowest-priority stream (0: everything equal)")
    ap.add_argument("--policy-mask", type=int, default=3,
                    help="1 AEG, 2 BELADY, 4 EVICT_ALL, 8 LRU, 16 LRU+Prefix (default 3: the metric's pair)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from gen import make, place_cfg_for
    from paper_2605_00528_b200 import pipeline, saga

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    # N > 1 default: SURVEY §8(e)'s partition -- rank r owns cache nodes w mod R of the one trace
    # (placement replicated, (W_lo, W_hi) max- and counters sum-all-reduced over NCCL: counters
    # bit-identical to N = 1).  --shard trials runs an independent seeded trial per rank instead.
    shard = args.shard or "nodes"
    trials = shard == "trials"
    seed = None
    if trials and rank > 0 and args.config != "C1":
        import inspect
        from gen import CONFIGS
        seed = inspect.signature(CONFIGS[args.config]).parameters["seed"].default + 1000 * rank
    desc = make(args.config, n_sessions=args.n_sessions, seed=seed)
    pc = place_cfg_for(desc)
    rcfg = dict(policy_mask=args.policy_mask)
    caps_fn = sweep_for(args.config)
    shard_caps = (not trials) and desc.n_nodes == 1 and world > 1
    # Steps in flight.  "overlap": a step's expansion / next use start as soon as the previous
    # step's replay kernel is queued (they fill the SMs its short items free), which
    # keeps up to inflight expanded traces resident -- only when they fit in ~60 % of the device
    # memory at ~48 B per owned access (node arrays + sort scratch): C1-C4; C5 chains a step's
    # expansion to the previous step's freed trace.
    # node-sharded ranks hold 1/R of the replay items but the same per-step placement and critical
    # path (one item's epoch chain), so more steps are kept in flight as R grows
    # (latency of one step ~ 2.4x a rank's SM-time per step at C2 when R ranks split the items)
    n_over = min(12, 3 if world == 1 or shard != "nodes" else 2 + 2 * world)
    owned_acc = desc.n_accesses / (world if shard == "nodes" and world > 1 else 1)
    fits = n_over * 48 * owned_acc < 0.6 * torch.cuda.get_device_properties(dev).total_memory
    overlap = (fits or args.overlap) and not args.no_overlap
    inflight = max(1, args.inflight or (n_over if overlap else 2))
    inflight = min(inflight, 12)
    # one stream, trace handle and communicator per in-flight step (see run_steps)
    comms = [saga.Comm(rank, world, local) for _ in range(inflight)] if world > 1 else [None] * inflight
    # (W_lo, W_hi) max over ranks as a host exchange (gloo, one group per step stream): the two values
    # are host-side after saga_sweep_range, and an NCCL kernel would wait for an SM held by replays
    range_groups = [dist.new_group(backend="gloo") for _ in range(inflight)] \
        if world > 1 and not args.range_nccl else [None] * inflight

    def range_reduce_for(i):
        if range_groups[i] is None:
            return None

        def red(wlo, whi):
            x = torch.tensor([wlo, whi], dtype=torch.int64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX, group=range_groups[i])
            return int(x[0]), int(x[1])
        return red
    comm = comms[0]
    p_rank, p_world = (0, 1) if trials else (rank, world)
    # high-priority step streams: the next step's short kernels take SMs freed by a running replay
    # ahead of another replay's queued CTAs, so a replay is always ready to fill the machine
    streams = [torch.cuda.Stream(device=dev, priority=args.stream_priority) for _ in range(inflight)]
    stream = streams[0]
    host_pinned = saga.HostDesc(desc, pinned=True)
    # device-resident descriptor for `value` (the library deep-copies it device-to-device)
    dev_keep = []
    dptrs = []
    for name, dt in saga.DESC_ARRAYS:
        if name in saga.OPTIONAL_ARRAYS and getattr(desc, name, None) is None:
            dptrs.append(None)
            continue
        a = np.ascontiguousarray(getattr(desc, name), dtype=dt)
        t = torch.from_numpy(a.view(np.uint8).copy() if a.size else np.zeros(1, np.uint8)).to(dev)
        dev_keep.append(t)
        dptrs.append(t.data_ptr())

    class DevDesc:
        pass
    dd = DevDesc()
    dd.keep = dev_keep
    dd.c = saga.TraceDescC(desc.n_calls, desc.n_sessions, desc.n_types, desc.n_aeg_nodes, desc.n_edges, desc.n_ranges,
                           desc.n_blocks, desc.n_nodes, desc.block_tokens, *dptrs)
    counters = [None] * inflight
    import threading
    order = {"cv": threading.Condition(), "done": {}}
    timeline = [] if os.environ.get("SAGA_TIMELINE") else None

    def mark(st, what, j):  # SAGA_TIMELINE=1: device-side timeline of the steps, printed to stderr
        if timeline is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            timeline.append((what, j, e, time.perf_counter()))

    def step(host, i=0, j=None):
        """One step on stream i.  With steps in flight (j = step index), step j's expansion,
        next use and replay start after step j-1's trace was replayed and freed (so at most one
        expanded trace is resident: C5's is ~90 GB), while its load and placement (a single warp
        on one SM) run beside that replay.  Every step does all of its work."""
        s_ = streams[i]
        before = after = None
        if j is not None and inflight > 1:
            def before(st):
                if j == 0 or (overlap and args.gate == "none"):
                    mark(st, "go", j)
                    return
                with order["cv"]:
                    if overlap:  # only after step j-1's replay kernel is queued (its CTAs take the SMs first)
                        order["cv"].wait_for(lambda: (j - 1) in order["launched"] or order.get("error"))
                    else:
                        order["cv"].wait_for(lambda: (j - 1) in order["done"] or order.get("error"))
                    if order.get("error"):
                        raise RuntimeError("another in-flight step failed")
                    ev = None if overlap else order["done"][j - 1]
                mark(st, "placed", j)
                if ev is not None:
                    st.wait_event(ev)
                mark(st, "go", j)

            def after(st):
                mark(st, "replayed", j)
                ev = torch.cuda.Event()
                ev.record(st)
                with order["cv"]:
                    order["ev"][j] = ev  # published once the trace is freed (run_steps.worker)
                    order["launched"].add(j)
                    order["cv"].notify_all()
        mark(s_, "start", j)
        with torch.cuda.stream(s_):
            t, caps, ctr = pipeline.run_step(desc, pc, rcfg, caps_fn, rank=p_rank, world=p_world,
                                             comm=None if trials else comms[i], device=local, stream=s_, host=host,
                                             counters=counters[i], shard_caps=shard_caps,
                                             before_expand=before, after_replay=after,
                                             mark=(lambda st, w: mark(st, w, j)) if timeline is not None else None,
                                             range_comm=comms[i] if trials else None, replay_wait=False,
                                             range_host_reduce=range_reduce_for(i))
            if trials and comms[i] is not None:  # A8: combine the per-trial counters over ranks
                comms[i].allreduce(ctr, op=0, stream=t.stream)
        counters[i] = ctr
        return t, caps, ctr

    def run_steps(k, host, d2h=None):
        """k steps, step j on stream j mod inflight (one host thread per stream).  Device-timed:
        every stream starts after ev0 on streams[0], which waits for all of them before ev1.
        Returns (ms per step, (caps, counters) of the last step on stream 0)."""
        import concurrent.futures as cf
        with order["cv"]:
            order["done"] = {}
            order["ev"] = {}
            order["launched"] = set()
            order["error"] = None
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(streams[0])
        order["h0"] = time.perf_counter()
        for s_ in streams[1:]:
            s_.wait_event(ev0)

        def worker(i):
            torch.cuda.set_device(local)
            last = None
            try:
                for j in range(i, k, inflight):
                    t, caps, ctr = step(host, i, j)
                    if d2h is not None:
                        d2h(i, ctr)
                    t.replay_wait()  # the step's replay is done and passed its internal checks
                    t.free()
                    with order["cv"]:  # step j's trace is gone: step j+1 may expand
                        order["done"][j] = order["ev"].get(j)
                        order["cv"].notify_all()
                    last = (caps, ctr)
            except BaseException as exc:  # wake the other stream's thread instead of leaving it waiting
                with order["cv"]:
                    order["error"] = exc
                    order["cv"].notify_all()
                raise
            return last

        if inflight == 1:
            outs = [worker(0)]
        else:
            with cf.ThreadPoolExecutor(inflight) as ex:
                outs = list(ex.map(worker, range(inflight)))
        for s_ in streams[1:]:
            e = torch.cuda.Event()
            e.record(s_)
            streams[0].wait_event(e)
        ev1.record(streams[0])
        torch.cuda.synchronize()
        if timeline:
            for what, j, e, h in timeline:
                print(f"timeline step {j} {what:9s} dev {ev0.elapsed_time(e):9.2f} ms  host {1e3 * (h - order['h0']):9.2f} ms",
                      file=sys.stderr)
            timeline.clear()
        return ev0.elapsed_time(ev1) / k, outs[0]

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    # ---- warm-up ----
    sampler = ClockSampler(local)
    sampler.start()
    run_steps(max(args.warmup, inflight), dd)
    # latency of one step alone (nothing else in flight)
    lat_ms, _ = run_steps(1, dd)
    # per-step work (access-replays over all ranks)
    t, caps, ctr = step(dd)
    stream.synchronize()
    mine = (list(range(desc.n_nodes)) if trials else pipeline.owned_nodes(desc.n_nodes, rank, world)) \
        if not shard_caps else [0]
    n_acc_local = sum(t.info(w)[0] for w in mine)
    n_pol = bin(args.policy_mask & 31).count("1")
    if shard_caps:
        n_caps_local = len([i for i in range(len(caps)) if i % world == rank])
        rep_local = n_acc_local * n_pol * n_caps_local
    else:
        rep_local = n_acc_local * n_pol * len(caps)
    t.free()
    tot = torch.tensor([rep_local, n_acc_local if not shard_caps or rank == 0 else 0], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    replay_accesses, n_access = int(tot[0]), int(tot[1])

    # ---- timed region (device-resident inputs) ----
    l0 = saga.kernel_launches()
    barrier()
    torch.cuda.synchronize()
    sampler.begin()
    ms, (caps, ctr) = run_steps(args.steps, dd)
    barrier()
    sampler.end()
    launches = saga.kernel_launches() - l0
    clocks = sampler.stop()
    # per-kernel-family device times: the same steps again, one at a time, with the library's event
    # profile on (CUDA events around every kernel family; kept out of the timed region above)
    import ctypes as C
    prof_steps = args.steps if desc.n_calls < 1_000_000 else 1
    saga.lib.saga_profile_enable(1)
    saga.lib.saga_profile_read(None, None)
    ms_prof = 0.0
    for _ in range(prof_steps):  # one step at a time: a kernel family's events must not span waits for SMs
        ms1, _ = run_steps(1, dd)
        ms_prof += ms1 / prof_steps
    pm = (C.c_double * len(PROF_NAMES))()
    pn = (C.c_uint64 * len(PROF_NAMES))()
    saga.lib.saga_profile_read(pm, pn)
    saga.lib.saga_profile_enable(0)
    mt = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
    ms = float(mt[0])
    value = replay_accesses / (ms / 1e3)
    counters_host = ctr.cpu().numpy()

    # ---- e2e: public API from pinned host buffers, H2D + D2H inside the timed region ----
    e2e = None
    if not args.no_e2e:
        barrier()
        torch.cuda.synchronize()
        out_host = [torch.empty(tuple(ctr.shape), dtype=torch.int64, pin_memory=True) for _ in range(inflight)]

        wrote = set()

        def d2h(i, c2):  # the step's result back to the host, inside the timed region
            with torch.cuda.stream(streams[i]):
                out_host[i].copy_(c2, non_blocking=True)
            streams[i].synchronize()
            wrote.add(i)

        ems, _ = run_steps(args.steps, host_pinned, d2h=d2h)
        barrier()
        et = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        ems = float(et[0])
        e2e = {"value": replay_accesses / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": host_pinned.nbytes,
               "d2h_bytes_per_step": int(out_host[0].numel() * 8), "ms_per_step": ems}
        for i in sorted(wrote):  # (streams without a step when steps < steps in flight hold nothing)
            assert np.array_equal(out_host[i].numpy(), counters_host), "e2e counters differ from the device-resident run"

    # ---- roofline of the dominant kernel family (per-launch, CUDA events on the launching stream) ----
    peak, peak_kind = hbm_peak()
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 0)) or None  # cudaDevAttrL2CacheSize
    ncu_cfg = {}
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):  # ncu dram__bytes_read + write per launch, by config and kernel family
        try:
            ncu_cfg = json.load(open(tfile)).get(args.config, {}) if args.policy_mask == 3 else {}
        except Exception:
            ncu_cfg = {}
    key_bits = int(np.ceil(np.log2(max(desc.n_blocks, 2))))
    kernels = {}
    for i, nm in enumerate(PROF_NAMES):
        if pn[i] == 0:
            continue
        ms_k = pm[i] / prof_steps
        n_loc = n_access / max(world, 1) if not shard_caps else n_access
        byt = algorithmic_bytes(nm, n_loc, replay_accesses / max(world, 1), desc.n_calls, key_bits,
                                args.policy_mask)  # per rank
        ib = input_bytes_per_launch(nm, n_loc)
        kernels[nm] = {"ms_per_step": ms_k, "launches_per_step": pn[i] / prof_steps, "share": ms_k / ms_prof,
                       "algorithmic_gb_s": (byt / (ms_k / 1e3) / 1e9) if byt and ms_k > 0 else None,
                       "algorithmic_bytes_per_step": byt or None,
                       "input_over_l2": (ib / l2_bytes) if ib and l2_bytes else None}
        tr = ncu_cfg.get(nm)
        if tr and byt:
            kernels[nm]["ncu_dram_bytes_per_step"] = tr * pn[i] / prof_steps
            kernels[nm]["traffic_over_algorithmic"] = tr * (pn[i] / prof_steps) / byt
    dom = max((k for k in kernels if k in ("sort", "segscan", "epoch_stats", "replay", "expand")),
              key=lambda k: kernels[k]["ms_per_step"], default=None)
    traffic = ncu_cfg.get(dom) if dom else None
    tinfo = ncu_cfg
    roof = None
    if dom:
        ach = kernels[dom]["algorithmic_gb_s"] or 0.0
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "peak_source": peak_kind,
                "note": "achieved = algorithmic bytes of the kernel family / its CUDA-event time per step"}
        inst = tinfo.get(dom + "_warp_inst")
        if inst:
            # the replay is issue/latency-bound: its warp-instruction rate against the SM issue peak
            # (148 SMs x 4 schedulers x 1 instruction per clock at the sampled SM clock), DESIGN.md §6
            ms_k = kernels[dom]["ms_per_step"]
            mhz = clocks.get("sm_mhz") or 1965.0
            peak_i = 148 * 4 * mhz * 1e6 / 1e9
            ach_i = inst / (ms_k / 1e3) / 1e9
            roof["issue"] = {"achieved": ach_i, "peak": peak_i, "unit": "G warp-inst/s", "frac": ach_i / peak_i,
                             "warp_inst_per_launch": inst, "source": "ncu smsp__inst_executed.sum of one launch"}

    bulk = pat = f4 = None
    if world == 1 and not args.no_bulk:  # single process: no collective may be issued by one rank
        with torch.cuda.stream(stream):
            t_b, _, _ = pipeline.run_step(desc, pc, rcfg, caps_fn, device=local, stream=stream, host=dd)
        stream.synchronize()
        bulk = bulk_score_select(t_b, desc, stream, dev)
        t_b.free()
        if bulk:
            n_cand = 1024 * 32768
            for kname, kv in bulk.items():
                if isinstance(kv, dict):
                    kv["frac"] = kv["algorithmic_gb_s"] / peak
                    kv["input_over_l2"] = (n_cand * (12 if kname == "score_aeg" else 8) / l2_bytes) if l2_bytes else None
                    tr = ncu_cfg.get(kname)  # ncu DRAM bytes of one launch of the same snapshot
                    if tr:
                        kv["ncu_dram_bytes"] = tr
                        kv["traffic_over_algorithmic"] = tr / (n_cand * kv["bytes_per_candidate"])
        pat = f3_pattern(stream, dev)
        pat["frac"] = pat["algorithmic_gb_s"] / peak
        f4 = f4_tool_stats(stream, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(desc, pc, caps, os.cpu_count() or 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if trials and world > 1 else "strong",
            "vs_baseline": None,
            "dtype": "int64/fp32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOADS.get(args.config, '')}", "trace": desc.name,
                       "nodes": desc.n_nodes, "caps": caps, "policies": [nm for b, nm in ((1, "AEG"), (2, "BELADY"), (4, "EVICT_ALL"), (8, "LRU"),
                                                                  (16, "LRU_PREFIX")) if args.policy_mask & b],
                       "trace_accesses": n_access, "access_replays_per_step": replay_accesses,
                       "trace_accesses_per_s": n_access / (ms / 1e3),
                       "l2_bytes": l2_bytes,
                       "l2": ("L2 not flushed between steps: every step loads a new trace and its per-access inputs "
                              "exceed L2 (kernels.*.input_over_l2 = main input bytes of one launch / L2 size)"),
                       "steps_in_flight": inflight, "overlap": overlap, "step_latency_ms": lat_ms,
                       "sharding": ("independent trials (seed + 1000 r), counters all-reduced" if trials and world > 1
                                    else ("capacity points" if shard_caps else "cache nodes w mod R"))},
            "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "roofline": roof, "cpu_baseline": cpu, "kernels": kernels, "bulk_score_select": bulk, "f3_pattern": pat, "f4_tool_stats": f4,
            "counters_checksum": int(np.bitwise_xor.reduce(counters_host.reshape(-1).view(np.uint64))),
        }
        print(json.dumps(line), flush=True)
    for c_ in comms:
        if c_ is not None:
            c_.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
