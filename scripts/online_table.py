"""Static per-node TTL / observation length vs the online statistics of F4 (Alg. 1 line 2).

For each config: saga_tool_stats on the generator's tool labels gives each call a TTL base (p95
of its tool's last 256 observed latencies) and an EMA of observation lengths; the trace is
reloaded with them as per-call overrides and replayed.  Reported per capacity: regenerated
blocks (MISSES - COMPULSORY_GLOBAL over nodes) of AEG, each relative to epoch-Belady of its own run.
Diagnostic only.

  python scripts/online_table.py [C2 C4]  -> markdown table, profiles/online_<cfg>.json
"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import TOOL_LABELS, make, place_cfg_for, sweep_caps, N_SWEEP, PHYSICAL_CAP, pattern_labels  # noqa: E402
from paper_2605_00528_b200 import pipeline, saga  # noqa: E402


def regen(ctr):
    c = ctr.cpu().numpy()
    return (c[:, :, :, saga.CI["MISSES"]] - c[:, :, :, saga.CI["COMPULSORY_GLOBAL"]]).sum(axis=2)


def main(cfgs):
    torch.cuda.set_device(0)
    print("| config | capacity | AEG regen / Belady, static TTL | online TTL + EMA | change | median TTL static / online (ms) |")
    print("|---|---|---|---|---|---|")
    for name in cfgs:
        d = make(name)
        pc = place_cfg_for(d)
        label = pattern_labels(d)
        t = saga.Trace(d, pc, defer_expand=True)
        ttl, obs = t.tool_stats(torch.from_numpy(label.view(np.int32)).cuda(), len(TOOL_LABELS))
        torch.cuda.synchronize()
        ttl = ttl.cpu().numpy()
        obs = obs.cpu().numpy().view(np.uint32)
        t.free()
        do = dataclasses.replace(d, call_ttl_base_us=ttl, call_obs_tokens=obs)
        caps_fn = lambda lo, hi: sweep_caps(lo, hi, N_SWEEP.get(name, 8), PHYSICAL_CAP.get(name))
        t1, caps, c1 = pipeline.run_step(d, pc, dict(policy_mask=3), caps_fn)
        r1 = regen(c1)
        t1.free()
        t2, _, c2 = pipeline.run_step(do, pc, dict(policy_mask=3), lambda lo, hi: caps)
        r2 = regen(c2)
        t2.free()
        med_s = float(np.median(np.asarray(d.node_ttl_base_us)[np.asarray(d.call_aeg_node)])) / 1e3
        med_o = float(np.median(ttl)) / 1e3
        rows = []
        for ci, cap in enumerate(caps):
            a, b = r1[0, ci] / max(int(r1[1, ci]), 1), r2[0, ci] / max(int(r2[1, ci]), 1)
            ch = (r2[0, ci] - r1[0, ci]) / max(int(r1[0, ci]), 1)
            print(f"| {name} | {cap} | {a:.3f} | {b:.3f} | {100 * ch:+.1f}% | {med_s:.0f} / {med_o:.0f} |")
            rows.append(dict(cap=cap, static=int(r1[0, ci]), online=int(r2[0, ci]), belady_static=int(r1[1, ci]),
                             belady_online=int(r2[1, ci])))
        with open(os.path.join(ROOT, "profiles", f"online_{name}.json"), "w") as f:
            json.dump(dict(config=name, median_ttl_ms_static=med_s, median_ttl_ms_online=med_o, rows=rows), f)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C4"])
