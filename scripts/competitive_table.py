"""Regeneration ratio of every policy against epoch-Belady on the synthetic traces (GPU path).

regen ratio = (MISSES - COMPULSORY_GLOBAL)_policy / (MISSES - COMPULSORY_GLOBAL)_BELADY, summed over nodes, per
capacity of the sweep (the analogue of the paper's competitive ratio, P:882 and
Table tab:competitive P:910-923).  Diagnostic only: the paper's 1.31 / 1.86 / 2.84 were measured
on production traces with a serving system in the loop.

  python scripts/competitive_table.py [C2 C3 ...]  -> prints a markdown table (one row per config
  and capacity) and writes profiles/competitive_<cfg>.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import make, place_cfg_for, sweep_caps, N_SWEEP, PHYSICAL_CAP  # noqa: E402
from paper_2605_00528_b200 import pipeline, saga  # noqa: E402

POLS = ["AEG (WA-LRU)", "BELADY", "EVICT_ALL", "LRU", "LRU+Prefix"]


def main(cfgs):
    torch.cuda.set_device(0)
    print("| config | capacity | " + " | ".join(p for p in POLS if p != "BELADY") + " |")
    print("|---|---|" + "---|" * (len(POLS) - 1))
    for name in cfgs:
        d = make(name)
        pc = place_cfg_for(d)
        caps_fn = lambda lo, hi: sweep_caps(lo, hi, N_SWEEP.get(name, 8), PHYSICAL_CAP.get(name))
        t, caps, ctr = pipeline.run_step(d, pc, dict(policy_mask=31), caps_fn)
        torch.cuda.synchronize()
        c = ctr.cpu().numpy()
        regen = (c[:, :, :, saga.CI["MISSES"]] - c[:, :, :, saga.CI["COMPULSORY_GLOBAL"]]).sum(axis=2)
        out = {"config": name, "caps": caps, "policies": POLS, "regen_blocks": regen.tolist()}
        for ci, cap in enumerate(caps):
            base = max(int(regen[1, ci]), 1)
            cells = [f"{regen[pi, ci] / base:.2f}" for pi in range(len(POLS)) if pi != 1]
            print(f"| {name} | {cap} | " + " | ".join(cells) + " |")
        with open(os.path.join(ROOT, "profiles", f"competitive_{name}.json"), "w") as f:
            json.dump(out, f)
        t.free()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3"])
