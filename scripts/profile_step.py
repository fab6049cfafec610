#!/usr/bin/env python
"""Exactly one pipeline step (A1-A8, policies AEG + BELADY, the bench's capacity sweep) of a config,
optionally followed by one launch each of the bulk score / select snapshot -- the command the ncu
traffic captures run (scripts/gpu_profile.sh), so that per-kernel DRAM bytes are per step."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--bulk", action="store_true")
    args = ap.parse_args()
    import torch
    import bench
    from gen import make, place_cfg_for
    from paper_2605_00528_b200 import pipeline
    d = make(args.config)
    pc = place_cfg_for(d)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        t, caps, ctr = pipeline.run_step(d, pc, dict(policy_mask=3), bench.sweep_for(args.config), stream=s)
    s.synchronize()
    if args.bulk:
        bench.bulk_score_select(t, d, s, torch.device("cuda", 0), reps=1)
    t.free()
    print("caps", caps, "checksum", int(ctr.cpu().numpy().view("uint64").sum()))


if __name__ == "__main__":
    main()
