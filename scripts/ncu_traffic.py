#!/usr/bin/env python
"""Fold an ncu --csv metrics log of scripts/profile_step.py (one step of a config) into
profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each kernel family."""
import collections
import csv
import json
import os
import sys

FAMILY = {"k_hist": "sort", "k_hist_scan": "sort", "k_onesweep": "sort", "k_segscan": "segscan",
          "k_ev_pos": "epoch_stats", "k_epoch_stats": "epoch_stats", "k_sweep": "epoch_stats",
          "k_replay": "replay", "k_score": "score_aeg", "k_key_belady": "score_belady", "k_select": "select",
          "k_fill_stream": "expand", "k_place": "place"}


def main(csv_path, config, out="profiles/ncu_traffic.json"):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        x = dict(zip(h, r))
        name = x["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].strip()
        per[(int(x["ID"]), name)][x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
    fam = collections.defaultdict(lambda: {"bytes": 0.0, "ns": 0.0, "launches": 0, "inst": 0.0})
    for (_, name), m in per.items():
        f = FAMILY.get(name)
        if f is None:
            continue
        fam[f]["bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        fam[f]["ns"] += m.get("gpu__time_duration.sum", 0)
        fam[f]["inst"] += m.get("smsp__inst_executed.sum", 0)
        fam[f]["launches"] += 1
    db = json.load(open(out)) if os.path.exists(out) else {}
    db = {k: v for k, v in db.items() if k.startswith("C")}
    cfg = {}
    bulk = {"score_aeg", "score_belady", "select"}   # per launch: the profiled command repeats these
    for f, v in fam.items():
        div = v["launches"] if f in bulk else 1          # pipeline families: per step (one step profiled)
        cfg[f] = v["bytes"] / div
        cfg[f + "_ms"] = v["ns"] / 1e6 / div
        if f == "replay" and v["inst"]:
            cfg["replay_warp_inst"] = v["inst"]
    cfg["_source"] = f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum " \
                     f"--clock-control none python scripts/profile_step.py --config {config} --bulk ({os.path.basename(csv_path)})"
    db[config] = cfg
    json.dump(db, open(out, "w"), indent=1, sort_keys=True)
    for f in sorted(fam):
        print(f"{config} {f:14s} {fam[f]['launches']:3d} launches  {fam[f]['ns'] / 1e6:9.3f} ms  {fam[f]['bytes'] / 1e9:8.3f} GB "
              f"{fam[f]['bytes'] / fam[f]['ns'] if fam[f]['ns'] else 0:8.1f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
