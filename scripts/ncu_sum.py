#!/usr/bin/env python
"""Summarise an ncu --csv metrics log per kernel: launches, total time, DRAM bytes, GB/s."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
d = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    x = dict(zip(h, r))
    name = x["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("saga::", "")
    d[(int(x["ID"]), name)][x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
per = collections.defaultdict(list)
for (i, n), m in sorted(d.items()):
    a = agg[n]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0)
    a[3] += m.get("dram__bytes_write.sum", 0)
    a[4] += m.get("lts__t_bytes.sum", 0)
    per[n].append((m.get("gpu__time_duration.sum", 0), m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)))
print(f"{'kernel':44s} {'n':>4s} {'ms total':>9s} {'ms/launch':>9s} {'DRAM GB/launch':>14s} {'DRAM GB/s':>9s}")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    t_ns = a[1]
    print(f"{n[:44]:44s} {a[0]:4d} {t_ns / 1e6:9.3f} {t_ns / 1e6 / a[0]:9.3f} {(a[2] + a[3]) / 1e9 / a[0]:14.4f} "
          f"{(a[2] + a[3]) / t_ns if t_ns else 0:9.1f}")
