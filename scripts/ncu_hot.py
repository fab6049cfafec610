#!/usr/bin/env python
"""Summarise an ncu report: headline metrics and the hottest source lines (stall samples)."""
import csv, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__block_size',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__average_warp_latency_per_inst_issued.ratio']
for row in r[2:]:
    print(row[4][:80] if len(row) > 4 else '')
    for i, name in enumerate(r[0]):
        if name in want:
            print(f"  {name:60s} {r[1][i]:>10s} {row[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; res = []
for row in csv.reader(src.splitlines()):
    if not row: continue
    if row[0] == 'File Path': cur = row[1].split('/')[-1]; continue
    if row[0] == 'Line No': hdr = row; continue
    if hdr and row[0] and row[0] != 'Function Name':
        try: samp = int(row[4])
        except Exception: continue
        d = dict(zip(hdr[4:], row[4:]))
        res.append((samp, cur, int(row[0]), row[1].strip()[:90], d.get('Instructions Executed', '0')))
tot = sum(x[0] for x in res) or 1
for x in sorted(res, reverse=True)[:n]:
    print(f"{100*x[0]/tot:5.1f}% {x[4]:>12} {x[1]}:{x[2]} {x[3]}")
