#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import paper_2605_00528_b200.build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
SAGA_REPLAY_TRACE=1 timeout 900 python scripts/profile_step.py --config C5 > gpurun_out/trace_c5.log 2>&1
grep "grid" gpurun_out/trace_c5.log | head -3
python - gpurun_out/trace_c5.log <<'PY'
import re, sys, collections
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, [0.0] * 8])
for l in open(sys.argv[1]):
    m = re.search(r"pol=(\d+) cap=(\d+) .* Mcycles=([\d.]+) phases=([\d.,]+)", l)
    if m:
        a = agg[int(m.group(1))]
        a[0] += 1; a[1] = max(a[1], float(m.group(3))); a[2] += float(m.group(3))
        for i, x in enumerate(m.group(4).split(",")): a[3][i] += float(x)
for p, a in sorted(agg.items()):
    print("C5 pol", p, "items", a[0], "max Mcycles", a[1], "sum Gcycles", round(a[2] / 1e3, 1), "mean phases", [round(x / a[0], 1) for x in a[3]])
PY
VARIANT="-DSAGA_REPLAY_LC=1" bash scripts/gpu_ab.sh
