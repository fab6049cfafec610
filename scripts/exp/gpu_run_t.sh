#!/bin/bash
# steps in flight at N=1 (C2, the driver's --steps 20 --warmup 5): 3 (default) vs 4 / 5 / 6, two runs each
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for f in 3 4 5 6; do for r in 1 2; do
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-bulk --inflight $f > gpurun_out/infl_${f}_$r.log 2>&1
  python - gpurun_out/infl_${f}_$r.log $f $r <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("inflight", sys.argv[2], "run", sys.argv[3], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step; e2e", round(d["e2e"]["value"] / 1e9, 3), "chk", d["counters_checksum"])
PY
done; done
