#!/bin/bash
# C4 with the default (memory-based) overlap decision, e2e on
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline --no-bulk > gpurun_out/c4_default.log 2>&1; echo "exit $?"
python - gpurun_out/c4_default.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step e2e", round(d["e2e"]["value"] / 1e9, 3), "inflight", d["config"]["steps_in_flight"], d["config"]["overlap"], d["counters_checksum"])
PY
tail -3 gpurun_out/c4_default.log | cut -c1-300
