#!/bin/bash
# C5 line with the final code
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-bulk > gpurun_out/bench_c5_final.log 2>&1
python - gpurun_out/bench_c5_final.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step e2e", round(((d.get("e2e") or {}).get("value") or 0) / 1e9, 3), {k: round(v["ms_per_step"], 1) for k, v in d["kernels"].items()}, d["clocks"], d["counters_checksum"])
PY
