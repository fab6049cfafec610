#!/bin/bash
# bench lines at every config (one GPU), logs in gpurun_out/cfg_*.log
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for CFG in ${CFGS:-C1 C3 C4 C5}; do
  S=5; [ "$CFG" = "C4" ] && S=3; [ "$CFG" = "C5" ] && S=2
  timeout 1800 python bench.py --config $CFG --steps $S --warmup ${W:-3} --no-cpu-baseline --no-bulk > gpurun_out/cfg_$CFG.log 2>&1
  python - gpurun_out/cfg_$CFG.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["config"]["trace"], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step",
              "lat", round(d["config"]["step_latency_ms"], 1), "inflight", d["config"]["steps_in_flight"],
              {k: round(v["ms_per_step"], 1) for k, v in d["kernels"].items()}, "e2e", (d.get("e2e") or {}).get("value"))
PY
  tail -2 gpurun_out/cfg_$CFG.log | grep -v "^{" | tail -2
done
