#!/bin/bash
# A3 expansion batched over nodes (two host reads of sizes for all), plus the earlier sync cuts (one h2d
# of the replay parameters, no pre-copy sync in d2h / h2d): GPU tier, driver command x3
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider -n 4 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for r in 1 2 3; do
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_exp_$r.log 2>&1
  python - gpurun_out/bench_exp_$r.log $r <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("run", sys.argv[2], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step e2e", round(d["e2e"]["value"] / 1e9, 3), "lat", round(d["config"]["step_latency_ms"], 1), d["counters_checksum"])
PY
done
SAGA_TIMELINE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-bulk --no-e2e > gpurun_out/tl_exp.log 2> gpurun_out/tl_exp.err
