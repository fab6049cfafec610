#!/bin/bash
# GPU parity (async replay) + default bench C2 (overlap, 3 in flight) vs --no-overlap, with a timeline
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -n 4 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "exit $?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --no-overlap --no-cpu-baseline --no-bulk > gpurun_out/bench_nooverlap.log 2>&1
SAGA_TIMELINE=1 timeout 900 python bench.py --steps 6 --no-cpu-baseline --no-e2e --no-bulk > gpurun_out/bench_timeline.log 2>&1
for f in bench_default bench_nooverlap bench_timeline; do python - gpurun_out/$f.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step", "lat",
              round(d["config"]["step_latency_ms"], 1), "inflight", d["config"]["steps_in_flight"], "overlap",
              d["config"].get("overlap"), "e2e", (d.get("e2e") or {}).get("value"), "chk", d.get("counters_checksum"))
PY
done
