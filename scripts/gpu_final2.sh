#!/bin/bash
# round-end style validation: smoke, the GPU test tier, the default bench line, a launch list
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -n 4 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_default.log
python - gpurun_out/bench_default.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step; e2e", round(d["e2e"]["value"] / 1e9, 3),
              "lat", round(d["config"]["step_latency_ms"], 1), "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 4),
              "issue", round(d["roofline"].get("issue", {}).get("frac", 0), 3), "cpu", d["cpu_baseline"]["value"],
              d["cpu_baseline"].get("single_thread"), "launches", d["gpu_launches"], "clocks", d["clocks"])
        print({k: (round(v["ms_per_step"], 2), round(v["algorithmic_gb_s"] or 0), v.get("traffic_over_algorithmic")) for k, v in d["kernels"].items()})
        print({k: (round(v["ms"], 4), round(v["algorithmic_gb_s"]), v.get("traffic_over_algorithmic")) for k, v in d["bulk_score_select"].items() if isinstance(v, dict)})
PY
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launches.log
tail -1 gpurun_out/ncu_launches.log
