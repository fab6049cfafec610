#!/bin/bash
# round-end style validation: smoke, the GPU test tier, the driver's bench command (twice), C3 / C4
# lines, a launch list of the default bench
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -n 4 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
summ() { python - "$1" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        e2e = d.get("e2e") or {}
        cb = d.get("cpu_baseline") or {}
        print(sys.argv[1], d["config"]["workload"][:3], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step; e2e",
              round((e2e.get("value") or 0) / 1e9, 3), "lat", round(d["config"].get("step_latency_ms", 0), 1),
              "roof", round(d["roofline"]["frac"], 4), "issue", round(d["roofline"].get("issue", {}).get("frac", 0), 3),
              "cpu", cb.get("value"), "launches", d["gpu_launches"], "clocks", d["clocks"], "chk", d["counters_checksum"])
        print("  ", {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
}
for r in 1 2; do
  timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver_$r.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_driver_$r.log
  summ gpurun_out/bench_driver_$r.log
done
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
summ gpurun_out/bench_c3.log
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-bulk > gpurun_out/bench_c4.log 2>&1
summ gpurun_out/bench_c4.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launches.log
tail -1 gpurun_out/ncu_launches.log
python scripts/ncu_sum.py gpurun_out/launches.csv | head -12
