#!/bin/bash
# placement rewrite + match.any sort default: parity (placement, sort, full size), C2/C4 bench, k_place ncu
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk > gpurun_out/bench_c5.log 2>&1
for f in bench_c2 bench_c4 bench_c5; do python - gpurun_out/$f.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"]/1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step lat", round(d["config"].get("step_latency_ms", 0), 1), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()}, "chk", d["counters_checksum"])
PY
done
KERNELS=k_place PROF_ARGS="--config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk --inflight 1" bash scripts/gpu_ncu_kernels.sh > /dev/null 2>&1
head -30 gpurun_out/hot_k_place.txt
