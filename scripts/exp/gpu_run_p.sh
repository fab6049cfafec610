#!/bin/bash
# lane-parallel hierarchical-bitmap take (BELADY / LRU victims): parity + bench + replay phases
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
VARIANTS="" bash scripts/gpu_ab2.sh
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_20.log 2>&1
python - gpurun_out/bench_c2_20.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("20 steps:", round(d["value"]/1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step; e2e", round(d["e2e"]["value"]/1e9, 3), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()}, "chk", d["counters_checksum"])
PY
