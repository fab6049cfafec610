#!/bin/bash
# AEG mono pivot taken block-wide (one round trip + one block scan per 16 K positions): parity + phases + bench
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
VARIANTS="" bash scripts/gpu_ab2.sh
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-bulk > gpurun_out/bench_c2_ag.log 2>&1
python - gpurun_out/bench_c2_ag.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print("20 steps", round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step e2e", round(d["e2e"]["value"] / 1e9, 3), d["counters_checksum"])
PY
