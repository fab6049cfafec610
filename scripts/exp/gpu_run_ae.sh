#!/bin/bash
# placement act masks maintained with the counts again (parity + C2/C5 placement time); AEG pivot-path counts
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-bulk > gpurun_out/bench_c2_ae.log 2>&1
timeout 1500 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-bulk --no-e2e > gpurun_out/bench_c5_ae.log 2>&1
for f in bench_c2_ae bench_c5_ae; do python - gpurun_out/$f.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step", {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()}, d["counters_checksum"])
PY
done
VARIANTS="-DSAGA_TRACE_COUNT_PIVOT" bash scripts/gpu_ab2.sh 2>&1 | grep COUNT
