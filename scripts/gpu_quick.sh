#!/bin/bash
# parity subset + one C2 bench line + ncu traffic of the bandwidth kernels
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_pins.py} -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
CFG=${CFG:-C2} bash scripts/gpu_k47.sh > /dev/null 2>&1
python scripts/ncu_sum.py gpurun_out/k47_${CFG:-C2}.csv
python - <<'PY'
import json
for l in open("gpurun_out/plain_C2.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(round(d["ms_per_step"], 1), {k: (round(v["ms_per_step"], 2), round(v["algorithmic_gb_s"])) for k, v in d["kernels"].items()})
        print({k: (round(v["ms"], 4), round(v["algorithmic_gb_s"])) for k, v in d["bulk_score_select"].items() if isinstance(v, dict)})
PY
