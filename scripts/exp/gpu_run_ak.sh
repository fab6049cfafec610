#!/bin/bash
# the driver's exact GPU-tier command (serial) and smoke
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
start=$(date +%s)
timeout 3000 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests_serial.log 2>&1; echo "pytest exit $? in $(( $(date +%s) - start )) s" >> gpurun_out/gpu_tests_serial.log
tail -3 gpurun_out/gpu_tests_serial.log
