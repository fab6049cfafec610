#!/bin/bash
# smoke + the GPU test tier (optionally a subset: TESTS="tests/test_gpu_pins.py ...")
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nproc > gpurun_out/nproc.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout ${T_LIMIT:-2400} python -m pytest ${TESTS:-tests} -m gpu -q --maxfail=40 -p no:cacheprovider -n ${NPROC:-4} \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/smoke.log; tail -40 gpurun_out/gpu_tests.log
