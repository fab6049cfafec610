#!/bin/bash
# hierarchical-bitmap cut placed inside the pivot c1 block by the take (one round trip fewer): parity + phases
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
VARIANTS="" bash scripts/gpu_ab2.sh
