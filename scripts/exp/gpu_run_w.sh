#!/bin/bash
# multi-GPU evidence with the final code: 2-process NCCL parity test, node-sharded scaling N = 1, 2, 4
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/multi_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/multi_tests.log
tail -3 gpurun_out/multi_tests.log
NG=4 STEPS=20 bash scripts/gpu_scale.sh
