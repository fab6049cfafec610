#!/bin/bash
# placement v3 parity + bench; replay A/B: L2 prefetch of the next epoch's nres words
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -n 4 \
   > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
VARIANTS="-DSAGA_REPLAY_PF_NRES" bash scripts/gpu_ab2.sh
KERNELS=k_place PROF_ARGS="--config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk --inflight 1" bash scripts/gpu_ncu_kernels.sh > /dev/null 2>&1
head -12 gpurun_out/hot_k_place.txt
