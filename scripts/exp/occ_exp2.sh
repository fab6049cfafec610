#!/bin/bash
# wide-shape variants on C4 / C5 (replay kernel ms per step)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk --inflight 1"
run() {  # name, extra flags
  SAGA_NVCC_EXTRA="$2" python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > gpurun_out/build_$1.log 2>&1 || { echo "build $1 failed"; tail -5 gpurun_out/build_$1.log; return; }
  for cfg in C4 C5; do
    timeout 900 python bench.py $A --config $cfg > gpurun_out/occ2_$1_$cfg.log 2>&1
    echo "$1 $cfg $(grep -o '"replay": {"ms_per_step": [0-9.]*' gpurun_out/occ2_$1_$cfg.log | head -1)"
  done
}
run w256x2 ""
run w128x4 "-DSAGA_WIDE_RT=128 -DSAGA_WIDE_MINB=4 -DSAGA_WIDE_PF=512 -DSAGA_WIDE_DYN_KB=16"
run w256x2d32 "-DSAGA_WIDE_RT=256 -DSAGA_WIDE_MINB=2 -DSAGA_WIDE_PF=1024 -DSAGA_WIDE_DYN_KB=32"
run w128x3 "-DSAGA_WIDE_RT=128 -DSAGA_WIDE_MINB=3 -DSAGA_WIDE_PF=1024 -DSAGA_WIDE_DYN_KB=24"
python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
