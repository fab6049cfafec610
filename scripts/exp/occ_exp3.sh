#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
A="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk --inflight 1"
run() {
  SAGA_NVCC_EXTRA="$2" python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > gpurun_out/build_$1.log 2>&1 || { echo "build $1 failed"; return; }
  for cfg in ${CFGS:-C4 C3}; do
    timeout 900 python bench.py $A --config $cfg > gpurun_out/occ3_$1_$cfg.log 2>&1
    echo "$1 $cfg $(grep -o '"replay": {"ms_per_step": [0-9.]*' gpurun_out/occ3_$1_$cfg.log | head -1)"
  done
}
run d32p1024 "-DSAGA_WIDE_RT=256 -DSAGA_WIDE_MINB=2 -DSAGA_WIDE_PF=1024 -DSAGA_WIDE_DYN_KB=32"
run d16p1024 "-DSAGA_WIDE_RT=256 -DSAGA_WIDE_MINB=2 -DSAGA_WIDE_PF=1024 -DSAGA_WIDE_DYN_KB=16"
run d32p512 "-DSAGA_WIDE_RT=256 -DSAGA_WIDE_MINB=2 -DSAGA_WIDE_PF=512 -DSAGA_WIDE_DYN_KB=32"
run d16p512 "-DSAGA_WIDE_RT=256 -DSAGA_WIDE_MINB=2 -DSAGA_WIDE_PF=512 -DSAGA_WIDE_DYN_KB=16"
python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
