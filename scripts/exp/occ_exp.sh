#!/bin/bash
# replay occupancy experiment: default (512 threads, 1 CTA/SM) vs 256 threads x 2 CTAs/SM
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
A="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk --inflight 1"
python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || exit 1
for cfg in C4 C2; do
  timeout 600 python bench.py $A --config $cfg > gpurun_out/occ_def_$cfg.log 2>&1
  SAGA_REPLAY_TRACE=1 timeout 600 python bench.py $A --config $cfg --steps 1 > gpurun_out/occ_def_trace_$cfg.log 2>&1
done
SAGA_NVCC_EXTRA="-DSAGA_REPLAY_RT=256 -DSAGA_REPLAY_MINB=2 -DSAGA_REPLAY_PF=1024" python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > gpurun_out/build2.log 2>&1 || exit 1
for cfg in C4 C2; do
  SAGA_REPLAY_SMEM_KB=${KB:-48} timeout 600 python bench.py $A --config $cfg > gpurun_out/occ_v2_$cfg.log 2>&1
  SAGA_REPLAY_SMEM_KB=${KB:-48} SAGA_REPLAY_TRACE=1 timeout 600 python bench.py $A --config $cfg > gpurun_out/occ_v2_trace_$cfg.log 2>&1
done
for f in gpurun_out/occ_*.log; do echo $f; grep -o '"replay": {"ms_per_step": [0-9.]*' $f | head -1; grep -m1 "saga replay\] grid" $f; done
