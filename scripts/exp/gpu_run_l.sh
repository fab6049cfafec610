#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
VARIANTS="-DSAGA_REPLAY_UNR=4;-DSAGA_SORT_MATCH_ANY" bash scripts/gpu_ab2.sh
python -c "import paper_2605_00528_b200.build as b; b.build(force=True)" > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launches.log
tail -2 gpurun_out/ncu_launches.log
KERNELS=k_place PROF_ARGS="--config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bulk --inflight 1" bash scripts/gpu_ncu_kernels.sh > /dev/null 2>&1
head -50 gpurun_out/hot_k_place.txt
