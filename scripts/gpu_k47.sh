#!/bin/bash
# ncu traffic + duration of the bandwidth kernels (K4 sort, K5 segscan / epoch stats, K6 score, K7 select)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
CFG=${CFG:-C2}
ARGS="--config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --inflight 1"
timeout 900 python bench.py $ARGS > gpurun_out/plain_$CFG.log 2>&1; rc=$?; echo "plain exit $rc" >> gpurun_out/plain_$CFG.log
if [ $rc -eq 0 ]; then
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
     --clock-control none --csv -k regex:'k_hist|k_onesweep|k_segscan|k_epoch_stats|k_score|k_select' \
     --log-file gpurun_out/k47_$CFG.csv python bench.py $ARGS > gpurun_out/ncu_k47_$CFG.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_k47_$CFG.log
fi
tail -2 gpurun_out/plain_$CFG.log; tail -3 gpurun_out/ncu_k47_$CFG.log
