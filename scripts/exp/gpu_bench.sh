#!/bin/bash
# bench + launch list on one B200 (run from the repo root under gpurun)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SMALL="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 python bench.py $SMALL > gpurun_out/bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py $SMALL > gpurun_out/ncu_launches.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launches.log
fi
tail -3 gpurun_out/bench.log
