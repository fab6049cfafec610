#!/bin/bash
# round-end check on one B200: build, smoke(), full GPU tests, default bench line, ncu launch list
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; rc=$?; echo "bench exit $rc" >> gpurun_out/bench_final.log
tail -c 600 gpurun_out/bench_final.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-bulk > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
  tail -1 gpurun_out/ncu_launches.log
fi
