#!/bin/bash
# one B200: build, full GPU tests, default bench line, ncu launch list, one ncu --set full capture of $KREGEX
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; rc=$?; echo "bench exit $rc" >> gpurun_out/bench_default.log
tail -c 400 gpurun_out/bench_default.log
if [ $rc -eq 0 ]; then
  ARGS="${NCU_ARGS:---steps 1 --warmup 3 --no-cpu-baseline --no-e2e}"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
  KREGEX="${KREGEX:-k_pat_count}"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 \
     -o gpurun_out/prof_$KREGEX -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?" >> gpurun_out/ncu_full.log
  tail -2 gpurun_out/ncu_launches.log; tail -2 gpurun_out/ncu_full.log
fi
