#!/bin/bash
# launch list + one `ncu --set full` capture of kernel $KREGEX (default k_replay) on one B200
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
ARGS="${PROF_ARGS:---steps 1 --warmup 1 --no-cpu-baseline --no-e2e}"
KREGEX="${KREGEX:-k_replay}"
timeout 600 python bench.py $ARGS > gpurun_out/plain.log 2>&1; rc=$?; echo "plain exit $rc" >> gpurun_out/plain.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c ${NCU_COUNT:-1} \
     -o gpurun_out/prof_$KREGEX -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?" >> gpurun_out/ncu_full.log
fi
tail -3 gpurun_out/plain.log; tail -3 gpurun_out/ncu_launches.log; tail -5 gpurun_out/ncu_full.log
