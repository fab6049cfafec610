#!/bin/bash
# one `ncu --set full` capture per kernel named in KERNELS (bench C2, 1 step), summaries in gpurun_out/
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
ARGS="${PROF_ARGS:---config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --inflight 1}"
for K in ${KERNELS:-k_score_aeg k_select_cl}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K -f \
     python bench.py $ARGS > gpurun_out/ncu_$K.log 2>&1
  python scripts/ncu_hot.py gpurun_out/prof_$K.ncu-rep 25 > gpurun_out/hot_$K.txt 2>&1
  ncu -i gpurun_out/prof_$K.ncu-rep --page details > gpurun_out/details_$K.txt 2>&1
done
ls gpurun_out
