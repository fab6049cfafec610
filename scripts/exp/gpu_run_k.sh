#!/bin/bash
# C5 bench (replay budget fix), per-config ncu traffic, onesweep / segscan ncu, sanitizer
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
CFGS="C5" W=1 bash scripts/gpu_configs2.sh
CFGS="C2 C3 C5" bash scripts/gpu_profile.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep --launch-skip 1 -c 1 \
   -o gpurun_out/prof_onesweep0 -f python scripts/profile_step.py --config C2 > gpurun_out/ncu_onesweep0.log 2>&1
python scripts/ncu_hot.py gpurun_out/prof_onesweep0.ncu-rep 30 > gpurun_out/hot_onesweep0.txt 2>&1
ncu -i gpurun_out/prof_onesweep0.ncu-rep --page details > gpurun_out/details_onesweep0.txt 2>&1
head -45 gpurun_out/hot_onesweep0.txt
bash scripts/gpu_sanitize.sh
