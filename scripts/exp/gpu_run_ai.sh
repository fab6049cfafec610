#!/bin/bash
# C4: overlapped steps (3 expanded traces resident, ~26 GB each) vs the chain
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config C4 --steps 4 --warmup 3 --no-cpu-baseline --no-bulk --no-e2e"
timeout 1200 python bench.py $A > gpurun_out/c4_chain.log 2>&1
timeout 1200 python bench.py $A --overlap > gpurun_out/c4_overlap.log 2>&1
timeout 1200 python bench.py $A --overlap --inflight 2 > gpurun_out/c4_overlap2.log 2>&1
nvidia-smi --query-gpu=memory.total --format=csv
for f in c4_chain c4_overlap c4_overlap2; do python - gpurun_out/$f.log $f <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[2], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step inflight", d["config"]["steps_in_flight"], d["counters_checksum"])
PY
tail -2 gpurun_out/$f.log | head -1
done
