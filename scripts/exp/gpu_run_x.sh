#!/bin/bash
# N = 2 node-sharded spread: stream priorities on / off, two runs each (20 steps)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-bulk"
for r in 1 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$r \
     bench.py $A --gpus 2 > gpurun_out/n2_prio_$r.log 2>&1
  SAGA_REPLAY_SAME_STREAM=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$r \
     bench.py $A --gpus 2 --stream-priority 0 > gpurun_out/n2_equal_$r.log 2>&1
done
for f in gpurun_out/n2_*.log; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["n_gpus"], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step inflight", d["config"]["steps_in_flight"], "chk", d.get("counters_checksum"), "e2e", round(((d.get("e2e") or {}).get("value") or 0) / 1e9, 3))
PY
done
