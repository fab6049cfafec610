#!/bin/bash
# scaling lines (node-sharded, the N > 1 default) at N = 1, 2, ..., NG on one box, plus trials at NG
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
NG=${NG:-4}
CFG=${CFG:-C2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config $CFG --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-bulk"
timeout 900 python bench.py $A > gpurun_out/scale_${CFG}_n1.log 2>&1
N=2
while [ $N -le $NG ]; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
     bench.py $A --gpus $N > gpurun_out/scale_${CFG}_n$N.log 2>&1
  N=$((N * 2))
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29599 \
   bench.py $A --gpus $NG --shard trials > gpurun_out/scale_${CFG}_n${NG}_trials.log 2>&1
for f in gpurun_out/scale_${CFG}_*.log; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["n_gpus"], d["config"].get("sharding")[:20], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1),
              "ms/step inflight", d["config"]["steps_in_flight"], "checksum", d.get("counters_checksum"),
              "e2e", round(((d.get("e2e") or {}).get("value") or 0) / 1e9, 3))
PY
done
