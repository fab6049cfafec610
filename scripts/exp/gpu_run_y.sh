#!/bin/bash
# expansion gating with overlap: after the previous step's replay is queued (default) vs none; N = 1 and 2
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-bulk"
for r in 1 2 3; do
  for G in queued none; do
    timeout 900 python bench.py $A --gate $G > gpurun_out/g1_${G}_$r.log 2>&1
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 295$r$((RANDOM % 9)) \
       bench.py $A --gpus 2 --gate $G > gpurun_out/g2_${G}_$r.log 2>&1
  done
done
for f in gpurun_out/g[12]_*.log; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["n_gpus"], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step chk", d.get("counters_checksum"), "e2e", round(((d.get("e2e") or {}).get("value") or 0) / 1e9, 3))
PY
done
