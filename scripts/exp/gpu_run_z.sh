#!/bin/bash
# clock sampler started before the warm-up (nvidia-smi start-up out of the timed region): spread at N = 1, 2
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-bulk"
for r in 1 2 3; do
  timeout 900 python bench.py $A > gpurun_out/z1_$r.log 2>&1
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$r \
     bench.py $A --gpus 2 > gpurun_out/z2_$r.log 2>&1
done
for f in gpurun_out/z[12]_*.log; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], d["n_gpus"], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step chk", d.get("counters_checksum"), "e2e", round(((d.get("e2e") or {}).get("value") or 0) / 1e9, 3), d["clocks"])
PY
done
