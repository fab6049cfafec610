#!/bin/bash
# (W_lo, W_hi) range as a host (gloo) exchange: spread at N = 2 (3 runs) and N = 4 (2 runs), one NCCL-range run
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-bulk"
run() {  # tag n extra
  local tag=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
     bench.py $A --gpus $n "$@" > gpurun_out/ab_$tag.log 2>&1
  python - gpurun_out/ab_$tag.log $tag <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[2], d["n_gpus"], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step chk", d.get("counters_checksum"), "e2e", round(((d.get("e2e") or {}).get("value") or 0) / 1e9, 3))
PY
}
run n2_host_1 2; run n2_host_2 2; run n2_host_3 2
run n4_host_1 4; run n4_host_2 4
run n2_nccl_1 2 --range-nccl
