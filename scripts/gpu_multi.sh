#!/bin/bash
# N-GPU evidence: the 2-process NCCL parity test, then node-sharded and trials bench
# lines at N = NG and N = 1 (counters_checksum of node-sharded N > 1 must equal N = 1).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
NG=${NG:-2}
CFG=${CFG:-C2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/multi_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/multi_tests.log
tail -3 gpurun_out/multi_tests.log
A="--config $CFG --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-bulk"
timeout 900 python bench.py $A --shard nodes > gpurun_out/multi_${CFG}_n1_nodes.log 2>&1
for SH in nodes trials; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 \
     bench.py $A --gpus $NG --shard $SH > gpurun_out/multi_${CFG}_n${NG}_$SH.log 2>&1
done
for f in gpurun_out/multi_${CFG}_*.log; do echo "== $f"; python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["n_gpus"], d["config"].get("sharding"), round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms",
              "checksum", d.get("counters_checksum"), "e2e", (d.get("e2e") or {}).get("value"))
PY
done
