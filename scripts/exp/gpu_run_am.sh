#!/bin/bash
# final code on 2 GPUs: the 2-process NCCL test and the node-sharded driver command
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/multi_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/multi_tests.log
tail -2 gpurun_out/multi_tests.log
for r in 1 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2966$r \
   bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/n2_final_$r.log 2>&1
python - gpurun_out/n2_final_$r.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(d["n_gpus"], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step e2e", round(d["e2e"]["value"] / 1e9, 3), d["counters_checksum"], d["clocks"])
PY
done
