#!/bin/bash
# N = 2 device timelines (rank 0 and 1), three runs
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-bulk --no-e2e"
for r in 1 2 3; do
  SAGA_TIMELINE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2958$r \
     --redirects 3 --log-dir gpurun_out/tl2_$r bench.py $A --gpus 2 > gpurun_out/tl2_$r.log 2>&1
  grep -h '^{' gpurun_out/tl2_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $r', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1))"
done
find gpurun_out/tl2_1 -type f | head
