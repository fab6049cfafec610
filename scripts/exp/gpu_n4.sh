#!/bin/bash
# 4 x B200: the driver's scaling launch at N=4 (trials, two steps in flight) and the reference arm
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.log 2>&1; echo "n4 exit $?" >> gpurun_out/bench_n4.log
tail -c 300 gpurun_out/bench_n4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --impl reference --gpus 4 --steps 1 --warmup 1 > gpurun_out/bench_n4_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_n4_ref.log
tail -c 200 gpurun_out/bench_n4_ref.log
