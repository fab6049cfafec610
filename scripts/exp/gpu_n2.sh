cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.log 2>&1; echo "n2 exit $?" >> gpurun_out/bench_n2.log
tail -c 700 gpurun_out/bench_n2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --shard nodes --no-e2e > gpurun_out/bench_n2_nodes.log 2>&1; echo "n2 nodes exit $?" >> gpurun_out/bench_n2_nodes.log
tail -c 500 gpurun_out/bench_n2_nodes.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_n2_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_n2_ref.log
tail -c 300 gpurun_out/bench_n2_ref.log
