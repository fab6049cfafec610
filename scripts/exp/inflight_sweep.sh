cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for inf in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --no-bulk --inflight $inf > gpurun_out/bench_inf$inf.log 2>&1; echo "exit $?" >> gpurun_out/bench_inf$inf.log
  tail -c 600 gpurun_out/bench_inf$inf.log; echo
done
timeout 600 python bench.py --no-cpu-baseline --no-bulk --config C3 > gpurun_out/bench_c3.log 2>&1; tail -c 400 gpurun_out/bench_c3.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
