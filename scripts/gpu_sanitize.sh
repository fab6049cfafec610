#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the small GPU parity cases
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for TOOL in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 20 \
     python -m pytest tests/test_gpu_pins.py -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitize_$TOOL.log 2>&1
  echo "$TOOL exit $?" >> gpurun_out/sanitize_$TOOL.log
  tail -3 gpurun_out/sanitize_$TOOL.log
done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 \
   python -m pytest "tests/test_gpu_parity.py" -m gpu -q -x -p no:cacheprovider -k "rand1 or C1 or obs1 or select" > gpurun_out/sanitize_parity.log 2>&1
echo "memcheck parity exit $?" >> gpurun_out/sanitize_parity.log
tail -3 gpurun_out/sanitize_parity.log
