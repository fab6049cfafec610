#!/bin/bash
# stream priorities: replay kernels on a lowest-priority stream, step streams high priority, vs all equal
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -n 4 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
one() {  # tag, inflight, run, extra env / args
  local tag=$1 f=$2 r=$3; shift 3
  env "$@" timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-bulk --inflight $f $PRIO_ARGS > gpurun_out/prio_${tag}_${f}_$r.log 2>&1
  python - gpurun_out/prio_${tag}_${f}_$r.log $tag $f $r <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[2], "inflight", sys.argv[3], "run", sys.argv[4], round(d["value"] / 1e9, 3), "G/s", round(d["ms_per_step"], 1), "ms/step; e2e", round(d["e2e"]["value"] / 1e9, 3), "chk", d["counters_checksum"])
PY
}
for f in 3 5; do for r in 1 2; do
  PRIO_ARGS="" one prio $f $r SAGA_X=1
  PRIO_ARGS="--stream-priority 0" one equal $f $r SAGA_REPLAY_SAME_STREAM=1
done; done
