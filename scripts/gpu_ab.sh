#!/bin/bash
# A/B of a compile-time variant of libsaga: bench C2 with the default build, then with
# SAGA_NVCC_EXTRA="$VARIANT" (forced rebuild); per-kernel ms and replay per-phase cycles
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
A="--config ${CFG:-C2} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-bulk"
summ() { python - "$1" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["ms_per_step"], 1), "ms/step", {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()},
              "chk", d["counters_checksum"])
PY
}
python -c "import paper_2605_00528_b200.build as b; b.build(force=True)" > gpurun_out/build_a.log 2>&1 || { tail gpurun_out/build_a.log; exit 1; }
timeout 900 python bench.py $A > gpurun_out/ab_a.log 2>&1; summ gpurun_out/ab_a.log
SAGA_REPLAY_TRACE=1 timeout 900 python scripts/profile_step.py --config ${CFG:-C2} > gpurun_out/ab_a_trace.log 2>&1
SAGA_NVCC_EXTRA="$VARIANT" python -c "import paper_2605_00528_b200.build as b; b.build(force=True)" > gpurun_out/build_b.log 2>&1 || { tail gpurun_out/build_b.log; exit 1; }
timeout 900 python bench.py $A > gpurun_out/ab_b.log 2>&1; summ gpurun_out/ab_b.log
SAGA_REPLAY_TRACE=1 timeout 900 python scripts/profile_step.py --config ${CFG:-C2} > gpurun_out/ab_b_trace.log 2>&1
for f in a b; do python - gpurun_out/ab_${f}_trace.log <<'PY'
import re, sys, collections
agg = collections.defaultdict(lambda: [0, 0.0, [0.0] * 8])
for l in open(sys.argv[1]):
    m = re.search(r"pol=(\d+) cap=(\d+) .* Mcycles=([\d.]+) phases=([\d.,]+)", l)
    if m:
        a = agg[int(m.group(1))]
        a[0] += 1; a[1] = max(a[1], float(m.group(3)))
        for i, x in enumerate(m.group(4).split(",")): a[2][i] += float(x)
for p, a in sorted(agg.items()):
    print(sys.argv[1], "pol", p, "items", a[0], "max Mcycles", a[1], "mean phases", [round(x / a[0], 1) for x in a[2]])
PY
done
