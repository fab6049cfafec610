#!/bin/bash
# several compile-time variants against the default: bench C2 (per-kernel ms) + replay phase cycles
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
A="--config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-bulk"
run() {  # $1 = tag, $2 = SAGA_NVCC_EXTRA
  SAGA_NVCC_EXTRA="$2" python -c "import paper_2605_00528_b200.build as b; b.build(force=True)" > gpurun_out/build_$1.log 2>&1 || { tail gpurun_out/build_$1.log; return; }
  timeout 900 python bench.py $A > gpurun_out/ab_$1.log 2>&1
  SAGA_REPLAY_TRACE=1 timeout 600 python scripts/profile_step.py --config C2 > gpurun_out/ab_$1_trace.log 2>&1
  python - gpurun_out/ab_$1.log gpurun_out/ab_$1_trace.log $1 <<'PY'
import json, re, sys, collections
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[3], round(d["ms_per_step"], 1), "ms/step", {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()}, "chk", d["counters_checksum"])
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, [0.0] * 8])
for l in open(sys.argv[2]):
    m = re.search(r"pol=(\d+) cap=(\d+) .* Mcycles=([\d.]+) phases=([\d.,]+)", l)
    if m:
        a = agg[int(m.group(1))]
        a[0] += 1; a[1] = max(a[1], float(m.group(3))); a[2] += float(m.group(3))
        for i, x in enumerate(m.group(4).split(",")): a[3][i] += float(x)
for p, a in sorted(agg.items()):
    print(sys.argv[3], "pol", p, "max Mcycles", a[1], "sum Gcycles", round(a[2] / 1e3, 2), "mean phases", [round(x / a[0], 1) for x in a[3]])
PY
}
run base ""
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do tag=$(echo "$v" | tr -c 'A-Za-z0-9' '_' | cut -c1-40); run "$tag" "$v"; done
python -c "import paper_2605_00528_b200.build as b; b.build(force=True)" > /dev/null 2>&1
