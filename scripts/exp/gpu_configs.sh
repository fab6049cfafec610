#!/bin/bash
# one B200: a bench line per config (no CPU baseline / bulk legs) for DESIGN.md's measurement table
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
A="--no-cpu-baseline --no-bulk"
timeout 600 python bench.py $A > gpurun_out/cfg_C2.log 2>&1
timeout 900 python bench.py $A --policy-mask 31 > gpurun_out/cfg_C2_all.log 2>&1
timeout 900 python bench.py $A --config C3 > gpurun_out/cfg_C3.log 2>&1
timeout 1200 python bench.py $A --config C4 --steps 3 > gpurun_out/cfg_C4.log 2>&1
timeout 1800 python bench.py $A --config C5 --steps 2 --warmup 3 --no-e2e > gpurun_out/cfg_C5.log 2>&1
for f in gpurun_out/cfg_*.log; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        k = d['kernels']
        print(sys.argv[1], f"value {d['value']:.3e} step {d['ms_per_step']:.1f} ms", "place", round(k['place']['ms_per_step'], 1),
              "replay", round(k['replay']['ms_per_step'], 1), "inflight", d['config'].get('steps_in_flight'),
              "e2e", d['e2e'] and round(d['e2e']['ms_per_step'], 1), d['clocks']['reasons'])
PY
done
