#!/bin/bash
# device timeline of the driver's bench command (20 steps), twice: where does the run-to-run spread come from?
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2 3; do
  SAGA_TIMELINE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-bulk --no-e2e > gpurun_out/tl_$r.log 2> gpurun_out/tl_$r.err
  grep -h '^{' gpurun_out/tl_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run $r', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1))"
done
