#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for kb in ${KBS:-16 64 128 200}; do
  SAGA_REPLAY_SMEM_KB=$kb SAGA_REPLAY_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/smem_$kb.log 2>&1
  echo "kb=$kb $(grep -o '"replay": {"ms_per_step": [0-9.]*' gpurun_out/smem_$kb.log | tail -1) $(grep -m1 'grid' gpurun_out/smem_$kb.log)"
done
