cd ${GRAFT_REPO_ROOT:-.}
A="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-bulk --inflight 1"
python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
for i in 1 2; do timeout 600 python bench.py $A > /tmp/s1.log 2>&1; echo "ballot $(grep -o '"sort": {"ms_per_step": [0-9.]*' /tmp/s1.log)"; done
SAGA_NVCC_EXTRA="-DSAGA_SORT_MATCH_ANY" python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
for i in 1 2; do timeout 600 python bench.py $A > /tmp/s2.log 2>&1; echo "match $(grep -o '"sort": {"ms_per_step": [0-9.]*' /tmp/s2.log)"; done
python -c "from paper_2605_00528_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "next_use" 2>&1 | tail -2
